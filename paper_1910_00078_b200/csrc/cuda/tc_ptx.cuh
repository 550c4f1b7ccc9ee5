// Thin inline-PTX wrappers for the sm_100a primitives used by the tcgen05
// convolution kernels: mbarriers, cp.async gathers, TMA tile loads, TMEM
// allocation, tcgen05.mma / commit / ld.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace pk::tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// ---- cp.async (LDGSTS) gathers ----
// 16-byte copy; src_bytes == 0 zero-fills the destination without reading.
__device__ __forceinline__ void cp_async_16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                 "r"(src_bytes)
                 : "memory");
}
// Arrive on `bar` once every cp.async previously issued by this thread has
// landed (does not increment the pending count: it is one of the expected
// arrivals).
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- TMA ----
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// L2 prefetch of a 4-D TMA box (no smem, no barrier): hides DRAM latency of
// loads issued a few tiles later.
__device__ __forceinline__ void tma_prefetch_4d(const CUtensorMap* map, int c0, int c1, int c2,
                                                int c3) {
    asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, uint32_t src, int c0, int c1,
                                             int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

// TMA tile store smem -> global (bulk async group of the issuing thread).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(src), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// Wait until at most N committed bulk groups of this thread still read smem.
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- TMEM ----
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ---- UMMA descriptors ----
// Shared-memory matrix descriptor, SWIZZLE_128B, sm_100 version bits.
//   K-major  : rows of 128 B (64 bf16 of K), 8-row atoms 1024 B apart (SBO)
//   MN-major : rows of 128 B (64 bf16 of M/N) per K index; LBO = distance
//              between 64-wide MN atoms, SBO = distance between 8-row K groups
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo_bytes,
                                                    uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;  // descriptor version (Blackwell)
    d |= 2ull << 61;  // SWIZZLE_128B
    return d;
}
// K-major SWIZZLE_NONE ("interleaved") descriptor: 8 x 16-byte core matrices,
// SBO = distance between 8-row groups along M/N, LBO = distance between the
// two core matrices along K of one MMA (K = 16 bf16 = 2 x 8).
__device__ __forceinline__ uint64_t umma_desc_noswz(uint32_t saddr, uint32_t lbo_bytes,
                                                    uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;  // descriptor version (Blackwell); layout type 0 = no swizzle
    return d;
}

// Instruction descriptor: kind::f16, A/B = fp16, D = f32 (bf16 bits 7/10 clear).
__host__ __device__ constexpr uint32_t idesc_f16_f32(int m, int n, bool a_mn_major, bool b_mn_major) {
    return (1u << 4) | ((a_mn_major ? 1u : 0u) << 15) | ((b_mn_major ? 1u : 0u) << 16) |
           (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

// Instruction descriptor: kind::tf32, A/B = tf32 (fp32 in shared memory), D = f32.
__host__ __device__ constexpr uint32_t idesc_tf32_f32(int m, int n, bool a_mn_major, bool b_mn_major) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn_major ? 1u : 0u) << 15) |
           ((b_mn_major ? 1u : 0u) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(m >> 4) << 24);
}

// Instruction descriptor: kind::f16, A/B = bf16, D = f32.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int m, int n, bool a_mn_major,
                                                      bool b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn_major ? 1u : 0u) << 15) |
           ((b_mn_major ? 1u : 0u) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Four back-to-back SS MMAs from one converged warp (elect.sync inside): the
// descriptors are computed up front so the per-instruction issue cost (64-bit
// descriptor math + R2UR moves, ~50-100 clk when chained) overlaps. Matters
// for N <= 128 tiles, whose MMAs execute in 44-64 clk.
__device__ __forceinline__ void mma4_bf16(uint32_t tmem_d, uint64_t a0, uint64_t a1, uint64_t a2,
                                          uint64_t a3, uint64_t b0, uint64_t b1, uint64_t b2,
                                          uint64_t b3, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %10, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %5, %9, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %6, %9, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %7, %9, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %8, %9, 1;\n\t}" ::"r"(tmem_d),
        "l"(a0), "l"(a1), "l"(a2), "l"(a3), "l"(b0), "l"(b1), "l"(b2), "l"(b3), "r"(idesc),
        "r"(accumulate)
        : "memory");
}
// Four tf32 MMAs (K = 8 fp32 = 32 bytes each, so the same descriptor steps as bf16).
__device__ __forceinline__ void mma4_tf32(uint32_t tmem_d, uint64_t a0, uint64_t a1, uint64_t a2,
                                          uint64_t a3, uint64_t b0, uint64_t b1, uint64_t b2,
                                          uint64_t b3, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %10, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %5, %9, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %2, %6, %9, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %3, %7, %9, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %4, %8, %9, 1;\n\t}" ::"r"(tmem_d),
        "l"(a0), "l"(a1), "l"(a2), "l"(a3), "l"(b0), "l"(b1), "l"(b2), "l"(b3), "r"(idesc),
        "r"(accumulate)
        : "memory");
}
// Two K=64 blocks (8 MMAs, K=16 each) with one elect: A/B descriptors of the
// first K=16 step of each block; later steps advance the start field by 32 B.
__device__ __forceinline__ void mma8_bf16(uint32_t tmem_d, uint64_t a0, uint64_t b0, uint64_t a1,
                                          uint64_t b1, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 x1, x2, x3, y1, y2, y3, u1, u2, u3, v1, v2, v3;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "add.s64 x1, %1, 2;\n\tadd.s64 x2, %1, 4;\n\tadd.s64 x3, %1, 6;\n\t"
        "add.s64 y1, %2, 2;\n\tadd.s64 y2, %2, 4;\n\tadd.s64 y3, %2, 6;\n\t"
        "add.s64 u1, %3, 2;\n\tadd.s64 u2, %3, 4;\n\tadd.s64 u3, %3, 6;\n\t"
        "add.s64 v1, %4, 2;\n\tadd.s64 v2, %4, 4;\n\tadd.s64 v3, %4, 6;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], x1, y1, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], x2, y2, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], x3, y3, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %4, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], u1, v1, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], u2, v2, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], u3, v3, %5, 1;\n\t}" ::"r"(tmem_d),
        "l"(a0), "l"(b0), "l"(a1), "l"(b1), "r"(idesc), "r"(accumulate)
        : "memory");
}

// ---- CTA pair (cta_group::2) ----
// TMA load by either CTA of a pair whose completion is signalled on the
// LEADER's barrier (bar = this CTA's barrier address with the peer bit cleared).
__device__ __forceinline__ void tma_load_4d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                                 int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                                 int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                                 int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
// Arrive on the leader CTA's copy of a barrier (this CTA's address mapped to rank 0).
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// Four M=256 MMAs (leader CTA; each CTA holds 128 A rows and half of B).
__device__ __forceinline__ void mma4_bf16_pair(uint32_t tmem_d, uint64_t a0, uint64_t a1, uint64_t a2,
                                               uint64_t a3, uint64_t b0, uint64_t b1, uint64_t b2,
                                               uint64_t b3, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %10, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %5, %9, p;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %6, %9, 1;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %3, %7, %9, 1;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %4, %8, %9, 1;\n\t}" ::"r"(tmem_d),
        "l"(a0), "l"(a1), "l"(a2), "l"(a3), "l"(b0), "l"(b1), "l"(b2), "l"(b3), "r"(idesc),
        "r"(accumulate)
        : "memory");
}
// Commit of the pair's MMAs, arriving on the barrier at this offset in BOTH CTAs.
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
        "[%0], %1;\n\t}" ::"r"(smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}

// mma8_bf16 with an explicit B k-step (K-major: 2, MN-major: 128 in 16-byte units).
__device__ __forceinline__ void mma8_bf16_bs(uint32_t tmem_d, uint64_t a0, uint64_t b0, uint64_t a1,
                                             uint64_t b1, uint64_t bs, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 x1, x2, x3, y1, y2, y3, u1, u2, u3, v1, v2, v3, s2, s3;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "add.s64 s2, %7, %7;\n\tadd.s64 s3, s2, %7;\n\t"
        "add.s64 x1, %1, 2;\n\tadd.s64 x2, %1, 4;\n\tadd.s64 x3, %1, 6;\n\t"
        "add.s64 y1, %2, %7;\n\tadd.s64 y2, %2, s2;\n\tadd.s64 y3, %2, s3;\n\t"
        "add.s64 u1, %3, 2;\n\tadd.s64 u2, %3, 4;\n\tadd.s64 u3, %3, 6;\n\t"
        "add.s64 v1, %4, %7;\n\tadd.s64 v2, %4, s2;\n\tadd.s64 v3, %4, s3;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], x1, y1, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], x2, y2, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], x3, y3, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %4, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], u1, v1, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], u2, v2, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], u3, v3, %5, 1;\n\t}" ::"r"(tmem_d),
        "l"(a0), "l"(b0), "l"(a1), "l"(b1), "r"(idesc), "r"(accumulate), "l"(bs)
        : "memory");
}

// mma8_bf16_bs for a CTA pair (leader CTA, cta_group::2, M = 256).
__device__ __forceinline__ void mma8_bf16_bs_pair(uint32_t tmem_d, uint64_t a0, uint64_t b0, uint64_t a1,
                                                  uint64_t b1, uint64_t bs, uint32_t idesc,
                                                  uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 x1, x2, x3, y1, y2, y3, u1, u2, u3, v1, v2, v3, s2, s3;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "add.s64 s2, %7, %7;\n\tadd.s64 s3, s2, %7;\n\t"
        "add.s64 x1, %1, 2;\n\tadd.s64 x2, %1, 4;\n\tadd.s64 x3, %1, 6;\n\t"
        "add.s64 y1, %2, %7;\n\tadd.s64 y2, %2, s2;\n\tadd.s64 y3, %2, s3;\n\t"
        "add.s64 u1, %3, 2;\n\tadd.s64 u2, %3, 4;\n\tadd.s64 u3, %3, 6;\n\t"
        "add.s64 v1, %4, %7;\n\tadd.s64 v2, %4, s2;\n\tadd.s64 v3, %4, s3;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], x1, y1, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], x2, y2, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], x3, y3, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %3, %4, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], u1, v1, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], u2, v2, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], u3, v3, %5, 1;\n\t}" ::"r"(tmem_d),
        "l"(a0), "l"(b0), "l"(a1), "l"(b1), "r"(idesc), "r"(accumulate), "l"(bs)
        : "memory");
}

// Two SS MMAs from one elected thread (accumulate).
__device__ __forceinline__ void mma2_bf16(uint32_t tmem_d, uint64_t a0, uint64_t a1, uint64_t b0,
                                          uint64_t b1, uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %3, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %4, %5, 1;\n\t}" ::"r"(tmem_d),
        "l"(a0), "l"(a1), "l"(b0), "l"(b1), "r"(idesc)
        : "memory");
}

__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

// 32 lanes x 16 columns of 32-bit TMEM -> 16 registers per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

}  // namespace pk::tc
