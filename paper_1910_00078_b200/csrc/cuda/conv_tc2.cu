// CTA-pair (cta_group::2) tcgen05 plain GEMM for 1x1 convolutions whose filter
// slice is too large to stay resident (conv_tc.cu PLAIN_RES covers the rest):
//
//   D[pixel][out] = sum_k A[pixel][k] * B[out][k]      (fwd: x / W, dgrad: dY / W^T)
//
// Why: the single-CTA plain kernel is TMA-throughput bound — with MMA, TMEM
// reads and stores disabled it still needs 26.5 us on ResNet conv4_2a for
// 303 MB of TMA traffic, 2/3 of it the filter (B) re-read per 128-pixel tile
// (profiles/r01_ncu_full.md). A CTA pair computes a 256 x 256 tile with M=256
// MMAs: each CTA loads its own 128 pixel rows of A and HALF of the 256 filter
// rows of B, and the pair's tensor cores read both halves — B bytes per FLOP
// through TMA halve (A 16 KB + B 16 KB per SM per k-block instead of 16 + 32).
//
// Roles per CTA (320 threads): warp 0 TMA producer (cta_group::2 loads signal
// the leader's stage barrier), warp 1 TMEM allocator (both CTAs) + MMA issuer
// (leader only; commits multicast to both CTAs), warps 2-9 epilogue (each CTA
// drains its own 128 TMEM lanes, fused per-channel affine / activation, TMA
// stores, then arrives remotely on the leader's TMEM-empty barrier).
// Validated first in tools/probes/cta2_probe.cu.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc_host.cuh"
#include "tc_internal.h"
#include "tc_ptx.cuh"

namespace pk {
namespace {

using namespace pk::tc;

constexpr int kThreads2 = 320;
constexpr int kStages2 = 5;
constexpr int kHalfA = 128 * 64 * 2;   // 128 pixel rows x 64 k (SW128)
constexpr int kHalfB = 128 * 64 * 2;   // 128 filter rows x 64 k
constexpr int kStage2 = kHalfA + kHalfB;
constexpr int kStaging2 = 8 * 2 * 4096;  // 8 epilogue warps x 2 buffers x (32 x 128 B)
constexpr int kStgOff2 = kStages2 * kStage2;
constexpr int kBarOff2 = kStgOff2 + kStaging2;
constexpr int kBytes2 = kBarOff2 + (2 * kStages2 + 4) * 8 + 16 + 1024;
static_assert(kBytes2 <= 227 * 1024, "smem");

struct Gemm2Args {
    int M;          // pixel rows
    int num_kb;     // 64-wide k-blocks
    int n_out, out_pitch;
    int m_pairs, n_tiles, total;  // pair tiles: (M / 256) x (N / 256)
    int P, Q;       // output image extent (per-activation epilogues)
    int b_mn;       // B MN-major: two 64-wide atoms (8 KB apart) per CTA half
    // Work items: the first full_items are 256 x 256 pair tiles; when the last
    // round of tiles would leave pairs idle (R = total mod pairs, 2R <= pairs)
    // those R tiles run as 2R half tiles of 256 x 128 (N=128 MMAs), so the tail
    // takes half a tile time (ResNet conv5 1x1: 98 tiles on 74 pairs)
    int items, full_items;
    unsigned long long* trace;  // PK_TC2_TRACE: summed wait clocks per role (profiling only)
};

__device__ __forceinline__ void commit_pair(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
        "[%0], %1;\n\t}" ::"r"(smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}
// Four K=16 M=256 MMAs of one 64-wide k-block (leader CTA, one elect).
__device__ __forceinline__ void mma4_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
        "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a3, b3, %3, 1;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

struct PairItem {
    int mp, nt, h;  // pair tile (M, N) and half (-1: the whole 256-wide tile)
};
__device__ __forceinline__ PairItem pair_item(const Gemm2Args& g, int u) {
    int t = u, h = -1;
    if (u >= g.full_items) {
        const int v = u - g.full_items;
        t = g.full_items + (v >> 1);
        h = v & 1;
    }
    const int mp = t / g.n_tiles;
    return {mp, t - mp * g.n_tiles, h};
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                     const __grid_constant__ CUtensorMap bmap_h, const __grid_constant__ CUtensorMap ymap,
                     const __grid_constant__ Gemm2Args g, const pk_epilogue epi) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kBarOff2);
    uint64_t* empty = full + kStages2;
    uint64_t* tmem_full = empty + kStages2;   // [2]
    uint64_t* tmem_empty = tmem_full + 2;     // [2] (leader's is the one used)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int pair_id = blockIdx.x >> 1, num_pairs = gridDim.x >> 1;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages2; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 16);  // 8 epilogue warps x 2 CTAs
        }
        fence_barrier_init();
        tma_prefetch(&amap);
        tma_prefetch(&bmap);
        if (g.items != g.full_items && !g.b_mn) tma_prefetch(&bmap_h);
        tma_prefetch(&ymap);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // peer barriers initialised before any remote signal
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();
    pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            long long tw = 0;
            const long long t0 = clock64();
            for (int u = pair_id; u < g.items; u += num_pairs) {
                const PairItem pi = pair_item(g, u);
                const int bh = pi.h < 0 ? 128 : 64;  // filter rows of B per CTA
                const int arow = pi.mp * 256 + (int)rank * 128;
                const int brow = pi.nt * 256 + (pi.h < 0 ? 0 : pi.h * 128) + (int)rank * bh;
                for (int kb = 0; kb < g.num_kb; ++kb) {
                    const long long w0 = clock64();
                    mbar_wait(&empty[stage], phase ^ 1);
                    tw += clock64() - w0;
                    uint8_t* sa = smem + stage * kStage2;
                    const uint32_t fb = smem_u32(&full[stage]) & 0xFEFFFFFFu;  // leader's barrier
                    if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (kHalfA + bh * 128));
                    tma_load_2d_pair(smem_u32(sa), &amap, fb, kb * 64, arow);
                    if (g.b_mn) {
                        tma_load_2d_pair(smem_u32(sa + kHalfA), &bmap, fb, brow, kb * 64);
                        if (bh == 128)
                            tma_load_2d_pair(smem_u32(sa + kHalfA + 8192), &bmap, fb, brow + 64, kb * 64);
                    } else {
                        tma_load_2d_pair(smem_u32(sa + kHalfA), bh == 128 ? &bmap : &bmap_h, fb, kb * 64,
                                         brow);
                    }
                    if (++stage == kStages2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
            if (g.trace) {
                atomicAdd(&g.trace[4], (unsigned long long)tw);
                atomicAdd(&g.trace[5], (unsigned long long)(clock64() - t0));
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            const uint32_t idesc_full = idesc_bf16_f32(256, 256, false, g.b_mn != 0);
            const uint32_t idesc_half = idesc_bf16_f32(256, 128, false, g.b_mn != 0);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            long long tf = 0, te = 0;
            const long long t0 = clock64();
            for (int u = pair_id; u < g.items; u += num_pairs, ++it) {
                const uint32_t idesc = pair_item(g, u).h < 0 ? idesc_full : idesc_half;
                const int a = it & 1;
                long long w0 = clock64();
                mbar_wait(&tmem_empty[a], ((it >> 1) & 1) ^ 1);
                te += clock64() - w0;
                tc_fence_after();
                const uint32_t d = tmem_base + a * 256;
                for (int kb = 0; kb < g.num_kb; ++kb) {
                    w0 = clock64();
                    mbar_wait(&full[stage], phase);
                    tf += clock64() - w0;
                    tc_fence_after();
                    const uint32_t sa = smem_u32(smem + stage * kStage2);
                    if (g.b_mn) {
                        const uint64_t ad = umma_desc_sw128(sa, 16, 1024);
                        const uint64_t bd = umma_desc_sw128(sa + kHalfA, 8192, 1024);
                        mma4_bf16_pair(d, ad, ad + 2, ad + 4, ad + 6, bd, bd + 128, bd + 256, bd + 384,
                                       idesc, kb != 0);
                    } else {
                        mma4_pair(d, umma_desc_sw128(sa, 16, 1024), umma_desc_sw128(sa + kHalfA, 16, 1024),
                                  idesc, kb != 0);
                    }
                    commit_pair(&empty[stage]);
                    if (kb == g.num_kb - 1) commit_pair(&tmem_full[a]);
                    if (++stage == kStages2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
            if (g.trace && lane == 0) {
                atomicAdd(&g.trace[0], (unsigned long long)tf);
                atomicAdd(&g.trace[1], (unsigned long long)te);
                atomicAdd(&g.trace[2], (unsigned long long)(clock64() - t0));
                atomicAdd(&g.trace[3], 1ull);
            }
        }
    } else {
        // ---------------- epilogue: this CTA's 128 TMEM lanes x 256 columns ----------
        const int ew = warp - 2, q = warp & 3, half = ew >> 2;
        uint8_t* stg_base = smem + kStgOff2 + ew * 2 * 4096;
        int sbuf = 0;
        const bool has_epi = epilogue_active(&epi);
        uint32_t leader_empty[2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;"
                         : "=r"(leader_empty[i])
                         : "r"(smem_u32(&tmem_empty[i])));
        int it = 0;
        for (int u = pair_id; u < g.items; u += num_pairs, ++it) {
            const PairItem pi = pair_item(g, u);
            const int m0 = pi.mp * 256 + (int)rank * 128, n0 = pi.nt * 256 + (pi.h < 0 ? 0 : pi.h * 128);
            const int a = it & 1;
            mbar_wait(&tmem_full[a], (it >> 1) & 1);
            tc_fence_after();
            const int span = min(pi.h < 0 ? 256 : 128, g.out_pitch - n0);
            const int nchunks = (span + 63) / 64;
            const int my_m = m0 + q * 32 + lane;
            int oy = 0, ox = 0;
            if (my_m < g.M) {
                const int rem = my_m % (g.P * g.Q);
                oy = rem / g.Q;
                ox = rem - oy * g.Q;
            }
#pragma unroll 1
            for (int ci = half; ci < nchunks; ci += 2) {
                const int c0 = ci * 64;
                uint32_t v[64];
                const uint32_t ta = tmem_base + a * 256 + c0 + (static_cast<uint32_t>(q * 32) << 16);
                tmem_ld16(ta + 0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
                tmem_ld16(ta + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
                tmem_ld16(ta + 32, *reinterpret_cast<uint32_t(*)[16]>(&v[32]));
                tmem_ld16(ta + 48, *reinterpret_cast<uint32_t(*)[16]>(&v[48]));
                tmem_ld_wait();
                const uint32_t stg_u = smem_u32(stg_base + sbuf * 4096);
                if (lane == 0) bulk_wait_read<1>();
                __syncwarp();
                float xf[64];
#pragma unroll
                for (int e = 0; e < 64; ++e) xf[e] = __uint_as_float(v[e]);
                if (has_epi) epilogue_chunk64(epi, xf, n0 + c0, g.n_out, oy, ox, g.P, g.Q);
                pack_stage64(xf, stg_u, lane, min(g.n_out - (n0 + c0), 64));
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_2d(&ymap, stg_u, n0 + c0, m0 + q * 32);
                    bulk_commit();
                }
                sbuf ^= 1;
            }
            // this warp's share of the accumulator is read: release it on the leader
            tc_fence_before();
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                 leader_empty[a])
                             : "memory");
        }
        if (lane == 0) bulk_wait_all();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
    }
}

}  // namespace
}  // namespace pk

using namespace pk;

// 1 when the pair kernel takes this plain GEMM: >= 256 output channels and
// enough 256 x 256 pair tiles to fill the SM pairs (PK_TC2=0 disables).
int pk_gemm_pair_eligible(int M, int kdim, int n_out, int out_pitch) {
    static const bool off = [] {
        const char* v = std::getenv("PK_TC2");
        return v && v[0] == '0';
    }();
    if (off || kdim % 64 || out_pitch % 256 || n_out < 256) return 0;
    const long long tiles = (long long)((M + 255) / 256) * (out_pitch / 256);
    return tiles >= 74;
}

cudaError_t pk_gemm_pair(const void* a, const void* b, void* y, int M, int kdim, int n_out,
                         int out_pitch, int P, int Q, const pk_epilogue* epi, cudaStream_t st,
                         int b_mn_pitch) {
    CUtensorMap amap{}, bmap{}, bmap_h{}, ymap{};
    const bool bmap_ok = b_mn_pitch > 0 ? tc::make_map_2d(&bmap, b, kdim, b_mn_pitch, b_mn_pitch, 64)
                                        : tc::make_map_2d(&bmap, b, n_out, kdim, kdim, 128) &&
                                              tc::make_map_2d(&bmap_h, b, n_out, kdim, kdim, 64);
    if (!tc::make_map_2d(&amap, a, M, kdim, kdim, 128) || !bmap_ok ||
        !tc::make_map_2d(&ymap, y, M, out_pitch, out_pitch, 32))
        return cudaErrorInvalidValue;
    Gemm2Args g{};
    g.M = M;
    g.num_kb = kdim / 64;
    g.n_out = n_out;
    g.out_pitch = out_pitch;
    g.m_pairs = (M + 255) / 256;
    g.n_tiles = out_pitch / 256;
    g.total = g.m_pairs * g.n_tiles;
    g.P = P;
    g.Q = Q;
    g.b_mn = b_mn_pitch > 0;
    static unsigned long long* trace = [] {
        unsigned long long* p = nullptr;
        if (std::getenv("PK_TC2_TRACE")) cudaMalloc(&p, 8 * 8);
        return p;
    }();
    g.trace = trace;
    if (trace) cudaMemsetAsync(trace, 0, 8 * 8, st);
    pk_epilogue e{};
    e.act = -1;
    if (epi) e = *epi;
    static int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
        cudaError_t err = cudaFuncSetAttribute(gemm_pair_kernel,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, kBytes2);
        if (err != cudaSuccess) return err;
        attr_dev = dev;
    }
    int grid = tc::num_sms_of_current_device() / 2 * 2;
    if (grid > 2 * g.total) grid = 2 * g.total;
    static const bool no_split = [] {  // PK_TC2_TAIL=0: whole tiles only (A/B)
        const char* v = std::getenv("PK_TC2_TAIL");
        return v && v[0] == '0';
    }();
    const int pairs = grid / 2, rem = g.total % pairs;
    g.full_items = g.items = g.total;
    if (!no_split && rem > 0 && 2 * rem <= pairs) {
        g.full_items = g.total - rem;
        g.items = g.full_items + 2 * rem;
    }
    const cudaError_t le = pk_launch(gemm_pair_kernel, dim3(grid), dim3(kThreads2), kBytes2, st, amap,
                                     bmap, bmap_h, ymap, g, e);
    count_launch();
    if (trace) {  // profiling only (PK_TC2_TRACE; not inside graph capture)
        unsigned long long h[8];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
        const double n = h[3] ? (double)h[3] : 1.0;
        fprintf(stderr,
                "tc2: pairs %llu, per pair: mma loop %.0f clk, wait full %.0f, wait tmem_empty %.0f | "
                "producer loop %.0f, wait empty %.0f (per CTA)\n",
                h[3], h[2] / n, h[0] / n, h[1] / n, h[5] / (2 * n), h[4] / (2 * n));
    }
    return le != cudaSuccess ? le : cudaGetLastError();
}
