#include <cstdio>
#include <cstdlib>
// Fused narrow-channel ("stem") convolutions on tcgen05 — ResNet conv1
// (3 -> 64, 7x7 stride 2) and VGG conv1_1 (3 -> 64, 3x3) — without the
// column matrix round trip through HBM.
//
// A 4-channel input has too little data per pixel for TMA boxes (16-byte
// rows re-read once per filter tap) and too much redundancy for an explicit
// im2col (49 taps x 8 bytes per output pixel written and re-read: 1.3 GB for
// conv1 at N=256). Instead each CTA stages the input HALO of its output
// rectangle (8 x 16 pixels) in shared memory once, split by column phase
// (c mod stride) so lanes reading neighbouring output pixels hit consecutive
// 8-byte words, and 8 builder warps expand it in shared memory into the
// tap-packed operand the tensor core reads:
//
//   kc = tap*4 + c (tap = r*S + s, c < 4), 16-byte unit = (2 taps x 4 ch)
//
//   forward   D[pixel][k]  = A[pixel][kc] . B[k][kc]      A K-major (built),
//             B = packed filter, resident in smem; fused epilogue + TMA store
//   backward  D[kc][k]    += A[kc][pixel] . dY[k][pixel]  A MN-major SW128
//   weights   (built), dY by TMA; every CTA accumulates its tiles in TMEM,
//             writes one fp32 partial; a fixed-order sum finishes (deterministic)
//
// Roofline: HBM (x read once, y / dY read or written once); the tensor work
// (2 * 128 * K * 208 FLOP per tile) is a few percent of the MMA peak.
#include "common.cuh"
#include "tc_host.cuh"
#include "tc_internal.h"
#include "tc_ptx.cuh"

namespace pk {
namespace {

using namespace pk::tc;

constexpr int kTile = 128;          // output pixels per tile (8 x 16 rectangle)
constexpr int kBw = 16, kBh = 8;
constexpr int kBuilders = 256;      // 8 builder warps
constexpr int kHaloPer = 4;         // halo pixels per builder thread (<= 1024)
constexpr int kMaxTaps = 64;

struct StemArgs {
    int N, H, W, x_pitch;
    int P, Q;
    int K, n_pad;             // output channels, MMA N (fprop) / dY channel pitch (wgrad)
    int R, S, sh, sw, dh, dw, ph, pw;
    int C;                    // real input channels (<= 4)
    int tiles_w, tiles_h, total_tiles;
    int HH, HW, HWp;          // halo rows, cols, cols per column phase
    int nchunks;              // 16-byte (2-tap) units per pixel, even
    int taps;
    int kcm;                  // wgrad: padded kc rows (multiple of 128)
    unsigned long long* trace;  // PK_STEM_TRACE: per-role clock64 stamps of CTA 0 (profiling only)
    int debug;                // PK_STEM_DEBUG bits (profiling only): 1 no MMA, 2 no build, 4 no store, 8 no TMEM drain, 16 no halo
    int tap_off[kMaxTaps];    // halo word offset of tap t
};

__device__ __forceinline__ void tile_origin(const StemArgs& g, int t, int& n, int& oy0, int& ox0) {
    const int tx = t % g.tiles_w;
    const int rest = t / g.tiles_w;
    const int ty = rest % g.tiles_h;
    n = rest / g.tiles_h;
    oy0 = ty * kBh;
    ox0 = tx * kBw;
}

// trace slot: [tile < 32][event < 16]
__device__ __forceinline__ void stamp(const StemArgs& g, int it, int ev) {
    if (g.trace && blockIdx.x == 0 && it < 32 && (threadIdx.x & 31) == 0)
        g.trace[it * 32 + ev] = clock64();
}

__device__ __forceinline__ void named_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Per builder thread: the halo pixels it loads (fixed across tiles).
struct HaloSlots {
    int hr[kHaloPer], hc[kHaloPer], word[kHaloPer];
};

__device__ __forceinline__ void halo_slots(const StemArgs& g, int b, HaloSlots& hs) {
#pragma unroll
    for (int u = 0; u < kHaloPer; ++u) {
        const int i = b + u * kBuilders;
        if (i < g.HH * g.HW) {
            hs.hr[u] = i / g.HW;
            hs.hc[u] = i - hs.hr[u] * g.HW;
            hs.word[u] = (hs.hc[u] % g.sw) * g.HH * g.HWp + hs.hr[u] * g.HWp + hs.hc[u] / g.sw;
        } else {
            hs.hr[u] = -1;
            hs.hc[u] = 0;
            hs.word[u] = 0;
        }
    }
}

// Halo ring: kHaloStages buffers of the compact (4-channel, column-phase
// split) input halo, filled by 8-byte cp.async copies (zero fill outside x)
// kHaloStages - 1 tiles ahead of the build, so ~3 tiles of input are in
// flight per SM (the stem is HBM-latency bound otherwise).
constexpr int kHaloStages = 4;
constexpr int kHaloStageBytes = 8192;

__device__ __forceinline__ void cp_async_8(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
                 "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Issue this thread's halo copies of tile t (none past the last tile) into
// the stage at dst_u and close one cp.async group (always, to keep counts).
__device__ __forceinline__ void halo_issue(const StemArgs& g, const __nv_bfloat16* __restrict__ x,
                                           int t, const HaloSlots& hs, uint32_t dst_u) {
    if (t < g.total_tiles && !(g.debug & 16)) {
        int n, oy0, ox0;
        tile_origin(g, t, n, oy0, ox0);
        const int iy0 = oy0 * g.sh - g.ph, ix0 = ox0 * g.sw - g.pw;
#pragma unroll
        for (int u = 0; u < kHaloPer; ++u) {
            if (hs.hr[u] < 0) continue;
            const int iy = iy0 + hs.hr[u], ix = ix0 + hs.hc[u];
            const bool in = iy >= 0 && iy < g.H && ix >= 0 && ix < g.W;
            const __nv_bfloat16* src = in ? x + (((size_t)n * g.H + iy) * g.W + ix) * g.x_pitch : x;
            cp_async_8(dst_u + hs.word[u] * 8, src, in ? 8u : 0u);
        }
    }
    cp_async_commit();
}

__device__ __forceinline__ void st_shared_v2(uint32_t addr, uint2 v) {
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ uint2 ld_shared_v2(uint32_t addr) {
    uint2 v;
    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

// Operand expansion plan of one builder warp: warp w owns the 16-byte units
// (2 taps x 4 channels) j = w, w + 8, w + 16, w + 24 of all 128 tile pixels;
// lanes walk 32 consecutive pixels (row groups g = 0..3), so halo reads are
// consecutive 8-byte words and operand stores consecutive 16-byte units.
constexpr int kUnitsPerWarp = 4;  // nchunks <= 32
struct BuildPlan {
    int count;                                   // units owned by this warp
    int src0[kUnitsPerWarp], src1[kUnitsPerWarp];  // halo byte offset of tap 2j / 2j+1 (-1: none)
    uint32_t dst[kUnitsPerWarp];                 // operand byte offset of unit j (+ lane term)
    uint32_t row[4];                             // halo byte offset of pixel g*32 + lane
    uint32_t rowdst[4];                          // operand byte offset of pixel g*32 + lane
};

// MN_MAJOR = false: forward A[pixel][kc] no-swizzle K-major, [j][128 px][16 B]
// MN_MAJOR = true : wgrad  A[kc][pixel] SWIZZLE_128B MN-major, 64-kc atoms of
//                   128 px x 128 B (unit j = 16-byte chunk j%8 of atom j/8)
template <bool MN_MAJOR>
__device__ __forceinline__ void build_plan(const StemArgs& g, int wib, int lane, BuildPlan& bp) {
    bp.count = 0;
#pragma unroll
    for (int c = 0; c < kUnitsPerWarp; ++c) {
        const int j = wib + 8 * c;
        const int t0 = 2 * j, t1 = t0 + 1;
        bp.src0[c] = (j < g.nchunks && t0 < g.taps) ? g.tap_off[t0] * 8 : -1;
        bp.src1[c] = (j < g.nchunks && t1 < g.taps) ? g.tap_off[t1] * 8 : -1;
        if (MN_MAJOR)
            bp.dst[c] = (j >> 3) * (kTile * 128) + (((j & 7) ^ (lane & 7)) << 4);
        else
            bp.dst[c] = j * (kTile * 16);
        if (j < g.nchunks) bp.count = c + 1;
    }
#pragma unroll
    for (int gi = 0; gi < 4; ++gi) {
        const int m = gi * 32 + lane;
        bp.row[gi] = ((m / kBw) * g.sh * g.HWp + (m % kBw)) * 8;
        bp.rowdst[gi] = MN_MAJOR ? m * 128 : m * 16;
    }
}

// Branch-free expansion: taps past R*S read the zero word at the end of
// the halo stage, so each unit is 8 independent loads then 4 stores.
constexpr uint32_t kHaloZero = kHaloStageBytes - 8;

__device__ __forceinline__ void build_tile(const BuildPlan& bp, uint32_t a_base, uint32_t halo_u) {
#pragma unroll
    for (int c = 0; c < kUnitsPerWarp; ++c) {
        if (c >= bp.count) break;
        const int s0 = bp.src0[c], s1 = bp.src1[c];
        const uint32_t d = a_base + bp.dst[c];
        uint2 v[8];
#pragma unroll
        for (int gi = 0; gi < 4; ++gi) {
            const uint32_t a0 = halo_u + (s0 >= 0 ? bp.row[gi] + s0 : kHaloZero);
            const uint32_t a1 = halo_u + (s1 >= 0 ? bp.row[gi] + s1 : kHaloZero);
            v[2 * gi] = ld_shared_v2(a0);
            v[2 * gi + 1] = ld_shared_v2(a1);
        }
#pragma unroll
        for (int gi = 0; gi < 4; ++gi)
            st_shared_v4(d + bp.rowdst[gi],
                         make_uint4(v[2 * gi].x, v[2 * gi].y, v[2 * gi + 1].x, v[2 * gi + 1].y));
    }
}

// Zero the reserved last word of every halo stage (never written by cp.async).
__device__ __forceinline__ void halo_zero_words(uint32_t halo0, int b) {
    if (b < kHaloStages) st_shared_v2(halo0 + b * kHaloStageBytes + kHaloZero, make_uint2(0u, 0u));
}

// Halo byte offsets (relative to the pixel's row base) of the two taps of each
// unit this warp expands: units [u0, u0 + 16); invalid taps -> the zero word.
struct UnitOffsets {
    uint32_t o0[16], o1[16];
};
__device__ __forceinline__ void unit_offsets(const StemArgs& g, int u0, int u1, uint32_t rowoff,
                                             UnitOffsets& uo) {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        const int j = u0 + e, t0 = 2 * j, t1 = t0 + 1;
        uo.o0[e] = (j < u1 && t0 < g.taps) ? g.tap_off[t0] * 8 : kHaloZero - rowoff;
        uo.o1[e] = (j < u1 && t1 < g.taps) ? g.tap_off[t1] * 8 : kHaloZero - rowoff;
    }
}

// ---------------------------------------------------------------------------
// forward: A built straight into TENSOR MEMORY (tcgen05.st), MMA with A from
// TMEM and the resident packed filter from smem. Keeping the 53 KB/tile
// operand out of shared memory halves the smem traffic per tile (it was the
// bound: build writes + MMA reads of A competed with everything else).
//   warp 0: MMA issuer (+ TMEM owner), warps 1-4: epilogue, warps 5-12: builders
//   (builder warp w writes TMEM lane quarter w % 4; the two warps of a quarter
//   split the 16-byte units of their 32 pixels)
constexpr int kFwdThreads = 32 * 13;
constexpr int kMaxAStages = 4;

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// Issued by the whole (converged) warp; elect.sync picks the one issuing lane,
// so the compiler emits no per-instruction divergence loop around UTCHMMA.
__device__ __forceinline__ void mma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Four back-to-back MMAs (operands computed up front, one elect): keeps the
// per-instruction issue cost (descriptor math + R2UR moves) out of the chain.
__device__ __forceinline__ void mma4_bf16_ts(uint32_t tmem_d, uint32_t a0, uint32_t a1, uint32_t a2,
                                             uint32_t a3, uint64_t b0, uint64_t b1, uint64_t b2,
                                             uint64_t b3, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %10, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %5, %9, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %6, %9, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%3], %7, %9, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%4], %8, %9, 1;\n\t}" ::"r"(tmem_d),
        "r"(a0), "r"(a1), "r"(a2), "r"(a3), "l"(b0), "l"(b1), "l"(b2), "l"(b3), "r"(idesc),
        "r"(accumulate)
        : "memory");
}


// Two builder groups (4 warps each, one per TMEM lane quarter) alternate
// tiles, so two independent halo -> operand chains are in flight; each group
// streams its halos with 8-byte cp.async copies (zero fill = padding) into its
// own ring of compact, column-phase-split halo stages.
constexpr int kGroupThreads = 128;
constexpr int kGroupHaloStages = 3;
constexpr int kSlots = 8;  // halo pixels per group thread (<= 1024 per tile)

struct GroupHalo {
    int goff[kSlots];   // element offset of the slot's pixel from the halo origin
    int hrc[kSlots];    // (row << 16) | col, -1 = unused slot
    int word[kSlots];   // compact word index
};

__device__ __forceinline__ void group_halo_slots(const StemArgs& g, int b, GroupHalo& gh) {
#pragma unroll
    for (int u = 0; u < kSlots; ++u) {
        const int i = b + u * kGroupThreads;
        if (i < g.HH * g.HW) {
            const int hr = i / g.HW, hc = i - hr * g.HW;
            gh.goff[u] = (hr * g.W + hc) * g.x_pitch;
            gh.hrc[u] = (hr << 16) | hc;
            gh.word[u] = ((hc % g.sw) * g.HH + hr) * g.HWp + hc / g.sw;
        } else {
            gh.goff[u] = 0;
            gh.hrc[u] = -1;
            gh.word[u] = 0;
        }
    }
}

// Tile walker: (n, ty, tx) of tile t, advanced by a fixed tile stride without
// divisions.
struct TileWalk {
    int t, n, ty, tx, dn, dty, dtx, step;
    __device__ __forceinline__ void init(const StemArgs& g, int t0, int stride) {
        t = t0;
        step = stride;
        tx = t0 % g.tiles_w;
        ty = (t0 / g.tiles_w) % g.tiles_h;
        n = t0 / (g.tiles_w * g.tiles_h);
        dtx = stride % g.tiles_w;
        dty = (stride / g.tiles_w) % g.tiles_h;
        dn = stride / (g.tiles_w * g.tiles_h);
    }
    __device__ __forceinline__ void next(const StemArgs& g) {
        t += step;
        tx += dtx;
        if (tx >= g.tiles_w) {
            tx -= g.tiles_w;
            ++ty;
        }
        ty += dty;
        if (ty >= g.tiles_h) {
            ty -= g.tiles_h;
            ++n;
        }
        n += dn;
    }
};

__device__ __forceinline__ void group_halo_issue(const StemArgs& g, const __nv_bfloat16* __restrict__ x,
                                                 const TileWalk& tw, const GroupHalo& gh,
                                                 uint32_t dst_u) {
    if (tw.t < g.total_tiles) {
        const int iy0 = tw.ty * kBh * g.sh - g.ph, ix0 = tw.tx * kBw * g.sw - g.pw;
        const __nv_bfloat16* base = x + (((size_t)tw.n * g.H + iy0) * g.W + ix0) * g.x_pitch;
#pragma unroll
        for (int u = 0; u < kSlots; ++u) {
            if (gh.hrc[u] < 0) continue;
            const int iy = iy0 + (gh.hrc[u] >> 16), ix = ix0 + (gh.hrc[u] & 0xffff);
            const bool in = (unsigned)iy < (unsigned)g.H && (unsigned)ix < (unsigned)g.W;
            cp_async_8(dst_u + gh.word[u] * 8, in ? base + gh.goff[u] : x, in ? 8u : 0u);
        }
    }
    cp_async_commit();
}

// smem: resident filter (SW128 K-major), halo ring, epilogue staging, barriers
struct FwdLayout {
    int halo_off, stg_off, bar_off, bytes;
    __host__ __device__ FwdLayout(int nchunks, int np) {
        const int atoms = (nchunks + 7) / 8;
        halo_off = atoms * np * 128;
        stg_off = halo_off + 2 * kGroupHaloStages * kHaloStageBytes;
        bar_off = stg_off + 4 * 2 * 4096;  // 4 epilogue warps x 2 staging buffers
        bytes = bar_off + 256 + 1024;
    }
};

template <int NP>
__global__ void __launch_bounds__(kFwdThreads, 1)
    stem_fprop_kernel(const __grid_constant__ CUtensorMap ymap, const __nv_bfloat16* __restrict__ x,
                      const __nv_bfloat16* __restrict__ w, const __grid_constant__ StemArgs g,
                      const pk_epilogue epi) {
    pdl_wait();
    pdl_trigger();
    const FwdLayout L(g.nchunks, NP);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* empty = full + kMaxAStages;
    uint64_t* tmem_full = empty + kMaxAStages;
    uint64_t* tmem_empty = tmem_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
    const uint32_t halo0 = smem_u32(smem + L.halo_off);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // TMEM columns: [0, 2*NP) accumulators, then A stages of 4 columns per unit
    const int a_cols = (g.nchunks + 3) / 4 * 16;  // whole 4-unit (16-column) store groups
    int a_stages = (512 - 2 * NP) / a_cols;
    if (a_stages > kMaxAStages) a_stages = kMaxAStages;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kMaxAStages; ++i) {
            mbar_init(&full[i], 4);  // the 4 warps of one builder group
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 4);
        }
        fence_barrier_init();
        tma_prefetch(&ymap);
    }
    if (warp == 0) tmem_alloc(tmem_slot, 512);
    if (warp >= 5) {
        // packed filter B[n][kc] (unit j = taps 2j, 2j+1 x 4 channels), K-major
        // SWIZZLE_128B, resident for the whole kernel
        const int b = threadIdx.x - 5 * 32;
        const uint32_t bbase = smem_u32(smem);
        for (int i = b; i < g.nchunks * NP; i += kBuilders) {
            const int j = i / NP, n = i - j * NP;
            __align__(16) __nv_bfloat16 v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int t = 2 * j + (e >> 2), c = e & 3;
                v[e] = (n < g.K && t < g.taps && c < g.C)
                           ? w[((size_t)n * g.taps + t) * g.x_pitch + c]
                           : __float2bfloat16_rn(0.0f);
            }
            st_shared_v4(bbase + (uint32_t)((j >> 3) * NP * 128 + n * 128 + (((j & 7) ^ (n & 7)) << 4)),
                         *reinterpret_cast<const uint4*>(v));
        }
        if (b < 2 * kGroupHaloStages)
            st_shared_v2(halo0 + b * kHaloStageBytes + kHaloZero, make_uint2(0u, 0u));
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ---------------- MMA issuer: D[pix][k] += A_tmem[pix][kc] . B[k][kc] ----
        constexpr uint32_t idesc = idesc_bf16_f32(kTile, NP, false, false);
        const uint64_t bd0 = umma_desc_sw128(smem_u32(smem), 16, 1024);
        const int nk = (g.debug & 1) ? 0 : g.nchunks / 2;
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int t = blockIdx.x; t < g.total_tiles; t += gridDim.x, ++it) {
            const int a = it & 1;
            stamp(g, it, 0);
            mbar_wait(&tmem_empty[a], ((it >> 1) & 1) ^ 1);
            stamp(g, it, 1);
            mbar_wait(&full[stage], phase);
            stamp(g, it, 2);
            tc_fence_after();
            {
                const uint32_t ta = tmem_base + 2 * NP + stage * a_cols;
                const uint32_t td = tmem_base + a * NP;
                int k = 0;
                for (; k + 4 <= nk; k += 4) {  // K16 steps k..k+3 share one 64-wide B atom
                    const uint64_t bk = bd0 + (uint64_t)((k >> 2) * (NP * 128 / 16));
                    mma4_bf16_ts(td, ta + k * 8, ta + k * 8 + 8, ta + k * 8 + 16, ta + k * 8 + 24, bk,
                                 bk + 2, bk + 4, bk + 6, idesc, k != 0);
                }
                for (; k < nk; ++k)
                    mma_bf16_ts(td, ta + k * 8,
                                bd0 + (uint64_t)((k >> 2) * (NP * 128 / 16) + (k & 3) * 2), idesc,
                                k != 0);
                if (g.trace && blockIdx.x == 0 && it < 32 && lane == 0)
                    g.trace[it * 32 + 16] = clock64();
                mma_commit_elect(&empty[stage]);
                mma_commit_elect(&tmem_full[a]);
            }
            stamp(g, it, 3);
            __syncwarp();
            if (++stage == a_stages) {
                stage = 0;
                phase ^= 1;
            }
        }
    } else if (warp <= 4) {
        // ---------------- epilogue (4 warps, one TMEM lane quarter each) ---------
        const int q = warp & 3;
        uint8_t* stg_base = smem + L.stg_off + (warp - 1) * 2 * 4096;
        int sbuf = 0;
        const bool has_epi = epilogue_active(&epi);
        const int row = q * 32 + lane;
        const int rw = row % kBw, rh = row / kBw;
        BnStatAcc bacc;
        bacc.init();
        int it = 0;
        for (int t = blockIdx.x; t < g.total_tiles; t += gridDim.x, ++it) {
            int n, oy0, ox0;
            tile_origin(g, t, n, oy0, ox0);
            const int a = it & 1;
            if (warp == 1) stamp(g, it, 4);
            mbar_wait(&tmem_full[a], (it >> 1) & 1);
            if (warp == 1) stamp(g, it, 5);
            tc_fence_after();
#pragma unroll 1
            for (int c0 = 0; c0 < NP; c0 += 64) {
                uint32_t v[64];
                const uint32_t ta = tmem_base + a * NP + c0 + (static_cast<uint32_t>(q * 32) << 16);
                tmem_ld16(ta + 0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
                tmem_ld16(ta + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
                tmem_ld16(ta + 32, *reinterpret_cast<uint32_t(*)[16]>(&v[32]));
                tmem_ld16(ta + 48, *reinterpret_cast<uint32_t(*)[16]>(&v[48]));
                tmem_ld_wait();
                if (warp == 1) stamp(g, it, 6);
                if (c0 + 64 >= NP) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tmem_empty[a]);
                }
                const uint32_t stg_u = smem_u32(stg_base + sbuf * 4096);
                if (lane == 0) bulk_wait_read<1>();
                __syncwarp();
                float xf[64];
#pragma unroll
                for (int e = 0; e < 64; ++e) xf[e] = __uint_as_float(v[e]);
                if (has_epi) epilogue_chunk64(epi, xf, c0, g.K, oy0 + rh, ox0 + rw, g.P, g.Q);
#pragma unroll
                for (int jj = 0; jj < 8; ++jj) {
                    uint32_t packed[4];
#pragma unroll
                    for (int e = 0; e < 8; e += 2) {
                        __nv_bfloat162 b2 = __floats2bfloat162_rn(xf[jj * 8 + e], xf[jj * 8 + e + 1]);
                        packed[e / 2] = *reinterpret_cast<uint32_t*>(&b2);
                    }
                    st_shared_v4(stg_u + lane * 128 + ((jj ^ (lane & 7)) << 4),
                                 make_uint4(packed[0], packed[1], packed[2], packed[3]));
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0 && !(g.debug & 4)) {
                    // this warp's 32 rows = 2 output rows of the 16-wide rectangle
                    tma_store_4d(&ymap, stg_u, c0, ox0, oy0 + q * 2, n);
                    bulk_commit();
                }
                if (epi.stats)
                    bacc.add(epi, stg_u, lane, oy0 + rh < g.P && ox0 + rw < g.Q, 0, (c0 >> 6) & 1, c0,
                             g.K, g.K);
                if (warp == 1) stamp(g, it, 7);
                sbuf ^= 1;
            }
        }
        if (epi.stats) bacc.finish(epi, lane, g.K);
        if (lane == 0) bulk_wait_all();
    } else {
        // ---------------- builders: 2 groups, cp.async halo -> A rows in TMEM --------
        const int grp = (warp - 5) >> 2;                    // tiles i with i % 2 == grp
        const int gb = (warp - 5 - 4 * grp) * 32 + lane;    // thread index in the group
        const int q = warp & 3;                             // TMEM lane quarter
        const int m = q * 32 + lane;                        // tile pixel = TMEM lane
        const uint32_t rowoff = ((m / kBw) * g.sh * g.HWp + (m % kBw)) * 8;
        UnitOffsets uo0, uo1;  // units [0, 16) and [16, 32)
        unit_offsets(g, 0, g.nchunks, rowoff, uo0);
        unit_offsets(g, 16, g.nchunks, rowoff, uo1);
        GroupHalo gh;
        group_halo_slots(g, gb, gh);
        const uint32_t ring = halo0 + grp * kGroupHaloStages * kHaloStageBytes;
        TileWalk pf;  // prefetch walker: this group's tiles
        pf.init(g, blockIdx.x + grp * gridDim.x, 2 * gridDim.x);
        for (int s2 = 0; s2 < kGroupHaloStages - 1; ++s2) {
            group_halo_issue(g, x, pf, gh, ring + s2 * kHaloStageBytes);
            pf.next(g);
        }
        int k = 0;
        for (int i = grp, t = blockIdx.x + grp * gridDim.x; t < g.total_tiles;
             i += 2, t += 2 * gridDim.x, ++k) {
            if (warp == 5) stamp(g, i, 8);
            cp_async_wait<kGroupHaloStages - 2>();
            named_sync(1 + grp, kGroupThreads);  // halo k landed; this group's build k-1 done
            if (warp == 5) stamp(g, i, 9);
            group_halo_issue(g, x, pf, gh,
                             ring + ((k + kGroupHaloStages - 1) % kGroupHaloStages) * kHaloStageBytes);
            pf.next(g);
            const int stage = i % a_stages;
            mbar_wait(&empty[stage], ((i / a_stages) & 1) ^ 1);
            tc_fence_after();
            if (warp == 5) stamp(g, i, 11);
            if (!(g.debug & 2)) {
                const uint32_t hbase = ring + (k % kGroupHaloStages) * kHaloStageBytes + rowoff;
                const uint32_t ta = tmem_base + 2 * NP + stage * a_cols + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll
                for (int g4 = 0; g4 < 8; ++g4) {
                    if (4 * g4 >= g.nchunks) break;
                    uint32_t v[16];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int u = 4 * g4 + e;
                        const uint32_t o0 = u < 16 ? uo0.o0[u] : uo1.o0[u - 16];
                        const uint32_t o1 = u < 16 ? uo0.o1[u] : uo1.o1[u - 16];
                        const uint2 lo = ld_shared_v2(hbase + o0);
                        const uint2 hi = ld_shared_v2(hbase + o1);
                        v[4 * e + 0] = lo.x;
                        v[4 * e + 1] = lo.y;
                        v[4 * e + 2] = hi.x;
                        v[4 * e + 3] = hi.y;
                    }
                    tmem_st16(ta + 16 * g4, v);
                }
                tmem_st_wait();
            }
            tc_fence_before();
            __syncwarp();
            if (warp == 5) stamp(g, i, 12);
            if (lane == 0) mbar_arrive(&full[stage]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

// ---------------------------------------------------------------------------
// backward weights
//   warp 0: MMA issuer, warps 1-4: final TMEM drain, warps 5-12: builders
//   (builder warp 5 lane 0 also issues the dY TMA loads)
constexpr int kWgThreads = 32 * 13;

template <int NP>
struct WgSmem {
    static constexpr int kAtom = kTile * 128;               // 64 kc x 128 pixels
    static constexpr int kA = 4 * kAtom;                     // kc rows up to 256
    static constexpr int kB = (NP / 64) * kAtom;             // dY: NP channels x 128 pixels
    static constexpr int kStage = kA + kB;
    static constexpr int kStages = 2;
    static constexpr int kHaloOff = kStages * kStage;
    static constexpr int kBarOff = kHaloOff + kHaloStages * kHaloStageBytes;
    static constexpr int kBytes = kBarOff + 128 + 1024;
};

template <int NP>
__global__ void __launch_bounds__(kWgThreads, 1)
    stem_wgrad_kernel(const __grid_constant__ CUtensorMap dymap, const __nv_bfloat16* __restrict__ x,
                      float* __restrict__ partial, const __grid_constant__ StemArgs g) {
    pdl_wait();
    pdl_trigger();
    using L = WgSmem<NP>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* empty = full + L::kStages;
    uint64_t* done = empty + L::kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    const uint32_t halo0 = smem_u32(smem + L::kHaloOff);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mtiles = g.kcm / 128;
    constexpr uint32_t kColsNeed = 2 * NP;  // up to 2 M tiles (kc <= 256)
    constexpr uint32_t kCols = kColsNeed <= 32 ? 32 : kColsNeed <= 64 ? 64 : kColsNeed <= 128 ? 128
                               : kColsNeed <= 256 ? 256 : 512;

    if (threadIdx.x == 0) {
        for (int i = 0; i < L::kStages; ++i) {
            mbar_init(&full[i], kBuilders / 32 + 1);  // 8 builder warps + the TMA arrival
            mbar_init(&empty[i], 1);
        }
        mbar_init(done, 1);
        fence_barrier_init();
        tma_prefetch(&dymap);
    }
    if (warp == 0) tmem_alloc(tmem_slot, kCols);
    if (warp >= 5) {
        // kc rows beyond 8*nchunks stay zero in every stage
        const int b = threadIdx.x - 5 * 32;
        for (int s = 0; s < L::kStages; ++s) {
            const uint32_t a_base = smem_u32(smem + s * L::kStage);
            for (int i = b; i < (4 * 8 - g.nchunks) * kTile; i += kBuilders) {
                const int j = g.nchunks + i / kTile, p = i % kTile;
                st_shared_v4(a_base + (j >> 3) * L::kAtom + p * 128 + (((j & 7) ^ (p & 7)) << 4),
                             make_uint4(0u, 0u, 0u, 0u));
            }
        }
        halo_zero_words(halo0, b);
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int my_tiles = blockIdx.x < g.total_tiles
                             ? (g.total_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

    if (warp == 0) {
        // ---------------- MMA issuer: D[kc][k] += A[kc][pix] . dY[k][pix] ---------
        constexpr uint32_t idesc = idesc_bf16_f32(kTile, NP, true, true);
        int stage = 0;
        uint32_t phase = 0;
        for (int i = 0; i < my_tiles; ++i) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            {
                const uint32_t a_base = smem_u32(smem + stage * L::kStage);
                const uint32_t b_base = a_base + L::kA;
                constexpr uint64_t ks = 2048 >> 4;  // 16 MN-major K rows (pixels)
                const uint64_t bd0 = umma_desc_sw128(b_base, L::kAtom, 1024);
                for (int mt = 0; mt < ((g.debug & 1) ? 0 : mtiles); ++mt) {  // PK_STEM_DEBUG=1: no MMA
                    const uint64_t ad0 = umma_desc_sw128(a_base + mt * 2 * L::kAtom, L::kAtom, 1024);
#pragma unroll
                    for (int k = 0; k < kTile / 16; k += 4)
                        mma4_bf16(tmem_base + mt * NP, ad0 + k * ks, ad0 + (k + 1) * ks,
                                  ad0 + (k + 2) * ks, ad0 + (k + 3) * ks, bd0 + k * ks,
                                  bd0 + (k + 1) * ks, bd0 + (k + 2) * ks, bd0 + (k + 3) * ks, idesc,
                                  (i | k) != 0);
                }
                mma_commit_elect(&empty[stage]);
                if (i == my_tiles - 1) mma_commit_elect(done);
            }
            if (++stage == L::kStages) {
                stage = 0;
                phase ^= 1;
            }
        }
    } else if (warp <= 4) {
        // ---------------- drain: partial[cta][k][kc] ------------------------------
        const int q = warp & 3;
        if (my_tiles > 0) {
            mbar_wait(done, 0);
            tc_fence_after();
        }
        for (int mt = 0; mt < mtiles; ++mt) {
            const int kc = mt * 128 + q * 32 + lane;
#pragma unroll 1
            for (int c0 = 0; c0 < NP; c0 += 16) {
                uint32_t v[16];
                if (my_tiles > 0) {
                    tmem_ld16(tmem_base + mt * NP + c0 + (static_cast<uint32_t>(q * 32) << 16), v);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = 0u;
                }
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    if (c0 + e < g.K)
                        partial[((size_t)blockIdx.x * g.K + c0 + e) * g.kcm + kc] =
                            __uint_as_float(v[e]);
            }
        }
    } else {
        // ---------------- builders: A[kc][pix] (MN-major, 128B swizzle) + dY TMA ---
        const int b = threadIdx.x - 5 * 32;
        HaloSlots hs;
        halo_slots(g, b, hs);
        BuildPlan bp;
        build_plan<true>(g, warp - 5, lane, bp);
        for (int i = 0; i < kHaloStages - 1; ++i)
            halo_issue(g, x, blockIdx.x + i * gridDim.x, hs, halo0 + i * kHaloStageBytes);
        int stage = 0;
        uint32_t phase = 0;
        int i = 0;
        for (int t = blockIdx.x; t < g.total_tiles; t += gridDim.x, ++i) {
            cp_async_wait<kHaloStages - 2>();
            named_sync(1, kBuilders);
            halo_issue(g, x, t + (kHaloStages - 1) * gridDim.x, hs,
                       halo0 + ((i + kHaloStages - 1) % kHaloStages) * kHaloStageBytes);
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sbase = smem + stage * L::kStage;
            if (b == 0) {
                int n, oy0, ox0;
                tile_origin(g, t, n, oy0, ox0);
                mbar_arrive_expect_tx(&full[stage], L::kB);
#pragma unroll
                for (int a = 0; a < NP / 64; ++a)
                    tma_load_4d(smem_u32(sbase + L::kA + a * L::kAtom), &dymap, &full[stage], a * 64,
                                ox0, oy0, n);
            }
            if (!(g.debug & 2))  // PK_STEM_DEBUG=2 (timing only): no operand build
                build_tile(bp, smem_u32(sbase), halo0 + (i % kHaloStages) * kHaloStageBytes);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[stage]);
            if (++stage == L::kStages) {
                stage = 0;
                phase ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kCols);
    }
}

// dw[k][r][s][c] = sum over CTAs of partial[cta][k][tap*4 + c]: one WARP per
// output element (lane l sums CTAs l, l + 32, ... in order, then a fixed xor
// tree), so the ~148 partial loads of an element are in flight together
// (one thread per element walked them serially: 28 us, latency-bound).
// Deterministic: the order depends on nothing but the CTA count.
__global__ void stem_wgrad_finish_kernel(const float* __restrict__ partial, int ctas, int K,
                                         int kcm, int taps, int f_pitch, int C,
                                         __nv_bfloat16* __restrict__ dw) {
    pdl_wait();
    pdl_trigger();
    const long long total = (long long)K * taps * f_pitch;
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * blockDim.x / 32;
    for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32; i < total; i += warps) {
        const int c = (int)(i % f_pitch);
        const long long kt = i / f_pitch;
        const int tap = (int)(kt % taps), k = (int)(kt / taps);
        float acc = 0.0f;
        if (c < C) {  // warp-uniform
            const float* p = partial + (size_t)k * kcm + tap * 4 + c;
#pragma unroll 4
            for (int s = lane; s < ctas; s += 32) acc += __ldcg(p + (size_t)s * K * kcm);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        }
        if (lane == 0) dw[i] = __float2bfloat16_rn(acc);
    }
}

// ---------------------------------------------------------------------------
// backward data (gather formulation, deterministic, no column matrix in HBM)
//
// A CTA owns a TY x TX rectangle of dX. The dY pixels whose taps reach it form
// an HY x WX halo (11 x 19 for conv1 at 16 x 32), loaded by one TMA box as the
// K-major A operand (K = the 64 dY channels). Two M=128 MMAs against the
// resident packed filter B[kc][k] (kc = tap*4 + c) give the column block
// colg[dY pixel][tap, c] in TMEM; 4 warps drain it to shared memory (fp32,
// compact tap*C + c, odd row stride: conflict-free), then 8 warps gather each
// dX pixel's taps (only those whose stride phase matches) and store 16-byte
// pixels. MMA of the next tile overlaps the gather.
//   warp 0: TMA producer + MMA issuer; warps 1-8: drain (1-4) + gather (1-8)
constexpr int kDgThreads = 32 * 9;

struct DgArgs {
    int N, H, W, x_pitch, P, Q, K;
    int R, S, sh, sw, dh, dw, ph, pw, C, taps;
    int TY, TX, HY, WX;         // dX tile, dY halo box
    int oy_lo0, ox_lo0;         // halo origin for tile (0, 0): oy_lo(Y0) = Y0/sh + oy_lo0
    int tiles_w, tiles_h, total_tiles;
    int npad;                   // MMA N = roundup(taps*4, 16)
    int cstride;                // colg row stride (words, odd)
    int v2;                     // 1: pipelined kernel (halo <= one M tile)
    int v3;                     // 1: row-strip kernel (ResNet conv1 geometry)
    int debug;                  // PK_STEM_DEBUG (v2, profiling only): 1 no MMA, 2 no drain, 4 no gather
    unsigned long long* trace;  // PK_STEM_TRACE (profiling only)
};
__device__ __forceinline__ void dstamp(const DgArgs& g, int it, int ev) {
    if (g.trace && blockIdx.x == 0 && it < 32 && (threadIdx.x & 31) == 0)
        g.trace[it * 32 + ev] = clock64();
}

struct DgLayout {
    int a_stage, b_off, colg_off, bar_off, bytes;
    __host__ __device__ DgLayout(const DgArgs& g) {
        a_stage = 2 * kTile * 128;                 // 2 M tiles of 128 halo pixels x 64 ch
        b_off = 2 * a_stage;                        // double-buffered A
        colg_off = b_off + g.npad * 128;
        bar_off = colg_off + (g.HY * g.WX * g.cstride * 4 + 1023) / 1024 * 1024;
        bytes = bar_off + 128 + 1024;
    }
};

__device__ __forceinline__ void st_shared_f32(uint32_t addr, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ float ld_shared_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ void dg_tile(const DgArgs& g, int t, int& n, int& Y0, int& X0) {
    const int tx = t % g.tiles_w, rest = t / g.tiles_w;
    Y0 = (rest % g.tiles_h) * g.TY;
    n = rest / g.tiles_h;
    X0 = tx * g.TX;
}

// C: input channels (<= 4); KR/KS/KSH/KSW: compile-time filter size and
// stride (0 = runtime values from g) so the ResNet conv1 gather unrolls.
template <int C, int KR, int KS, int KSH, int KSW>
__global__ void __launch_bounds__(kDgThreads, 1)
    stem_dgrad_kernel(const __grid_constant__ CUtensorMap dymap, const __nv_bfloat16* __restrict__ w,
                      __nv_bfloat16* __restrict__ dx, const __grid_constant__ DgArgs g) {
    pdl_wait();
    pdl_trigger();
    const DgLayout L(g);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* a_full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* a_empty = a_full + 2;
    uint64_t* tmem_full = a_empty + 2;
    uint64_t* tmem_empty = tmem_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);
    const uint32_t colg_u = smem_u32(smem + L.colg_off);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], 1);
        }
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, 4);
        fence_barrier_init();
        tma_prefetch(&dymap);
    }
    if (warp == 0) tmem_alloc(tmem_slot, 512);
    // packed filter B[kc][k] (kc = tap*4 + c, K-major SWIZZLE_128B, 64 k = one atom)
    for (int i = threadIdx.x; i < g.npad * 8; i += blockDim.x) {
        const int kc = i >> 3, j = i & 7;  // 16-byte unit j = k 8j..8j+7
        const int tap = kc >> 2, c = kc & 3;
        __align__(16) __nv_bfloat16 v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int k = j * 8 + e;
            v[e] = (tap < g.taps && c < g.C && k < g.K)
                       ? w[((size_t)k * g.taps + tap) * g.x_pitch + c]
                       : __float2bfloat16_rn(0.0f);
        }
        st_shared_v4(smem_u32(smem + L.b_off) + kc * 128 + ((j ^ (kc & 7)) << 4),
                     *reinterpret_cast<const uint4*>(v));
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer + MMA issuer --------------------------------
        constexpr int kBoxBytes = 0;  // (unused)
        (void)kBoxBytes;
        const uint32_t box_bytes = g.HY * g.WX * 128;
        const uint32_t idesc = idesc_bf16_f32(kTile, g.npad, false, false);
        const uint64_t bd0 = umma_desc_sw128(smem_u32(smem + L.b_off), 16, 1024);
        auto load = [&](int tt, int buf) {
            int n, Y0, X0;
            dg_tile(g, tt, n, Y0, X0);
            if (lane == 0) {
                mbar_arrive_expect_tx(&a_full[buf], box_bytes);
                tma_load_4d(smem_u32(smem + buf * L.a_stage), &dymap, &a_full[buf], 0,
                            X0 / g.sw + g.ox_lo0, Y0 / g.sh + g.oy_lo0, n);
            }
        };
        if (blockIdx.x < g.total_tiles) load(blockIdx.x, 0);
        int i = 0;
        for (int t = blockIdx.x; t < g.total_tiles; t += gridDim.x, ++i) {
            const int buf = i & 1;
            // prefetch tile i+1 once the MMA of tile i-1 released its buffer
            if (t + (int)gridDim.x < g.total_tiles) {
                if (i >= 1) mbar_wait(&a_empty[buf ^ 1], ((i - 1) >> 1) & 1);
                load(t + gridDim.x, buf ^ 1);
            }
            dstamp(g, i, 0);
            mbar_wait(&a_full[buf], (i >> 1) & 1);
            dstamp(g, i, 1);
            mbar_wait(tmem_empty, (i & 1) ^ 1);
            dstamp(g, i, 2);
            tc_fence_after();
            const uint64_t ad0 = umma_desc_sw128(smem_u32(smem + buf * L.a_stage), 16, 1024);
            for (int mt = 0; mt * kTile < g.HY * g.WX; ++mt) {
                const uint64_t am = ad0 + (uint64_t)(mt * (kTile * 128 / 16));
                mma4_bf16(tmem_base + mt * g.npad, am, am + 2, am + 4, am + 6, bd0, bd0 + 2, bd0 + 4,
                          bd0 + 6, idesc, 0);
            }
            mma_commit_elect(&a_empty[buf]);
            mma_commit_elect(tmem_full);
            dstamp(g, i, 3);
            __syncwarp();
        }
    } else {
        // ---------------- drain (warps 1-4) + gather (warps 1-8) -------------------
        const int rows = g.HY * g.WX;
        const int gt = threadIdx.x - 32;  // 0..255
        int i = 0;
        for (int t = blockIdx.x; t < g.total_tiles; t += gridDim.x, ++i) {
            int n, Y0, X0;
            dg_tile(g, t, n, Y0, X0);
            {
                // 8 drain warps: lane quarter q = warp % 4, column chunks split in two
                const int q = warp & 3, half = (warp - 1) >> 2;
                const int nch = g.npad / 16, ch0 = half ? (nch + 1) / 2 : 0,
                          ch1 = half ? nch : (nch + 1) / 2;
                if (warp == 1) dstamp(g, i, 4);
                mbar_wait(tmem_full, i & 1);
                if (warp == 1) dstamp(g, i, 5);
                tc_fence_after();
                // colg rows hold all npad/4 taps (the padding taps are never read),
                // so every chunk stores 4 taps x C values at immediate offsets
                for (int mt = 0; mt * kTile < rows; ++mt) {
                    const int row = mt * kTile + q * 32 + lane;
                    const uint32_t dst = colg_u + row * g.cstride * 4;
                    const bool live = row < rows;
                    int cb = ch0;
#pragma unroll 1
                    for (; cb + 2 <= ch1; cb += 2) {
                        uint32_t v[32];
                        const uint32_t ta = tmem_base + mt * g.npad + cb * 16 +
                                            (static_cast<uint32_t>(q * 32) << 16);
                        tmem_ld16(ta, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
                        tmem_ld16(ta + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
                        tmem_ld_wait();
                        if (live) {
                            const uint32_t d = dst + cb * 4 * C * 4;
#pragma unroll
                            for (int e = 0; e < 32; ++e)
                                if ((e & 3) < C) st_shared_f32(d + ((e >> 2) * C + (e & 3)) * 4, __uint_as_float(v[e]));
                        }
                    }
                    if (cb < ch1) {
                        uint32_t v[16];
                        tmem_ld16(tmem_base + mt * g.npad + cb * 16 + (static_cast<uint32_t>(q * 32) << 16), v);
                        tmem_ld_wait();
                        if (live) {
                            const uint32_t d = dst + cb * 4 * C * 4;
#pragma unroll
                            for (int e = 0; e < 16; ++e)
                                if ((e & 3) < C) st_shared_f32(d + ((e >> 2) * C + (e & 3)) * 4, __uint_as_float(v[e]));
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0 && warp <= 4) {
                    // tmem_empty counts 4 arrivals: one per quarter pair after both drained
                }
            }
            if (warp == 1) dstamp(g, i, 6);
            named_sync(1, 256);  // colg of tile i complete (all TMEM reads done too)
            if (warp == 1) dstamp(g, i, 7);
            if (warp <= 4 && lane == 0) mbar_arrive(tmem_empty);
            const int oy_lo = Y0 / g.sh + g.oy_lo0, ox_lo = X0 / g.sw + g.ox_lo0;
            const int TX = g.TX, npx = g.TY * TX;
            const int sh = KSH ? KSH : g.sh, sw = KSW ? KSW : g.sw, R = KR ? KR : g.R,
                      S = KS ? KS : g.S;
            const int WX = g.WX, cs4 = g.cstride * 4;
            for (int px = gt; px < npx; px += 256) {
                const int iy = Y0 + px / TX, ix = X0 + px % TX;
                if (iy >= g.H || ix >= g.W) continue;
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
                // taps reaching (iy, ix): r = r0, r0 + sh, ... (dil 1) with dY row
                // (iy + ph - r) / sh, i.e. one halo row up per step; dY outside the
                // image is zero in the halo box, so no bounds checks
                const int r0 = (iy + g.ph) % sh, s0 = (ix + g.pw) % sw;
                const int lr = (iy + g.ph - r0) / sh - oy_lo, lc = (ix + g.pw - s0) / sw - ox_lo;
                uint32_t rowa = colg_u + (lr * WX + lc) * cs4 + (r0 * S + s0) * C * 4;
                if (KR) {
                    // compile-time geometry: fixed trip counts, predicated tail taps
                    constexpr int NR = KR ? (KR + KSH - 1) / KSH : 1, NS = KS ? (KS + KSW - 1) / KSW : 1;
#pragma unroll
                    for (int ri = 0; ri < NR; ++ri) {
                        const bool rok = r0 + ri * KSH < KR;
#pragma unroll
                        for (int si = 0; si < NS; ++si) {
                            const bool ok = rok && s0 + si * KSW < KS;
                            const uint32_t a = rowa + ri * (KSH * KS * C * 4 - WX * cs4) +
                                               si * (KSW * C * 4 - cs4);
#pragma unroll
                            for (int c = 0; c < C; ++c)
                                if (ok) acc[c] += ld_shared_f32(a + c * 4);
                        }
                    }
                } else {
                    for (int r = r0; r < R; r += sh) {
                        uint32_t a = rowa;
                        for (int s = s0; s < S; s += sw) {
#pragma unroll
                            for (int c = 0; c < C; ++c) acc[c] += ld_shared_f32(a + c * 4);
                            a += sw * C * 4 - cs4;  // next tap in the row: one halo pixel left
                        }
                        rowa += sh * S * C * 4 - WX * cs4;  // next tap row: one halo row up
                    }
                }
                __align__(16) __nv_bfloat16 o[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) o[c] = __float2bfloat16_rn(c < 4 ? acc[c & 3] : 0.0f);
                *reinterpret_cast<uint4*>(dx + (((size_t)n * g.H + iy) * g.W + ix) * g.x_pitch) =
                    *reinterpret_cast<const uint4*>(o);
            }
            if (warp == 1) dstamp(g, i, 8);
            named_sync(1, 256);  // colg free for tile i+1
            if (warp == 1) dstamp(g, i, 9);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

// ---------------------------------------------------------------------------
// backward data, pipelined (v2): the halo of a tile fits one M=128 MMA, so the
// TMEM accumulator and the colg buffer are both double-buffered and the three
// stages run on separate warps, overlapping tile by tile:
//   warp 0     dY halo TMA (one tile ahead) + MMA issue into TMEM[buf]
//   warps 1-8  drain TMEM[buf] (lane quarter = warp % 4, column halves split
//              between the two warps of a quarter) -> colg[buf] (fp32)
//   warps 9-16 gather colg[buf] -> dX (each dX pixel sums its taps; bf16 store)
constexpr int kDg2Threads = 32 * 17;
constexpr int kDg2Stages = 3;    // dY halo ring: two tiles of TMA latency in flight
constexpr int kDg2Prefetch = 0;  // L2 prefetch distance beyond the ring (measured: no gain)

struct Dg2Layout {
    int a_stage, b_off, colg_off, colg_bytes, bar_off, bytes;
    __host__ __device__ Dg2Layout(const DgArgs& g) {
        a_stage = kTile * 128;                      // 128 halo pixels x 64 dY channels
        b_off = kDg2Stages * a_stage;
        colg_off = b_off + (g.npad * 128 + 1023) / 1024 * 1024;
        colg_bytes = (g.HY * g.WX * g.cstride * 4 + 127) / 128 * 128;
        bar_off = colg_off + 2 * colg_bytes;
        bytes = bar_off + 128 + 1024;
    }
};

template <int C, int KR, int KS, int KSH, int KSW>
__global__ void __launch_bounds__(kDg2Threads, 1)
    stem_dgrad2_kernel(const __grid_constant__ CUtensorMap dymap, const __nv_bfloat16* __restrict__ w,
                       __nv_bfloat16* __restrict__ dx, const __grid_constant__ DgArgs g) {
    pdl_wait();
    pdl_trigger();
    const Dg2Layout L(g);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* a_full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* a_empty = a_full + kDg2Stages;
    uint64_t* tmem_full = a_empty + kDg2Stages;
    uint64_t* tmem_empty = tmem_full + 2;
    uint64_t* colg_full = tmem_empty + 2;
    uint64_t* colg_empty = colg_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(colg_empty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kDg2Stages; ++i) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 8);
            mbar_init(&colg_full[i], 256);
            mbar_init(&colg_empty[i], 256);
        }
        fence_barrier_init();
        tma_prefetch(&dymap);
    }
    if (warp == 0) tmem_alloc(tmem_slot, 512);
    // packed filter B[kc][k] (kc = tap*C + c dense, K-major SWIZZLE_128B, 64 k = one atom):
    // the accumulator row of a halo pixel is then exactly its colg row
    for (int i = threadIdx.x; i < g.npad * 8; i += blockDim.x) {
        const int kc = i >> 3, j = i & 7;
        const int tap = kc / C, c = kc - tap * C;
        __align__(16) __nv_bfloat16 v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int k = j * 8 + e;
            v[e] = (tap < g.taps && c < g.C && k < g.K)
                       ? w[((size_t)k * g.taps + tap) * g.x_pitch + c]
                       : __float2bfloat16_rn(0.0f);
        }
        st_shared_v4(smem_u32(smem + L.b_off) + kc * 128 + ((j ^ (kc & 7)) << 4),
                     *reinterpret_cast<const uint4*>(v));
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ---------------- TMA producer + MMA issuer --------------------------------
        const uint32_t box_bytes = g.HY * g.WX * 128;
        const uint32_t idesc = idesc_bf16_f32(kTile, g.npad, false, false);
        const uint64_t bd0 = umma_desc_sw128(smem_u32(smem + L.b_off), 16, 1024);
        auto load = [&](int tt, int buf) {
            int n, Y0, X0;
            dg_tile(g, tt, n, Y0, X0);
            if (lane == 0) {
                mbar_arrive_expect_tx(&a_full[buf], box_bytes);
                tma_load_4d(smem_u32(smem + buf * L.a_stage), &dymap, &a_full[buf], 0,
                            X0 / g.sw + g.ox_lo0, Y0 / g.sh + g.oy_lo0, n);
            }
        };
        auto prefetch = [&](int tt) {
            int n, Y0, X0;
            dg_tile(g, tt, n, Y0, X0);
            if (lane == 0)
                tma_prefetch_4d(&dymap, 0, X0 / g.sw + g.ox_lo0, Y0 / g.sh + g.oy_lo0, n);
        };
        // L2 prefetch runs kDg2Prefetch tiles ahead of the smem loads
        for (int j = kDg2Stages - 1; j < kDg2Stages - 1 + kDg2Prefetch; ++j)
            if ((int)blockIdx.x + j * (int)gridDim.x < g.total_tiles) prefetch(blockIdx.x + j * gridDim.x);
        (void)prefetch;
        // ring of kDg2Stages halo buffers: tile j uses stage j % S (use count j / S)
        for (int j = 0; j < kDg2Stages - 1; ++j)
            if ((int)blockIdx.x + j * (int)gridDim.x < g.total_tiles)
                load(blockIdx.x + j * gridDim.x, j);
        int i = 0;
        for (int t = blockIdx.x; t < g.total_tiles; t += gridDim.x, ++i) {
            const int buf = i & 1;
            const uint32_t ph = (i >> 1) & 1;
            const int jn = i + kDg2Stages - 1;  // tile to prefetch now
            if (t + (kDg2Stages - 1) * (int)gridDim.x < g.total_tiles) {
                if (jn >= kDg2Stages) mbar_wait(&a_empty[jn % kDg2Stages], ((jn / kDg2Stages) - 1) & 1);
                load(t + (kDg2Stages - 1) * gridDim.x, jn % kDg2Stages);
            }
            if (kDg2Prefetch && t + (kDg2Stages - 1 + kDg2Prefetch) * (int)gridDim.x < g.total_tiles)
                prefetch(t + (kDg2Stages - 1 + kDg2Prefetch) * gridDim.x);
            const int as = i % kDg2Stages;
            mbar_wait(&a_full[as], (i / kDg2Stages) & 1);
            mbar_wait(&tmem_empty[buf], ph ^ 1);
            tc_fence_after();
            const uint64_t ad0 = umma_desc_sw128(smem_u32(smem + as * L.a_stage), 16, 1024);
            if (!(g.debug & 1))
                mma4_bf16(tmem_base + buf * 256, ad0, ad0 + 2, ad0 + 4, ad0 + 6, bd0, bd0 + 2,
                          bd0 + 4, bd0 + 6, idesc, 0);
            mma_commit_elect(&a_empty[as]);
            mma_commit_elect(&tmem_full[buf]);
            __syncwarp();
        }
    } else if (warp <= 8) {
        // ---------------- drain: TMEM[buf] -> colg[buf] ----------------------------
        const int q = warp & 3, half = (warp - 1) >> 2;
        const int rows = g.HY * g.WX;
        const int row = q * 32 + lane;
        const int nall = g.npad / 16, nh = ((nall + 1) / 2 + 1) & ~1;  // even split point
        const int cb0 = half ? nh : 0, nch = half ? nall : (nh < nall ? nh : nall);
        int i = 0;
        for (int t = blockIdx.x; t < g.total_tiles; t += gridDim.x, ++i) {
            const int buf = i & 1;
            const uint32_t ph = (i >> 1) & 1;
            mbar_wait(&tmem_full[buf], ph);
            tc_fence_after();
            mbar_wait(&colg_empty[buf], ph ^ 1);
            const uint32_t dst = smem_u32(smem + L.colg_off + buf * L.colg_bytes) + row * g.cstride * 4;
            const bool live = row < rows && !(g.debug & 2);
            const uint32_t ta0 = tmem_base + buf * 256 + (static_cast<uint32_t>(q * 32) << 16);
            int cb = cb0;
#pragma unroll 1
            for (; cb + 2 <= nch; cb += 2) {
                uint32_t v[32];
                tmem_ld16(ta0 + cb * 16, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
                tmem_ld16(ta0 + cb * 16 + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
                tmem_ld_wait();
                if (live) {
#pragma unroll
                    for (int q4 = 0; q4 < 8; ++q4)
                        if (cb * 16 + q4 * 4 < g.cstride)
                            st_shared_v4(dst + (cb * 16 + q4 * 4) * 4,
                                         make_uint4(v[q4 * 4], v[q4 * 4 + 1], v[q4 * 4 + 2], v[q4 * 4 + 3]));
                }
            }
            if (cb < nch) {
                uint32_t v[16];
                tmem_ld16(ta0 + cb * 16, v);
                tmem_ld_wait();
                if (live) {
#pragma unroll
                    for (int q4 = 0; q4 < 4; ++q4)
                        if (cb * 16 + q4 * 4 < g.cstride)
                            st_shared_v4(dst + (cb * 16 + q4 * 4) * 4,
                                         make_uint4(v[q4 * 4], v[q4 * 4 + 1], v[q4 * 4 + 2], v[q4 * 4 + 3]));
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tmem_empty[buf]);
            mbar_arrive(&colg_full[buf]);
        }
    } else {
        // ---------------- gather: colg[buf] -> dX ---------------------------------
        const int gt = threadIdx.x - 288;  // 0..255
        const int sh = KSH ? KSH : g.sh, sw = KSW ? KSW : g.sw, R = KR ? KR : g.R,
                  S = KS ? KS : g.S;
        const int WX = g.WX, cs4 = g.cstride * 4, TX = g.TX, npx = g.TY * g.TX;
        int i = 0;
        for (int t = blockIdx.x; t < g.total_tiles; t += gridDim.x, ++i) {
            const int buf = i & 1;
            const uint32_t ph = (i >> 1) & 1;
            int n, Y0, X0;
            dg_tile(g, t, n, Y0, X0);
            const int oy_lo = Y0 / g.sh + g.oy_lo0, ox_lo = X0 / g.sw + g.ox_lo0;
            const uint32_t colg_u = smem_u32(smem + L.colg_off + buf * L.colg_bytes);
            mbar_wait(&colg_full[buf], ph);
            for (int px = gt; px < (g.debug & 4 ? 0 : npx); px += 256) {
                const int iy = Y0 + px / TX, ix = X0 + px % TX;
                if (iy >= g.H || ix >= g.W) continue;
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
                const int r0 = (iy + g.ph) % sh, s0 = (ix + g.pw) % sw;
                const int lr = (iy + g.ph - r0) / sh - oy_lo, lc = (ix + g.pw - s0) / sw - ox_lo;
                uint32_t rowa = colg_u + (lr * WX + lc) * cs4 + (r0 * S + s0) * C * 4;
                if (KR) {
                    constexpr int NR = KR ? (KR + KSH - 1) / KSH : 1, NS = KS ? (KS + KSW - 1) / KSW : 1;
#pragma unroll
                    for (int ri = 0; ri < NR; ++ri) {
                        const bool rok = r0 + ri * KSH < KR;
#pragma unroll
                        for (int si = 0; si < NS; ++si) {
                            const bool ok = rok && s0 + si * KSW < KS;
                            const uint32_t a = rowa + ri * (KSH * KS * C * 4 - WX * cs4) +
                                               si * (KSW * C * 4 - cs4);
#pragma unroll
                            for (int c = 0; c < C; ++c)
                                if (ok) acc[c] += ld_shared_f32(a + c * 4);
                        }
                    }
                } else {
                    for (int r = r0; r < R; r += sh) {
                        uint32_t a = rowa;
                        for (int s2 = s0; s2 < S; s2 += sw) {
#pragma unroll
                            for (int c = 0; c < C; ++c) acc[c] += ld_shared_f32(a + c * 4);
                            a += sw * C * 4 - cs4;
                        }
                        rowa += sh * S * C * 4 - WX * cs4;
                    }
                }
                __align__(16) __nv_bfloat16 o[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) o[c] = __float2bfloat16_rn(c < 4 ? acc[c & 3] : 0.0f);
                *reinterpret_cast<uint4*>(dx + (((size_t)n * g.H + iy) * g.W + ix) * g.x_pitch) =
                    *reinterpret_cast<const uint4*>(o);
            }
            mbar_arrive(&colg_empty[buf]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

// ---------------------------------------------------------------------------
// forward v2 ("row strips"), ResNet conv1 geometry: 7x7, stride 2, pad 3,
// K = 64, Q <= 128. One output row p is ONE GEMM over the seven input rows
// 2p-3 .. 2p+3 it reads: TMEM lane = output column q, and with the input row
// stored as 8-byte pixels (4 channels) the 16-byte unit t of lane q — input
// pixels 2q-3+2t, 2q-2+2t — sits at byte 16q + 16t of the row. So the A operand of
// (input row, K step m) is the row itself read as a K-major no-swizzle matrix:
// start 32m, rows 16 B apart (SBO 128 per 8 lanes), the second K unit 16 B on
// (LBO 16). No im2col and no per-tile halo: each input row is staged once per
// band (8-byte cp.async, zero fill outside the image) and read by the MMAs of the
// four output rows that use it. B = packed filter [r][t][k][8] (t = tap-column
// pair, s = 2t + e/4, c = e%4; s = 7 and c >= C are zero), resident.
// Per output row: 7 rows x 2 K steps = 14 MMAs M=128 N=64 into one of four TMEM
// accumulators; the epilogue (bias/BN/activation/statistics as the tile kernels)
// stages each warp's 32 pixels and TMA-stores them.
//   warps 0-3: epilogue (lane quarter q), warp 4: input-row loader, warp 5: MMA
constexpr int kF2Threads = 32 * 6;
constexpr int kF2Band = 28;        // output rows per work unit (112 = 4 bands: 1024 units at N=256)
constexpr int kF2Ring = 24;        // staged input rows (8-byte pixels, 2 KB each)
constexpr int kF2RowBytes = 2048;  // input columns -3 .. 252
constexpr int kF2Bufs = 4;         // TMEM accumulator pairs (2 output rows x 64 columns)

struct F2Layout {
    int b_off, bp_off, ring_off, stg_off, bar_off, bytes;
    __host__ __device__ F2Layout() {
        b_off = 0;                                   // [r][t][64 k][16 B]: 7 x 4 x 1 KB
        bp_off = 28 * 1024;                          // [r' = 2..6][t][128 rows][16 B]: 5 x 4 x 2 KB
        ring_off = bp_off + 40 * 1024;
        stg_off = ring_off + kF2Ring * kF2RowBytes;
        bar_off = stg_off + 4 * 2 * 4096;            // 4 epilogue warps x 2 staging buffers
        bytes = bar_off + 512 + 1024;
    }
};

__global__ void __launch_bounds__(kF2Threads, 1)
    stem_fprop2_kernel(const __grid_constant__ CUtensorMap ymap, const __nv_bfloat16* __restrict__ x,
                       const __nv_bfloat16* __restrict__ w, const __grid_constant__ StemArgs g,
                       const pk_epilogue epi) {
    pdl_wait();
    pdl_trigger();
    const F2Layout L;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* row_full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* row_empty = row_full + kF2Ring;
    uint64_t* tmem_full = row_empty + kF2Ring;
    uint64_t* tmem_empty = tmem_full + kF2Bufs;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + kF2Bufs);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nb = (g.P + kF2Band - 1) / kF2Band;
    const int units = g.N * nb;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kF2Ring; ++i) {
            mbar_init(&row_full[i], 32);  // one cp.async arrive per loader lane
            mbar_init(&row_empty[i], 1);
        }
        for (int i = 0; i < kF2Bufs; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 4);
        }
        fence_barrier_init();
        tma_prefetch(&ymap);
    }
    if (warp == 5) tmem_alloc(tmem_slot, 512);
    // B[r][t][k][8]: unit t of filter row r = taps (r, 2t), (r, 2t+1) x 4 channels;
    // Bpair[r'][t][128]: rows 0..63 = B[r'][t], rows 64..127 = B[r'-2][t] (one N=128
    // MMA feeds output rows p (tap row r') and p+1 (tap row r'-2) from the same input row)
    for (int i = threadIdx.x; i < 7 * 4 * 64 + 5 * 4 * 128; i += blockDim.x) {
        int r, t, k, dst;
        if (i < 7 * 4 * 64) {
            k = i & 63;
            r = (i >> 6) >> 2;
            t = (i >> 6) & 3;
            dst = L.b_off + i * 16;
        } else {
            const int j = i - 7 * 4 * 64, row = j & 127, rt = j >> 7, rp = 2 + (rt >> 2);
            t = rt & 3;
            k = row & 63;
            r = row < 64 ? rp : rp - 2;
            dst = L.bp_off + j * 16;
        }
        __align__(16) __nv_bfloat16 v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int s = 2 * t + (e >> 2), c = e & 3;
            v[e] = (s < 7 && c < g.C && k < g.K) ? w[((size_t)k * 49 + r * 7 + s) * g.x_pitch + c]
                                                 : __float2bfloat16_rn(0.0f);
        }
        st_shared_v4(smem_u32(smem + dst), *reinterpret_cast<const uint4*>(v));
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t ring0 = smem_u32(smem + L.ring_off);

    if (warp == 4) {
        // ---------------- loader: input rows 2p0-3 .. 2(p0+band-1)+3 per unit ---------
        int rc = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            const int n = u / nb, p0 = (u - n * nb) * kF2Band;
            const int p1 = min(p0 + kF2Band, g.P);
            for (int rho = 2 * p0 - 3; rho <= 2 * (p1 - 1) + 3; ++rho, ++rc) {
                const int s = rc % kF2Ring;
                if (rc >= kF2Ring) mbar_wait(&row_empty[s], ((rc / kF2Ring) - 1) & 1);
                const bool row_in = rho >= 0 && rho < g.H;
                const __nv_bfloat16* src_row = x + ((size_t)n * g.H + (row_in ? rho : 0)) * g.W * g.x_pitch;
                if (g.debug & 2) {  // timing only: no input loads
                    mbar_arrive(&row_full[s]);
                    continue;
                }
#pragma unroll
                for (int e = 0; e < kF2RowBytes / 8 / 32; ++e) {
                    const int col = e * 32 + lane - 3;
                    const bool in = row_in && col >= 0 && col < g.W;
                    cp_async_8(ring0 + s * kF2RowBytes + (col + 3) * 8, in ? src_row + (size_t)col * g.x_pitch : x,
                               in ? 8u : 0u);
                }
                cp_async_arrive_noinc(&row_full[s]);
            }
        }
    } else if (warp == 5) {
        // ---------------- MMA issuer: output rows in pairs (p, p+1) --------------------
        // input rows 2p-3+k, k = 0..8: k = 7, 8 -> p+1 only (N=64, first: they start its
        // accumulator), k = 0, 1 -> p only (N=64, k = 0 starts it), k = 2..6 -> both
        // (N=128 over the adjacent accumulators, B = Bpair)
        const uint32_t id64 = idesc_bf16_f32(128, 64, false, false);
        const uint32_t id128 = idesc_bf16_f32(128, 128, false, false);
        const uint32_t b0 = smem_u32(smem + L.b_off), bp0 = smem_u32(smem + L.bp_off);
        int rc = 0, ready = 0, pc = 0;  // rc: ring index of this unit's first input row
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            const int n = u / nb, p0 = (u - n * nb) * kF2Band;
            const int p1 = min(p0 + kF2Band, g.P);
            const int rows = 2 * (p1 - p0) + 5;
            for (int p = p0; p < p1; p += 2, ++pc) {
                const int first = rc + 2 * (p - p0);  // ring index of input row 2p-3
                while (ready < first + 9) {
                    mbar_wait(&row_full[ready % kF2Ring], (ready / kF2Ring) & 1);
                    ++ready;
                }
                const int buf = pc % kF2Bufs;
                mbar_wait(&tmem_empty[buf], ((pc / kF2Bufs) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d0 = tmem_base + buf * 128;
                auto arow = [&](int k) {
                    return umma_desc_noswz(ring0 + ((first + k) % kF2Ring) * kF2RowBytes, 16, 128);
                };
                if (!(g.debug & 1)) {
                    {   // rows 7, 8: output row p+1, tap rows 5, 6 (k = 7 starts the accumulator)
                        const uint64_t a7 = arow(7), a8 = arow(8);
                        const uint64_t c5 = umma_desc_noswz(b0 + 5 * 4096, 1024, 128),
                                       c6 = umma_desc_noswz(b0 + 6 * 4096, 1024, 128);
                        mma4_bf16(d0 + 64, a7, a7 + 2, a8, a8 + 2, c5, c5 + 128, c6, c6 + 128, id64, 0);
                    }
                    {   // rows 0, 1: output row p, tap rows 0, 1 (k = 0 starts the accumulator)
                        const uint64_t a0 = arow(0), a1 = arow(1);
                        const uint64_t c0 = umma_desc_noswz(b0, 1024, 128), c1 = umma_desc_noswz(b0 + 4096, 1024, 128);
                        mma4_bf16(d0, a0, a0 + 2, a1, a1 + 2, c0, c0 + 128, c1, c1 + 128, id64, 0);
                    }
#pragma unroll
                    for (int k = 2; k < 7; k += 2) {  // rows 2..6: both output rows
                        const uint64_t ak = arow(k), bk = umma_desc_noswz(bp0 + (k - 2) * 8192, 2048, 128);
                        if (k + 1 < 7) {
                            const uint64_t ak1 = arow(k + 1), bk1 = umma_desc_noswz(bp0 + (k - 1) * 8192, 2048, 128);
                            mma4_bf16(d0, ak, ak + 2, ak1, ak1 + 2, bk, bk + 256, bk1, bk1 + 256, id128, 1);
                        } else {
                            mma2_bf16(d0, ak, ak + 2, bk, bk + 256, id128);
                        }
                    }
                }
                mma_commit_elect(&tmem_full[buf]);
                // input rows no later pair of this unit reads: 2p-3 .. 2p (or all at the end)
                const int done = p + 2 < p1 ? 4 : rows - 2 * (p - p0);
                for (int k = 0; k < done; ++k) mma_commit_elect(&row_empty[(first + k) % kF2Ring]);
                __syncwarp();
            }
            rc += rows;
        }
    } else {
        // ---------------- epilogue (4 warps, one TMEM lane quarter each) ---------
        const int q = warp;
        uint8_t* stg_base = smem + L.stg_off + warp * 2 * 4096;
        int sbuf = 0;
        const bool has_epi = epilogue_active(&epi);
        const int ox = q * 32 + lane;
        BnStatAcc bacc;
        bacc.init();
        int pc = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            const int n = u / nb, p0 = (u - n * nb) * kF2Band;
            const int p1 = min(p0 + kF2Band, g.P);
            for (int pp = p0; pp < p1; pp += 2, ++pc) {
                const int buf = pc % kF2Bufs;
                mbar_wait(&tmem_full[buf], (pc / kF2Bufs) & 1);
                tc_fence_after();
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {
                    const int p = pp + h;
                    uint32_t v[64];
                    const uint32_t ta = tmem_base + buf * 128 + h * 64 + (static_cast<uint32_t>(q * 32) << 16);
                    tmem_ld16(ta + 0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
                    tmem_ld16(ta + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
                    tmem_ld16(ta + 32, *reinterpret_cast<uint32_t(*)[16]>(&v[32]));
                    tmem_ld16(ta + 48, *reinterpret_cast<uint32_t(*)[16]>(&v[48]));
                    tmem_ld_wait();
                    if (h == 1) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tmem_empty[buf]);
                    }
                    if (q * 32 >= g.Q) continue;  // no output column in this lane quarter
                    const uint32_t stg_u = smem_u32(stg_base + sbuf * 4096);
                    if (lane == 0) bulk_wait_read<1>();
                    __syncwarp();
                    float xf[64];
#pragma unroll
                    for (int e = 0; e < 64; ++e) xf[e] = __uint_as_float(v[e]);
                    if (has_epi) epilogue_chunk64(epi, xf, 0, g.K, p, ox, g.P, g.Q);
                    pack_stage64(xf, stg_u, lane, 64);
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0 && !(g.debug & 4)) {
                        tma_store_4d(&ymap, stg_u, 0, q * 32, p, n);  // columns >= Q are clipped
                        bulk_commit();
                    }
                    if (epi.stats) bacc.add(epi, stg_u, lane, ox < g.Q, 0, 0, 0, g.K, g.K);
                    sbuf ^= 1;
                }
            }
        }
        if (epi.stats) bacc.finish(epi, lane, g.K);
        if (lane == 0) bulk_wait_all();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

// ---------------------------------------------------------------------------
// backward data v3 ("row strips"), ResNet conv1 geometry: 7x7, stride 2, pad 3,
// H = 2P, W = 2Q, Q <= 128.
//
// dX[y][x] = sum over dY rows i, columns j' of dY[i][j'] . W[r][s] with
// y = 2i + r - 3, x = 2j' + s - 3. For the dX pixel pair x = 2j + xp (xp = 0, 1)
// the tap columns s reaching it come from the four dY columns j' = j + d - 1
// (d = 0..3) with s = xp + 5 - 2d. So ONE GEMM per dY row gives, per dY column j
// (= TMEM lane), the row's whole contribution to dX pixels 2j and 2j+1 for all
// seven tap rows r:
//   D[j][(xp, r, c)] = sum_d sum_k dY[i][j + d - 1][k] . B_d[k][(xp, r, c)],
//   B_d = W[k][r][xp + 5 - 2d][c] (zero where s is outside 0..6)
// K = 4 x 64 (the four shifted copies of the row are the same shared-memory tile
// read from 128-byte row d: SWIZZLE_128B descriptors may start at any row), N = 48
// (2 x 7 x 3 = 42 used). The dY row lands as one in-bounds TMA box of the flat pixel
// array, pixels -1 .. 134 of the row; the three that belong to the neighbouring rows
// but are read (-1, Q, Q+1) are zeroed in shared memory by the MMA warp (partly
// out-of-bounds boxes stream at ~4 TB/s, in-bounds ones at the HBM rate). Rows
// outside the image are skipped by the gather. No cross-lane traffic: thread j adds
// its 42 columns into a window of the 7 dX rows the dY row reaches; rows 2i-3, 2i-2
// are then complete and leave as two 16-byte pixels each.
//
// A CTA owns a band of kDg3Band dX rows of one image and walks the dY rows reaching
// it two at a time (one TMA box, 8 MMA groups, one handshake per pair: per-row
// handshakes cost more than the row's MMAs). Rows outside the image are zero fill,
// so every band is the same 16 pairs (dY read once + ~4 rows per band, dX once).
//   warps 0-3: gather (lane quarter q = warp), warp 4: TMA producer, warp 5: MMA
constexpr int kDg3Threads = 32 * 6;
constexpr int kDg3Stages = 4;     // dY row pairs in flight (4 x 34 KB)
constexpr int kDg3Bufs = 3;       // TMEM accumulator pairs (2 x 64 columns each)
constexpr int kDg3Band = 56;      // dX rows per work unit (224 = 4 bands: 1024 units at N=256)
constexpr int kDg3N = 48;         // MMA N: (xp, r, c) columns, xp-major, 24 per xp
constexpr int kDg3BoxPx = 136;    // pixels -1 .. 134 of a dY row
constexpr int kDg3Steps = 16;     // dY row pairs per band: rows i_lo .. i_lo + 31 (band/2 + 3 used)
static_assert(2 * kDg3Steps >= kDg3Band / 2 + 3, "band rows");

struct Dg3Layout {
    int a_stage, b_off, bar_off, bytes;
    __host__ __device__ Dg3Layout() {
        a_stage = 2 * kDg3BoxPx * 128;               // two rows of 17 KB, 1024-aligned
        b_off = kDg3Stages * a_stage;
        bar_off = b_off + 4 * kDg3N * 128;           // four K blocks of N rows x 64 k
        bytes = bar_off + 256 + 1024;
    }
};

// Work unit u = (image, band): dY rows i_lo .. i_lo + 2 * kDg3Steps - 1.
struct Dg3Walk {
    int n, i_lo, Y0;
    __device__ Dg3Walk(const DgArgs& g, int u) {
        const int nb = (g.H + kDg3Band - 1) / kDg3Band;
        n = u / nb;
        Y0 = (u - n * nb) * kDg3Band;
        i_lo = Y0 / 2 - 1;
    }
};

template <int C>
__global__ void __launch_bounds__(kDg3Threads, 1)
    stem_dgrad3_kernel(const __grid_constant__ CUtensorMap dymap, const __nv_bfloat16* __restrict__ w,
                       __nv_bfloat16* __restrict__ dx, const __grid_constant__ DgArgs g) {
    pdl_wait();
    pdl_trigger();
    const Dg3Layout L;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* a_full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* a_empty = a_full + kDg3Stages;
    uint64_t* tmem_full = a_empty + kDg3Stages;
    uint64_t* tmem_empty = tmem_full + kDg3Bufs;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + kDg3Bufs);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int units = g.N * ((g.H + kDg3Band - 1) / kDg3Band);

    if (threadIdx.x == 0) {
        for (int i = 0; i < kDg3Stages; ++i) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], 1);
        }
        for (int i = 0; i < kDg3Bufs; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 4);
        }
        fence_barrier_init();
        tma_prefetch(&dymap);
    }
    if (warp == 5) tmem_alloc(tmem_slot, 512);
    // B_d[n][k], n = xp * 24 + r * C + c (K-major SWIZZLE_128B, 64 k = one atom)
    for (int i = threadIdx.x; i < 4 * kDg3N * 8; i += blockDim.x) {
        const int jj = i & 7, row = i >> 3, d = row / kDg3N, n = row - d * kDg3N;
        const int xp = n / 24, rc = n - xp * 24, r = rc / C, c = rc - r * C;
        const int s = xp + 5 - 2 * d;
        const bool ok = rc < 7 * C && s >= 0 && s < 7;
        __align__(16) __nv_bfloat16 v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int k = jj * 8 + e;
            v[e] = (ok && k < g.K) ? w[((size_t)k * 49 + r * 7 + s) * g.x_pitch + c] : __float2bfloat16_rn(0.0f);
        }
        st_shared_v4(smem_u32(smem + L.b_off) + row * 128 + ((jj ^ (row & 7)) << 4),
                     *reinterpret_cast<const uint4*>(v));
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 4) {
        // ---------------- TMA producer: one box of two dY rows per step ----------------
        int n = 0;
        for (int unit = blockIdx.x; unit < units; unit += gridDim.x) {
            const Dg3Walk wk(g, unit);
            for (int st = 0; st < kDg3Steps; ++st, ++n) {
                const int s = n % kDg3Stages;
                if (n >= kDg3Stages) mbar_wait(&a_empty[s], ((n / kDg3Stages) - 1) & 1);
                dstamp(g, n, 12);
                if (lane == 0 && (g.debug & 32)) {
                    mbar_arrive(&a_full[s]);
                } else if (lane == 0) {
                    // two in-bounds boxes of the flat pixel array: pixels -1 .. 134 of rows i, i+1
                    // (the MMA warp zeroes the neighbours' pixels -1, Q, Q+1 before use)
                    mbar_arrive_expect_tx(&a_full[s], 2 * kDg3BoxPx * 128);
                    const int base = (wk.n * g.P + wk.i_lo + 2 * st) * g.Q - 1;
                    tma_load_2d(smem_u32(smem + s * L.a_stage), &dymap, &a_full[s], 0, base);
                    tma_load_2d(smem_u32(smem + s * L.a_stage + kDg3BoxPx * 128), &dymap, &a_full[s], 0, base + g.Q);
                }
                __syncwarp();
            }
        }
    } else if (warp == 5) {
        // ---------------- MMA issuer: 2 rows x 4 shifted copies x 4 K steps ---------------
        const uint32_t idesc = idesc_bf16_f32(128, kDg3N, false, false);
        const uint32_t b0 = smem_u32(smem + L.b_off);
        const int steps = ((units - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x) * kDg3Steps;
        for (int n = 0; n < steps; ++n) {
            const int s = n % kDg3Stages, buf = n % kDg3Bufs;
            dstamp(g, n, 0);
            mbar_wait(&a_full[s], (n / kDg3Stages) & 1);
            dstamp(g, n, 1);
            // pixels -1, Q, Q+1 of each row are the neighbouring rows' data: zero them
            // (generic stores, then a proxy fence so the tensor core sees them)
            if (lane < 6 * 8) {
                const int rr = lane >> 3, row = rr / 3, e = rr % 3, q16 = lane & 7;
                const int prow = e == 0 ? 0 : g.Q + e;
                st_shared_v4(smem_u32(smem + s * L.a_stage + row * kDg3BoxPx * 128 + prow * 128 + q16 * 16),
                             make_uint4(0u, 0u, 0u, 0u));
            }
            if (lane < 16) {
                const int rr = 4 + (lane >> 3), row = rr / 3, e = rr % 3, q16 = lane & 7;
                const int prow = e == 0 ? 0 : g.Q + e;
                st_shared_v4(smem_u32(smem + s * L.a_stage + row * kDg3BoxPx * 128 + prow * 128 + q16 * 16),
                             make_uint4(0u, 0u, 0u, 0u));
            }
            fence_proxy_async_smem();
            __syncwarp();
            dstamp(g, n, 2);
            mbar_wait(&tmem_empty[buf], ((n / kDg3Bufs) & 1) ^ 1);
            dstamp(g, n, 3);
            tc_fence_after();
            if (!(g.debug & 1)) {
#pragma unroll
                for (int row = 0; row < 2; ++row) {
                    const uint32_t a0 = smem_u32(smem + s * L.a_stage + row * kDg3BoxPx * 128);
#pragma unroll
                    for (int d = 0; d < 4; ++d) {
                        // shifted copy d: box rows d .. d+127 (pixels j + d - 1), B block d
                        const uint64_t ad = umma_desc_sw128(a0 + d * 128, 16, 1024);
                        const uint64_t bd = umma_desc_sw128(b0 + d * kDg3N * 128, 16, 1024);
                        mma4_bf16(tmem_base + buf * 128 + row * 64, ad, ad + 2, ad + 4, ad + 6, bd, bd + 2,
                                  bd + 4, bd + 6, idesc, d > 0);
                    }
                }
            }
            dstamp(g, n, 4);
            mma_commit_elect(&a_empty[s]);
            mma_commit_elect(&tmem_full[buf]);
            __syncwarp();
            dstamp(g, n, 5);
        }
    } else {
        // ---------------- gather: lane j owns dX pixels 2j, 2j+1 ---------------------
        const int j = 32 * warp + lane;
        const bool owned = j < g.Q;
        const uint32_t ta_q = tmem_base + (static_cast<uint32_t>(warp * 32) << 16);
        int n = 0;
        for (int unit = blockIdx.x; unit < units; unit += gridDim.x) {
            const Dg3Walk wk(g, unit);
            // window of the 7 dX rows dY row i reaches: slot r <-> y = 2i + r - 3
            float acc[7][2][C];
#pragma unroll
            for (int r = 0; r < 7; ++r)
#pragma unroll
                for (int xp = 0; xp < 2; ++xp)
#pragma unroll
                    for (int c = 0; c < C; ++c) acc[r][xp][c] = 0.0f;
#pragma unroll 1
            for (int st = 0; st < kDg3Steps; ++st, ++n) {
                const int buf = n % kDg3Bufs;
                if (warp == 0) dstamp(g, n, 6);
                mbar_wait(&tmem_full[buf], (n / kDg3Bufs) & 1);
                if (warp == 0) dstamp(g, n, 7);
                tc_fence_after();
                uint32_t v[96];
#pragma unroll
                for (int k = 0; k < 6; ++k)
                    tmem_ld16(ta_q + buf * 128 + (k / 3) * 64 + (k % 3) * 16,
                              *reinterpret_cast<uint32_t(*)[16]>(&v[k * 16]));
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tmem_empty[buf]);
                dstamp(g, n, 8 + warp);
#pragma unroll
                for (int row = 0; row < 2; ++row) {
                    const int i = wk.i_lo + 2 * st + row;
                    if (!(g.debug & 2) && i >= 0 && i < g.P) {  // other rows are another image's
#pragma unroll
                        for (int r = 0; r < 7; ++r)
#pragma unroll
                            for (int xp = 0; xp < 2; ++xp)
#pragma unroll
                                for (int c = 0; c < C; ++c)
                                    acc[r][xp][c] += __uint_as_float(v[row * 48 + xp * 24 + r * C + c]);
                    }
                    // dX rows 2i-3 and 2i-2 (slots 0, 1) are complete: store (inside the band)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int y = 2 * i - 3 + e;
                        if (owned && y >= wk.Y0 && y < wk.Y0 + kDg3Band && y < g.H && !(g.debug & 4)) {
                            __align__(16) __nv_bfloat16 ob[16];
#pragma unroll
                            for (int xp = 0; xp < 2; ++xp)
#pragma unroll
                                for (int c = 0; c < 8; ++c)
                                    ob[xp * 8 + c] = __float2bfloat16_rn(c < C ? acc[e][xp][c < C ? c : 0] : 0.0f);
                            uint4* dst = reinterpret_cast<uint4*>(dx + (((size_t)wk.n * g.H + y) * g.W + 2 * j) * g.x_pitch);
                            dst[0] = reinterpret_cast<const uint4*>(ob)[0];
                            dst[1] = reinterpret_cast<const uint4*>(ob)[1];
                        }
                    }
                    // shift the window by two dX rows
#pragma unroll
                    for (int r = 0; r < 7; ++r)
#pragma unroll
                        for (int xp = 0; xp < 2; ++xp)
#pragma unroll
                            for (int c = 0; c < C; ++c) acc[r][xp][c] = r < 5 ? acc[r + 2 < 7 ? r + 2 : 0][xp][c] : 0.0f;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

__host__ __device__ inline int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

bool dg_args(const pk_conv_geom* g, DgArgs& a) {
    if (g->groups != 1 || g->transpose || g->c > 4 || g->x_pitch != 8 || g->f_pitch != 8 ||
        g->k != 64 || g->y_pitch != 64 || g->r * g->s > kMaxTaps || g->dil_h != 1 || g->dil_w != 1)
        return false;
    a = DgArgs{};
    a.N = g->n; a.H = g->h; a.W = g->w; a.x_pitch = g->x_pitch; a.P = g->p; a.Q = g->q; a.K = g->k;
    a.R = g->r; a.S = g->s; a.sh = g->str_h; a.sw = g->str_w; a.dh = g->dil_h; a.dw = g->dil_w;
    a.ph = g->pad_h; a.pw = g->pad_w; a.C = g->c; a.taps = g->r * g->s;
    a.npad = (a.taps * 4 + 15) / 16 * 16;
    if (2 * a.npad > 512) return false;
    a.cstride = ((a.npad / 4) * a.C) | 1;  // all padded taps stored; odd: conflict-free
    // v3 row strips: 7x7 stride 2 pad 3 with H = 2P, W = 2Q and a dY row within the 128 lanes
    static const int dg_ver = [] {
        const char* v = std::getenv("PK_STEM_DG");
        return v ? std::atoi(v) : 3;
    }();
    if (dg_ver >= 3 && a.R == 7 && a.S == 7 && a.sh == 2 && a.sw == 2 && a.ph == 3 && a.pw == 3 &&
        a.H == 2 * a.P && a.W == 2 * a.Q && a.Q <= 128 && a.C <= 3 &&
        Dg3Layout().bytes <= 227 * 1024) {
        a.v3 = 1;
        return true;
    }
    static const int cand[][2] = {{16, 32}, {8, 32}, {16, 16}, {8, 16}, {8, 8}, {4, 8}};
    // pipelined v2 first: the largest tile whose halo fits one 128-row MMA
    static const bool v2_off = std::getenv("PK_STEM_DG_V1") != nullptr || dg_ver == 1;
    for (const auto& c : cand) {
        if (v2_off || (a.taps * a.C + 15) / 16 * 16 > 256) break;
        const int TY = c[0], TX = c[1];
        if (TY % a.sh || TX % a.sw) continue;
        const int lo_y = -floor_div(-(a.ph - (a.R - 1) * a.dh), a.sh);
        const int hi_y = floor_div(TY - 1 + a.ph, a.sh);
        const int lo_x = -floor_div(-(a.pw - (a.S - 1) * a.dw), a.sw);
        const int hi_x = floor_div(TX - 1 + a.pw, a.sw);
        const int HY = hi_y - lo_y + 1, WX = hi_x - lo_x + 1;
        if (HY * WX > kTile || HY > 256 || WX > 256) continue;
        DgArgs b = a;
        // v2: dense kc = tap*C + c; colg rows of roundup4(taps*C) words with an odd
        // number of 16-byte units (conflict-free vector drain stores)
        b.npad = (a.taps * a.C + 15) / 16 * 16;
        b.cstride = (a.taps * a.C + 3) / 4 * 4;
        if ((b.cstride / 4) % 2 == 0) b.cstride += 4;
        b.TY = TY; b.TX = TX; b.HY = HY; b.WX = WX; b.oy_lo0 = lo_y; b.ox_lo0 = lo_x;
        b.tiles_w = (b.W + TX - 1) / TX;
        b.tiles_h = (b.H + TY - 1) / TY;
        b.total_tiles = b.tiles_w * b.tiles_h * b.N;
        b.v2 = 1;
        if (Dg2Layout(b).bytes > 227 * 1024) continue;
        a = b;
        return true;
    }
    for (const auto& c : cand) {
        const int TY = c[0], TX = c[1];
        if (TY % a.sh || TX % a.sw) continue;
        // dY rows reaching dX rows [Y0, Y0 + TY) for Y0 = 0 (pattern repeats every tile)
        const int lo_y = -floor_div(-(a.ph - (a.R - 1) * a.dh), a.sh);  // ceil
        const int hi_y = floor_div(TY - 1 + a.ph, a.sh);
        const int lo_x = -floor_div(-(a.pw - (a.S - 1) * a.dw), a.sw);
        const int hi_x = floor_div(TX - 1 + a.pw, a.sw);
        const int HY = hi_y - lo_y + 1, WX = hi_x - lo_x + 1;
        if (HY * WX > 2 * kTile || HY > 256 || WX > 256) continue;
        a.TY = TY; a.TX = TX; a.HY = HY; a.WX = WX; a.oy_lo0 = lo_y; a.ox_lo0 = lo_x;
        a.tiles_w = (a.W + TX - 1) / TX;
        a.tiles_h = (a.H + TY - 1) / TY;
        a.total_tiles = a.tiles_w * a.tiles_h * a.N;
        return DgLayout(a).bytes <= 227 * 1024;
    }
    return false;
}

// ---------------------------------------------------------------------------
// host

bool stem_args(const pk_conv_geom* g, StemArgs& a) {
    if (g->groups != 1 || g->transpose || g->c > 4 || g->x_pitch != 8 || g->f_pitch != 8)
        return false;
    if (g->r * g->s > kMaxTaps || (g->k != 64 && g->k != 128) || g->y_pitch != g->k)
        return false;
    a = StemArgs{};
    a.N = g->n;
    a.H = g->h;
    a.W = g->w;
    a.x_pitch = g->x_pitch;
    a.P = g->p;
    a.Q = g->q;
    a.K = g->k;
    a.n_pad = g->k;
    a.R = g->r;
    a.S = g->s;
    a.sh = g->str_h;
    a.sw = g->str_w;
    a.dh = g->dil_h;
    a.dw = g->dil_w;
    a.ph = g->pad_h;
    a.pw = g->pad_w;
    a.C = g->c;
    a.tiles_w = (g->q + kBw - 1) / kBw;
    a.tiles_h = (g->p + kBh - 1) / kBh;
    a.total_tiles = a.tiles_w * a.tiles_h * g->n;
    a.HH = (kBh - 1) * a.sh + (a.R - 1) * a.dh + 1;
    a.HW = (kBw - 1) * a.sw + (a.S - 1) * a.dw + 1;
    a.HWp = (a.HW + a.sw - 1) / a.sw;
    if (a.HH * a.HW > kBuilders * kHaloPer || a.sw * a.HH * a.HWp * 8 > kHaloStageBytes - 8) return false;
    a.taps = a.R * a.S;
    a.nchunks = (a.taps + 1) / 2;
    a.nchunks += a.nchunks & 1;
    a.kcm = (a.nchunks * 8 + 127) / 128 * 128;
    static const int dbg = [] {
        const char* v = std::getenv("PK_STEM_DEBUG");
        return v ? std::atoi(v) : 0;
    }();
    a.debug = dbg;
    static unsigned long long* trace = [] {
        unsigned long long* p = nullptr;
        if (std::getenv("PK_STEM_TRACE")) cudaMalloc(&p, 32 * 32 * 8);
        return p;
    }();
    a.trace = trace;
    for (int t = 0; t < a.taps; ++t) {
        const int r = t / a.S, s = t % a.S;
        a.tap_off[t] = ((s * a.dw) % a.sw) * a.HH * a.HWp + r * a.dh * a.HWp + (s * a.dw) / a.sw;
    }
    return true;
}

template <typename Kern>
cudaError_t set_smem(Kern kern, int bytes, int* attr_dev) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (*attr_dev != dev) {
        const cudaError_t err =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (err != cudaSuccess) return err;
        *attr_dev = dev;
    }
    return cudaSuccess;
}

template <int NP>
cudaError_t launch_stem_fprop(const CUtensorMap& ymap, const void* x, const void* w, const StemArgs& a, const pk_epilogue& e,
                              cudaStream_t st) {
    static int attr_dev = -1;
    auto kern = stem_fprop_kernel<NP>;
    const int bytes = FwdLayout(a.nchunks, NP).bytes;
    if (bytes > 227 * 1024) return cudaErrorNotSupported;
    cudaError_t err = set_smem(kern, 227 * 1024, &attr_dev);
    if (err != cudaSuccess) return err;
    int grid = num_sms_of_current_device();
    if (a.total_tiles < grid) grid = a.total_tiles;
    cudaError_t le = pk_launch(kern, dim3(grid), dim3(kFwdThreads), bytes, st, ymap,
                               (const __nv_bfloat16*)x, (const __nv_bfloat16*)w, a, e);
    if (le != cudaSuccess) return le;
    count_launch();
    if (a.trace) {
        unsigned long long h[32 * 32];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, a.trace, sizeof(h), cudaMemcpyDeviceToHost);
        const unsigned long long t0 = h[0];
        for (int i = 0; i < 32; ++i) {
            fprintf(stderr, "tile %2d:", i);
            for (int e = 0; e < 13; ++e) fprintf(stderr, " %7lld", (long long)(h[i * 32 + e] - t0));
            fprintf(stderr, " | mma:");
            for (int e = 16; e < 17; ++e)
                fprintf(stderr, " %5lld", (long long)(h[i * 32 + e] - h[i * 32 + 2]));
            fprintf(stderr, "\n");
        }
    }
    return cudaGetLastError();
}

int stem_wgrad_ctas(const StemArgs& a, int num_sms) {
    if (num_sms > 148) num_sms = 148;  // workspace is sized for 148 partials
    return a.total_tiles < num_sms ? a.total_tiles : num_sms;
}

template <int NP>
cudaError_t launch_stem_wgrad(const CUtensorMap& dymap, const void* x, float* partial,
                              const StemArgs& a, int ctas, cudaStream_t st) {
    static int attr_dev = -1;
    auto kern = stem_wgrad_kernel<NP>;
    cudaError_t err = set_smem(kern, WgSmem<NP>::kBytes, &attr_dev);
    if (err != cudaSuccess) return err;
    cudaError_t le = pk_launch(kern, dim3(ctas), dim3(kWgThreads), WgSmem<NP>::kBytes, st, dymap,
                               (const __nv_bfloat16*)x, partial, a);
    if (le != cudaSuccess) return le;
    count_launch();
    return cudaGetLastError();
}

}  // namespace
}  // namespace pk

using namespace pk;

extern "C" {

int pk_cuda_stem_fused_supported(const pk_conv_geom* g) {
    StemArgs a;
    return stem_args(g, a) && tc::encode_fn() != nullptr;
}

cudaError_t pk_cuda_stem_fused_fprop(const pk_conv_geom* g, const void* x, const void* w, void* y,
                                const pk_epilogue* epi, cudaStream_t st) {
    StemArgs a;
    if (!stem_args(g, a)) return cudaErrorNotSupported;
    CUtensorMap ymap{};
    // one epilogue warp stores 32 rows = 2 output rows of 16 pixels
    if (!tc::make_map_nhwc(&ymap, y, g->n, g->p, g->q, g->y_pitch, kBw, 2, 1))
        return cudaErrorNotSupported;
    pk_epilogue e{};
    e.act = -1;
    if (epi) e = *epi;
    static const bool f2_off = [] {
        const char* v = std::getenv("PK_STEM_FWD");
        return v && std::atoi(v) == 1;
    }();
    if (!f2_off && g->k == 64 && a.R == 7 && a.S == 7 && a.sh == 2 && a.sw == 2 && a.ph == 3 && a.pw == 3 &&
        a.Q <= 128 && a.W <= 2 * 128 && a.C <= 4 && a.dh == 1 && a.dw == 1 && a.P % 2 == 0) {
        // row strips: one TMA store box = one warp's 32 output columns of a row
        CUtensorMap ymap2{};
        if (!tc::make_map_nhwc(&ymap2, y, g->n, g->p, g->q, g->y_pitch, 32, 1, 1))
            return cudaErrorNotSupported;
        static int attr_f2 = -1;
        cudaError_t err = set_smem(stem_fprop2_kernel, F2Layout().bytes, &attr_f2);
        if (err != cudaSuccess) return err;
        int grid = num_sms_of_current_device();
        const int units = g->n * ((g->p + kF2Band - 1) / kF2Band);
        if (units < grid) grid = units;
        err = pk_launch(stem_fprop2_kernel, dim3(grid), dim3(kF2Threads), F2Layout().bytes, st, ymap2,
                        (const __nv_bfloat16*)x, (const __nv_bfloat16*)w, a, e);
        if (err != cudaSuccess) return err;
        count_launch();
        return cudaGetLastError();
    }
    switch (g->k) {
        case 64: return launch_stem_fprop<64>(ymap, x, w, a, e, st);
        case 128: return launch_stem_fprop<128>(ymap, x, w, a, e, st);
        default: return cudaErrorNotSupported;
    }
}

int pk_cuda_stem_fused_dgrad_supported(const pk_conv_geom* g) {
    DgArgs a;
    return dg_args(g, a) && tc::encode_fn() != nullptr;
}

cudaError_t pk_cuda_stem_fused_dgrad(const pk_conv_geom* g, const void* dy, const void* w, void* dx,
                                     cudaStream_t st) {
    DgArgs a;
    if (!dg_args(g, a)) return cudaErrorNotSupported;
    CUtensorMap dymap{};
    int grid = tc::num_sms_of_current_device();
    if (const char* v = std::getenv("PK_STEM_DEBUG")) a.debug = std::atoi(v);
    if (a.v3) {
        // flat pixel rows [N*P*Q][64]: boxes of pixels -1 .. 134 of a dY row
        if (!tc::make_map_2d(&dymap, dy, (long long)g->n * g->p * g->q, 64, g->y_pitch, kDg3BoxPx))
            return cudaErrorNotSupported;
        const int units = g->n * ((g->h + kDg3Band - 1) / kDg3Band);
        if (units < grid) grid = units;
        static int attr3[4] = {-1, -1, -1, -1};
        static unsigned long long* trace3 = [] {
            unsigned long long* p = nullptr;
            if (std::getenv("PK_STEM_TRACE")) cudaMalloc(&p, 32 * 32 * 8);
            return p;
        }();
        a.trace = trace3;
        auto go3 = [&](auto kern, int* attr_dev) {
            cudaError_t err = set_smem(kern, Dg3Layout().bytes, attr_dev);
            if (err != cudaSuccess) return err;
            err = pk_launch(kern, dim3(grid), dim3(kDg3Threads), Dg3Layout().bytes, st, dymap,
                            (const __nv_bfloat16*)w, (__nv_bfloat16*)dx, a);
            if (err != cudaSuccess) return err;
            count_launch();
            if (a.trace) {  // profiling only (PK_STEM_TRACE): per-step clock stamps of CTA 0
                unsigned long long h[32 * 32];
                cudaStreamSynchronize(st);
                cudaMemcpy(h, a.trace, sizeof(h), cudaMemcpyDeviceToHost);
                for (int i = 0; i < 32; ++i) {
                    fprintf(stderr, "dg3 step %2d:", i);
                    for (int e = 0; e < 13; ++e) fprintf(stderr, " %6lld", (long long)(h[i * 32 + e] - h[0]));
                    fprintf(stderr, "\n");
                }
            }
            return cudaGetLastError();
        };
        switch (a.C) {
            case 1: return go3(stem_dgrad3_kernel<1>, &attr3[1]);
            case 2: return go3(stem_dgrad3_kernel<2>, &attr3[2]);
            default: return go3(stem_dgrad3_kernel<3>, &attr3[3]);
        }
    }
    if (!tc::make_map_nhwc(&dymap, dy, g->n, g->p, g->q, g->y_pitch, a.WX, a.HY, 1))
        return cudaErrorNotSupported;
    if (a.total_tiles < grid) grid = a.total_tiles;
    static unsigned long long* trace = [] {
        unsigned long long* p = nullptr;
        if (std::getenv("PK_STEM_TRACE")) cudaMalloc(&p, 32 * 32 * 8);
        return p;
    }();
    a.trace = trace;
    auto go = [&](auto kern, int* attr_dev) {
        cudaError_t err = set_smem(kern, 227 * 1024, attr_dev);
        if (err != cudaSuccess) return err;
        if (a.v2)
            err = pk_launch(kern, dim3(grid), dim3(kDg2Threads), Dg2Layout(a).bytes, st, dymap,
                            (const __nv_bfloat16*)w, (__nv_bfloat16*)dx, a);
        else
            err = pk_launch(kern, dim3(grid), dim3(kDgThreads), DgLayout(a).bytes, st, dymap,
                            (const __nv_bfloat16*)w, (__nv_bfloat16*)dx, a);
        if (err != cudaSuccess) return err;
        count_launch();
        if (a.trace) {
            unsigned long long h[32 * 32];
            cudaStreamSynchronize(st);
            cudaMemcpy(h, a.trace, sizeof(h), cudaMemcpyDeviceToHost);
            for (int i = 0; i < 12; ++i) {
                fprintf(stderr, "dg tile %2d:", i);
                for (int e = 0; e < 10; ++e) fprintf(stderr, " %8lld", (long long)(h[i * 32 + e] - h[0]));
                fprintf(stderr, "\n");
            }
        }
        return cudaGetLastError();
    };
    static int dev0 = -1, dev1 = -1, dev2 = -1, dev3 = -1, dev4 = -1;
    static int e0 = -1, e1 = -1, e2 = -1, e3 = -1, e4 = -1;
    if (a.v2) {
        if (a.C == 3 && a.R == 7 && a.S == 7 && a.sh == 2 && a.sw == 2)  // ResNet conv1
            return go(stem_dgrad2_kernel<3, 7, 7, 2, 2>, &e0);
        switch (a.C) {
            case 1: return go(stem_dgrad2_kernel<1, 0, 0, 0, 0>, &e1);
            case 2: return go(stem_dgrad2_kernel<2, 0, 0, 0, 0>, &e2);
            case 3: return go(stem_dgrad2_kernel<3, 0, 0, 0, 0>, &e3);
            default: return go(stem_dgrad2_kernel<4, 0, 0, 0, 0>, &e4);
        }
    }
    if (a.C == 3 && a.R == 7 && a.S == 7 && a.sh == 2 && a.sw == 2)  // ResNet conv1
        return go(stem_dgrad_kernel<3, 7, 7, 2, 2>, &dev0);
    switch (a.C) {
        case 1: return go(stem_dgrad_kernel<1, 0, 0, 0, 0>, &dev1);
        case 2: return go(stem_dgrad_kernel<2, 0, 0, 0, 0>, &dev2);
        case 3: return go(stem_dgrad_kernel<3, 0, 0, 0, 0>, &dev3);
        default: return go(stem_dgrad_kernel<4, 0, 0, 0, 0>, &dev4);
    }
}

size_t pk_cuda_stem_fused_wgrad_workspace(const pk_conv_geom* g, int num_sms) {
    StemArgs a;
    if (!stem_args(g, a)) return 0;
    return (size_t)stem_wgrad_ctas(a, num_sms) * g->k * a.kcm * 4;
}

cudaError_t pk_cuda_stem_fused_wgrad(const pk_conv_geom* g, const void* dy, const void* x, void* dw,
                                void* workspace, int num_sms, cudaStream_t st) {
    StemArgs a;
    if (!stem_args(g, a) || a.kcm > 256) return cudaErrorNotSupported;
    CUtensorMap dymap{};
    if (!tc::make_map_nhwc(&dymap, dy, g->n, g->p, g->q, g->y_pitch, kBw, kBh, 1))
        return cudaErrorNotSupported;
    const int ctas = stem_wgrad_ctas(a, num_sms);
    float* partial = static_cast<float*>(workspace);
    cudaError_t err;
    switch (g->k) {
        case 64: err = launch_stem_wgrad<64>(dymap, x, partial, a, ctas, st); break;
        case 128: err = launch_stem_wgrad<128>(dymap, x, partial, a, ctas, st); break;
        default: return cudaErrorNotSupported;
    }
    if (err != cudaSuccess) return err;
    const long long total = (long long)g->k * a.taps * g->f_pitch;
    const unsigned blocks = (unsigned)std::min<long long>((total * 32 + 255) / 256, 148LL * 16);
    err = pk_launch(stem_wgrad_finish_kernel, dim3(blocks), dim3(256), 0, st, (const float*)partial,
                    ctas, g->k, a.kcm, a.taps, g->f_pitch, g->c, (__nv_bfloat16*)dw);
    count_launch();
    return err != cudaSuccess ? err : cudaGetLastError();
}

}  // extern "C"
