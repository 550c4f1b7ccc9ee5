#include <cstdio>
#include <cstdlib>
// tcgen05 implicit-GEMM convolution, forward and backward-data (sm_100a).
//
//   D[pixel][out_ch] = sum_{(r,s,ch)} A[pixel][(r,s,ch)] * B[out_ch][(r,s,ch)]
//
// This is the ImplicitGemm solver for bf16 ("composable
// kernels": blockwise tiles -> LDS -> threadwise MMA, re-designed for
// Blackwell) and the bf16 engine of the Im2colGemm backward-data path.
//
// Persistent, warp-specialised CTA (one per SM, 288 threads):
//   warps 0-3  producers: A tiles gathered from NHWC activations with 16-byte
//              cp.async (zero-fill = padding / stride holes) into the canonical
//              K-major SWIZZLE_128B layout, or loaded by TMA when the
//              convolution is a plain GEMM (1x1, stride 1, no padding); B
//              (filter [out][R][S][pitch]) is a 2-D TMA tile (OOB zero fill
//              covers the K tail and out-of-range output channels);
//   warp 4     TMEM allocator + MMA issuer: one elected lane issues
//              tcgen05.mma (M=128, N=BN, K=16) into a double-buffered TMEM
//              accumulator; tcgen05.commit recycles smem stages;
//   warps 5-8  epilogue: tcgen05.ld (32x32b) -> fused bias/BN/activation ->
//              bf16 -> swizzled smem staging -> fully coalesced 16-byte global
//              stores, overlapping the next tile's main loop.
// Backward data with stride > 1 uses sub-pixel (phase) decomposition: output
// pixels are grouped by (h mod s, w mod s) and each phase only iterates the
// filter taps that reach it, so no tensor-core work is spent on stride holes.
#include "common.cuh"
#include "tc_host.cuh"
#include "tc_internal.h"
#include "tc_ptx.cuh"

namespace pk {
namespace {

using namespace pk::tc;

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 416;  // 4 producer + 1 MMA + 8 epilogue warps
constexpr int kMaxPhases = 16;
constexpr int kMaxTaps = 1024;

// PLAIN_RES / PLAIN_RES_BIG: plain GEMM with the CTA's whole B slice (filter
// rows of its fixed N tile, <= kResB bytes) loaded once and kept resident in
// shared memory; the pipeline stages carry A only. Cuts the TMA traffic of 1x1
// layers (B was re-read for every 128-pixel tile) to the activations.
enum Mode { GATHER_FWD = 0, GATHER_DGRAD = 1, PHASE_DGRAD = 2, PLAIN = 3, PLAIN_RES = 4,
            PLAIN_RES_BIG = 5 };
template <int MODE>
constexpr bool is_plain() { return MODE == PLAIN || MODE == PLAIN_RES || MODE == PLAIN_RES_BIG; }
template <int MODE>
constexpr bool is_res() { return MODE == PLAIN_RES || MODE == PLAIN_RES_BIG; }

struct ConvTcArgs {
    int M;                 // output rows (non-phase modes)
    int Ho, Wo;            // output image extent
    int Hs, Ws;            // gathered source extent
    int src_pitch;         // channel pitch of the source
    int red_ch;            // reduction channels per tap (multiple of 8)
    int R, S, pad_h, pad_w, str_h, str_w, dil_h, dil_w;
    int kred, num_kb;      // non-phase modes
    int n_out, out_pitch;
    int n_tiles_n, total_tiles;
    // batched plain GEMM (Winograd): A/Y rows are [batch][rows_per_batch] with
    // rows_per_batch = b_batch_mtiles * BM; B rows of batch b start at
    // b * b_batch_rows. 0 = not batched.
    int b_batch_mtiles, b_batch_rows;
    // batched plain GEMM only: A, B and the output are IEEE fp16 (Winograd
    // transform domain), the accumulator fp32 as always
    int f16;
    // plain modes: B given MN-major (the filter W[K][C] itself for backward data,
    // no transpose launch): BN/64 atoms of 64 output channels x 64 k per k-block
    int b_mn;
    // phase decomposition (PHASE_DGRAD)
    int num_phases, cpt;   // cpt = red_ch / 64
    int ph_tile_start[kMaxPhases + 1];
    int ph_rows[kMaxPhases], ph_hp[kMaxPhases], ph_wp[kMaxPhases];
    int ph_h0[kMaxPhases], ph_w0[kMaxPhases];
    int ph_tap_start[kMaxPhases + 1];
    unsigned short taps[kMaxTaps];  // (r << 8) | s
    int debug_nores;       // PK_TC_NORES=1: disable the resident-B plain path (A/B comparisons)
    int debug;             // PK_TC_DEBUG (profiling only): 1 no MMA, 2 no TMEM load, 4 no store, 8 no math
    unsigned long long* trace;  // PK_TC_TRACE: clock64 stamps of CTA 0 (profiling only)
};
__device__ __forceinline__ void tcstamp(const ConvTcArgs& g, int it, int ev) {
    if (g.trace && blockIdx.x == 0 && it < 32 && (threadIdx.x & 31) == 0)
        g.trace[it * 16 + ev] = clock64();
}

template <int BN, int STAGES, int MODE = PLAIN>
struct Smem {
    static constexpr int kA = BM * BK * 2;
    static constexpr int kB = BN * BK * 2;
    static constexpr int kStage = is_res<MODE>() ? kA : kA + kB;
    // resident B slice (PLAIN_RES*): 64 KB, or 128 KB with single staging
    static constexpr int kResB = MODE == PLAIN_RES_BIG ? 128 * 1024 : MODE == PLAIN_RES ? 64 * 1024 : 0;
    static constexpr int kStgBufs = MODE == PLAIN_RES_BIG ? 1 : 2;
    static constexpr int kResOff = STAGES * kStage;
    static constexpr int kStaging = 8 * kStgBufs * 32 * 128;  // 8 epilogue warps x bufs x 32 x 128 B
    static constexpr int kStagingOff = kResOff + kResB;
    static constexpr int kBarOff = kStagingOff + kStaging;
    static constexpr int kBytes = kBarOff + (2 * STAGES + 9) * 8 + 16 + 1024;
};

struct TileInfo {
    int phase, m0, rows, n0, nkb;
};

template <int MODE>
__device__ __forceinline__ TileInfo tile_info(const ConvTcArgs& g, int t) {
    TileInfo ti;
    const int nt = t % g.n_tiles_n;
    int mt = t / g.n_tiles_n;
    ti.n0 = nt;  // N-tile index; callers scale by BN
    if (MODE == PHASE_DGRAD) {
        int ph = 0;
        while (ph + 1 < g.num_phases && mt >= g.ph_tile_start[ph + 1]) ++ph;
        ti.phase = ph;
        ti.m0 = (mt - g.ph_tile_start[ph]) * BM;
        ti.rows = g.ph_rows[ph];
        ti.nkb = (g.ph_tap_start[ph + 1] - g.ph_tap_start[ph]) * g.cpt;
    } else {
        ti.phase = 0;
        ti.m0 = mt * BM;
        ti.rows = g.M;
        ti.nkb = g.num_kb;
    }
    return ti;
}

// Output coordinates (n, oy, ox) of row m of a tile's phase.
template <int MODE>
__device__ __forceinline__ void row_coords(const ConvTcArgs& g, int phase, int m, int& n, int& oy,
                                           int& ox) {
    if (MODE == PHASE_DGRAD) {
        const int hp = g.ph_hp[phase], wp = g.ph_wp[phase];
        const int per = hp * wp;
        n = m / per;
        const int rem = m - n * per;
        const int hy = rem / wp;
        oy = hy * g.str_h + g.ph_h0[phase];
        ox = (rem - hy * wp) * g.str_w + g.ph_w0[phase];
    } else {
        const int per = g.Ho * g.Wo;
        n = m / per;
        const int rem = m - n * per;
        oy = rem / g.Wo;
        ox = rem - oy * g.Wo;
    }
}

template <int BN, int STAGES, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap amap,
                   const __grid_constant__ CUtensorMap bmap,
                   const __grid_constant__ CUtensorMap ymap,
                   const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ out,
                   const __grid_constant__ ConvTcArgs g, const pk_epilogue epi) {
    using L = Smem<BN, STAGES, MODE>;
    constexpr bool kPlain = is_plain<MODE>();
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* empty = full + STAGES;
    // Narrow tiles (BN <= 64: one 64-column chunk per tile) would leave half the
    // epilogue warps idle and make the per-tile epilogue latency the loop period
    // (PK_TC_TRACE: ~2200 clk per tile on a K=64 1x1 layer); there the two
    // epilogue halves take alternate TILES instead of alternate chunks, over
    // four accumulator buffers.
    constexpr bool kSplit = BN <= 64;
    constexpr int kAccBufs = kSplit ? 4 : 2;
    uint64_t* tmem_full = empty + STAGES;          // [kAccBufs]
    uint64_t* tmem_empty = tmem_full + kAccBufs;   // [kAccBufs]
    uint64_t* bfull = tmem_empty + kAccBufs;       // resident B loaded
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kAccCols = kAccBufs * BN;  // multi-buffered accumulator
    constexpr uint32_t kTmemCols = kAccCols <= 32 ? 32 : kAccCols <= 64 ? 64 : kAccCols <= 128 ? 128
                                   : kAccCols <= 256 ? 256 : 512;

    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], kPlain ? 1 : 128 + 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < kAccBufs; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], kSplit ? 4 : 8);  // the epilogue warps that read it
        }
        mbar_init(bfull, 1);
        fence_barrier_init();
        tma_prefetch(&bmap);
        if (kPlain) tma_prefetch(&amap);
        if (MODE != PHASE_DGRAD) tma_prefetch(&ymap);
    }
    if (warp == 4) tmem_alloc(tmem_slot, kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();  // predecessor complete: inputs ready, outputs free
    pdl_trigger();

    if (warp < 4) {
      // plain GEMMs: only thread 0 of warp 0 issues TMA; warps 1-3 stay idle
      // instead of polling the stage barriers
      if (!kPlain || warp == 0) {
        // ======================= producers ==================================
        int stage = 0;
        uint32_t phase = 0;
        const int j = lane & 7;
        const int rbase = warp * 32 + (lane >> 3);
        const int chunks_per_tap = g.red_ch >> 3;
        for (int t = blockIdx.x; t < g.total_tiles; t += gridDim.x) {
            const TileInfo ti = tile_info<MODE>(g, t);
            if (ti.nkb == 0) continue;
            const int n0 = ti.n0 * BN;
            int row_img[8], row_h[8], row_w[8];
            if (!kPlain) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int m = ti.m0 + rbase + 4 * i;
                    if (m < ti.rows) {
                        int n, oy, ox;
                        row_coords<MODE>(g, ti.phase, m, n, oy, ox);
                        row_img[i] = n * g.Hs;
                        if (MODE == GATHER_FWD) {
                            row_h[i] = oy * g.str_h - g.pad_h;
                            row_w[i] = ox * g.str_w - g.pad_w;
                        } else {
                            row_h[i] = oy + g.pad_h;
                            row_w[i] = ox + g.pad_w;
                        }
                    } else {
                        row_img[i] = -1;
                        row_h[i] = row_w[i] = 0;
                    }
                }
            }
            const int tap0 = MODE == PHASE_DGRAD ? g.ph_tap_start[ti.phase] : 0;
            for (int kb = 0; kb < ti.nkb; ++kb) {
                if (kb == 0 && warp == 0) tcstamp(g, (t - blockIdx.x) / gridDim.x, 0);
                mbar_wait(&empty[stage], phase ^ 1);
                if (kb == 0 && warp == 0) tcstamp(g, (t - blockIdx.x) / gridDim.x, 1);
                uint8_t* sa = smem + stage * L::kStage;
                int r = 0, s = 0, c8 = 0, bcol = kb * BK;
                bool kvalid = true;
                if (MODE == PHASE_DGRAD) {
                    const int tap = kb / g.cpt, chunk = kb - tap * g.cpt;
                    const unsigned short rs = g.taps[tap0 + tap];
                    r = rs >> 8;
                    s = rs & 0xff;
                    c8 = chunk * 8 + j;
                    bcol = (r * g.S + s) * g.red_ch + chunk * BK;
                } else if (!kPlain) {
                    const int k8 = kb * (BK / 8) + j;
                    kvalid = k8 * 8 < g.kred;
                    if (kvalid) {
                        const int rs = k8 / chunks_per_tap;
                        c8 = k8 - rs * chunks_per_tap;
                        r = rs / g.S;
                        s = rs - r * g.S;
                    }
                }
                if (threadIdx.x == 0) {
                    if (is_res<MODE>()) {
                        if (t == (int)blockIdx.x && kb == 0) {
                            // this CTA's N tile never changes (grid % n_tiles_n == 0):
                            // load its whole B slice once
                            mbar_arrive_expect_tx(bfull, ti.nkb * L::kB);
                            for (int k = 0; k < ti.nkb; ++k) {
                                if (g.b_mn) {
                                    for (int j = 0; j < BN / 64; ++j)
                                        tma_load_2d(smem_u32(smem + L::kResOff + k * L::kB + j * 8192),
                                                    &bmap, bfull, n0 + 64 * j, k * BK);
                                } else {
                                    tma_load_2d(smem_u32(smem + L::kResOff + k * L::kB), &bmap, bfull,
                                                k * BK, n0);
                                }
                            }
                        }
                        mbar_arrive_expect_tx(&full[stage], L::kA);
                    } else {
                        mbar_arrive_expect_tx(&full[stage], kPlain ? L::kA + L::kB : L::kB);
                        const int brow = kPlain && g.b_batch_mtiles
                                             ? (ti.m0 / BM / g.b_batch_mtiles) * g.b_batch_rows
                                             : 0;
                        if (kPlain && g.b_mn) {
                            for (int j = 0; j < BN / 64; ++j)
                                tma_load_2d(smem_u32(sa + L::kA + j * 8192), &bmap, &full[stage],
                                            n0 + 64 * j, kb * BK);
                        } else {
                            tma_load_2d(smem_u32(sa + L::kA), &bmap, &full[stage], bcol, n0 + brow);
                        }
                    }
                    if (kPlain) tma_load_2d(smem_u32(sa), &amap, &full[stage], kb * BK, ti.m0);
                }
                if (!kPlain) {
                    const uint32_t sa_u = smem_u32(sa);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int row = rbase + 4 * i;
                        const uint32_t dst = sa_u + row * 128 + ((j ^ (row & 7)) << 4);
                        const __nv_bfloat16* p = src;
                        uint32_t bytes = 0;
                        if (kvalid && row_img[i] >= 0) {
                            int ih, iw;
                            bool ok;
                            if (MODE == GATHER_FWD) {
                                ih = row_h[i] + r * g.dil_h;
                                iw = row_w[i] + s * g.dil_w;
                                ok = ih >= 0 && ih < g.Hs && iw >= 0 && iw < g.Ws;
                            } else {
                                const int nh = row_h[i] - r * g.dil_h, nw = row_w[i] - s * g.dil_w;
                                ok = nh >= 0 && nw >= 0;
                                if (MODE == GATHER_DGRAD) {
                                    if (g.str_h > 1) ok = ok && (nh % g.str_h) == 0;
                                    if (g.str_w > 1) ok = ok && (nw % g.str_w) == 0;
                                }
                                ih = nh / g.str_h;
                                iw = nw / g.str_w;
                                ok = ok && ih < g.Hs && iw < g.Ws;
                            }
                            if (ok) {
                                p = src + ((size_t)(row_img[i] + ih) * g.Ws + iw) * g.src_pitch +
                                    c8 * 8;
                                bytes = 16;
                            }
                        }
                        cp_async_16(dst, p, bytes);
                    }
                    cp_async_arrive_noinc(&full[stage]);
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
      }
    } else if (warp == 4) {
        // ======================= MMA issuer ==================================
        const uint32_t idesc = (kPlain && g.f16) ? idesc_f16_f32(BM, BN, false, false)
                                                 : idesc_bf16_f32(BM, BN, false, kPlain && g.b_mn);
        // B k-step (16 k): K-major +32 B, MN-major +16 rows (2048 B); atoms 8 KB apart
        const uint64_t bks = kPlain && g.b_mn ? 128 : 2;
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        if (is_res<MODE>() && (int)blockIdx.x < g.total_tiles) mbar_wait(bfull, 0);
        for (int t = blockIdx.x; t < g.total_tiles; t += gridDim.x) {
            const TileInfo ti = tile_info<MODE>(g, t);
            if (ti.nkb == 0) continue;
            const int a = it % kAccBufs;
            const uint32_t aphase = (it / kAccBufs) & 1;
            ++it;
            tcstamp(g, it - 1, 2);
            mbar_wait(&tmem_empty[a], aphase ^ 1);
            tcstamp(g, it - 1, 3);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + a * BN;
            for (int kb = 0; kb < ti.nkb; ++kb) {
                mbar_wait(&full[stage], phase);
                if (kb == 0) tcstamp(g, it - 1, 4);
                tc_fence_after();
                {
                    fence_proxy_async_smem();
                    const uint32_t a_base = smem_u32(smem + stage * L::kStage);
                    const uint32_t b_base = is_res<MODE>()
                                                ? smem_u32(smem + L::kResOff + kb * L::kB)
                                                : a_base + L::kA;
                    const uint64_t ad0 = umma_desc_sw128(a_base, 16, 1024);
                    const uint64_t bd0 = umma_desc_sw128(b_base, kPlain && g.b_mn ? 8192 : 16, 1024);
                    if (!(g.debug & 1))
                        mma4_bf16(d_tmem, ad0, ad0 + 2, ad0 + 4, ad0 + 6, bd0, bd0 + bks, bd0 + 2 * bks,
                                  bd0 + 3 * bks, idesc, kb != 0);
                    mma_commit_elect(&empty[stage]);
                    if (kb == ti.nkb - 1) mma_commit_elect(&tmem_full[a]);
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else {
        // ======================= epilogue ====================================
        // 8 warps: two per TMEM lane quarter (warp % 4), splitting the 64-column
        // chunks between them; each stages a 32 x 64 bf16 tile in swizzled smem
        // and hands it to a TMA store (double-buffered staging per warp).
        constexpr bool kTmaStore = MODE != PHASE_DGRAD;
        const int ew = warp - 5;
        const int q = warp & 3;
        const int half = ew >> 2;
        uint8_t* stg_base = smem + L::kStagingOff + ew * L::kStgBufs * 4096;
        int sbuf = 0;
        const bool has_epi = epilogue_active(&epi);
        BnStatAcc bacc;
        bacc.init();
        int it = 0;
        for (int t = blockIdx.x; t < g.total_tiles; t += gridDim.x) {
            const TileInfo ti = tile_info<MODE>(g, t);
            const bool live = ti.nkb > 0;
            // split mode: live tiles alternate between the halves (buffers a with
            // a % 2 == half); tiles without taps (zero output, no TMEM) go to half 0
            if (kSplit && (live ? (it & 1) != half : half != 0)) {
                if (live) ++it;
                continue;
            }
            const int n0 = ti.n0 * BN;
            const int my_m = ti.m0 + q * 32 + lane;
            int my_n = 0, my_oy = 0, my_ox = 0;  // (n unused: epilogue indexes by oy, ox)
            if (my_m < ti.rows) row_coords<MODE>(g, ti.phase, my_m, my_n, my_oy, my_ox);
            int a = 0;
            if (live) {
                a = it % kAccBufs;
                const uint32_t aphase = (it / kAccBufs) & 1;
                ++it;
                if (warp == 5) tcstamp(g, it - 1, 5);
                mbar_wait(&tmem_full[a], aphase);
                if (warp == 5) tcstamp(g, it - 1, 6);
                tc_fence_after();
            }
            // 64-column chunks that reach the output (warp-uniform)
            const int span = min(BN, g.out_pitch - n0);
            const int nchunks = (span + 63) / 64;
            int my_last = -1;
            const int ci0 = kSplit ? 0 : half, cstep = kSplit ? 1 : 2;
            for (int ci = ci0; ci < nchunks; ci += cstep) my_last = ci;
            if (live && my_last < 0) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tmem_empty[a]);
            }
            const int srow0 = lane >> 3, sj = lane & 7;
#pragma unroll 1
            for (int ci = ci0; ci < nchunks; ci += cstep) {
                const int c0 = ci * 64;
                uint32_t v[64];
                if (live && (g.debug & 2)) {
#pragma unroll
                    for (int e = 0; e < 64; ++e) v[e] = lane + e;
                    if (ci == my_last) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tmem_empty[a]);
                    }
                } else if (live) {
                    const uint32_t ta = tmem_base + a * BN + c0 + (static_cast<uint32_t>(q * 32) << 16);
                    tmem_ld16(ta + 0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
                    if (BN >= 32) tmem_ld16(ta + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
                    if (BN >= 64) {
                        tmem_ld16(ta + 32, *reinterpret_cast<uint32_t(*)[16]>(&v[32]));
                        tmem_ld16(ta + 48, *reinterpret_cast<uint32_t(*)[16]>(&v[48]));
                    }
                    tmem_ld_wait();
                    if (ci == my_last) {
                        // this warp's share of the accumulator is read: release
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&tmem_empty[a]);
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 64; ++e) v[e] = 0u;
                }
                uint8_t* stg = stg_base + sbuf * 4096;
                const uint32_t stg_u = smem_u32(stg);
                if (kTmaStore) {
                    // the store issued from this buffer two chunks ago must have
                    // finished reading it
                    if (lane == 0) {
                        if (L::kStgBufs == 2)
                            bulk_wait_read<1>();
                        else
                            bulk_wait_read<0>();
                    }
                    __syncwarp();
                }
                // math + pack into the swizzled staging row of this lane
                float xf[64];
#pragma unroll
                for (int e = 0; e < 64; ++e) xf[e] = __uint_as_float(v[e]);
                if (has_epi) epilogue_chunk64(epi, xf, n0 + c0, g.n_out, my_oy, my_ox, g.Ho, g.Wo);
                pack_stage64(xf, stg_u, lane, min(g.n_out - (n0 + c0), BN - c0), kPlain && g.f16);
                if (kTmaStore) {
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if (!(g.debug & 4)) tma_store_2d(&ymap, stg_u, n0 + c0, ti.m0 + q * 32);
                        bulk_commit();
                    }
                    if (epi.stats && live) {
                        long long pix = 0;
                        if (my_m < ti.rows) {
                            int pn, py, px;
                            row_coords<MODE>(g, ti.phase, my_m, pn, py, px);
                            pix = ((long long)pn * g.Ho + py) * g.Wo + px;
                        }
                        bacc.add(epi, stg_u, lane, my_m < ti.rows, pix, (ci >> 1) & 1, n0 + c0,
                                 g.n_out, g.out_pitch);
                    }
                    if (L::kStgBufs == 2) sbuf ^= 1;
                    if (warp == 5) tcstamp(g, it - 1, 7 + (ci >> 1));
                } else {
                    __syncwarp();
                    if (epi.stats && live) {
                        long long pix = 0;
                        if (my_m < ti.rows) {
                            int pn, py, px;
                            row_coords<MODE>(g, ti.phase, my_m, pn, py, px);
                            pix = ((long long)pn * g.Ho + py) * g.Wo + px;
                        }
                        bacc.add(epi, stg_u, lane, my_m < ti.rows, pix, (ci >> 1) & 1, n0 + c0,
                                 g.n_out, g.out_pitch);
                    }
                    // coalesced stores: 4 rows x 128 B per instruction
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int row = srow0 + 4 * i;
                        const int m = ti.m0 + q * 32 + row;
                        uint4 val;
                        const uint32_t srcs = stg_u + row * 128 + ((sj ^ (row & 7)) << 4);
                        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(val.x), "=r"(val.y), "=r"(val.z), "=r"(val.w)
                                     : "r"(srcs));
                        const int ch = n0 + c0 + sj * 8;
                        if (m < ti.rows && ch < g.out_pitch && c0 + sj * 8 < BN) {
                            int n, oy, ox;
                            row_coords<MODE>(g, ti.phase, m, n, oy, ox);
                            const size_t pix = ((size_t)n * g.Ho + oy) * g.Wo + ox;
                            *reinterpret_cast<uint4*>(out + pix * g.out_pitch + ch) = val;
                        }
                    }
                    __syncwarp();
                }
            }
        }
        if (epi.stats) bacc.finish(epi, lane, g.n_out);
        if (kTmaStore && lane == 0) bulk_wait_all();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kTmemCols);
    }
}

template <int BN, int STAGES, int MODE>
cudaError_t launch(const CUtensorMap& amap, const CUtensorMap& bmap, const CUtensorMap& ymap,
                   const void* src, void* out, const ConvTcArgs& g, const pk_epilogue& e,
                   cudaStream_t st) {
    using L = Smem<BN, STAGES, MODE>;
    static_assert(L::kBytes <= 227 * 1024, "smem");
    auto kern = conv_tc_kernel<BN, STAGES, MODE>;
    static int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
        cudaError_t err =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes);
        if (err != cudaSuccess) return err;
        attr_dev = dev;
    }
    int grid = num_sms_of_current_device();
    if (is_res<MODE>()) grid = grid / g.n_tiles_n * g.n_tiles_n;  // fixed N tile per CTA
    if (g.total_tiles < grid) grid = g.total_tiles;
    if (grid < 1) grid = 1;
    cudaError_t le = pk_launch(kern, dim3(grid), dim3(kThreads), L::kBytes, st, amap, bmap, ymap,
                               (const __nv_bfloat16*)src, (__nv_bfloat16*)out, g, e);
    if (le != cudaSuccess) return le;
    if (g.trace) {
        unsigned long long h[32 * 16];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, g.trace, sizeof(h), cudaMemcpyDeviceToHost);
        for (int i = 0; i < 12; ++i) {
            fprintf(stderr, "tc tile %2d:", i);
            for (int e = 0; e < 9; ++e) fprintf(stderr, " %7lld", (long long)(h[i * 16 + e] - h[0]));
            fprintf(stderr, "\n");
        }
    }
    count_launch();
    return cudaGetLastError();
}

template <int MODE>
cudaError_t dispatch_bn(int bn, const CUtensorMap& amap, const CUtensorMap& bmap, const void* src,
                        void* out, const ConvTcArgs& g, const pk_epilogue& e, cudaStream_t st) {
    CUtensorMap ymap{};
    if (MODE != PHASE_DGRAD &&
        !tc::make_map_2d(&ymap, out, g.M, g.out_pitch, g.out_pitch, 32))
        return cudaErrorInvalidValue;
    if (MODE == PLAIN && !g.b_batch_mtiles && !g.debug_nores && bn >= 64) {
        // resident B slice when it fits (num_kb x BN x 128 bytes)
        const long long resb = (long long)g.num_kb * bn * BK * 2;
        if (resb <= 64 * 1024) {
            if (bn == 64) return launch<64, 6, PLAIN_RES>(amap, bmap, ymap, src, out, g, e, st);
            if (bn == 128) return launch<128, 6, PLAIN_RES>(amap, bmap, ymap, src, out, g, e, st);
            return launch<256, 6, PLAIN_RES>(amap, bmap, ymap, src, out, g, e, st);
        }
        if (resb <= 128 * 1024) {
            if (bn == 64) return launch<64, 4, PLAIN_RES_BIG>(amap, bmap, ymap, src, out, g, e, st);
            if (bn == 128) return launch<128, 4, PLAIN_RES_BIG>(amap, bmap, ymap, src, out, g, e, st);
            return launch<256, 4, PLAIN_RES_BIG>(amap, bmap, ymap, src, out, g, e, st);
        }
    }
    if (bn == 32) return launch<32, 8, MODE>(amap, bmap, ymap, src, out, g, e, st);
    if (bn == 64) return launch<64, 6, MODE>(amap, bmap, ymap, src, out, g, e, st);
    if (bn == 128) return launch<128, 5, MODE>(amap, bmap, ymap, src, out, g, e, st);
    return launch<256, 3, MODE>(amap, bmap, ymap, src, out, g, e, st);
}

int pick_bn(int want, int out_pitch) {
    static const int env_bn = [] {  // PK_TC_BN: tile-width experiments only
        const char* v = std::getenv("PK_TC_BN");
        return v ? std::atoi(v) : 0;
    }();
    if (env_bn) want = env_bn;
    int bn = want <= 64 ? 64 : want <= 128 ? 128 : 256;
    const int need = out_pitch <= 32 ? 32 : out_pitch <= 64 ? 64 : out_pitch <= 128 ? 128 : 256;
    return bn < need ? bn : need;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

void base_args(ConvTcArgs& t, int bn) {
    t.n_tiles_n = (t.out_pitch + bn - 1) / bn;
    static const int dbg = [] {
        const char* v = std::getenv("PK_TC_DEBUG");
        return v ? std::atoi(v) : 0;
    }();
    t.debug = dbg;
    t.debug_nores = std::getenv("PK_TC_NORES") != nullptr;
    static unsigned long long* trace = [] {
        unsigned long long* p = nullptr;
        if (std::getenv("PK_TC_TRACE")) cudaMalloc(&p, 32 * 16 * 8);
        return p;
    }();
    t.trace = trace;
}

// Sub-pixel phase tables for backward data with stride > 1.
bool build_phases(ConvTcArgs& t, int n_img, int H, int W) {
    const int sh = t.str_h, sw = t.str_w;
    if (sh * sw > kMaxPhases || t.R * t.S > kMaxTaps || t.red_ch % BK != 0) return false;
    t.num_phases = sh * sw;
    t.cpt = t.red_ch / BK;
    int tiles = 0, taps = 0;
    for (int ph = 0; ph < sh; ++ph)
        for (int pw = 0; pw < sw; ++pw) {
            const int i = ph * sw + pw;
            const int hp = H > ph ? (H - ph + sh - 1) / sh : 0;
            const int wp = W > pw ? (W - pw + sw - 1) / sw : 0;
            t.ph_hp[i] = hp;
            t.ph_wp[i] = wp;
            t.ph_h0[i] = ph;
            t.ph_w0[i] = pw;
            t.ph_rows[i] = n_img * hp * wp;
            t.ph_tile_start[i] = tiles;
            tiles += (t.ph_rows[i] + BM - 1) / BM;
            t.ph_tap_start[i] = taps;
            for (int r = 0; r < t.R; ++r) {
                const int vh = ph + t.pad_h - r * t.dil_h;
                if (((vh % sh) + sh) % sh) continue;
                for (int s = 0; s < t.S; ++s) {
                    const int vw = pw + t.pad_w - s * t.dil_w;
                    if (((vw % sw) + sw) % sw) continue;
                    t.taps[taps++] = static_cast<unsigned short>((r << 8) | s);
                }
            }
        }
    t.ph_tile_start[t.num_phases] = tiles;
    t.ph_tap_start[t.num_phases] = taps;
    t.total_tiles = tiles * t.n_tiles_n;
    return true;
}

}  // namespace
}  // namespace pk

using namespace pk;

extern "C" {

int pk_tc_fwd_supported(const pk_conv_geom* g) {
    return g->groups == 1 && !g->transpose && g->x_pitch % 8 == 0 && g->f_pitch % 8 == 0 &&
           g->y_pitch % 8 == 0 && g->r < 256 && g->s < 256 && tc::encode_fn() != nullptr;
}

int pk_tc_dgrad_supported(const pk_conv_geom* g) {
    // outputs with very few channels waste most of a 64-wide MMA tile; the
    // CUDA-core path is faster there
    return g->groups == 1 && !g->transpose && g->r < 256 && g->s < 256 &&
           tc::encode_fn() != nullptr;
}

size_t pk_tc_dgrad_workspace(const pk_conv_geom* g) {
    return (size_t)g->c * g->r * g->s * pk_pitch(g->k) * 2;  // [C][R][S][pitch(K)] bf16
}

cudaError_t pk_cuda_igemm_tc_fwd(const pk_conv_geom* g, const void* x, const void* f, void* y,
                                 const pk_epilogue* epi, const pk_tc_config* cfg,
                                 cudaStream_t st) {
    if (!pk_tc_fwd_supported(g) || !aligned16(x) || !aligned16(f) || !aligned16(y))
        return cudaErrorNotSupported;
    const ActiveTcConfig active(cfg);
    const int want_bn = cfg && cfg->block_n ? cfg->block_n : 256;
    const int family = cfg ? cfg->family : 0, pair = cfg ? cfg->pair : 0;
    // narrow-channel stems: halo-staged fused kernel (stem_fused.cu)
    static const bool stem_on = [] {
        const char* v = std::getenv("PK_STEM_FUSED");
        return !(v && v[0] == '0');
    }();
    if (stem_on && pk_cuda_stem_fused_supported(g)) return pk_cuda_stem_fused_fprop(g, x, f, y, epi, st);
    ConvTcArgs t{};
    t.M = g->n * g->p * g->q;
    t.Ho = g->p;
    t.Wo = g->q;
    t.Hs = g->h;
    t.Ws = g->w;
    t.src_pitch = g->x_pitch;
    t.red_ch = g->f_pitch;
    t.R = g->r;
    t.S = g->s;
    t.pad_h = g->pad_h;
    t.pad_w = g->pad_w;
    t.str_h = g->str_h;
    t.str_w = g->str_w;
    t.dil_h = g->dil_h;
    t.dil_w = g->dil_w;
    t.kred = g->r * g->s * g->f_pitch;
    t.num_kb = (t.kred + BK - 1) / BK;
    t.n_out = g->k;
    t.out_pitch = g->y_pitch;
    const int bn = pick_bn(want_bn, g->y_pitch);
    base_args(t, bn);
    t.total_tiles = ((t.M + BM - 1) / BM) * t.n_tiles_n;
    pk_epilogue e{};
    e.act = -1;
    if (epi) e = *epi;
    CUtensorMap amap{}, bmap{};
    if (!tc::make_map_2d(&bmap, f, g->k, t.kred, t.kred, bn)) return cudaErrorInvalidValue;
    const bool plain = g->r == 1 && g->s == 1 && g->str_h == 1 && g->str_w == 1 &&
                       g->pad_h == 0 && g->pad_w == 0 && g->x_pitch == g->f_pitch;
    if (plain) {
        // filter slice too large to stay resident: CTA-pair kernel (half the B bytes)
        static const bool pair_all = std::getenv("PK_TC2_ALL") != nullptr;  // A/B experiments
        if (bn == 256 && pair != 1 && (t.kred > 256 || pair_all || pair == 2) && !e.stats &&
            !t.debug_nores && pk_gemm_pair_eligible(t.M, t.kred, g->k, g->y_pitch))
            return pk_gemm_pair(x, f, y, t.M, t.kred, g->k, g->y_pitch, g->p, g->q, &e, st);
        if (!tc::make_map_2d(&amap, x, t.M, g->x_pitch, g->x_pitch, BM)) return cudaErrorInvalidValue;
        return dispatch_bn<PLAIN>(bn, amap, bmap, x, y, t, e, st);
    }
    // stride-1 spatial filters: halo-reuse tiles (input loaded once per tile)
    if (family < 1) {
        const cudaError_t he = pk_halo_conv(g, false, x, f, y, &e, st);
        if (he != cudaErrorNotSupported) return he;
    }
    // TMA rectangle tiles when the channel pitch is a multiple of 64
    if (family < 2) {
        const cudaError_t te = pk_tma_conv(g, false, x, f, y, &e, want_bn, st);
        if (te != cudaErrorNotSupported) return te;
    }
    return dispatch_bn<GATHER_FWD>(bn, amap, bmap, x, y, t, e, st);
}

cudaError_t pk_cuda_gemm_tc_batched(const void* a, const void* b, void* y, int batch,
                                    int rows_per_batch, int kdim, int n_out, int b_rows_per_batch,
                                    int out_pitch, cudaStream_t st, int f16) {
    if (rows_per_batch % BM || kdim % 8 || out_pitch % 8 || !aligned16(a) || !aligned16(b) ||
        !aligned16(y) || tc::encode_fn() == nullptr)
        return cudaErrorNotSupported;
    ConvTcArgs t{};
    t.M = batch * rows_per_batch;
    t.Ho = t.M;
    t.Wo = 1;
    t.Hs = t.M;
    t.Ws = 1;
    t.src_pitch = kdim;
    t.red_ch = kdim;
    t.R = t.S = 1;
    t.str_h = t.str_w = t.dil_h = t.dil_w = 1;
    t.kred = kdim;
    t.num_kb = (kdim + BK - 1) / BK;
    t.n_out = n_out;
    t.out_pitch = out_pitch;
    const int bn = pick_bn(256, out_pitch);
    base_args(t, bn);
    t.total_tiles = (t.M / BM) * t.n_tiles_n;
    t.b_batch_mtiles = rows_per_batch / BM;
    t.b_batch_rows = b_rows_per_batch;
    t.f16 = f16;
    pk_epilogue e{};
    e.act = -1;
    CUtensorMap amap{}, bmap{};
    if (!tc::make_map_2d(&bmap, b, (long long)batch * b_rows_per_batch, kdim, kdim, bn) ||
        !tc::make_map_2d(&amap, a, t.M, kdim, kdim, BM))
        return cudaErrorInvalidValue;
    return dispatch_bn<PLAIN>(bn, amap, bmap, a, y, t, e, st);
}

cudaError_t pk_cuda_igemm_tc_dgrad(const pk_conv_geom* g, const void* dy, const void* f, void* dx,
                                   void* workspace, const pk_tc_config* cfg, cudaStream_t st,
                                   const pk_epilogue* stats_epi) {
    if (!pk_tc_dgrad_supported(g) || !aligned16(dy) || !aligned16(dx)) return cudaErrorNotSupported;
    const ActiveTcConfig active(cfg);
    const int want_bn = cfg && cfg->block_n ? cfg->block_n : 256;
    const int family = cfg ? cfg->family : 0, pair = cfg ? cfg->pair : 0;
    const int kp = pk_pitch(g->k);
    const bool plain1x1 = g->r == 1 && g->s == 1 && g->str_h == 1 && g->str_w == 1 &&
                          g->pad_h == 0 && g->pad_w == 0;
    static const bool no_mn = std::getenv("PK_DGRAD_TRANSPOSE") != nullptr;  // A/B experiments
    // 1x1: the filter W[K][C] is the MN-major B operand as is (no transpose launch);
    // others: B operand Wt[c][r][s][k] = W[k][r][s][c]
    const bool mn_ok = !no_mn && g->f_pitch % 64 == 0 && g->k == kp;
    const bool b_mn = plain1x1 && mn_ok;
    if (!plain1x1 && mn_ok) {
        // spatial / strided: halo or rectangle kernels reading W directly
        pk_epilogue se{};
        se.act = -1;
        if (stats_epi) {
            se.stats = stats_epi->stats;
            se.bnb_y = stats_epi->bnb_y;
            se.bnb_gamma = stats_epi->bnb_gamma;
            se.bnb_beta = stats_epi->bnb_beta;
            se.bnb_mean = stats_epi->bnb_mean;
            se.bnb_invstd = stats_epi->bnb_invstd;
            se.bnb_relu = stats_epi->bnb_relu;
        }
        if (family < 1) {
            const cudaError_t he = pk_halo_conv(g, true, dy, f, dx, stats_epi ? &se : nullptr, st, true);
            if (he != cudaErrorNotSupported) return he;
        }
        if (family < 2) {
            const cudaError_t te = pk_tma_conv(g, true, dy, f, dx, stats_epi ? &se : nullptr, want_bn,
                                               st, true);
            if (te != cudaErrorNotSupported) return te;
        }
    }
    cudaError_t err = b_mn ? cudaSuccess : pk_cuda_filter_to_dgrad(g, PK_BF16, f, workspace, st);
    if (err != cudaSuccess) return err;
    ConvTcArgs t{};
    t.M = g->n * g->h * g->w;
    t.Ho = g->h;
    t.Wo = g->w;
    t.Hs = g->p;
    t.Ws = g->q;
    t.src_pitch = g->y_pitch;
    t.red_ch = kp;
    t.R = g->r;
    t.S = g->s;
    t.pad_h = g->pad_h;
    t.pad_w = g->pad_w;
    t.str_h = g->str_h;
    t.str_w = g->str_w;
    t.dil_h = g->dil_h;
    t.dil_w = g->dil_w;
    t.kred = g->r * g->s * kp;
    t.num_kb = (t.kred + BK - 1) / BK;
    t.n_out = g->c;
    t.out_pitch = g->x_pitch;
    const int bn = pick_bn(want_bn, g->x_pitch);
    base_args(t, bn);
    t.total_tiles = ((t.M + BM - 1) / BM) * t.n_tiles_n;
    pk_epilogue e{};
    e.act = -1;
    if (stats_epi) {  // BN statistics only: the dgrad output is never transformed
        e.stats = stats_epi->stats;
        e.bnb_y = stats_epi->bnb_y;
        e.bnb_gamma = stats_epi->bnb_gamma;
        e.bnb_beta = stats_epi->bnb_beta;
        e.bnb_mean = stats_epi->bnb_mean;
        e.bnb_invstd = stats_epi->bnb_invstd;
        e.bnb_relu = stats_epi->bnb_relu;
    }
    CUtensorMap amap{}, bmap{};
    if (b_mn) {
        t.b_mn = 1;
        if (!tc::make_map_2d(&bmap, f, g->k, g->f_pitch, g->f_pitch, 64)) return cudaErrorInvalidValue;
    } else if (!tc::make_map_2d(&bmap, workspace, g->c, t.kred, t.kred, bn)) {
        return cudaErrorInvalidValue;
    }
    const bool plain = plain1x1;
    if (plain) {
        static const bool pair_all = std::getenv("PK_TC2_ALL") != nullptr;
        if (bn == 256 && pair != 1 && (t.kred > 256 || pair_all || pair == 2) && !e.stats &&
            !t.debug_nores && pk_gemm_pair_eligible(t.M, t.kred, g->c, g->x_pitch))
            return pk_gemm_pair(dy, b_mn ? f : workspace, dx, t.M, t.kred, g->c, g->x_pitch, g->h, g->w,
                                nullptr, st, b_mn ? g->f_pitch : 0);
        if (!tc::make_map_2d(&amap, dy, t.M, g->y_pitch, g->y_pitch, BM)) return cudaErrorInvalidValue;
        return dispatch_bn<PLAIN>(bn, amap, bmap, dy, dx, t, e, st);
    }
    if (family < 1) {
        const cudaError_t he = pk_halo_conv(g, true, dy, workspace, dx, stats_epi ? &e : nullptr, st);
        if (he != cudaErrorNotSupported) return he;
    }
    if (family < 2) {
        const cudaError_t te = pk_tma_conv(g, true, dy, workspace, dx, stats_epi ? &e : nullptr,
                                           want_bn, st);
        if (te != cudaErrorNotSupported) return te;
    }
    if ((g->str_h > 1 || g->str_w > 1) && build_phases(t, g->n, g->h, g->w))
        return dispatch_bn<PHASE_DGRAD>(bn, amap, bmap, dy, dx, t, e, st);
    return dispatch_bn<GATHER_DGRAD>(bn, amap, bmap, dy, dx, t, e, st);
}

}  // extern "C"
