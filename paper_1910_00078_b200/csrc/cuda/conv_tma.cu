#include <cstdio>
// TMA-fed tcgen05 convolution kernels (sm_100a) — the fast path for layers
// whose channel pitches are multiples of 64 (every ResNet-50 / VGG-16 layer
// except the 3-channel stem).
//
// Idea: tile the output as RECTANGLES of pixels (bw x bh x bn = 128) instead
// of linear pixel ranges. For a filter tap (r, s) the A operand of a
// rectangle is then itself a rectangle of the NHWC source, shifted by the tap
// (and traversed with the convolution stride), so one 4-D TMA box load with
// out-of-bounds zero fill performs the whole im2col gather — padding
// included — with no producer threads. A single elected thread streams A and
// B (filter, 2-D box) into a multi-stage SWIZZLE_128B ring; one thread issues
// tcgen05.mma into a double-buffered TMEM accumulator; 8 epilogue warps drain
// it (fused bias/BN/activation), stage bf16 tiles in swizzled smem and write
// them with 4-D TMA stores (hardware clips partial rectangles).
//
// Backward data reuses the kernel: stride 1 is a convolution of dY with the
// transposed filter (tap offsets pad - r*dil); stride > 1 is split into
// sub-pixel phases (h mod s, w mod s), each a dense convolution over only the
// taps that reach it, written back with strided global stores.
//
// Backward weights: rectangles of 64 pixels form the reduction blocks; dY and
// the tap-shifted X rectangles arrive by TMA as MN-major operands; split-K
// over rectangles with a fixed-order fp32 reduction.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "tc_host.cuh"
#include "tc_internal.h"
#include "tc_ptx.cuh"

namespace pk {
namespace {

using namespace pk::tc;

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kMaxPhases = 16;
constexpr int kMaxTaps = 1024;
constexpr int kFpropThreads = 320;  // producer, MMA, 8 epilogue warps

struct TmaConvArgs {
    int N;
    int red_ch, cpt;          // reduction channels per tap (pitch) and 64-chunks per tap
    int S;                    // filter width (B column = (r*S + s)*red_ch)
    int mult_h, mult_w;       // source coordinate multiplier (stride for fprop, 1 for dgrad)
    int n_out, out_pitch;
    int Ho, Wo;               // full output extent
    int str_h, str_w;         // output phase strides (dgrad) / 1
    int bw, bh, bn;           // rectangle tile
    int qbw, qbh, qbn;        // per-epilogue-warp quarter sub-box
    int n_tiles_n, total_tiles;
    int num_phases;
    int mt;                   // 128-pixel M tiles per rectangle (1 or 2)
    int m_tiles, total_pairs; // PAIR: rectangle tiles (M) and pair tiles ceil(m/2) x n
    int b_mn;                 // dgrad: B = the filter itself, MN-major 64 x 64 atoms
    int phase_tma;            // PHASED: 1 = per-phase TMA store maps (num_phases <= kStoreMaps)
    int ph_tw[kMaxPhases], ph_th[kMaxPhases], ph_tn[kMaxPhases];
    int ph_tile_start[kMaxPhases + 1];
    int ph_hp[kMaxPhases], ph_wp[kMaxPhases], ph_h0[kMaxPhases], ph_w0[kMaxPhases];
    int ph_tap_start[kMaxPhases + 1];
    unsigned short taps[kMaxTaps];   // (r << 8) | s
    short off_h[kMaxTaps], off_w[kMaxTaps];
};

// MT = 128-pixel M tiles per CTA tile (2: a 256-pixel rectangle whose two
// halves are two M=128 MMAs sharing every filter (B) stage — half the B bytes
// per FLOP through TMA; needs 2 x MT x BN <= 512 TMEM columns, so BN <= 128)
template <int BN, int STAGES, int MT = 1, bool PAIR = false>
struct FSmem {
    static constexpr int kA = MT * BM * BK * 2;
    static constexpr int kB = (PAIR ? BN / 2 : BN) * BK * 2;  // PAIR: this CTA's half of B
    static constexpr int kStage = kA + kB;
    // epilogue staging per warp: double-buffered, except BN=256 where the
    // smem goes to a 4th pipeline stage instead
    static constexpr int kStgBufs = BN >= 256 ? 1 : 2;
    static constexpr int kStaging = 8 * kStgBufs * 4096;
    static constexpr int kStagingOff = STAGES * kStage;
    static constexpr int kBarOff = kStagingOff + kStaging;
    static constexpr int kBytes = kBarOff + (2 * STAGES + 4) * 8 + 16 + 1024;
};

struct RectInfo {
    int phase, n0, h0, w0, nt, ntaps, tap0;
};

// Output store maps: one 4-D map per sub-pixel phase (strided views of dX,
// so phased backward-data tiles also leave through TMA stores); only m[0]
// for unphased convolutions.
constexpr int kStoreMaps = 4;
struct alignas(64) YMaps {
    CUtensorMap m[kStoreMaps];
};

__device__ __forceinline__ RectInfo rect_info(const TmaConvArgs& g, int t) {
    RectInfo ri;
    ri.nt = t % g.n_tiles_n;
    const int mt = t / g.n_tiles_n;
    int ph = 0;
    while (ph + 1 < g.num_phases && mt >= g.ph_tile_start[ph + 1]) ++ph;
    ri.phase = ph;
    int loc = mt - g.ph_tile_start[ph];
    const int tw = g.ph_tw[ph], th = g.ph_th[ph];
    const int wi = loc % tw;
    loc /= tw;
    const int hi = loc % th;
    const int ni = loc / th;
    ri.w0 = wi * g.bw;
    ri.h0 = hi * g.bh;
    ri.n0 = ni * g.bn;
    ri.tap0 = g.ph_tap_start[ph];
    ri.ntaps = g.ph_tap_start[ph + 1] - ri.tap0;
    return ri;
}

// k-blocks of a tile: (tap, 64-channel chunk) pairs, or for NARROW sources
// (channel pitch < 64) groups of eight (tap, 8-channel) slots.
template <bool NARROW>
__device__ __forceinline__ int tile_kblocks(const TmaConvArgs& g, const RectInfo& ri) {
    return NARROW ? (ri.ntaps * g.cpt + 7) / 8 : ri.ntaps * g.cpt;
}

// PAIR (cluster of 2, cta_group::2; BN = 256, unphased, MT = 1): the pair owns
// two consecutive rectangles of one output-channel tile; each CTA loads its own
// rectangle's tap boxes and HALF of the 256 filter rows, the leader issues
// M=256 MMAs, commits are multicast and both epilogues release the leader's
// accumulator remotely.
// F32: fp32 operands as tf32 MMAs (the 3xTF32 path: operands are the hi/lo
// concatenations of tf32x3_split, read as 32 fp32 per 128-byte row, so the
// descriptors are the bf16 kernel's) and an fp32 output written directly.
template <int BN, int STAGES, bool PHASED, bool NARROW, int MT, bool PAIR = false, bool F32 = false>
__global__ void __launch_bounds__(kFpropThreads, 1)
    conv_tma_fprop_kernel(const __grid_constant__ CUtensorMap amap,
                          const __grid_constant__ CUtensorMap bmap,
                          const __grid_constant__ YMaps ymaps, __nv_bfloat16* __restrict__ out,
                          const __grid_constant__ TmaConvArgs g, const pk_epilogue epi) {
    using L = FSmem<BN, STAGES, MT, PAIR>;
    static_assert(!PAIR || (!NARROW && ((MT == 1 && BN == 256) || (MT == 2 && BN == 128))),
                  "pair variant");
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
    // tile loop: this CTA's rectangle tile of pair tile pt (PAIR) or tile pt
    const int t_first = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int t_step = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    const int t_end = PAIR ? g.total_pairs : g.total_tiles;
    auto my_tile = [&](int pt) {
        return PAIR ? ((pt / g.n_tiles_n) * 2 + (int)rank) * g.n_tiles_n + pt % g.n_tiles_n : pt;
    };
    static_assert(2 * MT * BN <= 512, "TMEM");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint64_t* tmem_empty = tmem_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kAcc = 2 * MT * BN;
    constexpr uint32_t kTmemCols = kAcc <= 32 ? 32 : kAcc <= 64 ? 64 : kAcc <= 128 ? 128
                                   : kAcc <= 256 ? 256 : 512;

    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], PAIR ? 16 : 8);
        }
        fence_barrier_init();
        tma_prefetch(&amap);
        tma_prefetch(&bmap);
        if (!PHASED || g.phase_tma)
            for (int i = 0; i < (PHASED ? g.num_phases : 1); ++i) tma_prefetch(&ymaps.m[i]);
    }
    if (warp == 1) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(kTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            tmem_alloc(tmem_slot, kTmemCols);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();  // predecessor complete: inputs ready, outputs free
    pdl_trigger();

    if (warp == 0) {
        // ---------------- TMA producer (one elected lane) -------------------
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int pt = t_first; pt < t_end; pt += t_step) {
                const RectInfo ri = rect_info(g, my_tile(pt));
                const int nkb = tile_kblocks<NARROW>(g, ri);
                const int ys = ri.h0 * g.mult_h, xs = ri.w0 * g.mult_w;
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * L::kStage;
                    if (PAIR) {
                        const int tap = kb / g.cpt, chunk = kb - tap * g.cpt;
                        const int ti = ri.tap0 + tap;
                        const unsigned short rs = g.taps[ti];
                        const uint32_t fb = smem_u32(&full[stage]) & 0xFEFFFFFFu;  // leader's
                        if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (L::kA + L::kB));
                        tma_load_4d_pair(smem_u32(sa), &amap, fb, chunk * BK, xs + g.off_w[ti],
                                         ys + g.off_h[ti], ri.n0);
                        if (g.b_mn) {
                            for (int j = 0; j < BN / 128; ++j)
                                tma_load_3d_pair(smem_u32(sa + L::kA + j * 8192), &bmap, fb,
                                                 ri.nt * BN + (int)rank * (BN / 2) + 64 * j,
                                                 (rs >> 8) * g.S + (rs & 0xff), chunk * BK);
                        } else {
                            tma_load_2d_pair(smem_u32(sa + L::kA), &bmap, fb,
                                             ((rs >> 8) * g.S + (rs & 0xff)) * g.red_ch + chunk * BK,
                                             ri.nt * BN + (int)rank * (BN / 2));
                        }
                        if (++stage == STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                        continue;
                    }
                    mbar_arrive_expect_tx(&full[stage], L::kA + L::kB);
                    if (NARROW) {
                        // eight 16-byte-row boxes, one per (tap, 8-channel group);
                        // the K order (tap, c8) is exactly the dense filter order
                        const int slots = ri.ntaps * g.cpt;
#pragma unroll 1
                        for (int j = 0; j < 8; ++j) {
                            const int slot = kb * 8 + j;
                            int cx = 0, wx = -(1 << 20), hy = 0;  // far OOB -> zeros
                            if (slot < slots) {
                                const int tap = slot / g.cpt, c8 = slot - tap * g.cpt;
                                const int ti = ri.tap0 + tap;
                                cx = c8 * 8;
                                wx = xs + g.off_w[ti];
                                hy = ys + g.off_h[ti];
                            }
                            tma_load_4d(smem_u32(sa + j * (L::kA / 8)), &amap, &full[stage], cx,
                                        wx, hy, ri.n0);
                        }
                        tma_load_2d(smem_u32(sa + L::kA), &bmap, &full[stage], kb * BK,
                                    ri.nt * BN);
                    } else {
                        const int tap = kb / g.cpt, chunk = kb - tap * g.cpt;
                        const int ti = ri.tap0 + tap;
                        const unsigned short rs = g.taps[ti];
                        tma_load_4d(smem_u32(sa), &amap, &full[stage], chunk * BK,
                                    xs + g.off_w[ti], ys + g.off_h[ti], ri.n0);
                        if (g.b_mn) {
                            for (int j = 0; j < BN / 64; ++j)
                                tma_load_3d(smem_u32(sa + L::kA + j * 8192), &bmap, &full[stage],
                                            ri.nt * BN + 64 * j, (rs >> 8) * g.S + (rs & 0xff),
                                            chunk * BK);
                        } else {
                            tma_load_2d(smem_u32(sa + L::kA), &bmap, &full[stage],
                                        ((rs >> 8) * g.S + (rs & 0xff)) * g.red_ch + chunk * BK,
                                        ri.nt * BN);
                        }
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------------------------------
      if (!PAIR || rank == 0) {
        const uint32_t idesc = F32 ? idesc_tf32_f32(BM, BN, false, false)
                                   : idesc_bf16_f32(PAIR ? 2 * BM : BM, BN, false, g.b_mn != 0);
        const uint64_t bks = g.b_mn ? 128 : 2;  // B k-step: MN-major 16 rows, K-major 32 B
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int pt = t_first; pt < t_end; pt += t_step) {
            const RectInfo ri = rect_info(g, my_tile(pt));
            const int nkb = tile_kblocks<NARROW>(g, ri);
            if (nkb == 0) continue;
            const int a = it & 1;
            const uint32_t aphase = (it >> 1) & 1;
            ++it;
            mbar_wait(&tmem_empty[a], aphase ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + a * (MT * BN);
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                {
                    // whole warp: 4 MMAs per asm block (elect inside); descriptor
                    // start fields advance by byte offset >> 4
                    const uint32_t a_base = smem_u32(smem + stage * L::kStage);
                    const uint32_t b_base = a_base + L::kA;
                    const uint64_t bd0 = umma_desc_sw128(b_base, g.b_mn ? 8192 : 16, 1024);
                    if constexpr (PAIR) {
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            // MT = 2: each CTA's 256-pixel rectangle is two M=128 halves; the
                            // pair's M=256 MMA for half mt takes half mt of both CTAs
                            const uint64_t ad0 = umma_desc_sw128(a_base + mt * BM * 128, 16, 1024);
                            mma4_bf16_pair(d_tmem + mt * BN, ad0, ad0 + 2, ad0 + 4, ad0 + 6, bd0, bd0 + bks,
                                           bd0 + 2 * bks, bd0 + 3 * bks, idesc, kb != 0);
                        }
                        mma_commit_pair(&empty[stage]);
                        if (kb == nkb - 1) mma_commit_pair(&tmem_full[a]);
                        if (++stage == STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                        continue;
                    } else {
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        // NARROW: K step k covers boxes 2k, 2k+1 (2 KB apart, LBO),
                        // 16-row core-matrix groups are 128 B apart (SBO)
                        const uint64_t ad0 = NARROW ? umma_desc_noswz(a_base, L::kA / 8, 128)
                                                    : umma_desc_sw128(a_base + mt * BM * 128, 16, 1024);
                        constexpr uint64_t as = NARROW ? (2 * (L::kA / 8)) >> 4 : 2;
                        if constexpr (F32)
                            mma4_tf32(d_tmem + mt * BN, ad0, ad0 + as, ad0 + 2 * as, ad0 + 3 * as, bd0,
                                      bd0 + bks, bd0 + 2 * bks, bd0 + 3 * bks, idesc, kb != 0);
                        else
                            mma4_bf16(d_tmem + mt * BN, ad0, ad0 + as, ad0 + 2 * as, ad0 + 3 * as, bd0,
                                      bd0 + bks, bd0 + 2 * bks, bd0 + 3 * bks, idesc, kb != 0);
                    }
                    mma_commit_elect(&empty[stage]);
                    if (kb == nkb - 1) mma_commit_elect(&tmem_full[a]);
                    }
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
      }
    } else {
        // ---------------- epilogue (8 warps) ---------------------------------
        const int ew = warp - 2;
        const int q = warp & 3;       // TMEM lane quarter accessible to this warp
        const int half = ew >> 2;     // column-chunk parity handled by this warp
        uint8_t* stg_base = smem + L::kStagingOff + ew * L::kStgBufs * 4096;
        int sbuf = 0;
        const bool has_epi = epilogue_active(&epi);
        const bool tma_st = !F32 && (!PHASED || g.phase_tma);
        BnStatAcc bacc;
        bacc.init();
        int it = 0;
        for (int pt = t_first; pt < t_end; pt += t_step) {
            const RectInfo ri = rect_info(g, my_tile(pt));
            const int n0c = ri.nt * BN;
            const bool live = ri.ntaps > 0;
            int a = 0;
            if (live) {
                a = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                ++it;
                mbar_wait(&tmem_full[a], aphase);
                tc_fence_after();
            }
#pragma unroll 1
          for (int mt = 0; mt < MT; ++mt) {
            // this lane's row inside the rectangle, and the quarter's sub-box origin
            const int row = mt * BM + q * 32 + lane;
            const int rw = row % g.bw, rh = (row / g.bw) % g.bh, rn = row / (g.bw * g.bh);
            const int q0 = mt * BM + q * 32;
            const int qw = q0 % g.bw, qh = (q0 / g.bw) % g.bh, qn = q0 / (g.bw * g.bh);
            // output coordinates of this lane's row
            const int pn = ri.n0 + rn, ph_ = ri.h0 + rh, pw_ = ri.w0 + rw;
            int oy = ph_, ox = pw_;
            bool row_ok = pn < g.N && ph_ < g.ph_hp[ri.phase] && pw_ < g.ph_wp[ri.phase];
            if (PHASED) {
                oy = ph_ * g.str_h + g.ph_h0[ri.phase];
                ox = pw_ * g.str_w + g.ph_w0[ri.phase];
            }
            const int span = min(BN, g.out_pitch - n0c);
            const int nchunks = (span + 63) / 64;
            int my_last = -1;
            if (mt == MT - 1)
                for (int ci = half; ci < nchunks; ci += 2) my_last = ci;
            if (live && mt == MT - 1 && my_last < 0) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) { if (PAIR) mbar_arrive_leader(&tmem_empty[a]); else mbar_arrive(&tmem_empty[a]); }
            }
#pragma unroll 1
            for (int ci = half; ci < nchunks; ci += 2) {
                const int c0 = ci * 64;
                uint32_t v[64];
                if (live) {
                    const uint32_t ta = tmem_base + a * (MT * BN) + mt * BN + c0 +
                                        (static_cast<uint32_t>(q * 32) << 16);
                    tmem_ld16(ta + 0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
                    if (BN >= 32) tmem_ld16(ta + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
                    if (BN >= 64) {
                        tmem_ld16(ta + 32, *reinterpret_cast<uint32_t(*)[16]>(&v[32]));
                        tmem_ld16(ta + 48, *reinterpret_cast<uint32_t(*)[16]>(&v[48]));
                    }
                    tmem_ld_wait();
                    if (ci == my_last) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) { if (PAIR) mbar_arrive_leader(&tmem_empty[a]); else mbar_arrive(&tmem_empty[a]); }
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 64; ++e) v[e] = 0u;
                }
                const uint32_t stg_u = smem_u32(stg_base + sbuf * 4096);
                if (tma_st) {
                    if (lane == 0) {
                        if (L::kStgBufs == 2)
                            bulk_wait_read<1>();
                        else
                            bulk_wait_read<0>();
                    }
                    __syncwarp();
                }
                float xf[64];
#pragma unroll
                for (int e = 0; e < 64; ++e) xf[e] = __uint_as_float(v[e]);
                if (has_epi) epilogue_chunk64(epi, xf, n0c + c0, g.n_out, oy, ox, g.Ho, g.Wo);
                if constexpr (F32) {
                    // fp32 output: each lane writes its row's 64 values (pitch in floats)
                    if (row_ok) {
                        float* dst = reinterpret_cast<float*>(out) +
                                     (((size_t)pn * g.Ho + oy) * g.Wo + ox) * g.out_pitch + n0c + c0;
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj)
                            if (n0c + c0 + jj * 4 < g.out_pitch && c0 + jj * 4 < BN)
                                reinterpret_cast<float4*>(dst)[jj] =
                                    make_float4(xf[4 * jj], xf[4 * jj + 1], xf[4 * jj + 2], xf[4 * jj + 3]);
                    }
                    continue;
                }
                pack_stage64(xf, stg_u, lane, min(g.n_out - (n0c + c0), BN - c0));
                if (tma_st) {
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_4d(&ymaps.m[PHASED ? ri.phase : 0], stg_u, n0c + c0, ri.w0 + qw, ri.h0 + qh, ri.n0 + qn);
                        bulk_commit();
                    }
                    if (epi.stats && live)
                        bacc.add(epi, stg_u, lane, row_ok, ((long long)pn * g.Ho + oy) * g.Wo + ox,
                                 (ci >> 1) & 1, n0c + c0, g.n_out, g.out_pitch);
                    if (L::kStgBufs == 2) sbuf ^= 1;
                } else {
                    __syncwarp();
                    if (epi.stats && live)
                        bacc.add(epi, stg_u, lane, row_ok, ((long long)pn * g.Ho + oy) * g.Wo + ox,
                                 (ci >> 1) & 1, n0c + c0, g.n_out, g.out_pitch);
                    // each lane owns its row: write the 128-byte chunk back from
                    // staging as 8 x 16 B (rows are strided in the output)
                    if (row_ok) {
                        __nv_bfloat16* dst = out + (((size_t)pn * g.Ho + oy) * g.Wo + ox) * g.out_pitch +
                                             n0c + c0;
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) {
                            if (n0c + c0 + jj * 8 >= g.out_pitch || c0 + jj * 8 >= BN) break;
                            uint4 val;
                            const uint32_t srcs = stg_u + lane * 128 + ((jj ^ (lane & 7)) << 4);
                            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                         : "=r"(val.x), "=r"(val.y), "=r"(val.z), "=r"(val.w)
                                         : "r"(srcs));
                            reinterpret_cast<uint4*>(dst)[jj] = val;
                        }
                    }
                    __syncwarp();
                }
            }
          }  // mt
        }
        if (epi.stats) bacc.finish(epi, lane, g.n_out);
        if (tma_st && lane == 0) bulk_wait_all();
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        if (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(kTmemCols));
        else
            tmem_dealloc(tmem_base, kTmemCols);
    }
}

// ---------------------------------------------------------------------------
// wgrad: D[k][n], n = (r, s, c); reduction over 64-pixel rectangles.
// producer, MMA, 8 epilogue warps: the drain of the fp32 tile runs after the last
// MMA (one tile per CTA), so two warps per TMEM lane quarter halve it
// (PK_WG_TRACE: 15k clk for a 256 x 256 tile with one warp per quarter)
constexpr int kWgThreads = 320;

struct TmaWgArgs {
    int K, Nn;                 // GEMM M (out channels) and N (R*S*Cp)
    int Cp, S;
    int pad_h, pad_w, str_h, str_w, dil_h, dil_w;
    int rw, rh, rn;            // reduction rectangle (product 64)
    int tw, th;                // rectangles per row / column
    int num_kb, kb_per_split;
    unsigned long long* trace;  // PK_WG_TRACE: clock64 stamps of CTA (0,0,0) (profiling only)
    // in-kernel split-K finish (single-CTA tiles, co-resident grid): barrier slot,
    // output and split count; sync == nullptr -> the host launches wgrad_sum_kernel
    unsigned int* sync;
    __nv_bfloat16* dw;
    int splits;
    long long total;
};
__device__ __forceinline__ void wgstamp(const TmaWgArgs& g, int ev) {
    if (g.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (threadIdx.x & 31) == 0)
        g.trace[ev] = clock64();
}

// MT = output-channel tiles of 128 per CTA (2: M = 256 rows sharing every B
// load, halving the L2 bytes per FLOP — the kernel is L2/TMA-throughput bound)
template <int NB, int STAGES, int MT, bool PAIR = false>
struct WSmem {
    static constexpr int kA = MT * BM * BK * 2;   // 2*MT 64-channel MN atoms of dY
    static constexpr int kB = (PAIR ? NB / 2 : NB) * BK * 2;   // MN atoms of tap-shifted X
    static constexpr int kAtom = 64 * BK * 2;
    static constexpr int kStage = kA + kB;
    static constexpr int kBarOff = STAGES * kStage;
    static constexpr int kBytes = kBarOff + (2 * STAGES + 1) * 8 + 16 + 1024;
};

// PAIR: a CTA pair (cluster of 2, cta_group::2) owns a 256 x NB tile: each CTA
// loads its 128 output-channel rows of dY and HALF of the NB filter-position
// columns of X; the leader issues M=256 MMAs (half the TMA bytes per FLOP of
// the M=256 single-CTA form, which re-reads every X column per CTA).
template <int NB, int STAGES, int MT, bool PAIR>
__global__ void __launch_bounds__(kWgThreads, 1)
    conv_tma_wgrad_kernel(const __grid_constant__ CUtensorMap dymap,
                          const __grid_constant__ CUtensorMap xmap, float* __restrict__ partial,
                          const __grid_constant__ TmaWgArgs g) {
    using L = WSmem<NB, STAGES, MT, PAIR>;
    static_assert(!PAIR || MT == 1, "pair tiles: 128 rows per CTA");
    constexpr uint32_t kCols = MT * NB <= 128 ? 128 : MT * NB <= 256 ? 256 : 512;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t rank = 0;
    if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int m0 = PAIR ? (blockIdx.x >> 1) * 2 * BM + (int)rank * BM : blockIdx.x * BM * MT;
    const int n0 = blockIdx.y * NB;
    const int split = blockIdx.z;
    const int kb_begin = split * g.kb_per_split;
    const int kb_end = min(g.num_kb, kb_begin + g.kb_per_split);

    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tmem_full, 1);
        fence_barrier_init();
        tma_prefetch(&dymap);
        tma_prefetch(&xmap);
    }
    if (warp == 1) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(kCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            tmem_alloc(tmem_slot, kCols);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR)  // the peer's barriers exist before any cross-CTA signal
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                         : "memory");
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();  // predecessor complete: inputs ready, outputs free
    pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {
            // the column blocks of B this CTA loads: (tap, channel chunk) each
            constexpr int kAtoms = (PAIR ? NB / 2 : NB) / 64;
            int bc[kAtoms], bs[kAtoms], br[kAtoms];
#pragma unroll
            for (int a = 0; a < kAtoms; ++a) {
                const int nidx = n0 + (PAIR ? (int)rank * (NB / 2) : 0) + a * 64;
                const int tap = nidx / g.Cp;
                bc[a] = nidx - tap * g.Cp;
                br[a] = tap / g.S;
                bs[a] = tap - br[a] * g.S;
            }
            int stage = 0;
            uint32_t phase = 0;
            for (int kb = kb_begin; kb < kb_end; ++kb) {
                int loc = kb;
                const int wi = loc % g.tw;
                loc /= g.tw;
                const int hi = loc % g.th;
                const int ni = loc / g.th;
                const int q0 = wi * g.rw, p0 = hi * g.rh, img0 = ni * g.rn;
                mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* sa = smem + stage * L::kStage;
                if (PAIR) {
                    // both CTAs' loads complete on the leader's stage barrier
                    const uint32_t fb = smem_u32(&full[stage]) & 0xFEFFFFFFu;
                    if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (L::kA + L::kB));
#pragma unroll
                    for (int j = 0; j < 2; ++j)
                        tma_load_4d_pair(smem_u32(sa + j * L::kAtom), &dymap, fb, m0 + 64 * j, q0, p0,
                                         img0);
#pragma unroll
                    for (int a = 0; a < kAtoms; ++a)
                        tma_load_4d_pair(smem_u32(sa + L::kA + a * L::kAtom), &xmap, fb, bc[a],
                                         q0 * g.str_w - g.pad_w + bs[a] * g.dil_w,
                                         p0 * g.str_h - g.pad_h + br[a] * g.dil_h, img0);
                } else {
                // dY atoms past K (e.g. K = 64 in an M = 128 tile) are not loaded:
                // the MMA rows they feed are never stored
                const int a_atoms = min(2 * MT, (g.K - m0 + 63) / 64);
                mbar_arrive_expect_tx(&full[stage], a_atoms * L::kAtom + L::kB);
#pragma unroll
                for (int j = 0; j < 2 * MT; ++j)
                    if (j < a_atoms)
                        tma_load_4d(smem_u32(sa + j * L::kAtom), &dymap, &full[stage], m0 + 64 * j,
                                    q0, p0, img0);
#pragma unroll
                for (int a = 0; a < kAtoms; ++a)
                    tma_load_4d(smem_u32(sa + L::kA + a * L::kAtom), &xmap, &full[stage], bc[a],
                                q0 * g.str_w - g.pad_w + bs[a] * g.dil_w,
                                p0 * g.str_h - g.pad_h + br[a] * g.dil_h, img0);
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
      if (!PAIR || rank == 0) {
        constexpr uint32_t idesc = idesc_bf16_f32(PAIR ? 2 * BM : BM, NB, true, true);
        int stage = 0;
        uint32_t phase = 0;
        wgstamp(g, 0);
        for (int kb = kb_begin; kb < kb_end; ++kb) {
            mbar_wait(&full[stage], phase);
            if (kb - kb_begin < 8) wgstamp(g, 8 + kb - kb_begin);
            tc_fence_after();
            {
                const uint32_t a_base = smem_u32(smem + stage * L::kStage);
                const uint32_t b_base = a_base + L::kA;
                const uint64_t bd0 = umma_desc_sw128(b_base, L::kAtom, 1024);
                constexpr uint64_t ks = 2048 >> 4;  // 16 MN-major K rows
                if (PAIR) {
                    const uint64_t ad0 = umma_desc_sw128(a_base, L::kAtom, 1024);
                    mma4_bf16_pair(tmem_base, ad0, ad0 + ks, ad0 + 2 * ks, ad0 + 3 * ks, bd0, bd0 + ks,
                                   bd0 + 2 * ks, bd0 + 3 * ks, idesc, kb != kb_begin);
                    mma_commit_pair(&empty[stage]);
                    if (kb == kb_end - 1) mma_commit_pair(tmem_full);
                } else {
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    const uint64_t ad0 = umma_desc_sw128(a_base + mt * 2 * L::kAtom, L::kAtom, 1024);
                    mma4_bf16(tmem_base + mt * NB, ad0, ad0 + ks, ad0 + 2 * ks, ad0 + 3 * ks, bd0,
                              bd0 + ks, bd0 + 2 * ks, bd0 + 3 * ks, idesc, kb != kb_begin);
                }
                mma_commit_elect(&empty[stage]);
                if (kb == kb_end - 1) mma_commit_elect(tmem_full);
                }
            }
            if (kb == kb_end - 1) wgstamp(g, 1);
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }
      }
    } else {
        const int q = warp & 3;
        const bool live = kb_end > kb_begin;
        if (live) {
            mbar_wait(tmem_full, 0);
            if (warp == 2) wgstamp(g, 2);
            tc_fence_after();
        }
        // drain: 64 TMEM columns per round (one wait), staged through the now
        // idle pipeline smem so every global store writes two full 256-byte
        // row segments of the partial (coalesced) instead of 32 scattered 16 B;
        // the two warps of a lane quarter take alternate 64-column rounds
        // (per-lane 256-byte bulk copies instead were no faster: all CTAs drain at
        // once, so the drain runs at the aggregate write bandwidth either way)
        static_assert(8 * 32 * 68 * 4 <= L::kBarOff, "drain staging fits the pipeline smem");
        float* stg = reinterpret_cast<float*>(smem) + (warp - 2) * 32 * 68;
        const uint32_t stg_u = smem_u32(stg);
        const int half = (warp - 2) >> 2;
#pragma unroll 1
        for (int mt = 0; mt < MT; ++mt) {
#pragma unroll 1
            for (int c0 = 64 * half; c0 < NB; c0 += 128) {
                uint32_t v[64];
                if (live) {
                    const uint32_t ta = tmem_base + mt * NB + c0 + (static_cast<uint32_t>(q * 32) << 16);
                    tmem_ld16(ta + 0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
                    tmem_ld16(ta + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
                    tmem_ld16(ta + 32, *reinterpret_cast<uint32_t(*)[16]>(&v[32]));
                    tmem_ld16(ta + 48, *reinterpret_cast<uint32_t(*)[16]>(&v[48]));
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int e = 0; e < 64; ++e) v[e] = 0u;
                }
#pragma unroll
                for (int e = 0; e < 64; e += 4)
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                                     stg_u + (lane * 68 + e) * 4),
                                 "r"(v[e]), "r"(v[e + 1]), "r"(v[e + 2]), "r"(v[e + 3])
                                 : "memory");
                __syncwarp();
                const int col = (lane & 15) * 4, nn = n0 + c0 + col;
#pragma unroll 4
                for (int i = 0; i < 16; ++i) {
                    const int r = (lane >> 4) + 2 * i;
                    const int k = m0 + mt * BM + q * 32 + r;
                    float4 val;
                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(val.x), "=f"(val.y), "=f"(val.z), "=f"(val.w)
                                 : "r"(stg_u + (r * 68 + col) * 4));
                    if (k < g.K && nn < g.Nn) {
                        float* dst = partial + ((size_t)split * g.K + k) * g.Nn + nn;
                        if (nn + 4 <= g.Nn) {
                            *reinterpret_cast<float4*>(dst) = val;
                        } else {
                            const float vv[4] = {val.x, val.y, val.z, val.w};
                            for (int e = 0; e < 4 && nn + e < g.Nn; ++e) dst[e] = vv[e];
                        }
                    }
                }
                __syncwarp();
            }
        }
        if (warp == 2) wgstamp(g, 3);
    }
    if (!PAIR && g.sync) splitk_finish(partial, g.splits, g.total, g.dw, g.sync);
    tc_fence_before();
    __syncthreads();
    if (PAIR)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                         : "memory");
    if (warp == 1) {
        tc_fence_after();
        if (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(kCols));
        else
            tmem_dealloc(tmem_base, kCols);
    }
}

// dW = sum over splits of the fp32 partials (fixed order: deterministic), four
// outputs per thread and eight splits' loads in flight before the adds.
__global__ void wgrad_sum_kernel(const float* __restrict__ partial, int splits, long long total,
                                 __nv_bfloat16* __restrict__ dw) {
    pdl_wait();
    pdl_trigger();
    const long long quads = total / 4;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < quads;
         i += (long long)gridDim.x * blockDim.x) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4* p = reinterpret_cast<const float4*>(partial) + i;
        int s = 0;
        for (; s + 8 <= splits; s += 8) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(p + (size_t)(s + u) * quads);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                acc.x += v[u].x;
                acc.y += v[u].y;
                acc.z += v[u].z;
                acc.w += v[u].w;
            }
        }
        for (; s < splits; ++s) {
            const float4 v = __ldg(p + (size_t)s * quads);
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
        __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y), hi = __floats2bfloat162_rn(acc.z, acc.w);
        reinterpret_cast<uint2*>(dw)[i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo),
                                                     *reinterpret_cast<uint32_t*>(&hi));
    }
    // tail (total not a multiple of 4)
    for (long long i = quads * 4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        float a = 0.f;
        for (int s = 0; s < splits; ++s) a += partial[(size_t)s * total + i];
        dw[i] = __float2bfloat16_rn(a);
    }
}

// ---------------------------------------------------------------------------
// host

template <int BN, int STAGES, bool PHASED, bool NARROW, int MT = 1, bool PAIR = false, bool F32 = false>
cudaError_t launch_fprop(const CUtensorMap& amap, const CUtensorMap& bmap, const YMaps& ymap,
                         void* out, const TmaConvArgs& g, const pk_epilogue& e, cudaStream_t st) {
    using L = FSmem<BN, STAGES, MT, PAIR>;
    static_assert(L::kBytes <= 227 * 1024, "smem");
    auto kern = conv_tma_fprop_kernel<BN, STAGES, PHASED, NARROW, MT, PAIR, F32>;
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
    if (PAIR) {
        grid = grid / 2 * 2;
        if (2 * g.total_pairs < grid) grid = 2 * g.total_pairs;
    } else if (g.total_tiles < grid) {
        grid = g.total_tiles;
    }
    if (grid < 1) grid = 1;
    cudaError_t le = pk_launch(kern, dim3(grid), dim3(kFpropThreads), L::kBytes, st, PAIR ? 2 : 1,
                               amap, bmap, ymap, (__nv_bfloat16*)out, g, e);
    if (le != cudaSuccess) return le;
    count_launch();
    return cudaGetLastError();
}

template <bool PHASED, bool NARROW>
cudaError_t dispatch_fprop(int bn, const CUtensorMap& amap, const CUtensorMap& bmap,
                           const YMaps& ymap, void* out, const TmaConvArgs& g,
                           const pk_epilogue& e, cudaStream_t st) {
    if (g.total_pairs > 0 && !PHASED && !NARROW && bn == 256)
        return launch_fprop<256, 6, false, false, 1, true>(amap, bmap, ymap, out, g, e, st);
    if (g.total_pairs > 0 && !PHASED && !NARROW && bn == 128 && g.mt == 2)
        return launch_fprop<128, 4, false, false, 2, true>(amap, bmap, ymap, out, g, e, st);
    if (g.total_pairs > 0 && PHASED && !NARROW && bn == 256 && g.mt == 1)
        return launch_fprop<256, 6, true, false, 1, true>(amap, bmap, ymap, out, g, e, st);
    if (g.mt == 2 && !NARROW) {
        if (bn == 64) return launch_fprop<64, 4, PHASED, false, 2>(amap, bmap, ymap, out, g, e, st);
        if (bn == 128) return launch_fprop<128, 3, PHASED, false, 2>(amap, bmap, ymap, out, g, e, st);
    }
    if (bn == 64) return launch_fprop<64, 6, PHASED, NARROW>(amap, bmap, ymap, out, g, e, st);
    if (bn == 128) return launch_fprop<128, 5, PHASED, NARROW>(amap, bmap, ymap, out, g, e, st);
    return launch_fprop<256, 4, PHASED, NARROW>(amap, bmap, ymap, out, g, e, st);
}

int choose_bn(int want, int out_pitch) {
    int bn = want <= 64 ? 64 : want <= 128 ? 128 : 256;
    const int need = out_pitch <= 64 ? 64 : out_pitch <= 128 ? 128 : 256;
    return bn < need ? bn : need;
}

// Fill tile grid / tap tables. Phases: ph in [0, sh) x [0, sw) (1 x 1 for fprop).
// even_tiles (CTA pairs over phased grids): every phase gets an even tile count, the
// extra tile sitting past the batch (n0 >= N: zero loads, clipped stores), so no pair
// straddles two phases with different tap lists.
bool fill_phases(TmaConvArgs& t, int n_img, int Ho, int Wo, int sh, int sw, int R, int S,
                 int pad_h, int pad_w, int dil_h, int dil_w, bool dgrad, bool even_tiles = false) {
    if (sh * sw > kMaxPhases || R * S > kMaxTaps) return false;
    t.num_phases = sh * sw;
    int tiles = 0, taps = 0;
    for (int ph = 0; ph < sh; ++ph)
        for (int pw = 0; pw < sw; ++pw) {
            const int i = ph * sw + pw;
            const int hp = Ho > ph ? (Ho - ph + sh - 1) / sh : 0;
            const int wp = Wo > pw ? (Wo - pw + sw - 1) / sw : 0;
            t.ph_hp[i] = hp;
            t.ph_wp[i] = wp;
            t.ph_h0[i] = ph;
            t.ph_w0[i] = pw;
            t.ph_tw[i] = (wp + t.bw - 1) / t.bw;
            t.ph_th[i] = (hp + t.bh - 1) / t.bh;
            t.ph_tn[i] = (n_img + t.bn - 1) / t.bn;
            t.ph_tile_start[i] = tiles;
            if (hp > 0 && wp > 0) {
                const int c = t.ph_tw[i] * t.ph_th[i] * t.ph_tn[i];
                tiles += even_tiles ? c + (c & 1) : c;
            }
            t.ph_tap_start[i] = taps;
            for (int r = 0; r < R; ++r) {
                int oh;
                if (dgrad) {
                    const int vh = ph + pad_h - r * dil_h;
                    if (((vh % sh) + sh) % sh) continue;
                    oh = (vh - (((vh % sh) + sh) % sh)) / sh;  // exact division
                } else {
                    oh = r * dil_h - pad_h;
                }
                for (int s = 0; s < S; ++s) {
                    int ow;
                    if (dgrad) {
                        const int vw = pw + pad_w - s * dil_w;
                        if (((vw % sw) + sw) % sw) continue;
                        ow = (vw - (((vw % sw) + sw) % sw)) / sw;
                    } else {
                        ow = s * dil_w - pad_w;
                    }
                    t.taps[taps] = static_cast<unsigned short>((r << 8) | s);
                    t.off_h[taps] = static_cast<short>(oh);
                    t.off_w[taps] = static_cast<short>(ow);
                    ++taps;
                }
            }
        }
    t.ph_tile_start[t.num_phases] = tiles;
    t.ph_tap_start[t.num_phases] = taps;
    t.total_tiles = tiles * t.n_tiles_n;
    return true;
}

void quarter_box(TmaConvArgs& t) {
    t.qbw = t.bw >= 32 ? 32 : t.bw;
    const int rem = 32 / t.qbw;
    t.qbh = t.bh >= rem ? rem : t.bh;
    t.qbn = 32 / (t.qbw * t.qbh);
}

}  // namespace
}  // namespace pk

using namespace pk;

// Forward / backward-data through the TMA rectangle path. Returns
// cudaErrorNotSupported (without launching) when the geometry does not fit.
namespace pk {
namespace {
cudaError_t tma_conv_impl(const pk_conv_geom* g, bool dgrad, const void* src, const void* filt,
                          void* out, const pk_epilogue* epi, int bn_want, cudaStream_t st,
                          bool filt_mn, bool f32) {
    if (g->groups != 1 || g->transpose || g->r > 255 || g->s > 255) return cudaErrorNotSupported;
    if (f32 && (dgrad || filt_mn || g->x_pitch % 64)) return cudaErrorNotSupported;
    const int src_pitch = dgrad ? g->y_pitch : g->x_pitch;
    const int out_pitch = dgrad ? g->x_pitch : g->y_pitch;
    // narrow sources (pitch < 64, e.g. the 3-channel stem) use 16-byte-row boxes
    const bool narrow = src_pitch % 64 != 0;
    if (narrow && (src_pitch > 56 || src_pitch % 8 != 0)) return cudaErrorNotSupported;
    // narrow k-blocks assume the dense tap order (all taps): not for dgrad phases
    if (narrow && dgrad && (g->str_h > 1 || g->str_w > 1)) return cudaErrorNotSupported;
    if (!dgrad && g->f_pitch != g->x_pitch) return cudaErrorNotSupported;
    TmaConvArgs t{};
    t.N = g->n;
    t.red_ch = src_pitch;
    t.cpt = narrow ? src_pitch / 8 : src_pitch / 64;
    t.S = g->s;
    t.n_out = dgrad ? g->c : g->k;
    t.out_pitch = out_pitch;
    t.Ho = dgrad ? g->h : g->p;
    t.Wo = dgrad ? g->w : g->q;
    const int sh = dgrad ? g->str_h : 1, sw = dgrad ? g->str_w : 1;
    t.str_h = sh;
    t.str_w = sw;
    t.mult_h = dgrad ? 1 : g->str_h;
    t.mult_w = dgrad ? 1 : g->str_w;
    const int hp0 = (t.Ho + sh - 1) / sh, wp0 = (t.Wo + sw - 1) / sw;
    // PK_TMA_BN (64/128/256) overrides the tile width for tuning experiments
    static const int env_bn = [] {
        const char* v = std::getenv("PK_TMA_BN");
        return v ? std::atoi(v) : 0;
    }();
    const int bn = choose_bn(env_bn ? env_bn : bn_want, out_pitch);
    // 256-pixel rectangles (two M=128 MMAs per filter stage) when the tile
    // width leaves TMEM room for two double-buffered accumulators
    static const bool mt_off = std::getenv("PK_TMA_MT1") != nullptr;
    const int cfg_mt = cfg_field(&pk_tc_config::mt), cfg_pair = cfg_field(&pk_tc_config::pair);
    // phased (strided dgrad) tiles too: their few k-blocks (1-4 taps x chunks) leave the
    // per-tile handshakes dominant, and 256-pixel tiles halve them (PK_TMA_MT2_PHASED=0: off)
    static const bool mt_phased_off = [] {
        const char* v = std::getenv("PK_TMA_MT2_PHASED");
        return v && v[0] == '0';
    }();
    t.mt = (!f32 && !mt_off && cfg_mt != 1 && !narrow && ((sh == 1 && sw == 1) || !mt_phased_off) &&
            bn <= 128) ? 2 : 1;
    const RectTile rt = tc::best_rect(g->n, hp0, wp0, BM * t.mt);
    t.bw = rt.bw;
    t.bh = rt.bh;
    t.bn = rt.bn;
    quarter_box(t);
    t.n_tiles_n = (out_pitch + bn - 1) / bn;
    // CTA pairs over the sub-pixel phases of strided backward data, 256-wide tiles (measured
    // conv4_1b 60.6 -> 55.9, conv5_1b 58.9 -> 51.3, conv4_1ds 83.7 -> 78.0 us; PK_TMA_PAIR_PHASED=0: off)
    static const bool pair_phased_off = [] {
        const char* v = std::getenv("PK_TMA_PAIR_PHASED");
        return v && v[0] == '0';
    }();
    const int cfg_pair0 = cfg_field(&pk_tc_config::pair);
    const bool pair_phased = (sh > 1 || sw > 1) && !pair_phased_off && !f32 && !narrow && cfg_pair0 != 1 &&
                             !(std::getenv("PK_TMA_PAIR") && std::getenv("PK_TMA_PAIR")[0] == '0') &&
                             bn == 256 && t.mt == 1 &&  // 128-wide phased pairs measured slower (conv3_1b 86 -> 95 us)
                             (!epi || !epi->stats) && !(filt_mn && bn == 64);
    if (!fill_phases(t, g->n, t.Ho, t.Wo, sh, sw, g->r, g->s, g->pad_h, g->pad_w, g->dil_h,
                     g->dil_w, dgrad, pair_phased))
        return cudaErrorNotSupported;
    CUtensorMap amap{}, bmap{};
    YMaps ymap{};
    const int Hs = dgrad ? g->p : g->h, Ws = dgrad ? g->q : g->w;
    if (!tc::make_map_nhwc(&amap, src, g->n, Hs, Ws, src_pitch, t.bw, t.bh, t.bn, t.mult_w,
                           t.mult_h, narrow ? 8 : 64))
        return cudaErrorNotSupported;
    const long long kred = (long long)g->r * g->s * src_pitch;
    // CTA pairs for 256-wide tiles of unphased spatial convolutions (PK_TMA_PAIR=0 disables)
    static const bool pair_off = [] {
        const char* v = std::getenv("PK_TMA_PAIR");
        return v && v[0] == '0';
    }();
    t.m_tiles = t.n_tiles_n ? t.total_tiles / t.n_tiles_n : 0;
    t.total_pairs = 0;
    // 128-wide tiles with 256-pixel rectangles as CTA pairs: per SM the MMAs read A + B/2
    // instead of A + B from shared memory, which bounds the single-CTA form (measured ResNet
    // conv3_x 3x3 fwd and dgrad 57.3 -> 53.6 us; PK_TMA_PAIR_MT2=0 disables)
    static const bool pair_mt2 = !(std::getenv("PK_TMA_PAIR_MT2") && std::getenv("PK_TMA_PAIR_MT2")[0] == '0');
    if (pair_phased) {
        t.total_pairs = t.m_tiles / 2 * t.n_tiles_n;
    } else if (pair_mt2 && !f32 && !pair_off && cfg_pair != 1 && !narrow && sh == 1 && sw == 1 && bn == 128 &&
        t.mt == 2 && g->r * g->s > 1 && (!epi || !epi->stats))
        t.total_pairs = (t.m_tiles + 1) / 2 * t.n_tiles_n;
    else if (!f32 && !pair_off && cfg_pair != 1 && !narrow && sh == 1 && sw == 1 && bn == 256 && t.mt == 1 &&
        g->r * g->s > 1 && (!epi || !epi->stats) &&
        (cfg_pair == 2 || (long long)((t.m_tiles + 1) / 2) * t.n_tiles_n >= 74))
        t.total_pairs = (t.m_tiles + 1) / 2 * t.n_tiles_n;
    if (filt_mn) {
        // narrow sources use the dense tap order (not supported here); the filter
        // rows (output channels of the forward conv) must cover whole 64-k chunks
        if (!dgrad || narrow || g->f_pitch % 64 || (bn == 64 && t.total_pairs)) return cudaErrorNotSupported;
        t.b_mn = 1;
        if (!tc::make_map_filter_mn(&bmap, filt, g->k, g->r * g->s, g->f_pitch))
            return cudaErrorInvalidValue;
    } else if (!tc::make_map_2d(&bmap, filt, t.n_out, kred, kred, t.total_pairs ? bn / 2 : bn)) {
        return cudaErrorInvalidValue;
    }
    const bool phased = sh > 1 || sw > 1;
    if (!phased &&
        !tc::make_map_nhwc(&ymap.m[0], out, g->n, t.Ho, t.Wo, out_pitch, t.qbw, t.qbh, t.qbn))
        return cudaErrorInvalidValue;
    if (phased && t.num_phases <= kStoreMaps) {
        // phase (ph, pw) of dX as a strided 4-D view: dims (pitch, wp, hp, n)
        t.phase_tma = 1;
        for (int i = 0; i < t.num_phases; ++i) {
            if (t.ph_hp[i] == 0 || t.ph_wp[i] == 0) continue;  // no tiles in this phase
            const void* base = static_cast<const __nv_bfloat16*>(out) +
                               ((size_t)t.ph_h0[i] * t.Wo + t.ph_w0[i]) * out_pitch;
            if (!tc::make_map_nhwc_strided(&ymap.m[i], base, g->n, t.ph_hp[i], t.ph_wp[i],
                                           out_pitch, (long long)sw * out_pitch,
                                           (long long)sh * t.Wo * out_pitch,
                                           (long long)t.Ho * t.Wo * out_pitch, t.qbw, t.qbh, t.qbn)) {
                t.phase_tma = 0;
                break;
            }
        }
    }
    pk_epilogue e{};
    e.act = -1;
    if (epi) e = *epi;
    if (f32) {
        if (phased || narrow || e.stats) return cudaErrorNotSupported;
        if (bn == 64) return launch_fprop<64, 6, false, false, 1, false, true>(amap, bmap, ymap, out, t, e, st);
        if (bn == 128) return launch_fprop<128, 5, false, false, 1, false, true>(amap, bmap, ymap, out, t, e, st);
        return launch_fprop<256, 4, false, false, 1, false, true>(amap, bmap, ymap, out, t, e, st);
    }
    if (narrow)
        return phased ? dispatch_fprop<true, true>(bn, amap, bmap, ymap, out, t, e, st)
                      : dispatch_fprop<false, true>(bn, amap, bmap, ymap, out, t, e, st);
    return phased ? dispatch_fprop<true, false>(bn, amap, bmap, ymap, out, t, e, st)
                  : dispatch_fprop<false, false>(bn, amap, bmap, ymap, out, t, e, st);
}

// 3xTF32 operand split: x_cat[pix][3Cp] = (hi(x), hi(x), lo(x)), w_cat[k][tap][3Cp] =
// (hi(w), lo(w), hi(w)), hi = x rounded to tf32 (10-bit mantissa, low 13 bits zero),
// lo = x - hi (exact in fp32). One GEMM over the 3Cp "channels" then sums
// hi.hi + hi.lo + lo.hi: the fp32 product up to lo.lo (~2^-22 relative).
__device__ __forceinline__ float tf32_hi(float v) {
    uint32_t u = __float_as_uint(v);
    if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;  // RNE-ish (ties up)
    return __uint_as_float(u);
}
__global__ void tf32x3_split_kernel(const float4* __restrict__ src, float4* __restrict__ dst, long long rows,
                                    int cp4, int order) {
    const long long total = rows * cp4;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / cp4;
        const int c = (int)(i - r * cp4);
        const float4 v = src[i];
        const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
        const float4 l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        float4* row = dst + r * 3 * cp4 + c;
        row[0] = h;                        // block 0: hi (both operands)
        row[cp4] = order ? l : h;          // block 1: x: hi, w: lo
        row[2 * cp4] = order ? h : l;      // block 2: x: lo, w: hi
    }
}
}  // namespace
}  // namespace pk

cudaError_t pk_tma_conv(const pk_conv_geom* g, bool dgrad, const void* src, const void* filt,
                        void* out, const pk_epilogue* epi, int bn_want, cudaStream_t st,
                        bool filt_mn) {
    return pk::tma_conv_impl(g, dgrad, src, filt, out, epi, bn_want, st, filt_mn, false);
}

extern "C" {
// Reduction depth limit: the tensor core's fp32 accumulation is not round-to-nearest,
// and its error grows with the number of accumulated products. Measured: R*S*C = 576
// and 1152 stay inside the reference's max-rel 1e-4 (proj/tests/acceptance.cpp:137);
// 5x5 x 64 (1600, 4800 tf32 products) reached 2.6e-4, so deeper reductions stay on the
// fp32 FMA kernels.
int pk_tf32x3_fwd_supported(const pk_conv_geom* g) {
    return g->groups == 1 && !g->transpose && g->x_pitch % 32 == 0 && g->f_pitch == g->x_pitch &&
           g->r <= 255 && g->s <= 255 && g->y_pitch % 4 == 0 && g->r * g->s * g->x_pitch <= 1152 &&
           tc::encode_fn() != nullptr;
}

size_t pk_tf32x3_fwd_workspace(const pk_conv_geom* g) {
    const size_t xb = (size_t)g->n * g->h * g->w * 3 * g->x_pitch * 4;
    const size_t wb = (size_t)g->k * g->r * g->s * 3 * g->f_pitch * 4;
    return (xb + 255) / 256 * 256 + wb;
}

// fp32 forward convolution on the tensor cores with fp32-level accuracy (3xTF32).
cudaError_t pk_cuda_tf32x3_fwd(const pk_conv_geom* g, const void* x, const void* w, void* y,
                               const pk_epilogue* epi, void* workspace, size_t ws_bytes, cudaStream_t st) {
    if (!pk_tf32x3_fwd_supported(g) || ws_bytes < pk_tf32x3_fwd_workspace(g)) return cudaErrorNotSupported;
    const size_t xb = (size_t)g->n * g->h * g->w * 3 * g->x_pitch * 4;
    float* xcat = static_cast<float*>(workspace);
    float* wcat = reinterpret_cast<float*>(static_cast<char*>(workspace) + (xb + 255) / 256 * 256);
    const long long xrows = (long long)g->n * g->h * g->w, wrows = (long long)g->k * g->r * g->s;
    const int cp4 = g->x_pitch / 4;
    auto blocks = [](long long n) { return (unsigned)std::min<long long>((n + 255) / 256, 148LL * 16); };
    cudaError_t err = pk_launch(tf32x3_split_kernel, dim3(blocks(xrows * cp4)), dim3(256), 0, st,
                                (const float4*)x, (float4*)xcat, xrows, cp4, 0);
    if (err != cudaSuccess) return err;
    count_launch();
    err = pk_launch(tf32x3_split_kernel, dim3(blocks(wrows * cp4)), dim3(256), 0, st, (const float4*)w,
                    (float4*)wcat, wrows, cp4, 1);
    if (err != cudaSuccess) return err;
    count_launch();
    // the concatenations viewed as bf16 tensors of 6 x pitch elements per pixel / filter tap
    pk_conv_geom g2 = *g;
    g2.x_pitch = g2.f_pitch = 6 * g->x_pitch;
    return pk::tma_conv_impl(&g2, false, xcat, wcat, y, epi, 256, st, false, true);
}
}  // extern "C"

// One wave: split-K so that tiles x splits fills the SMs once (no tail wave);
// at least 4 k-blocks per split.
static int tma_wgrad_splits(int tiles_mn, int num_kb, int num_sms) {
    int splits = num_sms / tiles_mn;
    const int max_splits = num_kb / 4 > 1 ? num_kb / 4 : 1;
    if (splits > max_splits) splits = max_splits;
    if (splits < 1) splits = 1;
    // tuned split-K: scale the one-wave count by split/4 (at least 2 k-blocks per split)
    if (const int k = cfg_field(&pk_tc_config::split)) {
        splits = splits * k / 4;
        const int cap = num_kb / 2 > 1 ? num_kb / 2 : 1;
        if (splits > cap) splits = cap;
        if (splits < 1) splits = 1;
    }
    return splits;
}

// Filter-position tile width 256 and two output-channel tiles per CTA
// (M = 256) whenever the layer is wide enough: more MMA work per byte pulled
// through L2 (the bound of this kernel). PK_WG_TILE=128x1 etc. overrides.
struct WgTile {
    int nb, mt;
    bool pair;  // CTA-pair M=256 tiles (cta_group::2): nb = 256, mt = 1 per CTA
};
static WgTile wgrad_tile(const pk_conv_geom* g) {
    static const char* env = std::getenv("PK_WG_TILE");
    const int nn = g->r * g->s * g->x_pitch;
    WgTile t{nn >= 256 ? 256 : 128, g->k >= 256 ? 2 : 1, false};
    // 3 taps x 64 channels (3x3 filters on 64-channel inputs): 192-wide tiles
    // cover the 576 filter positions exactly (256-wide ones waste 25%)
    if (nn % 256 != 0 && nn % 192 == 0 && nn <= 768 && t.mt == 1) t.nb = 192;
    // measured (B200, all ResNet-50 layers): 1x1 stride-1 layers are fastest
    // with 128-wide filter tiles (smaller fp32 partials to drain and sum)
    if (g->r == 1 && g->s == 1 && g->str_h == 1 && g->str_w == 1) t.nb = 128;
    // ...except few pixels against wide filters (ResNet conv5 1x1: 12544 pixels, 512 x 2048):
    // 256-wide tiles halve the bytes per FLOP there (measured 35 -> 32 us)
    if (t.nb == 128 && t.mt == 2 && g->r == 1 && g->s == 1 && (long long)g->n * g->p * g->q <= 16384 &&
        nn >= 512)
        t.nb = 256;
    // tuned choices (pk_tc_config): tile width, one or two M tiles, CTA pairs
    if (const int bn = cfg_field(&pk_tc_config::block_n); bn == 128 || bn == 256) t.nb = bn;
    if (const int mt = cfg_field(&pk_tc_config::mt); mt == 1 || (mt == 2 && g->k >= 256)) t.mt = mt;
    if (t.nb == 192 && t.mt == 2) t.nb = 256;
    if (env) {
        int nb = 0, mt = 0;
        if (std::sscanf(env, "%dx%d", &nb, &mt) == 2 && (nb == 128 || nb == 256 || (nb == 192 && mt == 1)) &&
            (mt == 1 || mt == 2))
            t = {nb, mt, false};
    }
    // CTA pairs: each SM loads its 128 dY rows and half of a 256-wide X tile
    static const int pair_env = [] {
        const char* v = std::getenv("PK_WG_PAIR");
        return v ? std::atoi(v) : -1;
    }();
    // measured (ResNet-50 N=256): 1x1 layers gain 3-15% (conv3_1ds 71 -> 61 us), 3x3 lose
    const bool pair_ok = g->k % 256 == 0 && nn % 256 == 0;
    const int cfg_pair = cfg_field(&pk_tc_config::pair);
    if (pair_ok && cfg_pair != 1 &&
        (pair_env == 1 || cfg_pair == 2 || (pair_env != 0 && g->r * g->s == 1)))
        t = {256, 1, true};
    return t;
}

// 1x1, stride 1, no padding: the reduction runs over plain pixel ranges, so
// both operands are contiguous [pixels][channels] matrices (64-pixel boxes of
// 8 KB, no rectangle padding or short runs).
static bool wgrad_linear(const pk_conv_geom* g) {
    return g->r == 1 && g->s == 1 && g->str_h == 1 && g->str_w == 1 && g->pad_h == 0 &&
           g->pad_w == 0 && (long long)g->n * g->p * g->q < (1LL << 31);
}

static void wgrad_geometry(const pk_conv_geom* g, int* tiles_mn, int* num_kb, RectTile* rt) {
    if (wgrad_linear(g)) {
        *rt = RectTile{BK, 1, 1};
        *num_kb = (int)(((long long)g->n * g->p * g->q + BK - 1) / BK);
    } else {
        *rt = tc::best_rect(g->n, g->p, g->q, BK);
        const int tw = (g->q + rt->bw - 1) / rt->bw, th = (g->p + rt->bh - 1) / rt->bh;
        const int tn = (g->n + rt->bn - 1) / rt->bn;
        *num_kb = tw * th * tn;
    }
    const int nn = g->r * g->s * g->x_pitch;
    const WgTile wt = wgrad_tile(g);
    *tiles_mn = ((g->k + BM * wt.mt - 1) / (BM * wt.mt)) * ((nn + wt.nb - 1) / wt.nb);
}

template <int NB, int STAGES, int MT, bool PAIR = false>
cudaError_t launch_wgrad(const CUtensorMap& dymap, const CUtensorMap& xmap, float* partial,
                         const TmaWgArgs& w, int splits, cudaStream_t st) {
    using L = WSmem<NB, STAGES, MT, PAIR>;
    static_assert(L::kBytes <= 227 * 1024, "smem");
    static int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
        cudaError_t err = cudaFuncSetAttribute(conv_tma_wgrad_kernel<NB, STAGES, MT, PAIR>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               L::kBytes);
        if (err != cudaSuccess) return err;
        attr_dev = dev;
    }
    dim3 grid(PAIR ? 2 * ((w.K + 2 * BM - 1) / (2 * BM)) : (w.K + BM * MT - 1) / (BM * MT),
              (w.Nn + NB - 1) / NB, splits);
    cudaError_t le = pk_launch(conv_tma_wgrad_kernel<NB, STAGES, MT, PAIR>, grid, dim3(kWgThreads),
                               L::kBytes, st, PAIR ? 2 : 1, dymap, xmap, partial, w);
    if (le != cudaSuccess) return le;
    return cudaGetLastError();
}

size_t pk_tma_wgrad_workspace(const pk_conv_geom* g, int num_sms) {
    if (const int hs = pk_halo_wgrad_splits(g, num_sms))
        return (size_t)hs * g->k * g->r * g->s * g->x_pitch * 4;
    int tiles_mn, num_kb;
    RectTile rt;
    wgrad_geometry(g, &tiles_mn, &num_kb, &rt);
    return (size_t)tma_wgrad_splits(tiles_mn, num_kb, num_sms) * g->k * g->r * g->s * g->x_pitch * 4;
}

bool pk_tma_wgrad_supported(const pk_conv_geom* g) {
    // B column blocks must stay inside one tap unless the filter is 1x1; the
    // dY (M) and channel boxes tolerate ragged tails through OOB zero fill
    return g->groups == 1 && !g->transpose &&
           (g->x_pitch % 64 == 0 || (g->r == 1 && g->s == 1)) && g->y_pitch % 8 == 0 &&
           g->f_pitch == g->x_pitch && g->str_h * 1 <= 8 && g->str_w <= 8 &&
           tc::encode_fn() != nullptr;
}

cudaError_t pk_tma_wgrad(const pk_conv_geom* g, const void* dy, const void* x, void* dw,
                         void* workspace, int num_sms, cudaStream_t st) {
    if (!pk_tma_wgrad_supported(g)) return cudaErrorNotSupported;
    if (const int hs = pk_halo_wgrad_splits(g, num_sms)) {
        // 64-channel spatial filters: padded-grid halo kernel + deterministic split sum
        unsigned int* sync = splitk_sync_slot();
        cudaError_t le = pk_halo_wgrad(g, dy, x, static_cast<float*>(workspace), hs, st,
                                       static_cast<__nv_bfloat16*>(dw), sync);
        if (le != cudaErrorNotSupported) {
            if (le != cudaSuccess) return le;
            if (sync) return cudaSuccess;  // finished in-kernel
            const long long total = (long long)g->k * g->r * g->s * g->x_pitch;
            long long blocks = (total / 4 + 255) / 256;  // one float4 of output per thread
            if (blocks < 1) blocks = 1;
            if (blocks > 148 * 16) blocks = 148 * 16;
            le = pk_launch(wgrad_sum_kernel, dim3((unsigned)blocks), dim3(256), 0, st,
                           (const float*)workspace, hs, total, (__nv_bfloat16*)dw);
            count_launch();
            return le != cudaSuccess ? le : cudaGetLastError();
        }
    }
    int tiles_mn, num_kb;
    RectTile rt;
    wgrad_geometry(g, &tiles_mn, &num_kb, &rt);
    TmaWgArgs w{};
    w.K = g->k;
    w.Cp = g->x_pitch;
    w.S = g->s;
    w.Nn = g->r * g->s * g->x_pitch;
    w.pad_h = g->pad_h;
    w.pad_w = g->pad_w;
    w.str_h = g->str_h;
    w.str_w = g->str_w;
    w.dil_h = g->dil_h;
    w.dil_w = g->dil_w;
    const bool lin = wgrad_linear(g);
    // linear: one image of one row holding all N*P*Q pixels
    const int vn = lin ? 1 : g->n, vp = lin ? 1 : g->p, vq = lin ? g->n * g->p * g->q : g->q;
    w.rw = rt.bw;
    w.rh = rt.bh;
    w.rn = rt.bn;
    w.tw = (vq + rt.bw - 1) / rt.bw;
    w.th = (vp + rt.bh - 1) / rt.bh;
    w.num_kb = num_kb;
    static unsigned long long* trace = [] {
        unsigned long long* p = nullptr;
        if (std::getenv("PK_WG_TRACE")) cudaMalloc(&p, 32 * 8);
        return p;
    }();
    w.trace = trace;
    const int splits = tma_wgrad_splits(tiles_mn, num_kb, num_sms);
    w.kb_per_split = (num_kb + splits - 1) / splits;
    CUtensorMap dymap{}, xmap{};
    if (!tc::make_map_nhwc(&dymap, dy, vn, vp, vq, g->y_pitch, rt.bw, rt.bh, rt.bn))
        return cudaErrorNotSupported;
    if (!tc::make_map_nhwc(&xmap, x, lin ? 1 : g->n, lin ? 1 : g->h, lin ? vq : g->w, g->x_pitch,
                           rt.bw, rt.bh, rt.bn, g->str_w, g->str_h))
        return cudaErrorNotSupported;
    const WgTile wt = wgrad_tile(g);
    w.dw = static_cast<__nv_bfloat16*>(dw);
    w.splits = splits;
    w.total = (long long)w.K * w.Nn;
    // in-kernel finish pays for small outputs (launch saved); large ones want the
    // full-GPU sum kernel (measured: conv2 wgrads -7 us each, conv4/5 3x3 +8 us)
    static const long long fuse_max = [] {  // PK_SPLITK_FUSE_MAX: output-size cap (A/B only)
        const char* v = std::getenv("PK_SPLITK_FUSE_MAX");
        return v ? std::atoll(v) : 65536LL;
    }();
    if (!wt.pair && (long long)tiles_mn * splits <= num_sms && w.total <= fuse_max)
        w.sync = splitk_sync_slot();
    cudaError_t le;
    if (wt.mt == 2)
        le = wt.nb == 256 ? launch_wgrad<256, 3, 2>(dymap, xmap, (float*)workspace, w, splits, st)
                          : launch_wgrad<128, 4, 2>(dymap, xmap, (float*)workspace, w, splits, st);
    else if (wt.pair)
        le = launch_wgrad<256, 6, 1, true>(dymap, xmap, (float*)workspace, w, splits, st);
    else if (wt.nb == 192)
        le = launch_wgrad<192, 5, 1>(dymap, xmap, (float*)workspace, w, splits, st);
    else
        le = wt.nb == 256 ? launch_wgrad<256, 4, 1>(dymap, xmap, (float*)workspace, w, splits, st)
                          : launch_wgrad<128, 6, 1>(dymap, xmap, (float*)workspace, w, splits, st);
    if (le != cudaSuccess) return le;
    if (w.trace) {
        unsigned long long h[32];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, w.trace, sizeof(h), cudaMemcpyDeviceToHost);
        fprintf(stderr, "wg: kb/split %d, mma start 0, last commit %lld, drain start %lld end %lld | first kb fulls:",
                w.kb_per_split, (long long)(h[1] - h[0]), (long long)(h[2] - h[0]), (long long)(h[3] - h[0]));
        for (int e = 8; e < 16; ++e) fprintf(stderr, " %lld", (long long)(h[e] - h[0]));
        fprintf(stderr, "\n");
    }
    if (w.sync && !wt.pair) {  // finished in-kernel
        count_launch();
        return cudaGetLastError();
    }
    const long long total = (long long)w.K * w.Nn;
    long long blocks = (total / 4 + 255) / 256;  // one float4 of output per thread
    if (blocks < 1) blocks = 1;
    if (blocks > 148 * 16) blocks = 148 * 16;
    le = pk_launch(wgrad_sum_kernel, dim3((unsigned)blocks), dim3(256), 0, st, (const float*)workspace,
                   splits, total, (__nv_bfloat16*)dw);
    count_launch(2);
    return le != cudaSuccess ? le : cudaGetLastError();
}
