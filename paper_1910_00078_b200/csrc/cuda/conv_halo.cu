// Halo-reuse tcgen05 convolution for stride-1 spatial filters (3x3 layers of
// ResNet/VGG, forward and backward-data).
//
// The rectangle kernel (conv_tma.cu) fetches one shifted A box per filter
// tap, so a 3x3 layer pulls every input pixel through L2 nine times — the
// kernel is L2-bound for narrow layers (64-128 channels). Here the output is
// tiled along the ROW-MAJOR PADDED GRID of each image (rows H + 2*pad, columns
// Wg = W + 2*pad): tile = 128 consecutive grid positions p. The input of tap
// (r, s) for position p is grid position p + r*Wg + s, so for every tap the
// A operand is the SAME halo buffer (whole padded grid rows, one TMA box with
// out-of-bounds zero fill) viewed from a different starting row — the tensor
// core applies the 128B swizzle on absolute smem address bits, so a
// descriptor may start at any 128-byte row (verified, tools/probes/
// shift_probe.cu). Each 64-channel chunk of input is loaded once per tile;
// only the filter slice streams per tap. Positions in the last S-1 grid
// columns are not outputs (3.4% of a 56-wide tile row) and are dropped by the
// epilogue.
//
// Backward data at stride 1 is the same convolution of dY with the
// transposed filter, taps flipped (grid pad R-1-pad).
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc_host.cuh"
#include "tc_internal.h"
#include "tc_ptx.cuh"

namespace pk {
namespace {

using namespace pk::tc;

constexpr int kM = 128;
constexpr int kHThreads = 320;  // producer, MMA, 8 epilogue warps
constexpr int kHaloBufs = 2;

struct HaloArgs {
    int N, Hg, Wg, Ho, Wo;       // grid rows/cols per image, output extent
    int pad_h, pad_w;            // grid origin in input coordinates
    int R, S;
    int red_ch, cpt;             // reduction channel pitch, 64-channel chunks
    int n_out, out_pitch;
    int tiles_img, total_tiles, n_tiles_n;
    int NR;                      // halo rows per tile (box height)
    int flip;                    // dgrad: tap (r,s) uses filter tap (R-1-r, S-1-s)
    int debug;                   // PK_HALO_DEBUG (timing experiments only): 1 = 8-row-aligned tap views
    int b_mn;                    // dgrad: B = the filter itself (MN-major 64 x 64 atoms)
    unsigned long long* trace;   // PK_HALO_TRACE (profiling only): clock stamps of CTA 0 per tile
};
__device__ __forceinline__ void hstamp(const HaloArgs& g, int it, int ev) {
    if (g.trace && blockIdx.x == 0 && it < 32 && (threadIdx.x & 31) == 0) g.trace[it * 32 + ev] = clock64();
}

// RESB: the whole filter slice of the tile's output channels is resident in
// smem (loaded once per CTA) — used when it fits (taps x chunks x BN x 128 B
// <= kResMax) and the grid has one output-channel tile; streaming a small
// (tap, chunk) slice per MMA group leaves the tensor core waiting on TMA
// latency.
constexpr int kResMax = 80 * 1024;

// HB = halo buffers. 3 (BN = 64 only): a third halo load in flight — with two,
// the next tile's halo is requested only when the current tile's MMAs start,
// so every tile waited ~one TMA latency (measured 0.083 ms vs 0.041 of MMA on
// ResNet conv2_x); paid for by smaller halo buffers (352 rows), an exact-size
// resident filter (<= 74 KB) and staging for the 4 epilogue warps that work
// when BN = 64.
constexpr int kHaloRows3 = 352;
constexpr int kResMax3 = 74 * 1024;
// MT = 2: 256-position tiles (two M=128 MMAs per tap on views 128 rows apart in
// the same halo): a 3x3 halo over a 58-wide grid is 8 rows for 256 positions
// instead of 6 rows for 128, so the L2 -> SM halo bytes per output drop by a
// third (the 64-channel layers are bound by that stream, not by the MMAs:
// with the MMAs disabled the 128-position kernel still took 55.6 of 80 us on
// ResNet conv2_x). Two halo buffers, direct epilogue stores (no staging).
constexpr int kHaloRowsMT2 = 480;
// PAIR (MT = 2, BN = 64, K-major filter): a CTA pair (cta_group::2) runs the same
// 256-position tile of two images with M = 256 MMAs; each CTA keeps HALF of the
// filter resident (32 output channels), so the SS MMAs read 5 KB of operands per
// K step per SM instead of 6 KB and the freed 36 KB hold a third halo buffer.
constexpr int kResPair = 40 * 1024;
template <int BN, int BSTAGES, bool RESB, int HB = kHaloBufs, int MT = 1, bool PAIR = false>
struct HSmem {
    static constexpr int kHalo = (MT == 2 ? kHaloRowsMT2 : HB == 3 ? kHaloRows3 : 448) * 128;  // grid rows x 128 B
    static constexpr int kB = (PAIR ? BN / 2 : BN) * 128;  // one (tap, chunk) filter slice (this CTA's)
    static constexpr int kBOff = HB * kHalo;
    static constexpr int kStgOff =
        kBOff + (RESB ? (PAIR ? kResPair : HB == 3 ? kResMax3 : kResMax) : BSTAGES * kB);
    static constexpr int kStaging = MT == 2 ? 0 : (HB == 3 ? 4 : 8) * 4096;
    static constexpr int kBarOff = kStgOff + kStaging;
    static constexpr int kBytes = kBarOff + (2 * HB + 2 * BSTAGES + 4) * 8 + 16 + 1024;
};

struct HTile {
    int n, p0, nt, row0;
};
template <int MT = 1>
__device__ __forceinline__ HTile htile(const HaloArgs& g, int t) {
    HTile h;
    h.nt = t % g.n_tiles_n;
    const int mt = t / g.n_tiles_n;
    h.n = mt / g.tiles_img;
    h.p0 = (mt - h.n * g.tiles_img) * (kM * MT);
    h.row0 = h.p0 / g.Wg;
    return h;
}

template <int BN, int BSTAGES, bool RESB, int HB, int MT = 1, bool PAIR = false>
__global__ void __launch_bounds__(kHThreads, 1)
    conv_halo_kernel(const __grid_constant__ CUtensorMap amap,
                     const __grid_constant__ CUtensorMap bmap, __nv_bfloat16* __restrict__ out,
                     const __grid_constant__ HaloArgs g, const pk_epilogue epi) {
    using L = HSmem<BN, BSTAGES, RESB, HB, MT, PAIR>;
    static_assert(HB == 2 || BN == 64, "3 halo buffers: BN = 64 only");
    static_assert(MT == 1 || (BN == 64 && RESB && (HB == 2 || PAIR)), "256-position tiles: BN = 64");
    static_assert(!PAIR || (MT == 2 && BN == 64), "pairs: 256-position tiles, BN = 64");
    const uint32_t rank = PAIR ? cluster_ctarank() : 0u;
    // tile loop: PAIR CTAs run pair tile pt = (image pair, tile in image) on image 2j + rank
    const int t_first = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int t_step = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    const int t_end = PAIR ? g.total_tiles / 2 : g.total_tiles;
    auto my_tile = [&](int pt) {
        return PAIR ? (2 * (pt / g.tiles_img) + (int)rank) * g.tiles_img + pt % g.tiles_img : pt;
    };
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* h_full = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* h_empty = h_full + HB;
    uint64_t* b_full = h_empty + HB;
    uint64_t* b_empty = b_full + BSTAGES;
    uint64_t* tmem_full = b_empty + BSTAGES;
    uint64_t* tmem_empty = tmem_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t kCols = 2 * MT * BN <= 128 ? 128 : 2 * MT * BN <= 256 ? 256 : 512;
    const int taps = g.R * g.S;

    if (threadIdx.x == 0) {
        for (int i = 0; i < HB; ++i) {
            mbar_init(&h_full[i], 1);
            mbar_init(&h_empty[i], 1);
        }
        for (int i = 0; i < BSTAGES; ++i) {
            mbar_init(&b_full[i], 1);
            mbar_init(&b_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], PAIR ? 16 : 8);
        }
        fence_barrier_init();
        tma_prefetch(&amap);
        tma_prefetch(&bmap);
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
    if (PAIR) cluster_sync_all();  // the peer's barriers exist before any cross-CTA signal
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();  // predecessor complete: inputs ready, outputs free
    pdl_trigger();

    if (warp == 0) {
        // ---------------- TMA producer: halo per chunk, filter slice per tap ----
        if (lane == 0) {
            int hs = 0, bs = 0;
            uint32_t hph = 0, bph = 0;
            // PK_HALO_DEBUG=2 (timing only): in-bounds boxes of the unpadded width
            const bool inb = g.debug & 2;
            const uint32_t halo_bytes = g.NR * (inb ? g.Wg - 2 * g.pad_w : g.Wg) * 128;
            if (PAIR) {
                // this CTA's 32 filter rows of every (chunk, tap) slice; both CTAs'
                // loads complete on the leader's barrier
                const uint32_t fb = smem_u32(&b_full[0]) & 0xFEFFFFFFu;
                if (rank == 0) mbar_arrive_expect_tx(&b_full[0], 2 * g.cpt * taps * L::kB);
                for (int ck = 0; ck < g.cpt; ++ck)
                    for (int tap = 0; tap < taps; ++tap) {
                        const int ft = g.flip ? taps - 1 - tap : tap;
                        tma_load_2d_pair(smem_u32(smem + L::kBOff + (ck * taps + tap) * L::kB), &bmap, fb,
                                         ft * g.red_ch + ck * 64, (int)rank * (BN / 2));
                    }
            } else if (RESB) {  // whole filter slice once: (chunk, tap) blocks of BN x 128 B
                mbar_arrive_expect_tx(&b_full[0], g.cpt * taps * L::kB);
                for (int ck = 0; ck < g.cpt; ++ck)
                    for (int tap = 0; tap < taps; ++tap) {
                        const int ft = g.flip ? taps - 1 - tap : tap;
                        if (g.b_mn) {
                            for (int j = 0; j < BN / 64; ++j)
                                tma_load_3d(smem_u32(smem + L::kBOff + (ck * taps + tap) * L::kB + j * 8192),
                                            &bmap, &b_full[0], 64 * j, ft, ck * 64);
                        } else {
                            tma_load_2d(smem_u32(smem + L::kBOff + (ck * taps + tap) * L::kB), &bmap,
                                        &b_full[0], ft * g.red_ch + ck * 64, 0);
                        }
                    }
            }
            int pit = 0;
            for (int pt = t_first; pt < t_end; pt += t_step, ++pit) {
                const HTile ht = htile<MT>(g, my_tile(pt));
                for (int ck = 0; ck < g.cpt; ++ck) {
                    hstamp(g, pit, 8);
                    mbar_wait(&h_empty[hs], hph ^ 1);
                    hstamp(g, pit, 9);
                    if (PAIR) {
                        const uint32_t fb = smem_u32(&h_full[hs]) & 0xFEFFFFFFu;
                        if (rank == 0) mbar_arrive_expect_tx(&h_full[hs], 2 * halo_bytes);
                        tma_load_4d_pair(smem_u32(smem + hs * L::kHalo), &amap, fb, ck * 64, -g.pad_w,
                                         ht.row0 - g.pad_h, ht.n);
                        if (++hs == HB) {
                            hs = 0;
                            hph ^= 1;
                        }
                        continue;
                    }
                    mbar_arrive_expect_tx(&h_full[hs], halo_bytes);
                    if (inb)
                        tma_load_4d(smem_u32(smem + hs * L::kHalo), &amap, &h_full[hs], ck * 64, 0,
                                    max(0, min(ht.row0 - g.pad_h, g.Hg - 2 * g.pad_h - g.NR)), ht.n);
                    else
                        tma_load_4d(smem_u32(smem + hs * L::kHalo), &amap, &h_full[hs], ck * 64,
                                    -g.pad_w, ht.row0 - g.pad_h, ht.n);
                    if (++hs == HB) {
                        hs = 0;
                        hph ^= 1;
                    }
                    for (int tap = 0; tap < (RESB ? 0 : taps); ++tap) {
                        const int ft = g.flip ? taps - 1 - tap : tap;
                        mbar_wait(&b_empty[bs], bph ^ 1);
                        mbar_arrive_expect_tx(&b_full[bs], L::kB);
                        if (g.b_mn) {
                            for (int j = 0; j < BN / 64; ++j)
                                tma_load_3d(smem_u32(smem + L::kBOff + bs * L::kB + j * 8192), &bmap,
                                            &b_full[bs], ht.nt * BN + 64 * j, ft, ck * 64);
                        } else {
                            tma_load_2d(smem_u32(smem + L::kBOff + bs * L::kB), &bmap, &b_full[bs],
                                        ft * g.red_ch + ck * 64, ht.nt * BN);
                        }
                        if (++bs == BSTAGES) {
                            bs = 0;
                            bph ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
      if (!PAIR || rank == 0) {
        // ---------------- MMA issuer: A = shifted halo view per tap --------------
        const uint32_t idesc = idesc_bf16_f32(PAIR ? 2 * kM : kM, BN, false, g.b_mn != 0);
        const uint64_t bks = g.b_mn ? 128 : 2;  // B k-step (MN-major: 16 rows)
        const uint32_t blbo = g.b_mn ? 8192 : 16;
        int hs = 0, bs = 0;
        uint32_t hph = 0, bph = 0;
        int it = 0;
        if (RESB) mbar_wait(&b_full[0], 0);
        for (int pt = t_first; pt < t_end; pt += t_step, ++it) {
            const HTile ht = htile<MT>(g, my_tile(pt));
            const int a = it & 1;
            hstamp(g, it, 0);
            mbar_wait(&tmem_empty[a], ((it >> 1) & 1) ^ 1);
            hstamp(g, it, 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + a * (MT * BN);
            const int base_row = ht.p0 - ht.row0 * g.Wg;
            for (int ck = 0; ck < g.cpt; ++ck) {
                mbar_wait(&h_full[hs], hph);
                hstamp(g, it, 2);
                tc_fence_after();
                const uint32_t halo_u = smem_u32(smem + hs * L::kHalo);
                if (PAIR || (RESB && !(g.debug & ~56))) {
                    // resident filter: descriptors are the tile base plus a per-tap
                    // offset (start field in 16-byte units), two taps per issue block;
                    // keeps the issuing thread ahead of N=64 MMAs (48 clk each)
                    const uint64_t at = umma_desc_sw128(
                        halo_u + ((g.debug & 16) ? 0 : base_row * 128), 16, 1024);
                    const uint64_t bt = umma_desc_sw128(
                        smem_u32(smem + L::kBOff + ck * taps * L::kB), blbo, 1024);
#pragma unroll
                  for (int mt = 0; mt < MT; ++mt) {
                    // M tile mt: positions p0 + 128 mt, i.e. the halo view 128 rows further
                    const uint64_t atm = at + (uint64_t)(mt * 128 * 8);
                    const uint32_t dm = d_tmem + mt * BN;
                    int r0 = 0, s0 = 0;
                    int tap = 0;
                    for (; tap + 2 <= taps; tap += 2) {
                        const int al = (g.debug & 16) ? ~63 : ~0;  // timing: 8-row-aligned views
                        const uint64_t a0 = atm + (uint64_t)(((r0 * g.Wg + s0) * 8) & al);
                        if (++s0 == g.S) { s0 = 0; ++r0; }
                        const uint64_t a1 = atm + (uint64_t)(((r0 * g.Wg + s0) * 8) & al);
                        if (++s0 == g.S) { s0 = 0; ++r0; }
                        const uint64_t b0 = bt + (uint64_t)(tap * (L::kB >> 4));
                        if constexpr (PAIR)
                            mma8_bf16_bs_pair(dm, a0, b0, a1, b0 + (L::kB >> 4), bks, idesc, (ck | tap) != 0);
                        else
                            mma8_bf16_bs(dm, a0, b0, a1, b0 + (L::kB >> 4), bks, idesc, (ck | tap) != 0);
                    }
                    if (tap < taps) {
                        const uint64_t a0 = atm + (uint64_t)((r0 * g.Wg + s0) * 8);
                        const uint64_t b0 = bt + (uint64_t)(tap * (L::kB >> 4));
                        if constexpr (PAIR)
                            mma4_bf16_pair(dm, a0, a0 + 2, a0 + 4, a0 + 6, b0, b0 + bks, b0 + 2 * bks,
                                           b0 + 3 * bks, idesc, (ck | tap) != 0);
                        else
                            mma4_bf16(dm, a0, a0 + 2, a0 + 4, a0 + 6, b0, b0 + bks, b0 + 2 * bks,
                                      b0 + 3 * bks, idesc, (ck | tap) != 0);
                    }
                  }
                }
                for (int tap = 0; tap < ((PAIR || (RESB && !(g.debug & ~56))) ? 0 : taps); ++tap) {
                    const int r = tap / g.S, s = tap - r * g.S;
                    if (!RESB) {
                        mbar_wait(&b_full[bs], bph);
                        tc_fence_after();
                    }
                    const int arow = base_row + r * g.Wg + s;
                    const uint64_t ad0 =
                        umma_desc_sw128(halo_u + ((g.debug & 1) ? (arow & ~7) : arow) * 128, 16, 1024);
                    const uint64_t bd0 = umma_desc_sw128(
                        smem_u32(smem + L::kBOff + (RESB ? ck * taps + tap : bs) * L::kB), blbo, 1024);
                    if (!(g.debug & 4))
                        mma4_bf16(d_tmem, ad0, ad0 + 2, ad0 + 4, ad0 + 6, bd0, bd0 + bks, bd0 + 2 * bks,
                                  bd0 + 3 * bks, idesc, (ck | tap) != 0);
                    if (!RESB) {
                        mma_commit_elect(&b_empty[bs]);
                        if (++bs == BSTAGES) {
                            bs = 0;
                            bph ^= 1;
                        }
                    }
                }
                hstamp(g, it, 3);
                if (PAIR)
                    mma_commit_pair(&h_empty[hs]);
                else
                    mma_commit_elect(&h_empty[hs]);
                if (++hs == HB) {
                    hs = 0;
                    hph ^= 1;
                }
            }
            if (PAIR)
                mma_commit_pair(&tmem_full[a]);
            else
                mma_commit_elect(&tmem_full[a]);
        }
      }
    } else {
        // ---------------- epilogue (8 warps): direct 16-byte stores ---------------
        const int ew = warp - 2;
        const int q = warp & 3;
        const int half = ew >> 2;
        uint8_t* stg = smem + L::kStgOff + (HB == 3 ? q : ew) * 4096;
        const uint32_t stg_u = smem_u32(stg);
        const bool has_epi = epilogue_active(&epi);
        const bool direct = MT == 2 || (!epi.stats && !(g.debug & 32));  // PK_HALO_DEBUG=32: staged
        BnStatAcc bacc;
        bacc.init();
        int it = 0;
        for (int pt = t_first; pt < t_end; pt += t_step, ++it) {
            const HTile ht = htile<MT>(g, my_tile(pt));
            const int n0c = ht.nt * BN;
            const int a = it & 1;
            if (warp == 2) hstamp(g, it, 4);
            mbar_wait(&tmem_full[a], (it >> 1) & 1);
            if (warp == 2) hstamp(g, it, 5);
            tc_fence_after();
            const int span = min(BN, g.out_pitch - n0c);
            const int nchunks = (span + 63) / 64;
            // work units j = (M tile, 64-column chunk), alternating between the warp halves
            const int units = MT * nchunks;
            int my_last = -1;
            for (int j = half; j < units; j += 2) my_last = j;
            if (my_last < 0) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (PAIR)
                        mbar_arrive_leader(&tmem_empty[a]);
                    else
                        mbar_arrive(&tmem_empty[a]);
                }
            }
            if (g.debug & 8) {  // timing experiments: no epilogue work
                if (my_last >= 0) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                    if (PAIR)
                        mbar_arrive_leader(&tmem_empty[a]);
                    else
                        mbar_arrive(&tmem_empty[a]);
                }
                }
                continue;
            }
#pragma unroll 1
            for (int j = half; j < units; j += 2) {
                const int mt = j / nchunks, ci = j - mt * nchunks;
                const int c0 = ci * 64;
                const int p = ht.p0 + mt * kM + q * 32 + lane;  // this lane's grid position
                const int oy = p / g.Wg, ox = p - oy * g.Wg;
                const bool row_ok = oy < g.Ho && ox < g.Wo;
                const long long pix = ((long long)ht.n * g.Ho + oy) * g.Wo + ox;
                uint32_t v[64];
                const uint32_t ta = tmem_base + a * (MT * BN) + mt * BN + c0 +
                                    (static_cast<uint32_t>(q * 32) << 16);
                tmem_ld16(ta + 0, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
                tmem_ld16(ta + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
                tmem_ld16(ta + 32, *reinterpret_cast<uint32_t(*)[16]>(&v[32]));
                tmem_ld16(ta + 48, *reinterpret_cast<uint32_t(*)[16]>(&v[48]));
                tmem_ld_wait();
                if (j == my_last) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                    if (PAIR)
                        mbar_arrive_leader(&tmem_empty[a]);
                    else
                        mbar_arrive(&tmem_empty[a]);
                }
                }
                float xf[64];
#pragma unroll
                for (int e = 0; e < 64; ++e) xf[e] = __uint_as_float(v[e]);
                if (has_epi) epilogue_chunk64(epi, xf, n0c + c0, g.n_out, oy, ox, g.Ho, g.Wo);
                if (direct) {
                    // each lane stores its own position's 64 channels (8 x 16 B): no
                    // staging round trip through shared memory, whose bandwidth the
                    // N=64 SS MMAs and the halo TMA writes already saturate
                    const int valid = g.n_out - (n0c + c0);
                    __nv_bfloat16* dst = out + pix * g.out_pitch + n0c + c0;
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        uint32_t w[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int c = jj * 8 + 2 * e;
                            const __nv_bfloat162 b2 = __floats2bfloat162_rn(c < valid ? xf[c] : 0.0f,
                                                                            c + 1 < valid ? xf[c + 1] : 0.0f);
                            w[e] = *reinterpret_cast<const uint32_t*>(&b2);
                        }
                        if (row_ok && n0c + c0 + jj * 8 < g.out_pitch)
                            *reinterpret_cast<uint4*>(dst + jj * 8) = make_uint4(w[0], w[1], w[2], w[3]);
                    }
                    continue;
                }
                // stage the rounded 32 x 64 tile (128-byte rows, swizzled), then
                // store 4 full rows per instruction (8 lanes x 16 B per row)
                pack_stage64(xf, stg_u, lane, g.n_out - (n0c + c0));
                __syncwarp();
                {
                    const int sj = lane & 7;
                    const int ch = n0c + c0 + sj * 8;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int row = (lane >> 3) + 4 * i;
                        const int pr = ht.p0 + mt * kM + q * 32 + row;
                        const int ry = pr / g.Wg, rx = pr - ry * g.Wg;
                        uint4 val;
                        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(val.x), "=r"(val.y), "=r"(val.z), "=r"(val.w)
                                     : "r"(stg_u + row * 128 + ((sj ^ (row & 7)) << 4)));
                        if (ry < g.Ho && rx < g.Wo && ch < g.out_pitch)
                            *reinterpret_cast<uint4*>(
                                out + (((long long)ht.n * g.Ho + ry) * g.Wo + rx) * g.out_pitch + ch) = val;
                    }
                }
                if (epi.stats)
                    bacc.add(epi, stg_u, lane, row_ok, pix, (ci >> 1) & 1, n0c + c0, g.n_out,
                             g.out_pitch);
                __syncwarp();  // staging reused by the next chunk
                if (warp == 2) hstamp(g, it, 6);
            }
        }
        if (epi.stats) bacc.finish(epi, lane, g.n_out);
    }
    tc_fence_before();
    __syncthreads();
    if (PAIR) cluster_sync_all();
    if (warp == 1) {
        tc_fence_after();
        if (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                         "r"(kCols));
        else
            tmem_dealloc(tmem_base, kCols);
    }
}

template <int BN, int BSTAGES, bool RESB, int HB = kHaloBufs, int MT = 1, bool PAIR = false>
cudaError_t launch_halo(const CUtensorMap& amap, const CUtensorMap& bmap, void* out,
                        const HaloArgs& g, const pk_epilogue& e, cudaStream_t st) {
    using L = HSmem<BN, BSTAGES, RESB, HB, MT, PAIR>;
    static_assert(L::kBytes <= 227 * 1024, "smem");
    auto kern = conv_halo_kernel<BN, BSTAGES, RESB, HB, MT, PAIR>;
    static int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
        const cudaError_t err =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes);
        if (err != cudaSuccess) return err;
        attr_dev = dev;
    }
    int grid = num_sms_of_current_device();
    if (PAIR) grid = grid / 2 * 2;
    if (g.total_tiles < grid) grid = g.total_tiles;
    cudaError_t le = pk_launch(kern, dim3(grid), dim3(kHThreads), L::kBytes, st, PAIR ? 2 : 1, amap, bmap,
                               (__nv_bfloat16*)out, g, e);
    if (le != cudaSuccess) return le;
    count_launch();
    if (g.trace) {  // profiling only (PK_HALO_TRACE)
        unsigned long long h[32 * 32];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, g.trace, sizeof(h), cudaMemcpyDeviceToHost);
        for (int i = 0; i < 32; ++i) {
            fprintf(stderr, "halo tile %2d:", i);
            for (int ev = 0; ev < 10; ++ev) fprintf(stderr, " %7lld", (long long)(h[i * 32 + ev] - h[0]));
            fprintf(stderr, "\n");
        }
    }
    return cudaGetLastError();
}

}  // namespace
}  // namespace pk

using namespace pk;

// Stride-1 spatial convolution (forward, or backward data when dgrad) through
// the halo-reuse kernel. cudaErrorNotSupported (nothing launched) when the
// geometry does not fit: stride/dilation 1, filters > 1x1, channel pitches
// multiples of 64, padded grid width <= 256, halo <= 448 rows, N <= 256.
cudaError_t pk_halo_conv(const pk_conv_geom* g, bool dgrad, const void* src, const void* filt,
                         void* out, const pk_epilogue* epi, cudaStream_t st, bool filt_mn) {
    static const bool enabled = [] {
        const char* v = std::getenv("PK_HALO");
        return !(v && v[0] == '0');
    }();
    if (!enabled || g->groups != 1 || g->transpose || g->str_h != 1 || g->str_w != 1 ||
        g->dil_h != 1 || g->dil_w != 1 || g->r * g->s < 2)
        return cudaErrorNotSupported;
    const int src_pitch = dgrad ? g->y_pitch : g->x_pitch;
    const int out_pitch = dgrad ? g->x_pitch : g->y_pitch;
    const int n_out = dgrad ? g->c : g->k;
    if (src_pitch % 64 || out_pitch % 8 || n_out > 256) return cudaErrorNotSupported;
    // grid of the source (dgrad: dY padded by R-1-pad, which reproduces dX's extent)
    const int Hs = dgrad ? g->p : g->h, Ws = dgrad ? g->q : g->w;
    const int pad_h = dgrad ? g->r - 1 - g->pad_h : g->pad_h;
    const int pad_w = dgrad ? g->s - 1 - g->pad_w : g->pad_w;
    if (pad_h < 0 || pad_w < 0) return cudaErrorNotSupported;
    HaloArgs a{};
    a.N = g->n;
    a.Hg = Hs + 2 * pad_h;
    a.Wg = Ws + 2 * pad_w;
    a.Ho = a.Hg - g->r + 1;
    a.Wo = a.Wg - g->s + 1;
    if (a.Ho != (dgrad ? g->h : g->p) || a.Wo != (dgrad ? g->w : g->q)) return cudaErrorNotSupported;
    a.pad_h = pad_h;
    a.pad_w = pad_w;
    a.R = g->r;
    a.S = g->s;
    a.red_ch = src_pitch;
    a.cpt = src_pitch / 64;
    a.n_out = n_out;
    a.out_pitch = out_pitch;
    a.flip = dgrad ? 1 : 0;
    if (const char* v = std::getenv("PK_HALO_DEBUG")) a.debug = std::atoi(v);
    static unsigned long long* trace = [] {
        unsigned long long* p = nullptr;
        if (std::getenv("PK_HALO_TRACE")) cudaMalloc(&p, 32 * 32 * 8);
        return p;
    }();
    a.trace = trace;
    // 256-position tiles (MT = 2) for 64-wide outputs without a statistics epilogue
    // (PK_HALO_MT2=0: 128-position tiles)
    static const bool mt2_off = [] {
        const char* v = std::getenv("PK_HALO_MT2");
        return v && v[0] == '0';
    }();
    const int bn0 = out_pitch <= 64 ? 64 : out_pitch <= 128 ? 128 : 256;
    int mt = 1;
    if (!mt2_off && bn0 == 64 && !(epi && epi->stats)) {
        const int nr2 = (2 * kM - 1 + (g->r - 1) * a.Wg + g->s - 1 + a.Wg - 1) / a.Wg + 1;
        if (a.Wg <= 256 && nr2 * a.Wg <= kHaloRowsMT2 &&
            (long long)src_pitch / 64 * g->r * g->s * 64 * 128 <= kResMax)
            mt = 2;
    }
    // halo of 128 MT positions: rows touched by [p0, p0 + 128 MT - 1 + (R-1)Wg + S-1]
    a.NR = (kM * mt - 1 + (g->r - 1) * a.Wg + g->s - 1 + a.Wg - 1) / a.Wg + 1;
    if (a.Wg > 256 || a.NR > 256 || a.NR * a.Wg > (mt == 2 ? kHaloRowsMT2 : 448)) return cudaErrorNotSupported;
    a.tiles_img = (a.Ho * a.Wg + kM * mt - 1) / (kM * mt);
    // small images waste most of a tile on padding columns: leave them to the
    // rectangle kernel (valid fraction below ~80%)
    if ((long long)a.Ho * a.Wo * 10 < (long long)a.tiles_img * kM * mt * 8) return cudaErrorNotSupported;
    const int bn = out_pitch <= 64 ? 64 : out_pitch <= 128 ? 128 : 256;
    a.n_tiles_n = (out_pitch + bn - 1) / bn;
    a.total_tiles = a.tiles_img * g->n * a.n_tiles_n;
    CUtensorMap amap{}, bmap{};
    if (!tc::make_map_nhwc(&amap, src, g->n, Hs, Ws, src_pitch, (a.debug & 2) ? Ws : a.Wg, a.NR, 1))
        return cudaErrorNotSupported;
    const long long kred = (long long)g->r * g->s * src_pitch;
    // CTA pairs over image pairs (K-major filter only; PK_HALO_PAIR=1)
    static const bool pair_on = std::getenv("PK_HALO_PAIR") && std::getenv("PK_HALO_PAIR")[0] == '1';
    const bool pair = pair_on && mt == 2 && !filt_mn && g->n % 2 == 0 && a.n_tiles_n == 1 &&
                      (long long)a.cpt * g->r * g->s * 32 * 128 <= kResPair && a.debug == 0;
    if (pair) {
        if (!tc::make_map_2d(&bmap, filt, n_out, kred, kred, bn / 2)) return cudaErrorNotSupported;
        pk_epilogue e{};
        e.act = -1;
        if (epi) e = *epi;
        return launch_halo<64, 8, true, 3, 2, true>(amap, bmap, out, a, e, st);
    }
    if (filt_mn) {
        if (!dgrad || g->f_pitch % 64 || bn % 64) return cudaErrorNotSupported;
        a.b_mn = 1;
        if (!tc::make_map_filter_mn(&bmap, filt, g->k, g->r * g->s, g->f_pitch))
            return cudaErrorNotSupported;
    } else if (!tc::make_map_2d(&bmap, filt, n_out, kred, kred, bn)) {
        return cudaErrorNotSupported;
    }
    pk_epilogue e{};
    e.act = -1;
    if (epi) e = *epi;
    // only the resident-filter form beats the rectangle kernel (measured: the
    // streamed per-tap filter slices leave the MMA waiting on TMA latency)
    const bool resb = a.n_tiles_n == 1 && (long long)a.cpt * g->r * g->s * bn * 128 <= kResMax;
    if (!resb) return cudaErrorNotSupported;
    if (mt == 2) return launch_halo<64, 8, true, 2, 2>(amap, bmap, out, a, e, st);
    static const bool hb2 = std::getenv("PK_HALO_HB2") != nullptr;
    if (bn == 64 && !hb2 && a.NR * a.Wg <= kHaloRows3 &&
        (long long)a.cpt * g->r * g->s * bn * 128 <= kResMax3)
        return launch_halo<64, 8, true, 3>(amap, bmap, out, a, e, st);
    if (bn == 64) return launch_halo<64, 8, true>(amap, bmap, out, a, e, st);
    return launch_halo<128, 4, true>(amap, bmap, out, a, e, st);
}
