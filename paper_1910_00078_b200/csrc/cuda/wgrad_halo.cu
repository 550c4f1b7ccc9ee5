// Backward weights of stride-1 spatial convolutions on 64-channel tensors
// (ResNet conv2_x 3x3) from a padded-grid HALO, the wgrad counterpart of
// conv_halo.cu:
//
//   dW^T[(tap, c)][k] = sum_g  Xg[g + r*Wg + s][c] * dYg[g][k]
//
// over grid positions g of the padded input grid (row width Wg = W + 2 pad),
// with dYg = dY at the valid positions and 0 in the padding columns (TMA OOB
// fill of a Wg-wide box over the Q-wide dY rows). A k-block is KBR whole grid
// rows (<= 128 positions, zero-padded to 128): ONE X halo box of
// KBR + R - 1 rows and one dY box per k-block; every tap's A operand is the
// same halo viewed from a shifted row (the K-major trick of conv_halo.cu, here
// MN-major: M = (tap pair, channel), the second tap of a pair reached through
// the descriptor's leading-byte offset). The single-CTA rectangle wgrad
// re-loads X once per tap (9x) and wastes half of every M=128 MMA on K = 64;
// this form loads X ~1.8x and fills M with two taps.
//
// Accumulators: ceil(taps / 2) M-tiles x 64 columns of TMEM; split-K over
// k-blocks, one fp32 partial per CTA in the [split][K][R*S*Cp] layout the
// deterministic wgrad_sum_kernel (conv_tma.cu) finishes.
#include <cstdlib>

#include "common.cuh"
#include "tc_host.cuh"
#include "tc_internal.h"
#include "tc_ptx.cuh"

namespace pk {
namespace {

using namespace pk::tc;

constexpr int kHwThreads = 320;         // producer, MMA, 8 epilogue warps (two per lane quarter)
constexpr int kHwStages = 4;
constexpr int kHaloRowsMax = 256;       // halo buffer rows (128 B each)
constexpr int kHaloBytes = kHaloRowsMax * 128;
constexpr int kDyBytes = 128 * 128;     // 128 positions x 64 channels
constexpr int kHwStage = kHaloBytes + kDyBytes;
constexpr int kHwBarOff = kHwStages * kHwStage;
constexpr int kHwBytes = kHwBarOff + (2 * kHwStages + 1) * 8 + 16 + 1024;
constexpr int kMaxMTiles = 5;           // taps <= 10

struct HwArgs {
    int N, P, Q, Wg, R, S, pad_h, pad_w, K, Nn;  // Nn = R*S*64
    int KBR;                 // grid rows per k-block
    int blocks_img, total_kb, kb_per;
    int taps, mtiles;
    int tap_off[16];         // grid-row offset r*Wg + s of tap t
    unsigned int* sync;      // in-kernel split-K finish (nullptr: separate sum kernel)
    __nv_bfloat16* dw;
    int splits;
};

__global__ void __launch_bounds__(kHwThreads, 1)
    wgrad_halo_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap dymap,
                      float* __restrict__ partial, const __grid_constant__ HwArgs g) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kHwBarOff);
    uint64_t* empty = full + kHwStages;
    uint64_t* tmem_full = empty + kHwStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kb_begin = blockIdx.x * g.kb_per;
    const int kb_end = min(g.total_kb, kb_begin + g.kb_per);

    // the rows no TMA box writes (halo tail read by shifted views, dY rows past
    // KBR*Wg) must be zero: clear every stage once
    for (int i = threadIdx.x; i < kHwStages * kHwStage / 16; i += blockDim.x)
        asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(smem_u32(smem) + i * 16), "r"(0)
                     : "memory");
    fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        for (int i = 0; i < kHwStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tmem_full, 1);
        fence_barrier_init();
        tma_prefetch(&xmap);
        tma_prefetch(&dymap);
    }
    if (warp == 1) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();
    pdl_trigger();

    if (warp == 0) {
        if (lane == 0) {
            const uint32_t halo_bytes = (g.KBR + g.R - 1) * g.Wg * 128;
            const uint32_t dy_bytes = g.KBR * g.Wg * 128;
            int stage = 0;
            uint32_t phase = 0;
            for (int kb = kb_begin; kb < kb_end; ++kb) {
                const int n = kb / g.blocks_img, p0 = (kb - n * g.blocks_img) * g.KBR;
                mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* sa = smem + stage * kHwStage;
                mbar_arrive_expect_tx(&full[stage], halo_bytes + dy_bytes);
                tma_load_4d(smem_u32(sa), &xmap, &full[stage], 0, -g.pad_w, p0 - g.pad_h, n);
                tma_load_4d(smem_u32(sa + kHaloBytes), &dymap, &full[stage], 0, 0, p0, n);
                if (++stage == kHwStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = idesc_bf16_f32(128, 64, true, true);
        constexpr uint64_t ks = 2048 >> 4;  // 16 MN-major K rows (positions)
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = kb_begin; kb < kb_end; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t halo_u = smem_u32(smem + stage * kHwStage);
            const uint64_t bd = umma_desc_sw128(halo_u + kHaloBytes, 8192, 1024);
#pragma unroll 1
            for (int m = 0; m < g.mtiles; ++m) {
                // M rows 0-63: tap 2m, rows 64-127: tap 2m+1 (a shifted row of the
                // same halo: the leading byte offset is the row distance)
                const int t0 = 2 * m, t1 = 2 * m + 1 < g.taps ? 2 * m + 1 : 2 * m;
                const int o0 = g.tap_off[t0];
                const int lbo = (t1 == t0 ? 1 : g.tap_off[t1] - o0) * 128;
                const uint64_t ad = umma_desc_sw128(halo_u + o0 * 128, lbo, 1024);
                const uint32_t d = tmem_base + m * 64;
                const uint32_t acc = kb != kb_begin;
                mma4_bf16(d, ad, ad + ks, ad + 2 * ks, ad + 3 * ks, bd, bd + ks, bd + 2 * ks, bd + 3 * ks,
                          idesc, acc);
                mma4_bf16(d, ad + 4 * ks, ad + 5 * ks, ad + 6 * ks, ad + 7 * ks, bd + 4 * ks, bd + 5 * ks,
                          bd + 6 * ks, bd + 7 * ks, idesc, 1);
            }
            mma_commit_elect(&empty[stage]);
            if (kb == kb_end - 1) mma_commit_elect(tmem_full);
            if (++stage == kHwStages) {
                stage = 0;
                phase ^= 1;
            }
        }
    } else {
        // ---------------- epilogue: TMEM lane = (tap, c), column = k -------------
        const int q = warp & 3, half = (warp - 2) >> 2;  // the two warps of a quarter: alternate M tiles
        const bool live = kb_end > kb_begin;
        if (live) {
            mbar_wait(tmem_full, 0);
            tc_fence_after();
        }
        const int row = q * 32 + lane;
        float* dst0 = partial + (size_t)blockIdx.x * g.K * g.Nn;
#pragma unroll 1
        for (int m = half; m < g.mtiles; m += 2) {
            const int tap = 2 * m + (row >> 6), c = row & 63;
            const bool ok = tap < g.taps;
#pragma unroll 1
            for (int c0 = 0; c0 < 64; c0 += 32) {
                uint32_t v[32];
                if (live) {
                    const uint32_t ta = tmem_base + m * 64 + c0 + (static_cast<uint32_t>(q * 32) << 16);
                    tmem_ld16(ta, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
                    tmem_ld16(ta + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) v[e] = 0u;
                }
                if (ok) {
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const int k = c0 + e;
                        if (k < g.K) dst0[(size_t)k * g.Nn + tap * 64 + c] = __uint_as_float(v[e]);
                    }
                }
            }
        }
    }
    if (g.sync) splitk_finish(partial, g.splits, (long long)g.K * g.Nn, g.dw, g.sync);
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

bool halo_args(const pk_conv_geom* g, HwArgs& a) {
    static const bool off = [] {
        const char* v = std::getenv("PK_WG_HALO");
        return v && v[0] == '0';
    }();
    if (off || g->groups != 1 || g->transpose || g->str_h != 1 || g->str_w != 1 || g->dil_h != 1 ||
        g->dil_w != 1 || g->x_pitch != 64 || g->f_pitch != 64 || g->y_pitch != 64 || g->k > 64 ||
        g->r * g->s < 2 || g->r * g->s > 2 * kMaxMTiles)
        return false;
    a = HwArgs{};
    a.N = g->n;
    a.P = g->p;
    a.Q = g->q;
    a.Wg = g->w + 2 * g->pad_w;
    a.R = g->r;
    a.S = g->s;
    a.pad_h = g->pad_h;
    a.pad_w = g->pad_w;
    a.K = g->k;
    a.Nn = g->r * g->s * 64;
    if (a.Q + g->s - 1 != a.Wg || a.Wg > 128) return false;
    a.KBR = 128 / a.Wg;
    const int halo_rows = (a.KBR + a.R - 1) * a.Wg;
    const int reach = (a.R - 1) * a.Wg + a.S - 1 + 128;
    if (halo_rows > kHaloRowsMax || reach > kHaloRowsMax) return false;
    a.taps = a.R * a.S;
    a.mtiles = (a.taps + 1) / 2;
    for (int t = 0; t < a.taps; ++t) a.tap_off[t] = (t / a.S) * a.Wg + t % a.S;
    a.blocks_img = (a.P + a.KBR - 1) / a.KBR;
    a.total_kb = a.N * a.blocks_img;
    return true;
}

}  // namespace
}  // namespace pk

using namespace pk;

int pk_halo_wgrad_splits(const pk_conv_geom* g, int num_sms) {
    if (cfg_field(&pk_tc_config::family) >= 1) return 0;  // tuned: no halo kernels
    HwArgs a;
    if (!halo_args(g, a)) return 0;
    return a.total_kb < num_sms ? a.total_kb : num_sms;
}

cudaError_t pk_halo_wgrad(const pk_conv_geom* g, const void* dy, const void* x, float* partial,
                          int splits, cudaStream_t st, void* dw, unsigned int* sync) {
    HwArgs a;
    if (!halo_args(g, a) || splits < 1) return cudaErrorNotSupported;
    a.kb_per = (a.total_kb + splits - 1) / splits;
    a.sync = sync;  // grid = splits <= SMs, one CTA per SM: co-resident
    a.dw = static_cast<__nv_bfloat16*>(dw);
    a.splits = splits;
    CUtensorMap xmap{}, dymap{};
    if (!tc::make_map_nhwc(&xmap, x, g->n, g->h, g->w, 64, a.Wg, a.KBR + a.R - 1, 1) ||
        !tc::make_map_nhwc(&dymap, dy, g->n, g->p, g->q, 64, a.Wg, a.KBR, 1))
        return cudaErrorNotSupported;
    static int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
        cudaError_t err = cudaFuncSetAttribute(wgrad_halo_kernel,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, kHwBytes);
        if (err != cudaSuccess) return err;
        attr_dev = dev;
    }
    // CTAs whose k-block range is empty still write (zero) partials
    const cudaError_t le = pk_launch(wgrad_halo_kernel, dim3(splits), dim3(kHwThreads), kHwBytes, st,
                                     xmap, dymap, partial, a);
    count_launch();
    return le != cudaSuccess ? le : cudaGetLastError();
}
