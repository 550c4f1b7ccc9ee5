// tcgen05 implicit-GEMM backward-weights convolution (sm_100a): the bf16
// engine of the Im2colGemm backward-weights path.
//
//   dW[k][(r,s,c)] = sum_{npq} dY[npq][k] * X[npq shifted by (r,s)][c]
//
// Both operands are MN-major (the reduction index npq is the strided one):
// dY tiles arrive by TMA as [64 npq][64 k] SWIZZLE_128B atoms, X rows are
// gathered by 4 producer warps with 16-byte cp.async into [64 npq][64 (r,s,c)]
// atoms. One elected thread issues tcgen05.mma (M=128 output channels,
// N=128 filter positions, K=16) into TMEM. The npq reduction is split over
// CTAs (split-K) into fp32 partials that a second kernel sums in a fixed
// order, so results are deterministic and independent of the split.
#include "common.cuh"
#include "tc_host.cuh"
#include "tc_internal.h"
#include "tc_ptx.cuh"

namespace pk {
namespace {

using namespace pk::tc;

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kProducerThreads = 128;
constexpr int kThreads = 160;

// ---------------------------------------------------------------------------
// wgrad: D[k][n] with n = (r, s, c); reduction over npq in [kb_begin, kb_end).
constexpr int WBN = 128;

struct WgGeom {
    int K;             // output channels (M of the GEMM)
    int Nn;            // R * S * Cp (N of the GEMM)
    int NPQ;           // reduction length
    int P, Q, H, W, Cp;
    int R, S, pad_h, pad_w, str_h, str_w, dil_h, dil_w;
    int num_kb;        // ceil(NPQ / BK)
    int kb_per_split;
};

template <int STAGES>
struct WgSmem {
    static constexpr int kA = BM * BK * 2;   // 2 MN atoms of [64 npq][64 k]
    static constexpr int kB = WBN * BK * 2;  // 2 MN atoms of [64 npq][64 n]
    static constexpr int kStage = kA + kB;
    static constexpr int kBarOff = STAGES * kStage;
    static constexpr int kBytes = kBarOff + (2 * STAGES + 1) * 8 + 16 + 1024;
};

template <int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    igemm_tc_wgrad_kernel(const __grid_constant__ CUtensorMap amap,
                          const __nv_bfloat16* __restrict__ x, float* __restrict__ partial,
                          WgGeom g) {
    using L = WgSmem<STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * BM;     // output channel k
    const int n0 = blockIdx.y * WBN;    // (r, s, c)
    const int split = blockIdx.z;
    const int kb_begin = split * g.kb_per_split;
    const int kb_end = min(g.num_kb, kb_begin + g.kb_per_split);

    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], kProducerThreads + 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tmem_full, 1);
        fence_barrier_init();
        tma_prefetch(&amap);
    }
    if (warp == 4) tmem_alloc(tmem_slot, WBN);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp < 4) {
        const int j = threadIdx.x & 7;       // 16-byte chunk (8 channels)
        const int rsub = threadIdx.x >> 3;   // 0..15
        // (r, s, c) of this thread's chunk in each of the two 64-wide atoms
        int tap_r[2], tap_s[2], tap_c[2];
        bool tap_ok[2];
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            const int nidx = n0 + a * 64 + j * 8;
            tap_ok[a] = nidx < g.Nn;
            const int rs = nidx / g.Cp;
            tap_c[a] = nidx - rs * g.Cp;
            tap_r[a] = rs / g.S;
            tap_s[a] = rs - tap_r[a] * g.S;
        }
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = kb_begin; kb < kb_end; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * L::kStage;
            const uint32_t sb_u = smem_u32(sa + L::kA);
            if (threadIdx.x == 0) {
                mbar_arrive_expect_tx(&full[stage], L::kA);
                tma_load_2d(smem_u32(sa), &amap, &full[stage], m0, kb * BK);
                tma_load_2d(smem_u32(sa + L::kA / 2), &amap, &full[stage], m0 + 64, kb * BK);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int row = rsub + 16 * i;           // npq within the stage
                const int npq = kb * BK + row;
                int n = 0, p = 0, q = 0;
                const bool rv = npq < g.NPQ;
                if (rv) {
                    const int pq = g.P * g.Q;
                    n = npq / pq;
                    const int rem = npq - n * pq;
                    p = rem / g.Q;
                    q = rem - p * g.Q;
                }
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    const uint32_t dst = sb_u + a * (L::kB / 2) + row * 128 + ((j ^ (row & 7)) << 4);
                    const __nv_bfloat16* ptr = x;
                    uint32_t bytes = 0;
                    if (rv && tap_ok[a]) {
                        const int ih = p * g.str_h - g.pad_h + tap_r[a] * g.dil_h;
                        const int iw = q * g.str_w - g.pad_w + tap_s[a] * g.dil_w;
                        if (ih >= 0 && ih < g.H && iw >= 0 && iw < g.W) {
                            ptr = x + (((size_t)n * g.H + ih) * g.W + iw) * g.Cp + tap_c[a];
                            bytes = 16;
                        }
                    }
                    cp_async_16(dst, ptr, bytes);
                }
            }
            cp_async_arrive_noinc(&full[stage]);
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }
        // epilogue: fp32 partial tile [k][n] of this split
        if (kb_end > kb_begin) {
            mbar_wait(tmem_full, 0);
            tc_fence_after();
        }
        const int row = warp * 32 + lane;
        const int k = m0 + row;
#pragma unroll 1
        for (int c0 = 0; c0 < WBN; c0 += 16) {
            uint32_t v[16];
            if (kb_end > kb_begin) {
                tmem_ld16(tmem_base + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
                tmem_ld_wait();
            } else {
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = 0u;
            }
            const int nn = n0 + c0;
            if (k >= g.K || nn >= g.Nn) continue;
            float* dst = partial + ((size_t)split * g.K + k) * g.Nn + nn;
            if (nn + 16 <= g.Nn) {
#pragma unroll
                for (int e = 0; e < 16; e += 4)
                    *reinterpret_cast<float4*>(dst + e) =
                        make_float4(__uint_as_float(v[e]), __uint_as_float(v[e + 1]),
                                    __uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
            } else {
                for (int e = 0; e < 16 && nn + e < g.Nn; ++e) dst[e] = __uint_as_float(v[e]);
            }
        }
    } else if (warp == 4) {
        constexpr uint32_t idesc = idesc_bf16_f32(BM, WBN, true, true);
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = kb_begin; kb < kb_end; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            {
                fence_proxy_async_smem();
                const uint32_t a_base = smem_u32(smem + stage * L::kStage);
                const uint32_t b_base = a_base + L::kA;
                // MN-major: 16 K rows = 2 core groups of 8 rows (SBO 1024 B);
                // the two 64-wide MN atoms are LBO = 8 KB apart.
                const uint64_t ad0 = umma_desc_sw128(a_base, L::kA / 2, 1024);
                const uint64_t bd0 = umma_desc_sw128(b_base, L::kB / 2, 1024);
                constexpr uint64_t ks = 2048 >> 4;
                mma4_bf16(tmem_base, ad0, ad0 + ks, ad0 + 2 * ks, ad0 + 3 * ks, bd0, bd0 + ks,
                          bd0 + 2 * ks, bd0 + 3 * ks, idesc, kb != kb_begin);
                mma_commit_elect(&empty[stage]);
                if (kb == kb_end - 1) mma_commit_elect(tmem_full);
            }
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        tc_fence_after();
        tmem_dealloc(tmem_base, WBN);
    }
}

// dW[k][n] = sum over splits (fixed order) -> bf16, filter layout [K][R][S][Cp].
__global__ void wgrad_reduce_kernel(const float* __restrict__ partial, int splits, int K, int Nn,
                                    __nv_bfloat16* __restrict__ dw) {
    const long long total = (long long)K * Nn;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        float acc = 0.0f;
        for (int s = 0; s < splits; ++s) acc += partial[(size_t)s * total + i];
        dw[i] = __float2bfloat16_rn(acc);
    }
}

}  // namespace
}  // namespace pk

using namespace pk;

extern "C" {

int pk_tc_wgrad_supported(const pk_conv_geom* g) {
    return g->groups == 1 && !g->transpose && pk_pitch(g->k) % 8 == 0 && tc::encode_fn() != nullptr;
}

static int wgrad_splits(const pk_conv_geom* g, int num_sms) {
    const int mt = (g->k + BM - 1) / BM;
    const int nt = (g->r * g->s * pk_pitch(g->cg) + WBN - 1) / WBN;
    const long long npq = (long long)g->n * g->p * g->q;
    const int num_kb = (int)((npq + BK - 1) / BK);
    int splits = (2 * num_sms + mt * nt - 1) / (mt * nt);
    const int max_splits = num_kb / 8 > 1 ? num_kb / 8 : 1;  // >= 8 k-blocks per split
    if (splits > max_splits) splits = max_splits;
    if (splits < 1) splits = 1;
    return splits;
}

size_t pk_tc_wgrad_workspace(const pk_conv_geom* g, int num_sms, const pk_tc_config* cfg) {
    const ActiveTcConfig active(cfg);
    if (pk_tma_wgrad_supported(g)) return pk_tma_wgrad_workspace(g, num_sms);
    return (size_t)wgrad_splits(g, num_sms) * g->k * g->r * g->s * pk_pitch(g->cg) * 4;
}

cudaError_t pk_cuda_igemm_tc_wgrad(const pk_conv_geom* g, const void* dy, const void* x, void* dw,
                                   void* workspace, int num_sms, const pk_tc_config* cfg,
                                   cudaStream_t st) {
    if (!pk_tc_wgrad_supported(g)) return cudaErrorNotSupported;
    const ActiveTcConfig active(cfg);
    if (pk_tma_wgrad_supported(g)) return pk_tma_wgrad(g, dy, x, dw, workspace, num_sms, st);
    WgGeom w{};
    w.K = g->k;
    w.Cp = g->x_pitch;
    w.Nn = g->r * g->s * g->f_pitch;
    if (g->f_pitch != g->x_pitch) return cudaErrorNotSupported;
    w.NPQ = g->n * g->p * g->q;
    w.P = g->p;
    w.Q = g->q;
    w.H = g->h;
    w.W = g->w;
    w.R = g->r;
    w.S = g->s;
    w.pad_h = g->pad_h;
    w.pad_w = g->pad_w;
    w.str_h = g->str_h;
    w.str_w = g->str_w;
    w.dil_h = g->dil_h;
    w.dil_w = g->dil_w;
    w.num_kb = (w.NPQ + BK - 1) / BK;
    const int splits = wgrad_splits(g, num_sms);
    w.kb_per_split = (w.num_kb + splits - 1) / splits;
    CUtensorMap amap;  // dY viewed as [NPQ][pitch(K)], box {64 channels, 64 rows}
    if (!tc::make_map_2d(&amap, dy, w.NPQ, g->y_pitch, g->y_pitch, BK)) return cudaErrorInvalidValue;
    constexpr int STAGES = 4;
    using L = WgSmem<STAGES>;
    static int attr_dev = -1;  // the attribute is per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
        cudaError_t err = cudaFuncSetAttribute(igemm_tc_wgrad_kernel<STAGES>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               L::kBytes);
        if (err != cudaSuccess) return err;
        attr_dev = dev;
    }
    dim3 grid((w.K + BM - 1) / BM, (w.Nn + WBN - 1) / WBN, splits);
    igemm_tc_wgrad_kernel<STAGES><<<grid, kThreads, L::kBytes, st>>>(
        amap, (const __nv_bfloat16*)x, (float*)workspace, w);
    const long long total = (long long)w.K * w.Nn;
    long long blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    wgrad_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>((const float*)workspace, splits, w.K,
                                                          w.Nn, (__nv_bfloat16*)dw);
    count_launch(2);
    return cudaGetLastError();
}

}  // extern "C"
