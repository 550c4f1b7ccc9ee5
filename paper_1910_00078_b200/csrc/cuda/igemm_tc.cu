// tcgen05 implicit-GEMM convolution kernels for sm_100a (bf16 in, fp32
// accumulate in TMEM, bf16 out). This is the ImplicitGemm solver for bf16
// (the "composable kernels" blockwise -> LDS -> threadwise
// decomposition, re-designed for Blackwell) and the GEMM engine behind the
// bf16 Im2colGemm paths.
//
// Forward / backward-data ("fprop/dgrad" kernel):
//   D[pixel][out_ch] = sum_{(r,s,ch)} A[pixel][(r,s,ch)] * B[out_ch][(r,s,ch)]
//   * A (activations, NHWC) is gathered tile-by-tile straight from HBM/L2 by
//     4 producer warps with 16-byte cp.async (zero-fill for padding / stride
//     holes) into the canonical K-major SWIZZLE_128B layout;
//   * B (filter, [out][R][S][pitch]) is a plain 2-D TMA tile load (zero OOB
//     fill covers the K tail and out-of-range output channels);
//   * one elected thread of warp 4 issues tcgen05.mma (M=128, N=BLOCK_N, K=16)
//     into a TMEM accumulator; tcgen05.commit releases smem stages;
//   * the 4 producer warps then drain TMEM (tcgen05.ld 32x32b), apply the
//     fused epilogue (bias -> BN -> activation) and store bf16 NHWC.
//   dgrad gathers dY with the transposed index map (h + pad - r*dil) / stride
//   and uses the filter re-laid out as [C][R][S][pitch(K)].
//
// Backward-weights ("wgrad" kernel): D[k][(r,s,c)] = sum_{npq} dY[npq][k] *
//   X[npq shifted by (r,s)][c]; both operands are MN-major (the reduction
//   index npq is the strided one): dY tiles arrive by TMA, X rows by cp.async
//   gather. Split-K over npq with a deterministic fixed-order reduction.
#include <cuda.h>

#include <mutex>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace pk {
namespace {

using namespace pk::tc;

constexpr int BM = 128;      // UMMA M: output pixels (fprop/dgrad) or channels (wgrad)
constexpr int BK = 64;       // reduction elements per stage (128 bytes of bf16)
constexpr int kProducerThreads = 128;
constexpr int kThreads = 160;  // 4 producer/epilogue warps + 1 MMA warp

struct TcGeom {
    int M;                 // output rows
    int Ho, Wo;            // output image extent (row decode)
    int Hs, Ws;            // source image extent
    int src_pitch;         // channel pitch of the gathered source
    int red_ch;            // reduction channels per tap (multiple of 8)
    int R, S, pad_h, pad_w, str_h, str_w, dil_h, dil_w;
    int kred;              // R * S * red_ch
    int num_kb;            // ceil(kred / BK)
    int n_out;             // valid output channels
    int out_pitch;
    int P, Q;              // epilogue BN indexing extents
    int raster;
};

template <int BN, int STAGES>
struct FpropSmem {
    static constexpr int kA = BM * BK * 2;   // 16 KB
    static constexpr int kB = BN * BK * 2;
    static constexpr int kStage = kA + kB;
    static constexpr int kBarOff = STAGES * kStage;
    static constexpr int kBytes = kBarOff + (2 * STAGES + 1) * 8 + 16 + 1024;  // + align slack
};

template <int BN, int STAGES, bool DGRAD>
__global__ void __launch_bounds__(kThreads, 1)
    igemm_tc_fprop_kernel(const __grid_constant__ CUtensorMap bmap,
                          const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ out,
                          TcGeom g, pk_epilogue epi) {
    using L = FpropSmem<BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // rasterise: `raster` consecutive M tiles share one N tile sweep
    const int m_tiles = (g.M + BM - 1) / BM;
    int mt = blockIdx.x, nt = blockIdx.y;
    (void)m_tiles;
    const int m0 = mt * BM, n0 = nt * BN;

    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], kProducerThreads + 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tmem_full, 1);
        fence_barrier_init();
        tma_prefetch(&bmap);
    }
    if (warp == 4) tmem_alloc(tmem_slot, BN < 32 ? 32 : BN);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp < 4) {
        // ---------------- producers: A gather (+ B TMA by thread 0) ----------
        const int j = lane & 7;                   // 16-byte chunk within a 128-byte row
        const int rbase = warp * 32 + (lane >> 3);
        int row_img[8], row_h[8], row_w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int m = m0 + rbase + 4 * i;
            if (m < g.M) {
                const int hw = g.Ho * g.Wo;
                const int n = m / hw, rem = m - n * hw;
                const int oy = rem / g.Wo, ox = rem - oy * g.Wo;
                row_img[i] = n * g.Hs;
                if (DGRAD) {
                    row_h[i] = oy + g.pad_h;
                    row_w[i] = ox + g.pad_w;
                } else {
                    row_h[i] = oy * g.str_h - g.pad_h;
                    row_w[i] = ox * g.str_w - g.pad_w;
                }
            } else {
                row_img[i] = -1;
                row_h[i] = row_w[i] = 0;
            }
        }
        const int chunks_per_tap = g.red_ch >> 3;
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = 0; kb < g.num_kb; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * L::kStage;
            if (threadIdx.x == 0) {
                mbar_arrive_expect_tx(&full[stage], L::kB);
                tma_load_2d(smem_u32(sa + L::kA), &bmap, &full[stage], kb * BK, n0);
            }
            const int k8 = kb * (BK / 8) + j;
            const bool kvalid = k8 * 8 < g.kred;
            int r = 0, s = 0, c8 = 0;
            if (kvalid) {
                const int rs = k8 / chunks_per_tap;
                c8 = k8 - rs * chunks_per_tap;
                r = rs / g.S;
                s = rs - r * g.S;
            }
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
                    if (DGRAD) {
                        const int nh = row_h[i] - r * g.dil_h, nw = row_w[i] - s * g.dil_w;
                        ok = nh >= 0 && nw >= 0;
                        if (g.str_h > 1) ok = ok && (nh % g.str_h) == 0;
                        if (g.str_w > 1) ok = ok && (nw % g.str_w) == 0;
                        ih = nh / g.str_h;
                        iw = nw / g.str_w;
                        ok = ok && ih < g.Hs && iw < g.Ws;
                    } else {
                        ih = row_h[i] + r * g.dil_h;
                        iw = row_w[i] + s * g.dil_w;
                        ok = ih >= 0 && ih < g.Hs && iw >= 0 && iw < g.Ws;
                    }
                    if (ok) {
                        p = src + ((size_t)(row_img[i] + ih) * g.Ws + iw) * g.src_pitch + c8 * 8;
                        bytes = 16;
                    }
                }
                cp_async_16(dst, p, bytes);
            }
            cp_async_arrive_noinc(&full[stage]);
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }

        // ---------------- epilogue: TMEM -> registers -> global ---------------
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        const int row = warp * 32 + lane;
        const int m = m0 + row;
        const bool row_ok = m < g.M;
        int oy = 0, ox = 0;
        if (row_ok) {
            const int hw = g.Ho * g.Wo;
            const int rem = m % hw;
            oy = rem / g.Wo;
            ox = rem - oy * g.Wo;
        }
        const bool has_epi = epilogue_active(&epi);
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
            uint32_t v[16];
            tmem_ld16(tmem_base + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
            tmem_ld_wait();
            const int ch0 = n0 + c0;
            if (!row_ok || ch0 >= g.out_pitch) continue;
            __align__(16) __nv_bfloat16 o[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int ch = ch0 + e;
                float a = __uint_as_float(v[e]);
                if (ch >= g.n_out) {
                    a = 0.0f;
                } else if (has_epi) {
                    a = apply_epilogue(epi, a, ch, oy, ox, g.P, g.Q);
                }
                o[e] = __float2bfloat16_rn(a);
            }
            __nv_bfloat16* dst = out + (size_t)m * g.out_pitch + ch0;
            const uint4* ov = reinterpret_cast<const uint4*>(o);
            if (ch0 + 16 <= g.out_pitch) {
                reinterpret_cast<uint4*>(dst)[0] = ov[0];
                reinterpret_cast<uint4*>(dst)[1] = ov[1];
            } else {
                reinterpret_cast<uint4*>(dst)[0] = ov[0];  // pitch is a multiple of 8
            }
        }
    } else if (warp == 4) {
        // ---------------- MMA issuer ------------------------------------------
        constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, false, false);
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = 0; kb < g.num_kb; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            if (lane == 0) {
                fence_proxy_async_smem();
                const uint32_t a_base = smem_u32(smem + stage * L::kStage);
                const uint32_t b_base = a_base + L::kA;
#pragma unroll
                for (int k = 0; k < BK / 16; ++k) {
                    const uint64_t ad = umma_desc_sw128(a_base + k * 32, 16, 1024);
                    const uint64_t bd = umma_desc_sw128(b_base + k * 32, 16, 1024);
                    mma_bf16(tmem_base, ad, bd, idesc, (kb | k) != 0);
                }
                mma_commit(&empty[stage]);
                if (kb == g.num_kb - 1) mma_commit(tmem_full);
            }
            __syncwarp();
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
        tmem_dealloc(tmem_base, BN < 32 ? 32 : BN);
    }
}

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
            if (lane == 0) {
                fence_proxy_async_smem();
                const uint32_t a_base = smem_u32(smem + stage * L::kStage);
                const uint32_t b_base = a_base + L::kA;
#pragma unroll
                for (int k = 0; k < BK / 16; ++k) {
                    // MN-major: 16 K rows = 2 core groups of 8 rows (SBO 1024 B);
                    // the two 64-wide MN atoms are LBO = 8 KB apart.
                    const uint64_t ad = umma_desc_sw128(a_base + k * 2048, L::kA / 2, 1024);
                    const uint64_t bd = umma_desc_sw128(b_base + k * 2048, L::kB / 2, 1024);
                    mma_bf16(tmem_base, ad, bd, idesc, (kb != kb_begin) || (k != 0));
                }
                mma_commit(&empty[stage]);
                if (kb == kb_end - 1) mma_commit(tmem_full);
            }
            __syncwarp();
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

// ---------------------------------------------------------------------------
// host helpers

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 2-D bf16 row-major [rows][cols] (row stride in elements), 128-byte swizzle,
// box {64 cols, box_rows}, zero fill out of bounds.
bool make_map_2d(CUtensorMap* map, const void* base, long long rows, long long cols,
                 long long row_stride, int box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)row_stride * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int STAGES, bool DGRAD>
cudaError_t launch_fprop(const CUtensorMap& bmap, const void* src, void* out, const TcGeom& g,
                         const pk_epilogue& e, cudaStream_t st) {
    using L = FpropSmem<BN, STAGES>;
    auto kern = igemm_tc_fprop_kernel<BN, STAGES, DGRAD>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t err =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kBytes);
        if (err != cudaSuccess) return err;
        attr_set = true;
    }
    dim3 grid((g.M + BM - 1) / BM, (g.out_pitch + BN - 1) / BN);
    kern<<<grid, kThreads, L::kBytes, st>>>(bmap, (const __nv_bfloat16*)src, (__nv_bfloat16*)out,
                                            g, e);
    count_launch();
    return cudaGetLastError();
}

template <bool DGRAD>
cudaError_t dispatch_fprop(int bn, int stages, const CUtensorMap& bmap, const void* src, void* out,
                           const TcGeom& g, const pk_epilogue& e, cudaStream_t st) {
    if (bn <= 64) return launch_fprop<64, 4, DGRAD>(bmap, src, out, g, e, st);
    if (bn <= 128)
        return stages <= 3 ? launch_fprop<128, 3, DGRAD>(bmap, src, out, g, e, st)
                           : launch_fprop<128, 4, DGRAD>(bmap, src, out, g, e, st);
    return stages <= 3 ? launch_fprop<256, 3, DGRAD>(bmap, src, out, g, e, st)
                       : launch_fprop<256, 4, DGRAD>(bmap, src, out, g, e, st);
}

int pick_bn(int want, int n_out) {
    int bn = want <= 64 ? 64 : want <= 128 ? 128 : 256;
    int need = n_out <= 64 ? 64 : n_out <= 128 ? 128 : 256;
    return bn < need ? bn : need;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace
}  // namespace pk

using namespace pk;

extern "C" {

int pk_tc_fwd_supported(const pk_conv_geom* g) {
    return g->groups == 1 && !g->transpose && g->x_pitch % 8 == 0 && g->f_pitch % 8 == 0 &&
           g->y_pitch % 8 == 0 && encode_fn() != nullptr;
}

int pk_tc_dgrad_supported(const pk_conv_geom* g) {
    return g->groups == 1 && !g->transpose && encode_fn() != nullptr;
}

int pk_tc_wgrad_supported(const pk_conv_geom* g) {
    return g->groups == 1 && !g->transpose && pk_pitch(g->k) % 8 == 0 && encode_fn() != nullptr;
}

size_t pk_tc_dgrad_workspace(const pk_conv_geom* g) {
    // re-laid-out filter [C][R][S][pitch(K)] in bf16
    return (size_t)g->c * g->r * g->s * pk_pitch(g->k) * 2;
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

size_t pk_tc_wgrad_workspace(const pk_conv_geom* g, int num_sms) {
    return (size_t)wgrad_splits(g, num_sms) * g->k * g->r * g->s * pk_pitch(g->cg) * 4;
}

cudaError_t pk_cuda_igemm_tc_fwd(const pk_conv_geom* g, const void* x, const void* f, void* y,
                                 const pk_epilogue* epi, const pk_tc_config* cfg,
                                 cudaStream_t st) {
    if (!pk_tc_fwd_supported(g) || !aligned16(x) || !aligned16(f) || !aligned16(y))
        return cudaErrorNotSupported;
    TcGeom t{};
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
    t.P = g->p;
    t.Q = g->q;
    t.raster = cfg ? cfg->raster : 1;
    const int bn = pick_bn(cfg ? cfg->block_n : 256, g->k);
    CUtensorMap bmap;
    if (!make_map_2d(&bmap, f, g->k, t.kred, t.kred, bn)) return cudaErrorInvalidValue;
    pk_epilogue e{};
    e.act = -1;
    if (epi) e = *epi;
    return dispatch_fprop<false>(bn, cfg ? cfg->stages : 4, bmap, x, y, t, e, st);
}

cudaError_t pk_cuda_igemm_tc_dgrad(const pk_conv_geom* g, const void* dy, const void* f, void* dx,
                                   void* workspace, const pk_tc_config* cfg, cudaStream_t st) {
    if (!pk_tc_dgrad_supported(g)) return cudaErrorNotSupported;
    // B operand for dgrad: Wt[c][r][s][k] = W[k][r][s][c]
    cudaError_t err = pk_cuda_filter_to_dgrad(g, PK_BF16, f, workspace, st);
    if (err != cudaSuccess) return err;
    const int kp = pk_pitch(g->k);
    TcGeom t{};
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
    t.P = g->h;
    t.Q = g->w;
    const int bn = pick_bn(cfg ? cfg->block_n : 256, g->c);
    CUtensorMap bmap;
    if (!make_map_2d(&bmap, workspace, g->c, t.kred, t.kred, bn)) return cudaErrorInvalidValue;
    pk_epilogue e{};
    e.act = -1;
    return dispatch_fprop<true>(bn, cfg ? cfg->stages : 4, bmap, dy, dx, t, e, st);
}

cudaError_t pk_cuda_igemm_tc_wgrad(const pk_conv_geom* g, const void* dy, const void* x, void* dw,
                                   void* workspace, int num_sms, const pk_tc_config* cfg,
                                   cudaStream_t st) {
    (void)cfg;
    if (!pk_tc_wgrad_supported(g)) return cudaErrorNotSupported;
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
    if (!make_map_2d(&amap, dy, w.NPQ, g->y_pitch, g->y_pitch, BK)) return cudaErrorInvalidValue;
    constexpr int STAGES = 4;
    using L = WgSmem<STAGES>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t err = cudaFuncSetAttribute(igemm_tc_wgrad_kernel<STAGES>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               L::kBytes);
        if (err != cudaSuccess) return err;
        attr_set = true;
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
