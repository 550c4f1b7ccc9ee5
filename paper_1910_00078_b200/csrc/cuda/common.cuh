// Shared device helpers for the primkit-b200 kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace pk {

// Process-wide count of kernels launched by this library (pk_cuda_launch_count).
void count_launch(int n = 1);

template <typename T>
struct Elt;
template <>
struct Elt<float> {
    static __device__ __forceinline__ float load(const float* p) { return *p; }
    static __device__ __forceinline__ void store(float* p, float v) { *p = v; }
};
template <>
struct Elt<__nv_bfloat16> {
    static __device__ __forceinline__ float load(const __nv_bfloat16* p) {
        return __bfloat162float(*p);
    }
    // Round-to-nearest-even, the reference's round_bf16 (tensor.cpp:44-54)
    // for every non-NaN input.
    static __device__ __forceinline__ void store(__nv_bfloat16* p, float v) {
        *p = __float2bfloat16_rn(v);
    }
};

template <typename T>
__device__ __forceinline__ float ld(const T* p) { return Elt<T>::load(p); }
template <typename T>
__device__ __forceinline__ void st(T* p, float v) { Elt<T>::store(p, v); }

// The reference's activation_apply (primitives.cpp:154-164).
__device__ __forceinline__ float activate(int act, float alpha, float v) {
    switch (act) {
        case 0: return v > 0.0f ? v : 0.0f;
        case 1: return v > 0.0f ? v : alpha * v;
        case 2: return 1.0f / (1.0f + expf(-v));
        case 3: return tanhf(v);
        default: return v;
    }
}

// Fusion epilogue on one fp32 accumulator for output channel k at output
// pixel (oh, ow) of a P x Q image (fusion.cpp:384-398 order).
__device__ __forceinline__ float apply_epilogue(const pk_epilogue& e, float acc, int k, int oh,
                                                int ow, int P, int Q) {
    if (e.bias) acc += e.bias[k];
    if (e.bn_mean) {
        const int bi = e.bn_per_activation ? (k * P + oh) * Q + ow : k;
        if (e.bn_standalone) {
            const float inv = 1.0f / sqrtf(e.bn_var[bi] + e.bn_eps);
            acc = e.bn_gamma[bi] * (acc - e.bn_mean[bi]) * inv + e.bn_beta[bi];
        } else {
            acc = (acc - e.bn_mean[bi]) / sqrtf(e.bn_var[bi] + e.bn_eps) * e.bn_gamma[bi] +
                  e.bn_beta[bi];
        }
    }
    if (e.act >= 0) acc = activate(e.act, e.act_alpha, acc);
    return acc;
}

__host__ __device__ inline bool epilogue_active(const pk_epilogue* e) {
    return e && (e->bias || e->bn_mean || e->act >= 0 || e->ch_scale);
}

// Activation on the tensor-core epilogue path (bf16 outputs): ReLU/LeakyReLU
// exactly as the reference; sigmoid/tanh through the MUFU exp2 unit (relative
// error ~1e-6, far below the bf16 output rounding) so the unrolled epilogue
// stays compact in the instruction cache.
__device__ __forceinline__ float activate_fast(int act, float alpha, float v) {
    switch (act) {
        case 0: return v > 0.0f ? v : 0.0f;
        case 1: return v > 0.0f ? v : alpha * v;
        case 2: return __frcp_rn(1.0f + __expf(-v));
        case 3: return 2.0f * __frcp_rn(1.0f + __expf(-2.0f * v)) - 1.0f;
        default: return v;
    }
}

// Fused epilogue for 64 consecutive output channels [ch0, ch0 + 64) of one
// output pixel (oy, ox) of a P x Q image, in place on fp32 accumulators.
// ch_scale / ch_shift must be readable up to ch0 + 64 (host pads them);
// the unfolded form only touches channels below n_out.
__device__ __forceinline__ void epilogue_chunk64(const pk_epilogue& e, float (&x)[64], int ch0,
                                                 int n_out, int oy, int ox, int P, int Q) {
    if (e.ch_scale) {
        const float4* sc = reinterpret_cast<const float4*>(e.ch_scale + ch0);
        const float4* sh = reinterpret_cast<const float4*>(e.ch_shift + ch0);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const float4 s = __ldg(sc + j), t = __ldg(sh + j);
            x[4 * j + 0] = fmaf(x[4 * j + 0], s.x, t.x);
            x[4 * j + 1] = fmaf(x[4 * j + 1], s.y, t.y);
            x[4 * j + 2] = fmaf(x[4 * j + 2], s.z, t.z);
            x[4 * j + 3] = fmaf(x[4 * j + 3], s.w, t.w);
        }
    } else if (e.bias || e.bn_mean) {
        // general form (per-activation BN): rare, kept out of the fast path
#pragma unroll
        for (int j = 0; j < 64; ++j) {
            float a = x[j];
            const int k = ch0 + j;
            if (k >= n_out) continue;
            if (e.bias) a += __ldg(e.bias + k);
            if (e.bn_mean) {
                const int bi = e.bn_per_activation ? (k * P + oy) * Q + ox : k;
                a = (a - __ldg(e.bn_mean + bi)) / sqrtf(__ldg(e.bn_var + bi) + e.bn_eps) *
                        __ldg(e.bn_gamma + bi) +
                    __ldg(e.bn_beta + bi);
            }
            x[j] = a;
        }
    }
    const float alpha = e.act_alpha;
    if (e.act == 0) {
#pragma unroll
        for (int j = 0; j < 64; ++j) x[j] = activate_fast(0, alpha, x[j]);
    } else if (e.act == 1) {
#pragma unroll
        for (int j = 0; j < 64; ++j) x[j] = activate_fast(1, alpha, x[j]);
    } else if (e.act == 2) {
#pragma unroll
        for (int j = 0; j < 64; ++j) x[j] = activate_fast(2, alpha, x[j]);
    } else if (e.act == 3) {
#pragma unroll
        for (int j = 0; j < 64; ++j) x[j] = activate_fast(3, alpha, x[j]);
    }
}

// BN statistics of a staged 32-row x 64-channel bf16 tile (128-byte rows,
// 16-byte chunks XOR-swizzled by row & 7, as the tcgen05 epilogues stage
// them): lane l sums channels ch0 + 2l, ch0 + 2l + 1 over the rows set in
// `rows_ok` and adds (sum, sumsq) into part[channel][2].
__device__ __forceinline__ void epilogue_stats64(uint32_t stg_u, int lane, unsigned rows_ok,
                                                 float* part, int ch0, int n_out) {
    float s0 = 0.f, s1 = 0.f, q0 = 0.f, q1 = 0.f;
    const uint32_t wb = (lane & 3) << 2;
#pragma unroll 8
    for (int r = 0; r < 32; ++r) {
        if (!((rows_ok >> r) & 1u)) continue;
        uint32_t wv;
        asm volatile("ld.shared.b32 %0, [%1];"
                     : "=r"(wv)
                     : "r"(stg_u + r * 128 + ((((lane >> 2) ^ (r & 7)) << 4) | wb)));
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv));
        s0 += f.x;
        q0 = fmaf(f.x, f.x, q0);
        s1 += f.y;
        q1 = fmaf(f.y, f.y, q1);
    }
    const int ch = ch0 + 2 * lane;
    if (ch < n_out) {
        atomicAdd(part + 2 * ch, s0);
        atomicAdd(part + 2 * ch + 1, q0);
    }
    if (ch + 1 < n_out) {
        atomicAdd(part + 2 * ch + 2, s1);
        atomicAdd(part + 2 * ch + 3, q1);
    }
}

// Backward variant: dz from the staged tile, y (the preceding BN's input) from
// global memory at the same pixel / channels (lane l: channels ch0+2l, +1;
// `pix` = this lane's own row pixel, broadcast per row).
__device__ __forceinline__ void epilogue_bnbwd_stats64(const pk_epilogue& e, uint32_t stg_u,
                                                       int lane, unsigned rows_ok, long long pix,
                                                       float* part, int ch0, int n_out,
                                                       int pitch) {
    const int ch = ch0 + 2 * lane;
    const bool v0 = ch < n_out, v1 = ch + 1 < n_out;
    const float g0 = v0 ? e.bnb_gamma[ch] : 0.f, g1 = v1 ? e.bnb_gamma[ch + 1] : 0.f;
    const float b0 = v0 ? e.bnb_beta[ch] : 0.f, b1 = v1 ? e.bnb_beta[ch + 1] : 0.f;
    const float m0 = v0 ? e.bnb_mean[ch] : 0.f, m1 = v1 ? e.bnb_mean[ch + 1] : 0.f;
    const float i0 = v0 ? e.bnb_invstd[ch] : 0.f, i1 = v1 ? e.bnb_invstd[ch + 1] : 0.f;
    const __nv_bfloat16* y = static_cast<const __nv_bfloat16*>(e.bnb_y);
    float s0 = 0.f, s1 = 0.f, t0 = 0.f, t1 = 0.f;
    const uint32_t wb = (lane & 3) << 2;
#pragma unroll 4
    for (int r = 0; r < 32; ++r) {
        const long long rp = __shfl_sync(0xffffffffu, pix, r);
        if (!((rows_ok >> r) & 1u)) continue;
        uint32_t wv, yv = 0u;
        asm volatile("ld.shared.b32 %0, [%1];"
                     : "=r"(wv)
                     : "r"(stg_u + r * 128 + ((((lane >> 2) ^ (r & 7)) << 4) | wb)));
        if (v0) yv = __ldg(reinterpret_cast<const unsigned int*>(y + rp * pitch + ch));
        const float2 dz = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&wv));
        const float2 yy = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&yv));
        float d0 = dz.x, d1 = dz.y;
        if (e.bnb_relu) {
            // the forward mask, recomputed exactly as bn_apply_bf16x8_kernel does
            if (!(g0 * (yy.x - m0) * i0 + b0 > 0.0f)) d0 = 0.f;
            if (!(g1 * (yy.y - m1) * i1 + b1 > 0.0f)) d1 = 0.f;
        }
        s0 += d0;
        t0 = fmaf(d0, (yy.x - m0) * i0, t0);
        s1 += d1;
        t1 = fmaf(d1, (yy.y - m1) * i1, t1);
    }
    if (v0) {
        atomicAdd(part + 2 * ch, s0);
        atomicAdd(part + 2 * ch + 1, t0);
    }
    if (v1) {
        atomicAdd(part + 2 * ch + 2, s1);
        atomicAdd(part + 2 * ch + 3, t1);
    }
}

// Forward or backward BN statistics of a staged tile (see pk_epilogue).
__device__ __forceinline__ void epilogue_bn_stats(const pk_epilogue& e, uint32_t stg_u, int lane,
                                                  bool row_ok, long long pix, int ch0, int n_out,
                                                  int pitch) {
    const unsigned ok = __ballot_sync(0xffffffffu, row_ok);
    float* part = e.stats + (size_t)blockIdx.x * n_out * 2;
    if (e.bnb_y)
        epilogue_bnbwd_stats64(e, stg_u, lane, ok, pix, part, ch0, n_out, pitch);
    else
        epilogue_stats64(stg_u, lane, ok, part, ch0, n_out);
}

inline unsigned ceil_div(long long a, long long b) { return (unsigned)((a + b - 1) / b); }

}  // namespace pk

// Dispatch on the storage element type.
#define PK_DISPATCH_DTYPE(dtype, T, ...)        \
    do {                                        \
        if ((dtype) == PK_BF16) {               \
            using T = __nv_bfloat16;            \
            __VA_ARGS__;                        \
        } else {                                \
            using T = float;                    \
            __VA_ARGS__;                        \
        }                                       \
    } while (0)
