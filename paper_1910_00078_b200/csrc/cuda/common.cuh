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
