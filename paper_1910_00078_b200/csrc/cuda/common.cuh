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
    return e && (e->bias || e->bn_mean || e->act >= 0);
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
