// Pooling and softmax (the ops around the convolutions
// in a ResNet training step), reference semantics of
// proj/src/core/primitives.cpp:204-370.
//
// Pooling runs on the device activation layout (NHWC, channel pitch, f32 or
// bf16): a thread owns 8 consecutive channels of one pixel, so every window tap
// is one 16-byte (bf16) / 32-byte (f32) load per thread and a warp reads
// contiguous channel vectors. HBM-bound; each input is read once per window
// it falls in (window / stride overlap).
// * forward: max keeps the FIRST maximum in window scan order (strict >), its
//   linear NCHW input index (int64, -1 for an empty window), average divides
//   the double sum of the valid taps by their count — exactly the reference.
// * backward is a gather: each input element sums, in increasing output
//   order, the contributions of the windows that cover it (max: only windows
//   whose argmax is this element; avg: dy / count). The reference scatters in
//   that same output order with a rounding store per addition, which the
//   gather reproduces (bf16: round after every add), so results are identical
//   and the kernel needs no atomics (deterministic).
//
// Softmax runs on a packed tensor viewed as [outer][axis][inner]: a warp per
// row when inner == 1 (the classifier case), a thread per (outer, inner)
// column otherwise; max in float, denominator in double (reference
// primitives.cpp:329-351), backward dot in double (353-370).
#include "common.cuh"

namespace pk {
namespace {

template <typename T>
struct Vec8;
template <>
struct Vec8<float> {
    static __device__ __forceinline__ void load(const float* p, float v[8]) {
        const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
    static __device__ __forceinline__ void store(float* p, const float v[8]) {
        reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
    static __device__ __forceinline__ float round(float v) { return v; }
};
template <>
struct Vec8<__nv_bfloat16> {
    static __device__ __forceinline__ void load(const __nv_bfloat16* p, float v[8]) {
        const uint4 u = *reinterpret_cast<const uint4*>(p);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __bfloat1622float2(h[i]);
            v[2 * i] = f.x;
            v[2 * i + 1] = f.y;
        }
    }
    static __device__ __forceinline__ void store(__nv_bfloat16* p, const float v[8]) {
        uint4 u;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
        *reinterpret_cast<uint4*>(p) = u;
    }
    static __device__ __forceinline__ float round(float v) {
        return __bfloat162float(__float2bfloat16_rn(v));
    }
};

__device__ __forceinline__ int out_extent_lo(int i_in, int pad, int win, int str) {
    // smallest output index whose window [o*str - pad, o*str - pad + win) covers i_in
    const int t = i_in + pad - win + 1;
    return t <= 0 ? 0 : (t + str - 1) / str;
}

template <typename T, bool MAX>
__global__ void __launch_bounds__(256) pool_fwd_kernel(pk_pool_geom g, const T* __restrict__ x,
                                                       T* __restrict__ y, long long* __restrict__ idx) {
    const int cv = g.pitch / 8;  // channel vectors per pixel
    const long long total = (long long)g.n * g.oh * g.ow * cv;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int v = (int)(t % cv);
        long long pix = t / cv;
        const int j = (int)(pix % g.ow);
        pix /= g.ow;
        const int i = (int)(pix % g.oh);
        const int n = (int)(pix / g.oh);
        float best[8];
        long long bidx[8];
        double sum[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            best[e] = -INFINITY;
            bidx[e] = -1;
            sum[e] = 0.0;
        }
        int count = 0;
        for (int p = 0; p < g.win_h; ++p) {
            const int ih = i * g.str_h - g.pad_h + p;
            if (ih < 0 || ih >= g.h) continue;
            for (int q = 0; q < g.win_w; ++q) {
                const int iw = j * g.str_w - g.pad_w + q;
                if (iw < 0 || iw >= g.w) continue;
                float xv[8];
                Vec8<T>::load(x + (((long long)n * g.h + ih) * g.w + iw) * g.pitch + v * 8, xv);
                ++count;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    if (MAX) {
                        if (xv[e] > best[e]) {
                            best[e] = xv[e];
                            bidx[e] = (((long long)n * g.c + v * 8 + e) * g.h + ih) * g.w + iw;
                        }
                    } else {
                        sum[e] += xv[e];
                    }
                }
            }
        }
        float out[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const bool real = v * 8 + e < g.c;
            out[e] = !real || !count ? 0.0f : MAX ? best[e] : (float)(sum[e] / count);
        }
        Vec8<T>::store(y + (((long long)n * g.oh + i) * g.ow + j) * g.pitch + v * 8, out);
        if (MAX && idx) {
            long long* o = idx + (((long long)n * g.oh + i) * g.ow + j) * g.c;
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (v * 8 + e < g.c) o[v * 8 + e] = count ? bidx[e] : -1;
        }
    }
}

template <typename T, bool MAX>
__global__ void __launch_bounds__(256) pool_bwd_kernel(pk_pool_geom g, const T* __restrict__ dy,
                                                       const long long* __restrict__ idx,
                                                       T* __restrict__ dx) {
    const int cv = g.pitch / 8;
    const long long total = (long long)g.n * g.h * g.w * cv;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int v = (int)(t % cv);
        long long pix = t / cv;
        const int iw = (int)(pix % g.w);
        pix /= g.w;
        const int ih = (int)(pix % g.h);
        const int n = (int)(pix / g.h);
        float acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
        const int i0 = out_extent_lo(ih, g.pad_h, g.win_h, g.str_h);
        const int i1 = min(g.oh - 1, (ih + g.pad_h) / g.str_h);
        const int j0 = out_extent_lo(iw, g.pad_w, g.win_w, g.str_w);
        const int j1 = min(g.ow - 1, (iw + g.pad_w) / g.str_w);
        for (int i = i0; i <= i1; ++i)
            for (int j = j0; j <= j1; ++j) {
                float dv[8];
                Vec8<T>::load(dy + (((long long)n * g.oh + i) * g.ow + j) * g.pitch + v * 8, dv);
                if (MAX) {
                    const long long* o = idx + (((long long)n * g.oh + i) * g.ow + j) * g.c;
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int c = v * 8 + e;
                        if (c < g.c && o[c] == (((long long)n * g.c + c) * g.h + ih) * g.w + iw)
                            acc[e] = Vec8<T>::round(acc[e] + dv[e]);
                    }
                } else {
                    // valid taps of window (i, j) (the reference's count)
                    const int h0 = max(0, i * g.str_h - g.pad_h), h1 = min(g.h, i * g.str_h - g.pad_h + g.win_h);
                    const int w0 = max(0, j * g.str_w - g.pad_w), w1 = min(g.w, j * g.str_w - g.pad_w + g.win_w);
                    const float cnt = (float)((h1 - h0) * (w1 - w0));
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        if (v * 8 + e < g.c) acc[e] = Vec8<T>::round(acc[e] + dv[e] / cnt);
                }
            }
        Vec8<T>::store(dx + (((long long)n * g.h + ih) * g.w + iw) * g.pitch + v * 8, acc);
    }
}

template <typename T>
__global__ void __launch_bounds__(256) softmax_rows_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                           long long rows, int axis) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x / 32);
    for (long long r = blockIdx.x * (long long)(blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
        const T* xr = x + r * axis;
        float mx = -INFINITY;
        for (int a = lane; a < axis; a += 32) mx = fmaxf(mx, ld(xr + a));
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        double den = 0.0;
        for (int a = lane; a < axis; a += 32) den += exp((double)(ld(xr + a) - mx));
#pragma unroll
        for (int o = 16; o; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
        for (int a = lane; a < axis; a += 32) st(y + r * axis + a, (float)(exp((double)(ld(xr + a) - mx)) / den));
    }
}

template <typename T>
__global__ void __launch_bounds__(256) softmax_cols_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                           long long outer, int axis, long long inner) {
    const long long total = outer * inner;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long o = t / inner, i = t % inner;
        const T* xc = x + o * axis * inner + i;
        float mx = ld(xc);
        for (int a = 1; a < axis; ++a) mx = fmaxf(mx, ld(xc + a * inner));
        double den = 0.0;
        for (int a = 0; a < axis; ++a) den += exp((double)(ld(xc + a * inner) - mx));
        for (int a = 0; a < axis; ++a)
            st(y + o * axis * inner + i + a * inner, (float)(exp((double)(ld(xc + a * inner) - mx)) / den));
    }
}

template <typename T>
__global__ void __launch_bounds__(256) softmax_bwd_rows_kernel(const T* __restrict__ y, const T* __restrict__ dy,
                                                               T* __restrict__ dx, long long rows, int axis) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x / 32);
    for (long long r = blockIdx.x * (long long)(blockDim.x / 32) + threadIdx.x / 32; r < rows; r += warps) {
        const long long b = r * axis;
        double dot = 0.0;
        for (int a = lane; a < axis; a += 32) dot += (double)ld(dy + b + a) * ld(y + b + a);
#pragma unroll
        for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        for (int a = lane; a < axis; a += 32)
            st(dx + b + a, (float)(ld(y + b + a) * ((double)ld(dy + b + a) - dot)));
    }
}

template <typename T>
__global__ void __launch_bounds__(256) softmax_bwd_cols_kernel(const T* __restrict__ y, const T* __restrict__ dy,
                                                               T* __restrict__ dx, long long outer, int axis,
                                                               long long inner) {
    const long long total = outer * inner;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long b = (t / inner) * axis * inner + t % inner;
        double dot = 0.0;
        for (int a = 0; a < axis; ++a) dot += (double)ld(dy + b + a * inner) * ld(y + b + a * inner);
        for (int a = 0; a < axis; ++a)
            st(dx + b + a * inner, (float)(ld(y + b + a * inner) * ((double)ld(dy + b + a * inner) - dot)));
    }
}

unsigned grid_for(long long work, int per_block = 256) {
    long long b = (work + per_block - 1) / per_block;
    if (b < 1) b = 1;
    if (b > 148 * 32) b = 148 * 32;
    return (unsigned)b;
}

}  // namespace
}  // namespace pk

using namespace pk;

extern "C" {

int pk_pool_supported(const pk_pool_geom* g) {
    return g->pitch % 8 == 0 && g->pitch >= g->c && g->win_h >= 1 && g->win_w >= 1 && g->str_h >= 1 &&
           g->str_w >= 1 && g->pad_h >= 0 && g->pad_w >= 0 && g->oh >= 1 && g->ow >= 1;
}

cudaError_t pk_cuda_pool_fwd(const pk_pool_geom* g, int dtype, int is_max, const void* x, void* y,
                             long long* indices, cudaStream_t st) {
    if (!pk_pool_supported(g) || (reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15)
        return cudaErrorNotSupported;
    const unsigned grid = grid_for((long long)g->n * g->oh * g->ow * (g->pitch / 8));
    PK_DISPATCH_DTYPE(dtype, T, {
        if (is_max)
            pool_fwd_kernel<T, true><<<grid, 256, 0, st>>>(*g, (const T*)x, (T*)y, indices);
        else
            pool_fwd_kernel<T, false><<<grid, 256, 0, st>>>(*g, (const T*)x, (T*)y, nullptr);
    });
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_pool_bwd(const pk_pool_geom* g, int dtype, int is_max, const void* dy,
                             const long long* indices, void* dx, cudaStream_t st) {
    if (!pk_pool_supported(g) || (is_max && !indices) ||
        (reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(dx)) & 15)
        return cudaErrorNotSupported;
    const unsigned grid = grid_for((long long)g->n * g->h * g->w * (g->pitch / 8));
    PK_DISPATCH_DTYPE(dtype, T, {
        if (is_max)
            pool_bwd_kernel<T, true><<<grid, 256, 0, st>>>(*g, (const T*)dy, indices, (T*)dx);
        else
            pool_bwd_kernel<T, false><<<grid, 256, 0, st>>>(*g, (const T*)dy, nullptr, (T*)dx);
    });
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_softmax_fwd(int dtype, const void* x, void* y, long long outer, int axis,
                                long long inner, cudaStream_t st) {
    if (outer < 1 || axis < 1 || inner < 1) return cudaSuccess;
    PK_DISPATCH_DTYPE(dtype, T, {
        if (inner == 1)
            softmax_rows_kernel<T><<<grid_for(outer * 32), 256, 0, st>>>((const T*)x, (T*)y, outer, axis);
        else
            softmax_cols_kernel<T><<<grid_for(outer * inner), 256, 0, st>>>((const T*)x, (T*)y, outer, axis,
                                                                            inner);
    });
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_softmax_bwd(int dtype, const void* y, const void* dy, void* dx, long long outer,
                                int axis, long long inner, cudaStream_t st) {
    if (outer < 1 || axis < 1 || inner < 1) return cudaSuccess;
    PK_DISPATCH_DTYPE(dtype, T, {
        if (inner == 1)
            softmax_bwd_rows_kernel<T><<<grid_for(outer * 32), 256, 0, st>>>((const T*)y, (const T*)dy, (T*)dx,
                                                                             outer, axis);
        else
            softmax_bwd_cols_kernel<T><<<grid_for(outer * inner), 256, 0, st>>>((const T*)y, (const T*)dy,
                                                                                (T*)dx, outer, axis, inner);
    });
    count_launch();
    return cudaGetLastError();
}

}  // extern "C"
