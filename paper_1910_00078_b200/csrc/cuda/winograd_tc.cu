// Winograd F(m x m, 3 x 3) forward convolution on the tensor cores (bf16 storage,
// fp32 arithmetic), m = 2 (the reference's F(2,3), proj/src/core/conv.cpp:269-365)
// or m = 4 (F(4,3), alpha = 6).
//
//   U[xi][k][c]  = (G g G^T)[xi]              filter transform   (winograd_filter_kernel)
//   V[xi][t][c]  = (B^T d B)[xi]              input transform    (winograd_input_kernel)
//   M[xi][t][k]  = sum_c V[xi][t][c] U[xi][k][c]   alpha^2 tcgen05 GEMMs in ONE batched launch
//                                                  (conv_tc.cu PLAIN mode, pk_cuda_gemm_tc_batched)
//   y[tile]      = epilogue((A^T M A))        output transform   (winograd_output_kernel)
//
// Transforms: one thread owns a (tile, channel pair) and keeps the whole
// alpha x alpha patch of both channels in registers (bf16x2 loads: a warp reads
// 128 contiguous bytes of one pixel row, so every patch load is coalesced),
// applies the separable transform in fp32 and rounds once to bf16. Edge tiles
// are zero padded on input and cropped on output exactly as the reference.
// V and M live in the caller's workspace; large problems are processed in
// chunks of tiles so the workspace stays bounded (pk_winograd_tc_workspace).
//
// Transform-domain precision: F(2,3) stores U, V, M in bf16 (the reference's
// round-on-store element type). F(4,3) amplifies every rounding through its
// 6x6 transforms (B^T entries up to 5, A^T up to 8): in bf16 the U, V and M
// roundings alone each cost ~1.8e-2 relative L2, so F(4,3) runs its transform
// domain in IEEE fp16 (8x finer mantissa, kind::f16 MMAs with fp32
// accumulation at the same rate), valid while |V| and |M| stay below 65504.
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace pk {
namespace {

template <int M_>
struct Wino;

template <>
struct Wino<2> {
    static constexpr int A = 4;
    // B^T (alpha x alpha), G (alpha x 3), A^T (m x alpha)
    static __device__ __forceinline__ float bt(int i, int j) {
        constexpr float t[4][4] = {{1, 0, -1, 0}, {0, 1, 1, 0}, {0, -1, 1, 0}, {0, 1, 0, -1}};
        return t[i][j];
    }
    static __device__ __forceinline__ float gm(int i, int j) {
        constexpr float t[4][3] = {{1, 0, 0}, {.5f, .5f, .5f}, {.5f, -.5f, .5f}, {0, 0, 1}};
        return t[i][j];
    }
    static __device__ __forceinline__ float at(int i, int j) {
        constexpr float t[2][4] = {{1, 1, 1, 0}, {0, 1, -1, -1}};
        return t[i][j];
    }
};

template <>
struct Wino<4> {
    static constexpr int A = 6;
    static __device__ __forceinline__ float bt(int i, int j) {
        constexpr float t[6][6] = {{4, 0, -5, 0, 1, 0},  {0, -4, -4, 1, 1, 0},
                                   {0, 4, -4, -1, 1, 0}, {0, -2, -1, 2, 1, 0},
                                   {0, 2, -1, -2, 1, 0}, {0, 4, 0, -5, 0, 1}};
        return t[i][j];
    }
    static __device__ __forceinline__ float gm(int i, int j) {
        constexpr float t[6][3] = {{1.f / 4, 0, 0},
                                   {-1.f / 6, -1.f / 6, -1.f / 6},
                                   {-1.f / 6, 1.f / 6, -1.f / 6},
                                   {1.f / 24, 1.f / 12, 1.f / 6},
                                   {1.f / 24, -1.f / 12, 1.f / 6},
                                   {0, 0, 1}};
        return t[i][j];
    }
    static __device__ __forceinline__ float at(int i, int j) {
        constexpr float t[4][6] = {
            {1, 1, 1, 1, 1, 0}, {0, 1, -1, 2, -2, 0}, {0, 1, 1, 4, 4, 0}, {0, 1, -1, 8, -8, 1}};
        return t[i][j];
    }
};

__device__ __forceinline__ float2 ld_bf2(const __nv_bfloat16* p) {
    const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(p);
    return __bfloat1622float2(v);
}
__device__ __forceinline__ float2 ld_bf2(const __half* p) {
    return __half22float2(*reinterpret_cast<const __half2*>(p));
}
__device__ __forceinline__ void st_bf2(__nv_bfloat16* p, float a, float b) {
    *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(a, b);
}
__device__ __forceinline__ void st_bf2(__half* p, float a, float b) {
    *reinterpret_cast<__half2*>(p) = __floats2half2_rn(a, b);
}

// element type of U, V, M for F(m x m, 3 x 3)
template <int M_>
using TDom = typename std::conditional<M_ == 4, __half, __nv_bfloat16>::type;

struct WinoArgs {
    int n, h, w, p, q, pad_h, pad_w;
    int th, tw;           // tiles per image row / column
    long long t0, tc;     // first tile and tile count of this chunk
    int rows;             // rows per transform position in V / M (tc rounded up to 128)
    int cp, k, kp;        // input channel pitch, output channels, output pitch
};

// V[xi][t - t0][c] = (B^T d B)[xi] for one channel pair; rows tc..rows-1 are zero.
template <int M_>
__global__ void __launch_bounds__(256) winograd_input_kernel(WinoArgs a,
                                                             const __nv_bfloat16* __restrict__ x,
                                                             TDom<M_>* __restrict__ v) {
    using W = Wino<M_>;
    constexpr int AL = W::A;
    const int c2n = a.cp / 2;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long lt = idx / c2n;
    const int c = (int)(idx - lt * c2n) * 2;
    if (lt >= a.rows) return;
    const size_t plane = (size_t)a.rows * a.cp;
    TDom<M_>* vo = v + (size_t)lt * a.cp + c;
    if (lt >= a.tc) {
#pragma unroll
        for (int xi = 0; xi < AL * AL; ++xi) st_bf2(vo + xi * plane, 0.f, 0.f);
        return;
    }
    const long long t = a.t0 + lt;
    const int tj = (int)(t % a.tw);
    const long long r = t / a.tw;
    const int ti = (int)(r % a.th);
    const int n = (int)(r / a.th);
    const int h0 = ti * M_ - a.pad_h, w0 = tj * M_ - a.pad_w;
    const __nv_bfloat16* xp = x + (size_t)n * a.h * a.w * a.cp + c;
    float d0[AL][AL], d1[AL][AL];
#pragma unroll
    for (int i = 0; i < AL; ++i) {
        const int ih = h0 + i;
        const bool rok = ih >= 0 && ih < a.h;
#pragma unroll
        for (int j = 0; j < AL; ++j) {
            const int iw = w0 + j;
            float2 vv = make_float2(0.f, 0.f);
            if (rok && iw >= 0 && iw < a.w) vv = ld_bf2(xp + ((size_t)ih * a.w + iw) * a.cp);
            d0[i][j] = vv.x;
            d1[i][j] = vv.y;
        }
    }
    // rows: T = B^T d
    float t0[AL][AL], t1[AL][AL];
#pragma unroll
    for (int i = 0; i < AL; ++i)
#pragma unroll
        for (int j = 0; j < AL; ++j) {
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int l = 0; l < AL; ++l) {
                const float b = W::bt(i, l);
                if (b != 0.f) {
                    s0 += b * d0[l][j];
                    s1 += b * d1[l][j];
                }
            }
            t0[i][j] = s0;
            t1[i][j] = s1;
        }
    // columns: V = T B
#pragma unroll
    for (int i = 0; i < AL; ++i)
#pragma unroll
        for (int j = 0; j < AL; ++j) {
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int l = 0; l < AL; ++l) {
                const float b = W::bt(j, l);
                if (b != 0.f) {
                    s0 += t0[i][l] * b;
                    s1 += t1[i][l] * b;
                }
            }
            st_bf2(vo + (i * AL + j) * plane, s0, s1);
        }
}

// U[xi][k][c] = (G g G^T)[xi] for filter f [K][3][3][cp]; one thread per (k, channel pair).
template <int M_>
__global__ void __launch_bounds__(256) winograd_filter_kernel(int K, int cp,
                                                              const __nv_bfloat16* __restrict__ f,
                                                              TDom<M_>* __restrict__ u) {
    using W = Wino<M_>;
    constexpr int AL = W::A;
    const int c2n = cp / 2;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= K * c2n) return;
    const int k = idx / c2n, c = (idx - k * c2n) * 2;
    float g0[3][3], g1[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            const float2 v = ld_bf2(f + ((size_t)(k * 3 + r) * 3 + s) * cp + c);
            g0[r][s] = v.x;
            g1[r][s] = v.y;
        }
    float t0[AL][3], t1[AL][3];
#pragma unroll
    for (int i = 0; i < AL; ++i)
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            float a0 = 0.f, a1 = 0.f;
#pragma unroll
            for (int r = 0; r < 3; ++r) {
                a0 += W::gm(i, r) * g0[r][s];
                a1 += W::gm(i, r) * g1[r][s];
            }
            t0[i][s] = a0;
            t1[i][s] = a1;
        }
    const size_t plane = (size_t)K * cp;
#pragma unroll
    for (int i = 0; i < AL; ++i)
#pragma unroll
        for (int j = 0; j < AL; ++j) {
            float a0 = 0.f, a1 = 0.f;
#pragma unroll
            for (int s = 0; s < 3; ++s) {
                a0 += t0[i][s] * W::gm(j, s);
                a1 += t1[i][s] * W::gm(j, s);
            }
            st_bf2(u + (i * AL + j) * plane + (size_t)k * cp + c, a0, a1);
        }
}

// y[n][m*ti + i][m*tj + j][k] = epilogue((A^T M A)[i][j]), cropped at the edges.
template <int M_>
__global__ void __launch_bounds__(256) winograd_output_kernel(WinoArgs a,
                                                              const TDom<M_>* __restrict__ mm,
                                                              __nv_bfloat16* __restrict__ y,
                                                              pk_epilogue e) {
    using W = Wino<M_>;
    constexpr int AL = W::A;
    const int k2n = a.kp / 2;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long lt = idx / k2n;
    const int k = (int)(idx - lt * k2n) * 2;
    if (lt >= a.tc || k >= a.k) return;
    const size_t plane = (size_t)a.rows * a.kp;
    const TDom<M_>* mp = mm + (size_t)lt * a.kp + k;
    float m0[AL][AL], m1[AL][AL];
#pragma unroll
    for (int xi = 0; xi < AL * AL; ++xi) {
        const float2 v = ld_bf2(mp + xi * plane);
        m0[xi / AL][xi % AL] = v.x;
        m1[xi / AL][xi % AL] = v.y;
    }
    float t0[M_][AL], t1[M_][AL];
#pragma unroll
    for (int i = 0; i < M_; ++i)
#pragma unroll
        for (int j = 0; j < AL; ++j) {
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int l = 0; l < AL; ++l) {
                const float c = W::at(i, l);
                if (c != 0.f) {
                    s0 += c * m0[l][j];
                    s1 += c * m1[l][j];
                }
            }
            t0[i][j] = s0;
            t1[i][j] = s1;
        }
    const long long t = a.t0 + lt;
    const int tj = (int)(t % a.tw);
    const long long r = t / a.tw;
    const int ti = (int)(r % a.th);
    const int n = (int)(r / a.th);
    const bool epi = epilogue_active(&e);
    const bool k1 = k + 1 < a.k;
#pragma unroll
    for (int i = 0; i < M_; ++i) {
        const int oh = ti * M_ + i;
        if (oh >= a.p) break;
#pragma unroll
        for (int j = 0; j < M_; ++j) {
            const int ow = tj * M_ + j;
            if (ow >= a.q) break;
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int l = 0; l < AL; ++l) {
                const float c = W::at(j, l);
                if (c != 0.f) {
                    s0 += t0[i][l] * c;
                    s1 += t1[i][l] * c;
                }
            }
            if (epi) {
                s0 = apply_epilogue(e, s0, k, oh, ow, a.p, a.q);
                s1 = k1 ? apply_epilogue(e, s1, k + 1, oh, ow, a.p, a.q) : 0.f;
            } else if (!k1) {
                s1 = 0.f;
            }
            st_bf2(y + (((size_t)n * a.p + oh) * a.q + ow) * a.kp + k, s0, s1);
        }
    }
}

constexpr size_t kChunkBudget = size_t(1) << 31;  // V + M bytes per chunk

size_t align256(size_t v) { return (v + 255) / 256 * 256; }

long long tiles_of(const pk_conv_geom* g, int m) {
    return (long long)g->n * ((g->p + m - 1) / m) * ((g->q + m - 1) / m);
}

size_t u_bytes(const pk_conv_geom* g, int m) {
    return align256((size_t)(m + 2) * (m + 2) * g->k * g->x_pitch * 2);
}

size_t bytes_per_tile(const pk_conv_geom* g, int m) {
    return (size_t)(m + 2) * (m + 2) * (g->x_pitch + g->y_pitch) * 2;
}

template <int M_>
cudaError_t run(const pk_conv_geom* g, const void* x, const void* f, void* y,
                const pk_epilogue* epi, void* ws, size_t ws_bytes, cudaStream_t st) {
    constexpr int AL = M_ + 2;
    const size_t ub = u_bytes(g, M_);
    if (ws_bytes < ub + 128 * bytes_per_tile(g, M_)) return cudaErrorNotSupported;
    auto* u = static_cast<TDom<M_>*>(ws);
    auto* v = reinterpret_cast<TDom<M_>*>(static_cast<char*>(ws) + ub);
    {
        const int total = g->k * (g->x_pitch / 2);
        winograd_filter_kernel<M_><<<ceil_div(total, 256), 256, 0, st>>>(
            g->k, g->x_pitch, static_cast<const __nv_bfloat16*>(f), u);
        count_launch();
    }
    WinoArgs a{};
    a.n = g->n;
    a.h = g->h;
    a.w = g->w;
    a.p = g->p;
    a.q = g->q;
    a.pad_h = g->pad_h;
    a.pad_w = g->pad_w;
    a.th = (g->p + M_ - 1) / M_;
    a.tw = (g->q + M_ - 1) / M_;
    a.cp = g->x_pitch;
    a.k = g->k;
    a.kp = g->y_pitch;
    const long long T = tiles_of(g, M_);
    long long chunk = (long long)((ws_bytes - ub) / bytes_per_tile(g, M_)) / 128 * 128;
    if (chunk > (T + 127) / 128 * 128) chunk = (T + 127) / 128 * 128;
    pk_epilogue e{};
    e.act = -1;
    if (epi) e = *epi;
    for (long long t0 = 0; t0 < T; t0 += chunk) {
        a.t0 = t0;
        a.tc = T - t0 < chunk ? T - t0 : chunk;
        a.rows = (int)((a.tc + 127) / 128 * 128);
        TDom<M_>* mm = v + (size_t)AL * AL * a.rows * a.cp;
        const long long nin = (long long)a.rows * (a.cp / 2);
        winograd_input_kernel<M_><<<ceil_div(nin, 256), 256, 0, st>>>(
            a, static_cast<const __nv_bfloat16*>(x), v);
        count_launch();
        cudaError_t err = pk_cuda_gemm_tc_batched(v, u, mm, AL * AL, a.rows, a.cp, g->k, g->k,
                                                  a.kp, st, M_ == 4);
        if (err != cudaSuccess) return err;
        const long long nout = a.tc * (a.kp / 2);
        winograd_output_kernel<M_><<<ceil_div(nout, 256), 256, 0, st>>>(
            a, mm, static_cast<__nv_bfloat16*>(y), e);
        count_launch();
    }
    return cudaGetLastError();
}

}  // namespace
}  // namespace pk

using namespace pk;

extern "C" {

int pk_winograd_tc_supported(const pk_conv_geom* g) {
    return g->groups == 1 && !g->transpose && g->r == 3 && g->s == 3 && g->str_h == 1 &&
           g->str_w == 1 && g->dil_h == 1 && g->dil_w == 1 && g->f_pitch == g->x_pitch &&
           g->x_pitch % 8 == 0 && g->y_pitch % 8 == 0;
}

size_t pk_winograd_tc_workspace(const pk_conv_geom* g, int m) {
    const long long T = tiles_of(g, m);
    size_t full = (size_t)((T + 127) / 128 * 128) * bytes_per_tile(g, m);
    if (full > kChunkBudget) full = kChunkBudget;
    const size_t one = 128 * bytes_per_tile(g, m);
    if (full < one) full = one;
    return u_bytes(g, m) + full;
}

cudaError_t pk_cuda_winograd_tc(const pk_conv_geom* g, int m, const void* x, const void* f,
                                void* y, const pk_epilogue* epi, void* ws, size_t ws_bytes,
                                cudaStream_t st) {
    if (!pk_winograd_tc_supported(g)) return cudaErrorNotSupported;
    if (m == 4) return run<4>(g, x, f, y, epi, ws, ws_bytes, st);
    if (m == 2) return run<2>(g, x, f, y, epi, ws, ws_bytes, st);
    return cudaErrorInvalidValue;
}

}  // extern "C"
