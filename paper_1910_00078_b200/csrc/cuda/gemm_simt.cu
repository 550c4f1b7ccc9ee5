// CUDA-core (fp32 FMA) GEMM-shaped kernels:
//  * im2col / col2im for the Im2colGemm solver (proj/src/core/conv.cpp:178-220,
//    :757-791) with a strided tiled GEMM (tensor.cpp:163-205 semantics:
//    C = A*B (+C), fp32 accumulate),
//  * an fp32 implicit-GEMM forward (the f32 ImplicitGemm solver and the f32
//    fused conv+bias+BN+activation executor; conv.cpp:516-600 semantics).
// The bf16 paths of the same solvers run on tcgen05 (igemm_tc.cu).
#include "common.cuh"

namespace pk {

template <typename T>
__global__ void im2col_kernel(pk_conv_geom g, const T* __restrict__ x, int image, int group,
                              T* __restrict__ col) {
    const int rowp = g.r * g.s * g.f_pitch;
    const long long total = (long long)g.p * g.q * rowp;
    const T* xn = x + (size_t)image * g.h * g.w * g.x_pitch + group * g.cg;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % g.f_pitch);
        long long t = i / g.f_pitch;
        const int s = (int)(t % g.s);
        t /= g.s;
        const int r = (int)(t % g.r);
        const long long pix = t / g.r;
        const int ow = (int)(pix % g.q), oh = (int)(pix / g.q);
        const int ih = oh * g.str_h - g.pad_h + r * g.dil_h;
        const int iw = ow * g.str_w - g.pad_w + s * g.dil_w;
        float v = 0.0f;
        if (c < g.cg && ih >= 0 && ih < g.h && iw >= 0 && iw < g.w)
            v = ld(xn + ((size_t)ih * g.w + iw) * g.x_pitch + c);
        st(col + i, v);
    }
}

template <typename T>
__global__ void col2im_kernel(pk_conv_geom g, const float* __restrict__ col, int image,
                              int group, T* __restrict__ dx) {
    const int rowp = g.r * g.s * g.f_pitch;
    const long long total = (long long)g.h * g.w * g.cg;
    T* dxn = dx + (size_t)image * g.h * g.w * g.x_pitch + group * g.cg;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % g.cg);
        const long long pix = i / g.cg;
        const int iw = (int)(pix % g.w), ih = (int)(pix / g.w);
        float acc = 0.0f;
        for (int r = 0; r < g.r; ++r) {
            const int nh = ih + g.pad_h - r * g.dil_h;
            if (nh < 0 || nh % g.str_h) continue;
            const int oh = nh / g.str_h;
            if (oh >= g.p) continue;
            for (int s = 0; s < g.s; ++s) {
                const int nw = iw + g.pad_w - s * g.dil_w;
                if (nw < 0 || nw % g.str_w) continue;
                const int ow = nw / g.str_w;
                if (ow >= g.q) continue;
                acc += col[((size_t)oh * g.q + ow) * rowp + (r * g.s + s) * g.f_pitch + c];
            }
        }
        st(dxn + (size_t)pix * g.x_pitch + c, acc);
    }
}

// Transpose-mode scatter (conv.cpp:224-242) in gather form.
template <typename T>
__global__ void col2im_transpose_kernel(pk_conv_geom g, const float* __restrict__ col, int image,
                                        int group, T* __restrict__ out) {
    const long long hw = (long long)g.h * g.w;
    const long long total = (long long)g.p * g.q * g.kg;
    T* on = out + (size_t)image * g.p * g.q * g.y_pitch + group * g.kg;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int kk = (int)(i % g.kg);
        const long long pix = i / g.kg;
        const int ow = (int)(pix % g.q), oh = (int)(pix / g.q);
        float acc = 0.0f;
        for (int r = 0; r < g.r; ++r) {
            const int nh = oh + g.pad_h - r;
            if (nh < 0 || nh % g.str_h) continue;
            const int ih = nh / g.str_h;
            if (ih >= g.h) continue;
            for (int s = 0; s < g.s; ++s) {
                const int nw = ow + g.pad_w - s;
                if (nw < 0 || nw % g.str_w) continue;
                const int iw = nw / g.str_w;
                if (iw >= g.w) continue;
                acc += col[((long long)(r * g.s + s) * g.f_pitch + kk) * hw + (long long)ih * g.w + iw];
            }
        }
        st(on + (size_t)pix * g.y_pitch + kk, acc);
    }
}

// 64x64 output tile, 16-deep K slices, 256 threads x (4x4) micro-tile.
constexpr int TM = 64, TN = 64, TK = 16;

template <typename T>
__global__ void __launch_bounds__(256) gemm_strided_kernel(int m, int n, int k,
                                                           const T* __restrict__ a, long long sam,
                                                           long long sak, const T* __restrict__ b,
                                                           long long sbk, long long sbn,
                                                           float* __restrict__ c, long long ldc,
                                                           int accumulate) {
    __shared__ float As[TK][TM + 4];
    __shared__ float Bs[TK][TN + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int m0 = blockIdx.x * TM, n0 = blockIdx.y * TN;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < k; k0 += TK) {
        for (int i = threadIdx.x; i < TM * TK; i += 256) {
            // consecutive threads walk the contiguous operand dimension
            int mm, kk;
            if (sak == 1) { kk = i % TK; mm = i / TK; } else { mm = i % TM; kk = i / TM; }
            const int gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < m && gk < k) ? ld(a + gm * sam + gk * sak) : 0.0f;
        }
        for (int i = threadIdx.x; i < TN * TK; i += 256) {
            int nn, kk;
            if (sbk == 1) { kk = i % TK; nn = i / TK; } else { nn = i % TN; kk = i / TN; }
            const int gn = n0 + nn, gk = k0 + kk;
            Bs[kk][nn] = (gn < n && gk < k) ? ld(b + gk * sbk + gn * sbn) : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
            float av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] += av[i] * bv[j];
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gm = m0 + ty * 4 + i;
        if (gm >= m) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gn = n0 + tx * 4 + j;
            if (gn >= n) continue;
            float* cp = c + gm * ldc + gn;
            *cp = accumulate ? *cp + acc[i][j] : acc[i][j];
        }
    }
}

// fp32 implicit GEMM forward: M = output pixels, N = output channels of one
// group (blockIdx.z), K = (r, s, c) with c fastest, the reference reduction
// order within every (r, s) tap being over channels.
template <typename T>
__global__ void __launch_bounds__(256) igemm_simt_fwd_kernel(pk_conv_geom g,
                                                             const T* __restrict__ x,
                                                             const T* __restrict__ f,
                                                             T* __restrict__ y, pk_epilogue e) {
    __shared__ float As[TK][TM + 4];
    __shared__ float Bs[TK][TN + 4];
    const int grp = blockIdx.z;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const long long npix = (long long)g.n * g.p * g.q;
    const long long m0 = (long long)blockIdx.x * TM;
    const int n0 = blockIdx.y * TN;
    const int kred = g.r * g.s * g.cg;
    // Each thread loads the same (pixel, k-slot) pair every slice: decode the
    // pixel once.
    const int a_k = threadIdx.x % TK, a_m = threadIdx.x / TK;  // 16 x 16 per pass
    float acc[4][4] = {};
    for (int k0 = 0; k0 < kred; k0 += TK) {
        {
            const int gk = k0 + a_k;
            int c = 0, r = 0, s = 0;
            const bool kv = gk < kred;
            if (kv) {
                c = gk % g.cg;
                const int rs = gk / g.cg;
                s = rs % g.s;
                r = rs / g.s;
            }
#pragma unroll
            for (int pass = 0; pass < TM / 16; ++pass) {
                const int mm = a_m + pass * 16;
                const long long gm = m0 + mm;
                float v = 0.0f;
                if (kv && gm < npix) {
                    const int ow = (int)(gm % g.q);
                    const int oh = (int)((gm / g.q) % g.p);
                    const int n = (int)(gm / ((long long)g.q * g.p));
                    const int ih = oh * g.str_h - g.pad_h + r * g.dil_h;
                    const int iw = ow * g.str_w - g.pad_w + s * g.dil_w;
                    if (ih >= 0 && ih < g.h && iw >= 0 && iw < g.w)
                        v = ld(x + (((size_t)n * g.h + ih) * g.w + iw) * g.x_pitch +
                               grp * g.cg + c);
                }
                As[a_k][mm] = v;
            }
        }
        for (int i = threadIdx.x; i < TN * TK; i += 256) {
            const int kk = i % TK, nn = i / TK;
            const int gn = n0 + nn, gk = k0 + kk;
            float v = 0.0f;
            if (gn < g.kg && gk < kred) {
                const int c = gk % g.cg, rs = gk / g.cg;
                v = ld(f + ((size_t)(grp * g.kg + gn) * g.r * g.s + rs) * g.f_pitch + c);
            }
            Bs[kk][nn] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
            float av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] += av[i] * bv[j];
        }
        __syncthreads();
    }
    const bool epi = epilogue_active(&e);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const long long gm = m0 + ty * 4 + i;
        if (gm >= npix) continue;
        const int ow = (int)(gm % g.q);
        const int oh = (int)((gm / g.q) % g.p);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gn = n0 + tx * 4 + j;
            if (gn >= g.kg) continue;
            const int k = grp * g.kg + gn;
            st(y + (size_t)gm * g.y_pitch + k,
               epi ? apply_epilogue(e, acc[i][j], k, oh, ow, g.p, g.q) : acc[i][j]);
        }
    }
}

inline unsigned grid1d(long long total) {
    long long b = (total + 255) / 256;
    if (b > 148LL * 64) b = 148LL * 64;
    return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace pk

using namespace pk;

extern "C" {

cudaError_t pk_cuda_im2col(const pk_conv_geom* g, int dtype, const void* x, int image, int group,
                           void* col, cudaStream_t st) {
    const long long total = (long long)g->p * g->q * g->r * g->s * g->f_pitch;
    PK_DISPATCH_DTYPE(dtype, T,
                      im2col_kernel<T><<<grid1d(total), 256, 0, st>>>(*g, (const T*)x, image,
                                                                       group, (T*)col));
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_col2im(const pk_conv_geom* g, int dtype, const float* col, int image,
                           int group, void* dx, cudaStream_t st) {
    const long long total = (long long)g->h * g->w * g->cg;
    PK_DISPATCH_DTYPE(dtype, T,
                      col2im_kernel<T><<<grid1d(total), 256, 0, st>>>(*g, col, image, group,
                                                                       (T*)dx));
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_col2im_transpose(const pk_conv_geom* g, int dtype, const float* col,
                                     int image, int group, void* out, cudaStream_t st) {
    const long long total = (long long)g->p * g->q * g->kg;
    PK_DISPATCH_DTYPE(dtype, T,
                      col2im_transpose_kernel<T><<<grid1d(total), 256, 0, st>>>(*g, col, image,
                                                                                 group, (T*)out));
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_gemm_simt(int m, int n, int k, int dtype_ab, const void* a, long long sam,
                              long long sak, const void* b, long long sbk, long long sbn,
                              float* c, long long ldc, int accumulate, cudaStream_t st) {
    dim3 grid(ceil_div(m, TM), ceil_div(n, TN));
    PK_DISPATCH_DTYPE(dtype_ab, T,
                      gemm_strided_kernel<T><<<grid, 256, 0, st>>>(m, n, k, (const T*)a, sam, sak,
                                                                   (const T*)b, sbk, sbn, c, ldc,
                                                                   accumulate));
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_igemm_simt_fwd(const pk_conv_geom* g, int dtype, const void* x, const void* f,
                                   void* y, const pk_epilogue* epi, cudaStream_t st) {
    pk_epilogue none{};
    none.act = -1;
    const pk_epilogue e = epi ? *epi : none;
    const long long npix = (long long)g->n * g->p * g->q;
    dim3 grid(ceil_div(npix, TM), ceil_div(g->kg, TN), g->groups);
    PK_DISPATCH_DTYPE(dtype, T,
                      igemm_simt_fwd_kernel<T><<<grid, 256, 0, st>>>(*g, (const T*)x,
                                                                     (const T*)f, (T*)y, e));
    count_launch();
    return cudaGetLastError();
}

}  // extern "C"
