// FFT convolution (forward, stride 1, dilation 1).
//
// Same method as the reference fft_forward (proj/src/core/conv.cpp:371-493):
// zero-pad image and filter to the next power of two covering the full linear
// correlation, transform, accumulate in(c) * conj(filter(k, c)) over c,
// inverse transform, crop. The reference computes in complex<double>; here the
// spectra are complex<float> (the FFT solver's tolerance is 1e-3 relative, the
// fp32 transforms stay ~1e-6), images are batched (a chunk of images per pass,
// sized to a workspace cap) instead of one image at a time, the line transforms
// run one warp per line, and the per-frequency channel reduction is a tiled
// complex GEMM (n x c) . (c x k)^H over blocks of 32 frequencies in shared memory.
#include <cuComplex.h>

#include <algorithm>

#include "common.cuh"

namespace pk {

struct FftDims {
    int ph, pw;
};

inline int next_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

inline FftDims fft_dims(const pk_conv_geom& g) {
    return {next_pow2(g.h + 2 * g.pad_h + g.r - 1), next_pow2(g.w + 2 * g.pad_w + g.s - 1)};
}

constexpr size_t kFftChunkCap = size_t(512) << 20;  // spectra bytes per image chunk

// images per pass: as many as fit the cap (at least one)
inline int fft_chunk_images(const pk_conv_geom& g) {
    const FftDims d = fft_dims(g);
    const size_t per_img = (size_t)(g.cg + g.kg) * d.ph * d.pw * sizeof(cuFloatComplex);
    size_t nb = kFftChunkCap / (per_img ? per_img : 1);
    if (nb < 1) nb = 1;
    if (nb > (size_t)g.n) nb = (size_t)g.n;
    return (int)nb;
}

// In-place radix-2 FFT of `len` points in shared memory by one warp.
__device__ void fft_line_warp(cuFloatComplex* a, int len, int inverse) {
    const int lane = threadIdx.x & 31;
    int bits = 0;
    while ((1 << bits) < len) ++bits;
    for (int i = lane; i < len; i += 32) {
        const int j = bits ? (int)(__brev((unsigned)i) >> (32 - bits)) : 0;
        if (i < j) {
            const cuFloatComplex t = a[i];
            a[i] = a[j];
            a[j] = t;
        }
    }
    __syncwarp();
    for (int half = 1; half < len; half <<= 1) {
        for (int i = lane; i < len / 2; i += 32) {
            const int grp = i / half, pos = i % half;
            const int i0 = grp * 2 * half + pos, i1 = i0 + half;
            float sn, cs;
            // angle = -/+ 2*pi*pos/(2*half)
            sincospif((inverse ? 1.0f : -1.0f) * (float)pos / (float)half, &sn, &cs);
            const cuFloatComplex w = make_cuFloatComplex(cs, sn);
            const cuFloatComplex u = a[i0];
            const cuFloatComplex v = cuCmulf(a[i1], w);
            a[i0] = cuCaddf(u, v);
            a[i1] = cuCsubf(u, v);
        }
        __syncwarp();
    }
}

// planes: [count][ph][pw]; one warp per (plane, row) or (plane, column), lpc per CTA.
__global__ void fft_pass_kernel(cuFloatComplex* planes, long long count, int ph, int pw, int columns,
                                int inverse, int lpc) {
    extern __shared__ cuFloatComplex lines[];
    const int len = columns ? ph : pw;
    const int per_plane = columns ? pw : ph;
    const long long line = (long long)blockIdx.x * lpc + (threadIdx.x >> 5);
    if (line >= count * per_plane) return;
    cuFloatComplex* buf = lines + (threadIdx.x >> 5) * len;
    const long long plane = line / per_plane;
    const int li = (int)(line - plane * per_plane);
    cuFloatComplex* base = planes + plane * (long long)ph * pw;
    const long long stride = columns ? pw : 1;
    cuFloatComplex* start = columns ? base + li : base + (long long)li * pw;
    const int lane = threadIdx.x & 31;
    for (int i = lane; i < len; i += 32) buf[i] = start[i * stride];
    __syncwarp();
    fft_line_warp(buf, len, inverse);
    const float scale = inverse ? 1.0f / len : 1.0f;
    for (int i = lane; i < len; i += 32)
        start[i * stride] = make_cuFloatComplex(buf[i].x * scale, buf[i].y * scale);
}

template <typename T>
__global__ void fft_load_input(pk_conv_geom g, const T* __restrict__ x, int n0, int nb, int grp,
                               cuFloatComplex* spec, int ph, int pw) {
    const long long total = (long long)nb * g.cg * ph * pw;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int col = (int)(i % pw);
        const int row = (int)((i / pw) % ph);
        const long long pl = i / ((long long)pw * ph);
        const int c = (int)(pl % g.cg), n = n0 + (int)(pl / g.cg);
        const int ih = row - g.pad_h, iw = col - g.pad_w;
        float v = 0.0f;
        if (ih >= 0 && ih < g.h && iw >= 0 && iw < g.w)
            v = ld(x + (((size_t)n * g.h + ih) * g.w + iw) * g.x_pitch + grp * g.cg + c);
        spec[i] = make_cuFloatComplex(v, 0.0f);
    }
}

template <typename T>
__global__ void fft_load_filter(pk_conv_geom g, const T* __restrict__ f, int grp,
                                cuFloatComplex* spec, int ph, int pw) {
    const long long total = (long long)g.kg * g.cg * ph * pw;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int col = (int)(i % pw);
        const int row = (int)((i / pw) % ph);
        const long long pl = i / ((long long)pw * ph);
        const int c = (int)(pl % g.cg), kk = (int)(pl / g.cg);
        float v = 0.0f;
        if (row < g.r && col < g.s)
            v = ld(f + (((size_t)(grp * g.kg + kk) * g.r + row) * g.s + col) * g.f_pitch + c);
        spec[i] = make_cuFloatComplex(v, 0.0f);
    }
}

// acc[n][k][e] = sum_c in[n][c][e] * conj(flt[k][c][e]): a CTA owns 32 frequencies x
// 8 images x 16 output channels and walks the channels 8 at a time through shared
// memory; thread (group g = image, lane = frequency) accumulates its 16 k.
constexpr int kAccE = 32, kAccN = 8, kAccK = 16, kAccC = 8;
__global__ void __launch_bounds__(256) fft_accumulate(const cuFloatComplex* __restrict__ in_spec,
                                                      const cuFloatComplex* __restrict__ flt_spec,
                                                      cuFloatComplex* __restrict__ acc, int nb, int kg,
                                                      int cg, long long plane) {
    __shared__ cuFloatComplex sin_[kAccN][kAccC][kAccE];
    __shared__ cuFloatComplex sfl[kAccK][kAccC][kAccE];
    const long long e0 = (long long)blockIdx.x * kAccE;
    const int k0 = blockIdx.y * kAccK, n0 = blockIdx.z * kAccN;
    const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;  // grp = image in the tile
    cuFloatComplex a[kAccK];
#pragma unroll
    for (int k = 0; k < kAccK; ++k) a[k] = make_cuFloatComplex(0.0f, 0.0f);
    for (int c0 = 0; c0 < cg; c0 += kAccC) {
        for (int i = threadIdx.x; i < kAccN * kAccC * kAccE; i += 256) {
            const int e = i % kAccE, c = (i / kAccE) % kAccC, n = i / (kAccE * kAccC);
            const bool ok = n0 + n < nb && c0 + c < cg && e0 + e < plane;
            sin_[n][c][e] = ok ? in_spec[((long long)(n0 + n) * cg + c0 + c) * plane + e0 + e]
                               : make_cuFloatComplex(0.0f, 0.0f);
        }
        for (int i = threadIdx.x; i < kAccK * kAccC * kAccE; i += 256) {
            const int e = i % kAccE, c = (i / kAccE) % kAccC, k = i / (kAccE * kAccC);
            const bool ok = k0 + k < kg && c0 + c < cg && e0 + e < plane;
            sfl[k][c][e] = ok ? flt_spec[((long long)(k0 + k) * cg + c0 + c) * plane + e0 + e]
                              : make_cuFloatComplex(0.0f, 0.0f);
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < kAccC; ++c) {
            const cuFloatComplex x = sin_[grp][c][lane];
#pragma unroll
            for (int k = 0; k < kAccK; ++k) {
                const cuFloatComplex f = sfl[k][c][lane];
                // x * conj(f)
                a[k].x = fmaf(x.x, f.x, fmaf(x.y, f.y, a[k].x));
                a[k].y = fmaf(x.y, f.x, fmaf(-x.x, f.y, a[k].y));
            }
        }
        __syncthreads();
    }
    if (n0 + grp < nb && e0 + lane < plane)
#pragma unroll
        for (int k = 0; k < kAccK; ++k)
            if (k0 + k < kg) acc[((long long)(n0 + grp) * kg + k0 + k) * plane + e0 + lane] = a[k];
}

template <typename T>
__global__ void fft_store(pk_conv_geom g, const cuFloatComplex* __restrict__ acc, int n0, int nb,
                          int grp, T* __restrict__ y, int ph, int pw) {
    const long long total = (long long)nb * g.kg * g.p * g.q;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int kk = (int)(i % g.kg);
        const long long pix = i / g.kg;
        const int ow = (int)(pix % g.q), oh = (int)((pix / g.q) % g.p), n = (int)(pix / ((long long)g.q * g.p));
        const float v = acc[(((long long)n * g.kg + kk) * ph + oh) * pw + ow].x;
        st(y + (((size_t)(n0 + n) * g.p + oh) * g.q + ow) * g.y_pitch + grp * g.kg + kk, v);
    }
}

inline unsigned g1(long long total) {
    long long b = (total + 255) / 256;
    if (b > 148LL * 32) b = 148LL * 32;
    return (unsigned)(b < 1 ? 1 : b);
}

cudaError_t fft_transform(cuFloatComplex* planes, long long count, int ph, int pw, int inverse,
                          cudaStream_t st) {
    // lines per CTA (one warp each) within 48 KB of staging
    auto lpc = [](int len) { return (int)std::max<size_t>(1, std::min<size_t>(8, (48 * 1024) / (len * sizeof(cuFloatComplex)))); };
    const int lr = lpc(pw), lc = lpc(ph);
    fft_pass_kernel<<<(unsigned)((count * ph + lr - 1) / lr), 32 * lr, lr * pw * sizeof(cuFloatComplex), st>>>(
        planes, count, ph, pw, 0, inverse, lr);
    fft_pass_kernel<<<(unsigned)((count * pw + lc - 1) / lc), 32 * lc, lc * ph * sizeof(cuFloatComplex), st>>>(
        planes, count, ph, pw, 1, inverse, lc);
    count_launch(2);
    return cudaGetLastError();
}

}  // namespace pk

using namespace pk;

extern "C" {

size_t pk_cuda_fft_scratch_bytes(const pk_conv_geom* g) {
    const FftDims d = fft_dims(*g);
    const size_t plane = (size_t)d.ph * d.pw;
    const size_t nb = (size_t)fft_chunk_images(*g);
    const size_t planes = nb * g->cg + (size_t)g->kg * g->cg + nb * g->kg;
    return planes * plane * sizeof(cuFloatComplex);
}

cudaError_t pk_cuda_fft_fwd(const pk_conv_geom* g, int dtype, const void* x, const void* f,
                            void* y, void* scratch, cudaStream_t st) {
    if (g->str_h != 1 || g->str_w != 1 || g->dil_h != 1 || g->dil_w != 1 || g->transpose)
        return cudaErrorInvalidValue;
    const FftDims d = fft_dims(*g);
    const long long plane = (long long)d.ph * d.pw;
    const int chunk = fft_chunk_images(*g);
    cuFloatComplex* in_spec = (cuFloatComplex*)scratch;
    cuFloatComplex* flt_spec = in_spec + (long long)chunk * g->cg * plane;
    cuFloatComplex* acc = flt_spec + (long long)g->kg * g->cg * plane;
    if ((size_t)std::max(d.ph, d.pw) * sizeof(cuFloatComplex) > 48 * 1024) return cudaErrorInvalidValue;
    cudaError_t err = cudaSuccess;
    for (int grp = 0; grp < g->groups && err == cudaSuccess; ++grp) {
        PK_DISPATCH_DTYPE(dtype, T,
                          fft_load_filter<T><<<g1((long long)g->kg * g->cg * plane), 256, 0, st>>>(
                              *g, (const T*)f, grp, flt_spec, d.ph, d.pw));
        count_launch();
        err = fft_transform(flt_spec, (long long)g->kg * g->cg, d.ph, d.pw, 0, st);
        for (int n0 = 0; n0 < g->n && err == cudaSuccess; n0 += chunk) {
            const int nb = std::min(chunk, g->n - n0);
            PK_DISPATCH_DTYPE(dtype, T,
                              fft_load_input<T><<<g1((long long)nb * g->cg * plane), 256, 0, st>>>(
                                  *g, (const T*)x, n0, nb, grp, in_spec, d.ph, d.pw));
            count_launch();
            err = fft_transform(in_spec, (long long)nb * g->cg, d.ph, d.pw, 0, st);
            if (err != cudaSuccess) break;
            const dim3 ag((unsigned)((plane + kAccE - 1) / kAccE), (unsigned)((g->kg + kAccK - 1) / kAccK),
                          (unsigned)((nb + kAccN - 1) / kAccN));
            fft_accumulate<<<ag, 256, 0, st>>>(in_spec, flt_spec, acc, nb, g->kg, g->cg, plane);
            count_launch();
            err = fft_transform(acc, (long long)nb * g->kg, d.ph, d.pw, 1, st);
            if (err != cudaSuccess) break;
            PK_DISPATCH_DTYPE(dtype, T,
                              fft_store<T><<<g1((long long)nb * g->kg * g->p * g->q), 256, 0, st>>>(
                                  *g, acc, n0, nb, grp, (T*)y, d.ph, d.pw));
            count_launch();
            err = cudaGetLastError();
        }
    }
    return err;
}

}  // extern "C"
