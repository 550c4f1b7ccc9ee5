// FFT convolution (forward, stride 1, dilation 1) in complex<double>.
//
// Same method as the reference fft_forward (proj/src/core/conv.cpp:371-493):
// zero-pad image and filter to the next power of two covering the full linear
// correlation, transform, accumulate in(c) * conj(filter(k, c)) over c,
// inverse transform, crop. Correctness path (perf irrelevant per SURVEY
// §2.1): radix-2 row and column passes, one CTA per line with the line staged
// in shared memory, twiddles from sincospi (exact angles, no recurrence).
#include <cuComplex.h>

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

// In-place radix-2 FFT of `len` points in shared memory by the whole CTA.
__device__ void fft_line(cuDoubleComplex* a, int len, int inverse) {
    // bit reversal
    int bits = 0;
    while ((1 << bits) < len) ++bits;
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
        const int j = bits ? (int)(__brev((unsigned)i) >> (32 - bits)) : 0;
        if (i < j) {
            const cuDoubleComplex t = a[i];
            a[i] = a[j];
            a[j] = t;
        }
    }
    __syncthreads();
    for (int half = 1; half < len; half <<= 1) {
        for (int i = threadIdx.x; i < len / 2; i += blockDim.x) {
            const int grp = i / half, pos = i % half;
            const int i0 = grp * 2 * half + pos, i1 = i0 + half;
            double sn, cs;
            // angle = -/+ 2*pi*pos/(2*half)
            sincospi((inverse ? 1.0 : -1.0) * (double)pos / (double)half, &sn, &cs);
            const cuDoubleComplex w = make_cuDoubleComplex(cs, sn);
            const cuDoubleComplex u = a[i0];
            const cuDoubleComplex v = cuCmul(a[i1], w);
            a[i0] = cuCadd(u, v);
            a[i1] = cuCsub(u, v);
        }
        __syncthreads();
    }
}

// planes: [count][ph][pw]; one CTA per (plane, row) or (plane, column).
__global__ void fft_pass_kernel(cuDoubleComplex* planes, int ph, int pw, int columns,
                                int inverse) {
    extern __shared__ cuDoubleComplex line[];
    const int len = columns ? ph : pw;
    const int lines = columns ? pw : ph;
    const long long plane = blockIdx.x / lines;
    const int li = blockIdx.x % lines;
    cuDoubleComplex* base = planes + plane * (long long)ph * pw;
    const long long stride = columns ? pw : 1;
    cuDoubleComplex* start = columns ? base + li : base + (long long)li * pw;
    for (int i = threadIdx.x; i < len; i += blockDim.x) line[i] = start[i * stride];
    __syncthreads();
    fft_line(line, len, inverse);
    const double scale = inverse ? 1.0 / len : 1.0;
    for (int i = threadIdx.x; i < len; i += blockDim.x)
        start[i * stride] = make_cuDoubleComplex(line[i].x * scale, line[i].y * scale);
}

template <typename T>
__global__ void fft_load_input(pk_conv_geom g, const T* __restrict__ x, int n, int grp,
                               cuDoubleComplex* spec, int ph, int pw) {
    const long long total = (long long)g.cg * ph * pw;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int col = (int)(i % pw);
        const int row = (int)((i / pw) % ph);
        const int c = (int)(i / ((long long)pw * ph));
        const int ih = row - g.pad_h, iw = col - g.pad_w;
        double v = 0.0;
        if (ih >= 0 && ih < g.h && iw >= 0 && iw < g.w)
            v = ld(x + (((size_t)n * g.h + ih) * g.w + iw) * g.x_pitch + grp * g.cg + c);
        spec[i] = make_cuDoubleComplex(v, 0.0);
    }
}

template <typename T>
__global__ void fft_load_filter(pk_conv_geom g, const T* __restrict__ f, int grp,
                                cuDoubleComplex* spec, int ph, int pw) {
    const long long total = (long long)g.kg * g.cg * ph * pw;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int col = (int)(i % pw);
        const int row = (int)((i / pw) % ph);
        const long long pl = i / ((long long)pw * ph);
        const int c = (int)(pl % g.cg), kk = (int)(pl / g.cg);
        double v = 0.0;
        if (row < g.r && col < g.s)
            v = ld(f + (((size_t)(grp * g.kg + kk) * g.r + row) * g.s + col) * g.f_pitch + c);
        spec[i] = make_cuDoubleComplex(v, 0.0);
    }
}

__global__ void fft_accumulate(const cuDoubleComplex* __restrict__ in_spec,
                               const cuDoubleComplex* __restrict__ flt_spec,
                               cuDoubleComplex* __restrict__ acc, int kg, int cg, long long plane) {
    const long long total = (long long)kg * plane;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long e = i % plane;
        const int kk = (int)(i / plane);
        cuDoubleComplex a = make_cuDoubleComplex(0.0, 0.0);
        for (int c = 0; c < cg; ++c)
            a = cuCadd(a, cuCmul(in_spec[c * plane + e],
                                 cuConj(flt_spec[((long long)kk * cg + c) * plane + e])));
        acc[i] = a;
    }
}

template <typename T>
__global__ void fft_store(pk_conv_geom g, const cuDoubleComplex* __restrict__ acc, int n,
                          int grp, T* __restrict__ y, int ph, int pw) {
    const long long total = (long long)g.kg * g.p * g.q;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int kk = (int)(i % g.kg);
        const long long pix = i / g.kg;
        const int ow = (int)(pix % g.q), oh = (int)(pix / g.q);
        const double v = acc[((long long)kk * ph + oh) * pw + ow].x;
        st(y + (((size_t)n * g.p + oh) * g.q + ow) * g.y_pitch + grp * g.kg + kk, (float)v);
    }
}

inline unsigned g1(long long total) {
    long long b = (total + 255) / 256;
    if (b > 148LL * 32) b = 148LL * 32;
    return (unsigned)(b < 1 ? 1 : b);
}

cudaError_t fft_transform(cuDoubleComplex* planes, long long count, int ph, int pw, int inverse,
                          cudaStream_t st) {
    const int threads = 128;
    fft_pass_kernel<<<(unsigned)(count * ph), threads, pw * sizeof(cuDoubleComplex), st>>>(
        planes, ph, pw, 0, inverse);
    fft_pass_kernel<<<(unsigned)(count * pw), threads, ph * sizeof(cuDoubleComplex), st>>>(
        planes, ph, pw, 1, inverse);
    count_launch(2);
    return cudaGetLastError();
}

}  // namespace pk

using namespace pk;

extern "C" {

size_t pk_cuda_fft_scratch_bytes(const pk_conv_geom* g) {
    const FftDims d = fft_dims(*g);
    const size_t plane = (size_t)d.ph * d.pw;
    const size_t planes = (size_t)g->cg + (size_t)g->kg * g->cg + (size_t)g->kg;
    return planes * plane * sizeof(cuDoubleComplex);
}

cudaError_t pk_cuda_fft_fwd(const pk_conv_geom* g, int dtype, const void* x, const void* f,
                            void* y, void* scratch, cudaStream_t st) {
    if (g->str_h != 1 || g->str_w != 1 || g->dil_h != 1 || g->dil_w != 1 || g->transpose)
        return cudaErrorInvalidValue;
    const FftDims d = fft_dims(*g);
    const long long plane = (long long)d.ph * d.pw;
    cuDoubleComplex* in_spec = (cuDoubleComplex*)scratch;
    cuDoubleComplex* flt_spec = in_spec + (long long)g->cg * plane;
    cuDoubleComplex* acc = flt_spec + (long long)g->kg * g->cg * plane;
    cudaError_t err = cudaSuccess;
    for (int grp = 0; grp < g->groups && err == cudaSuccess; ++grp) {
        PK_DISPATCH_DTYPE(dtype, T,
                          fft_load_filter<T><<<g1((long long)g->kg * g->cg * plane), 256, 0, st>>>(
                              *g, (const T*)f, grp, flt_spec, d.ph, d.pw));
        count_launch();
        err = fft_transform(flt_spec, (long long)g->kg * g->cg, d.ph, d.pw, 0, st);
        for (int n = 0; n < g->n && err == cudaSuccess; ++n) {
            PK_DISPATCH_DTYPE(dtype, T,
                              fft_load_input<T><<<g1((long long)g->cg * plane), 256, 0, st>>>(
                                  *g, (const T*)x, n, grp, in_spec, d.ph, d.pw));
            count_launch();
            err = fft_transform(in_spec, g->cg, d.ph, d.pw, 0, st);
            if (err != cudaSuccess) break;
            fft_accumulate<<<g1((long long)g->kg * plane), 256, 0, st>>>(in_spec, flt_spec, acc,
                                                                         g->kg, g->cg, plane);
            count_launch();
            err = fft_transform(acc, g->kg, d.ph, d.pw, 1, st);
            if (err != cudaSuccess) break;
            PK_DISPATCH_DTYPE(dtype, T,
                              fft_store<T><<<g1((long long)g->kg * g->p * g->q), 256, 0, st>>>(
                                  *g, acc, n, grp, (T*)y, d.ph, d.pw));
            count_launch();
            err = cudaGetLastError();
        }
    }
    return err;
}

}  // extern "C"
