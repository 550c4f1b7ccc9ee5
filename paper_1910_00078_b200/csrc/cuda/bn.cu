// Training-mode batch normalisation over NHWC activations.
//
// Semantics follow the reference (proj/src/core/primitives.cpp:61-152):
// statistics accumulated in double, biased variance var = max(0, E[x^2]-mu^2),
// invstd = float(1/sqrt(var+eps)), running <- (1-m)*running + m*stat,
// y = gamma*(x-mu)*invstd + beta; backward dbeta = sum dy, dgamma = sum dy*xhat,
// dx = gamma*invstd/m * (m*dy - dbeta - xhat*dgamma).
//
// Schedule (HBM-bound): spatial mode is a two-level deterministic reduction —
// CTAs own a 32-channel slice x a row chunk of the [N*H*W][pitch] matrix, warps
// stride rows (coalesced channel-contiguous loads), per-thread double
// accumulators, fixed-order smem + chunk combine — then one elementwise pass.
#include "common.cuh"

namespace pk {

struct BnPlan {
    int chunks;
};

inline int bn_chunks(long long rows, int c) {
    const int cslices = (c + 31) / 32;
    long long want = (148LL * 8 + cslices - 1) / cslices;
    long long maxc = (rows + 63) / 64;
    if (want > maxc) want = maxc;
    if (want < 1) want = 1;
    return (int)want;
}

// Mode 0: sums of x and x^2. Mode 1 (backward): sums of dy' and dy'*xhat,
// dy' = dy masked by (y > 0) when relu.
template <typename T, int MODE>
__global__ void __launch_bounds__(256) bn_partial_kernel(const T* __restrict__ x,
                                                         const T* __restrict__ y,
                                                         const T* __restrict__ dy, long long rows,
                                                         int c, int pitch, int chunks,
                                                         const float* __restrict__ mean,
                                                         const float* __restrict__ invstd,
                                                         int relu, double* __restrict__ part) {
    __shared__ double s0[8][33], s1[8][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ch = blockIdx.x * 32 + lane;
    const int chunk = blockIdx.y;
    const long long per = (rows + chunks - 1) / chunks;
    const long long r0 = chunk * per, r1 = min(rows, r0 + per);
    double a = 0.0, b = 0.0;
    if (ch < c) {
        float mu = 0.0f, inv = 0.0f;
        if (MODE == 1) {
            mu = mean[ch];
            inv = invstd[ch];
        }
        for (long long r = r0 + warp; r < r1; r += 8) {
            const size_t i = (size_t)r * pitch + ch;
            if (MODE == 0) {
                const double v = ld(x + i);
                a += v;
                b += v * v;
            } else {
                float d = ld(dy + i);
                if (relu && !(ld(y + i) > 0.0f)) d = 0.0f;
                const double xhat = (double)((ld(x + i) - mu) * inv);
                a += d;
                b += (double)d * xhat;
            }
        }
    }
    s0[warp][lane] = a;
    s1[warp][lane] = b;
    __syncthreads();
    if (warp == 0 && ch < c) {
        double ta = 0.0, tb = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            ta += s0[w][lane];
            tb += s1[w][lane];
        }
        part[((size_t)chunk * c + ch) * 2 + 0] = ta;
        part[((size_t)chunk * c + ch) * 2 + 1] = tb;
    }
}

// Per-activation mode: one thread per statistic (c, hw), reducing over n.
template <typename T, int MODE>
__global__ void bn_partial_peract_kernel(const T* __restrict__ x, const T* __restrict__ y,
                                         const T* __restrict__ dy, int n, int c, int hw,
                                         int pitch, const float* __restrict__ mean,
                                         const float* __restrict__ invstd, int relu,
                                         double* __restrict__ part) {
    const long long total = (long long)c * hw;
    for (long long si = blockIdx.x * (long long)blockDim.x + threadIdx.x; si < total;
         si += (long long)gridDim.x * blockDim.x) {
        const int ch = (int)(si / hw), px = (int)(si % hw);
        double a = 0.0, b = 0.0;
        float mu = 0.0f, inv = 0.0f;
        if (MODE == 1) {
            mu = mean[si];
            inv = invstd[si];
        }
        for (int i = 0; i < n; ++i) {
            const size_t off = ((size_t)i * hw + px) * pitch + ch;
            if (MODE == 0) {
                const double v = ld(x + off);
                a += v;
                b += v * v;
            } else {
                float d = ld(dy + off);
                if (relu && !(ld(y + off) > 0.0f)) d = 0.0f;
                const double xhat = (double)((ld(x + off) - mu) * inv);
                a += d;
                b += (double)d * xhat;
            }
        }
        part[si * 2 + 0] = a;
        part[si * 2 + 1] = b;
    }
}

__global__ void bn_finalize_fwd_kernel(const double* __restrict__ part, int chunks, int nstat,
                                       double m, float eps, float momentum,
                                       float* __restrict__ running_mean,
                                       float* __restrict__ running_var,
                                       float* __restrict__ saved_mean,
                                       float* __restrict__ saved_invstd) {
    const int si = blockIdx.x * blockDim.x + threadIdx.x;
    if (si >= nstat) return;
    double s = 0.0, sq = 0.0;
    for (int k = 0; k < chunks; ++k) {
        s += part[((size_t)k * nstat + si) * 2 + 0];
        sq += part[((size_t)k * nstat + si) * 2 + 1];
    }
    const double mu = s / m;
    const double var = fmax(0.0, sq / m - mu * mu);
    saved_mean[si] = (float)mu;
    saved_invstd[si] = (float)(1.0 / sqrt(var + (double)eps));
    if (running_mean) {
        running_mean[si] = (1.0f - momentum) * running_mean[si] + momentum * (float)mu;
        running_var[si] = (1.0f - momentum) * running_var[si] + momentum * (float)var;
    }
}

__global__ void bn_finalize_bwd_kernel(double* __restrict__ part, int chunks, int nstat,
                                       float* __restrict__ dgamma, float* __restrict__ dbeta,
                                       int round_bf16) {
    const int si = blockIdx.x * blockDim.x + threadIdx.x;
    if (si >= nstat) return;
    double db = 0.0, dg = 0.0;
    for (int k = 0; k < chunks; ++k) {
        db += part[((size_t)k * nstat + si) * 2 + 0];
        dg += part[((size_t)k * nstat + si) * 2 + 1];
    }
    // totals kept (unrounded, double) for the dx pass in chunk slot 0
    part[(size_t)si * 2 + 0] = db;
    part[(size_t)si * 2 + 1] = dg;
    float fdg = (float)dg, fdb = (float)db;
    if (round_bf16) {
        fdg = __bfloat162float(__float2bfloat16_rn(fdg));
        fdb = __bfloat162float(__float2bfloat16_rn(fdb));
    }
    if (dgamma) dgamma[si] = fdg;
    if (dbeta) dbeta[si] = fdb;
}

template <typename T>
__global__ void bn_apply_kernel(const T* __restrict__ x, T* __restrict__ y, long long rows, int c,
                                int hw, int pitch, int per_act,
                                const float* __restrict__ gamma, const float* __restrict__ beta,
                                const float* __restrict__ mean, const float* __restrict__ invstd,
                                int relu) {
    const long long total = rows * pitch;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int ch = (int)(i % pitch);
        float v = 0.0f;
        if (ch < c) {
            const long long si = per_act ? (long long)ch * hw + (i / pitch) % hw : ch;
            v = gamma[si] * (ld(x + i) - mean[si]) * invstd[si] + beta[si];
            if (relu && !(v > 0.0f)) v = 0.0f;
        }
        st(y + i, v);
    }
}

template <typename T>
__global__ void bn_dx_kernel(const T* __restrict__ x, const T* __restrict__ y,
                             const T* __restrict__ dy, T* __restrict__ dx, long long rows, int c,
                             int hw, int pitch, int per_act, double m,
                             const float* __restrict__ gamma, const float* __restrict__ mean,
                             const float* __restrict__ invstd, const double* __restrict__ tot,
                             int relu) {
    const long long total = rows * pitch;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int ch = (int)(i % pitch);
        float out = 0.0f;
        if (ch < c) {
            const long long si = per_act ? (long long)ch * hw + (i / pitch) % hw : ch;
            float d = ld(dy + i);
            if (relu && !(ld(y + i) > 0.0f)) d = 0.0f;
            const double xhat = (double)((ld(x + i) - mean[si]) * invstd[si]);
            const double v = ((double)(gamma[si] * invstd[si]) / m) *
                             (m * d - tot[si * 2 + 0] - xhat * tot[si * 2 + 1]);
            out = (float)v;
        }
        st(dx + i, out);
    }
}

// Per-CTA fp32 partials (sum, sumsq) of the conv epilogue -> batch stats.
__global__ void bn_finalize_partials_kernel(const float* __restrict__ part, int slots, int c,
                                            double m, float eps, float momentum,
                                            float* __restrict__ running_mean,
                                            float* __restrict__ running_var,
                                            float* __restrict__ saved_mean,
                                            float* __restrict__ saved_invstd) {
    const int ch = blockIdx.x * blockDim.x + threadIdx.x;
    if (ch >= c) return;
    double s = 0.0, sq = 0.0;
    for (int k = 0; k < slots; ++k) {
        s += part[((size_t)k * c + ch) * 2 + 0];
        sq += part[((size_t)k * c + ch) * 2 + 1];
    }
    const double mu = s / m;
    const double var = fmax(0.0, sq / m - mu * mu);
    saved_mean[ch] = (float)mu;
    saved_invstd[ch] = (float)(1.0 / sqrt(var + (double)eps));
    if (running_mean) {
        running_mean[ch] = (1.0f - momentum) * running_mean[ch] + momentum * (float)mu;
        running_var[ch] = (1.0f - momentum) * running_var[ch] + momentum * (float)var;
    }
}

// y = gamma * (x - mu) * invstd + beta (+ReLU) on bf16 NHWC, 8 channels (16 B)
// per thread; pad lanes stay zero.
__global__ void bn_apply_bf16x8_kernel(const uint4* __restrict__ x, uint4* __restrict__ y,
                                       long long vecs, int c, int pitch_vecs,
                                       const float* __restrict__ gamma,
                                       const float* __restrict__ beta,
                                       const float* __restrict__ mean,
                                       const float* __restrict__ invstd, int relu) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < vecs;
         i += (long long)gridDim.x * blockDim.x) {
        const int c0 = (int)(i % pitch_vecs) * 8;
        uint4 v = __ldg(x + i);
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            float2 f = __bfloat1622float2(h[e]);
            const int ch = c0 + 2 * e;
            float a = 0.f, b = 0.f;
            if (ch < c) {
                a = gamma[ch] * (f.x - mean[ch]) * invstd[ch] + beta[ch];
                if (relu && !(a > 0.0f)) a = 0.0f;
            }
            if (ch + 1 < c) {
                b = gamma[ch + 1] * (f.y - mean[ch + 1]) * invstd[ch + 1] + beta[ch + 1];
                if (relu && !(b > 0.0f)) b = 0.0f;
            }
            h[e] = __floats2bfloat162_rn(a, b);
        }
        y[i] = v;
    }
}

// dgrad-epilogue partials -> dbeta = sum d, dgamma = sum d*xhat (double),
// rounded to the element type like the reference (primitives.cpp:145-146).
__global__ void bn_bwd_finalize_partials_kernel(const float* __restrict__ part, int slots, int c,
                                                int round_bf16, float* __restrict__ dgamma,
                                                float* __restrict__ dbeta,
                                                float* __restrict__ tot) {
    const int ch = blockIdx.x * blockDim.x + threadIdx.x;
    if (ch >= c) return;
    double s = 0.0, t = 0.0;
    for (int k = 0; k < slots; ++k) {
        s += part[((size_t)k * c + ch) * 2 + 0];
        t += part[((size_t)k * c + ch) * 2 + 1];
    }
    float fs = (float)s, ft = (float)t;
    tot[2 * ch] = fs;
    tot[2 * ch + 1] = ft;
    if (round_bf16) {
        fs = __bfloat162float(__float2bfloat16_rn(fs));
        ft = __bfloat162float(__float2bfloat16_rn(ft));
    }
    if (dbeta) dbeta[ch] = fs;
    if (dgamma) dgamma[ch] = ft;
}

// dx = gamma*invstd/m * (m*d - sum d - xhat * sum d*xhat), d = dz * mask,
// 8 bf16 channels per thread.
__global__ void bn_bwd_apply_bf16x8_kernel(const uint4* __restrict__ dz, const uint4* __restrict__ y,
                                           uint4* __restrict__ dx, long long vecs, int c,
                                           int pitch_vecs, float m, const float* __restrict__ gamma,
                                           const float* __restrict__ beta,
                                           const float* __restrict__ mean,
                                           const float* __restrict__ invstd,
                                           const float* __restrict__ tot, int relu) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < vecs;
         i += (long long)gridDim.x * blockDim.x) {
        const int c0 = (int)(i % pitch_vecs) * 8;
        uint4 dv = __ldg(dz + i), yv = __ldg(y + i), ov;
        const __nv_bfloat162* dh = reinterpret_cast<const __nv_bfloat162*>(&dv);
        const __nv_bfloat162* yh = reinterpret_cast<const __nv_bfloat162*>(&yv);
        __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&ov);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float2 d2 = __bfloat1622float2(dh[e]), y2 = __bfloat1622float2(yh[e]);
            float o[2] = {0.f, 0.f};
            const float dd[2] = {d2.x, d2.y}, yy[2] = {y2.x, y2.y};
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int ch = c0 + 2 * e + u;
                if (ch >= c) continue;
                float d = dd[u];
                const float g = gamma[ch], mu = mean[ch], inv = invstd[ch];
                if (relu && !(g * (yy[u] - mu) * inv + beta[ch] > 0.0f)) d = 0.f;
                const float xhat = (yy[u] - mu) * inv;
                o[u] = (g * inv / m) * (m * d - tot[2 * ch] - xhat * tot[2 * ch + 1]);
            }
            oh[e] = __floats2bfloat162_rn(o[0], o[1]);
        }
        dx[i] = ov;
    }
}

inline unsigned gsz(long long total) {
    long long b = (total + 255) / 256;
    if (b > 148LL * 32) b = 148LL * 32;
    return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace pk

using namespace pk;

extern "C" {

cudaError_t pk_cuda_bn_finalize_apply(const float* part, int slots, const void* x, void* y, int n,
                                      int c, int hw, int pitch, int dtype, const float* gamma,
                                      const float* beta, float* running_mean, float* running_var,
                                      float eps, float momentum, float* saved_mean,
                                      float* saved_invstd, int relu, cudaStream_t st) {
    const long long rows = (long long)n * hw;
    bn_finalize_partials_kernel<<<(c + 127) / 128, 128, 0, st>>>(
        part, slots, c, (double)rows, eps, momentum, running_mean, running_var, saved_mean,
        saved_invstd);
    if (dtype == PK_BF16 && pitch % 8 == 0) {
        const long long vecs = rows * pitch / 8;
        bn_apply_bf16x8_kernel<<<gsz(vecs), 256, 0, st>>>((const uint4*)x, (uint4*)y, vecs, c,
                                                            pitch / 8, gamma, beta, saved_mean,
                                                            saved_invstd, relu);
    } else {
        PK_DISPATCH_DTYPE(dtype, T,
                          bn_apply_kernel<T><<<gsz(rows * pitch), 256, 0, st>>>(
                              (const T*)x, (T*)y, rows, c, hw, pitch, 0, gamma, beta, saved_mean,
                              saved_invstd, relu));
    }
    count_launch(2);
    return cudaGetLastError();
}

cudaError_t pk_cuda_bn_bwd_finalize_apply(const float* part, int slots, const void* dz,
                                          const void* y, void* dx, int n, int c, int hw, int pitch,
                                          int dtype, const float* gamma, const float* beta,
                                          const float* mean, const float* invstd, int relu,
                                          float* dgamma, float* dbeta, float* tot_scratch,
                                          cudaStream_t st) {
    if (dtype != PK_BF16 || pitch % 8) return cudaErrorNotSupported;
    const long long rows = (long long)n * hw;
    bn_bwd_finalize_partials_kernel<<<(c + 127) / 128, 128, 0, st>>>(part, slots, c, 1, dgamma,
                                                                      dbeta, tot_scratch);
    const long long vecs = rows * pitch / 8;
    bn_bwd_apply_bf16x8_kernel<<<gsz(vecs), 256, 0, st>>>(
        (const uint4*)dz, (const uint4*)y, (uint4*)dx, vecs, c, pitch / 8, (float)rows, gamma, beta,
        mean, invstd, tot_scratch, relu);
    count_launch(2);
    return cudaGetLastError();
}

cudaError_t pk_cuda_bn_apply_stats(const void* x, void* y, int n, int c, int hw, int pitch,
                                   int dtype, const float* gamma, const float* beta,
                                   const float* mean, const float* invstd, int relu,
                                   cudaStream_t st) {
    const long long rows = (long long)n * hw;
    if (dtype == PK_BF16 && pitch % 8 == 0) {
        const long long vecs = rows * pitch / 8;
        bn_apply_bf16x8_kernel<<<gsz(vecs), 256, 0, st>>>((const uint4*)x, (uint4*)y, vecs, c,
                                                            pitch / 8, gamma, beta, mean, invstd,
                                                            relu);
    } else {
        PK_DISPATCH_DTYPE(dtype, T,
                          bn_apply_kernel<T><<<gsz(rows * pitch), 256, 0, st>>>(
                              (const T*)x, (T*)y, rows, c, hw, pitch, 0, gamma, beta, mean, invstd,
                              relu));
    }
    count_launch();
    return cudaGetLastError();
}

size_t pk_bn_scratch_bytes(int n, int c, int hw, int per_act) {
    if (per_act) return (size_t)c * hw * 2 * sizeof(double);
    return (size_t)bn_chunks((long long)n * hw, c) * c * 2 * sizeof(double);
}

cudaError_t pk_cuda_bn_fwd_train(const void* x, void* y, int n, int c, int hw, int pitch,
                                 int dtype, int per_act, const float* gamma, const float* beta,
                                 float* running_mean, float* running_var, float eps,
                                 float momentum, float* saved_mean, float* saved_invstd,
                                 int relu, void* scratch, cudaStream_t st) {
    const long long rows = (long long)n * hw;
    double* part = (double*)scratch;
    int chunks = 1, nstat = c;
    double m = (double)rows;
    if (per_act) {
        nstat = c * hw;
        m = (double)n;
        PK_DISPATCH_DTYPE(dtype, T,
                          bn_partial_peract_kernel<T, 0><<<gsz(nstat), 256, 0, st>>>(
                              (const T*)x, nullptr, nullptr, n, c, hw, pitch, nullptr, nullptr, 0,
                              part));
    } else {
        chunks = bn_chunks(rows, c);
        dim3 grid((c + 31) / 32, chunks);
        PK_DISPATCH_DTYPE(dtype, T,
                          bn_partial_kernel<T, 0><<<grid, 256, 0, st>>>(
                              (const T*)x, nullptr, nullptr, rows, c, pitch, chunks, nullptr,
                              nullptr, 0, part));
    }
    bn_finalize_fwd_kernel<<<(nstat + 255) / 256, 256, 0, st>>>(
        part, chunks, nstat, m, eps, momentum, running_mean, running_var, saved_mean,
        saved_invstd);
    PK_DISPATCH_DTYPE(dtype, T,
                      bn_apply_kernel<T><<<gsz(rows * pitch), 256, 0, st>>>(
                          (const T*)x, (T*)y, rows, c, hw, pitch, per_act, gamma, beta,
                          saved_mean, saved_invstd, relu));
    count_launch(3);
    return cudaGetLastError();
}

cudaError_t pk_cuda_bn_bwd(const void* x, const void* y, const void* dy, void* dx, int n, int c,
                           int hw, int pitch, int dtype, int per_act, const float* gamma,
                           const float* saved_mean, const float* saved_invstd, float* dgamma,
                           float* dbeta, int relu, int round_params_bf16, void* scratch,
                           cudaStream_t st) {
    const long long rows = (long long)n * hw;
    double* part = (double*)scratch;
    int chunks = 1, nstat = c;
    double m = (double)rows;
    if (per_act) {
        nstat = c * hw;
        m = (double)n;
        PK_DISPATCH_DTYPE(dtype, T,
                          bn_partial_peract_kernel<T, 1><<<gsz(nstat), 256, 0, st>>>(
                              (const T*)x, (const T*)y, (const T*)dy, n, c, hw, pitch,
                              saved_mean, saved_invstd, relu, part));
    } else {
        chunks = bn_chunks(rows, c);
        dim3 grid((c + 31) / 32, chunks);
        PK_DISPATCH_DTYPE(dtype, T,
                          bn_partial_kernel<T, 1><<<grid, 256, 0, st>>>(
                              (const T*)x, (const T*)y, (const T*)dy, rows, c, pitch, chunks,
                              saved_mean, saved_invstd, relu, part));
    }
    bn_finalize_bwd_kernel<<<(nstat + 255) / 256, 256, 0, st>>>(part, chunks, nstat, dgamma,
                                                                 dbeta, round_params_bf16);
    PK_DISPATCH_DTYPE(dtype, T,
                      bn_dx_kernel<T><<<gsz(rows * pitch), 256, 0, st>>>(
                          (const T*)x, (const T*)y, (const T*)dy, (T*)dx, rows, c, hw, pitch,
                          per_act, m, gamma, saved_mean, saved_invstd, part, relu));
    count_launch(3);
    return cudaGetLastError();
}

}  // extern "C"
