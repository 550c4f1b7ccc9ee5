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

// Fixed-order (deterministic) warp reduction of (a, b) pairs over chunks:
// lane l sums chunks l, l+32, ...; then a butterfly in double.
template <typename P>
__device__ __forceinline__ void warp_sum_pairs(const P* __restrict__ part, int chunks, int nstat,
                                               int si, double& a, double& b) {
    const int lane = threadIdx.x & 31;
    a = 0.0;
    b = 0.0;
    for (int k = lane; k < chunks; k += 32) {
        a += (double)part[((size_t)k * nstat + si) * 2 + 0];
        b += (double)part[((size_t)k * nstat + si) * 2 + 1];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
}

__global__ void bn_finalize_fwd_kernel(const double* __restrict__ part, int chunks, int nstat,
                                       double m, float eps, float momentum,
                                       float* __restrict__ running_mean,
                                       float* __restrict__ running_var,
                                       float* __restrict__ saved_mean,
                                       float* __restrict__ saved_invstd) {
    const int si = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // one warp per statistic
    if (si >= nstat) return;
    double s, sq;
    warp_sum_pairs(part, chunks, nstat, si, s, sq);
    if ((threadIdx.x & 31) != 0) return;
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
    const int si = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // one warp per statistic
    if (si >= nstat) return;
    double db, dg;
    warp_sum_pairs(part, chunks, nstat, si, db, dg);
    if ((threadIdx.x & 31) != 0) return;
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
    const int ch = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // one warp per channel
    if (ch >= c) return;
    double s, sq;
    warp_sum_pairs(part, slots, c, ch, s, sq);
    if ((threadIdx.x & 31) != 0) return;
    const double mu = s / m;
    const double var = fmax(0.0, sq / m - mu * mu);
    saved_mean[ch] = (float)mu;
    saved_invstd[ch] = (float)(1.0 / sqrt(var + (double)eps));
    if (running_mean) {
        running_mean[ch] = (1.0f - momentum) * running_mean[ch] + momentum * (float)mu;
        running_var[ch] = (1.0f - momentum) * running_var[ch] + momentum * (float)var;
    }
}

// ---- vectorised bf16 passes (16 B = 8 channels per access) ----------------
// Thread layout: thread t owns channel vector v = t % vpr (vpr = pitch / 8, a
// power of two <= 256) for the whole kernel, so its per-channel constants
// live in registers; rows advance by 256 / vpr per block step. The folded
// affine y = fma(x, gamma*invstd, beta - mean*gamma*invstd) is used by the
// forward apply AND by the backward ReLU-mask recomputation (bn_fold), so the
// two always agree on the mask.

__device__ __forceinline__ void bn_fold(float g, float b, float mu, float inv, float& sc, float& sh) {
    sc = g * inv;
    sh = b - mu * sc;
}

__global__ void __launch_bounds__(256) bn_apply_bf16x8_kernel(
    const uint4* __restrict__ x, uint4* __restrict__ y, long long rows, int c, int vpr,
    const float* __restrict__ gamma, const float* __restrict__ beta,
    const float* __restrict__ mean, const float* __restrict__ invstd, int relu) {
    const int v = threadIdx.x & (vpr - 1), rpb = 256 / vpr;
    float sc[8], sh[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int ch = v * 8 + e;
        sc[e] = sh[e] = 0.f;
        if (ch < c) bn_fold(gamma[ch], beta[ch], mean[ch], invstd[ch], sc[e], sh[e]);
    }
    // 4 rows per thread in flight (the pass is latency-bound otherwise)
    const long long step = (long long)gridDim.x * rpb;
    for (long long r0 = (long long)blockIdx.x * rpb + threadIdx.x / vpr; r0 < rows; r0 += 4 * step) {
        uint4 val[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long r = r0 + u * step;
            val[u] = r < rows ? __ldg(x + r * vpr + v) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long r = r0 + u * step;
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&val[u]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h[e]);
                float a = fmaf(f.x, sc[2 * e], sh[2 * e]), b = fmaf(f.y, sc[2 * e + 1], sh[2 * e + 1]);
                if (relu) {
                    a = a > 0.f ? a : 0.f;
                    b = b > 0.f ? b : 0.f;
                }
                h[e] = __floats2bfloat162_rn(a, b);
            }
            if (r < rows) y[r * vpr + v] = val[u];
        }
    }
}

// dgrad-epilogue partials -> dbeta = sum d, dgamma = sum d*xhat (double),
// rounded to the element type like the reference (primitives.cpp:145-146).
__global__ void bn_bwd_finalize_partials_kernel(const float* __restrict__ part, int slots, int c,
                                                int round_bf16, float* __restrict__ dgamma,
                                                float* __restrict__ dbeta,
                                                float* __restrict__ tot) {
    const int ch = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // one warp per channel
    if (ch >= c) return;
    double s, t;
    warp_sum_pairs(part, slots, c, ch, s, t);
    if ((threadIdx.x & 31) != 0) return;
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

// dx = gamma*invstd/m * (m*d - sum d - xhat * sum d*xhat), d = dz * mask
__global__ void __launch_bounds__(256) bn_bwd_apply_bf16x8_kernel(
    const uint4* __restrict__ dz, const uint4* __restrict__ y, uint4* __restrict__ dx,
    long long rows, int c, int vpr, float m, const float* __restrict__ gamma,
    const float* __restrict__ beta, const float* __restrict__ mean,
    const float* __restrict__ invstd, const float* __restrict__ tot, int relu) {
    const int v = threadIdx.x & (vpr - 1), rpb = 256 / vpr;
    float sc[8], sh[8], mu[8], inv[8], k1[8], k0[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int ch = v * 8 + e;
        sc[e] = sh[e] = mu[e] = inv[e] = k1[e] = k0[e] = 0.f;
        if (ch < c) {
            bn_fold(gamma[ch], beta[ch], mean[ch], invstd[ch], sc[e], sh[e]);
            mu[e] = mean[ch];
            inv[e] = invstd[ch];
            k1[e] = gamma[ch] * inv[e] / m;  // dx = k1 * (m*d - tot0 - xhat*tot1)
            k0[e] = tot[2 * ch];
        }
    }
    float t1[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) t1[e] = (v * 8 + e < c) ? tot[2 * (v * 8 + e) + 1] : 0.f;
    const long long step = (long long)gridDim.x * rpb;
    for (long long r0 = (long long)blockIdx.x * rpb + threadIdx.x / vpr; r0 < rows; r0 += 2 * step) {
        uint4 dvs[2], yvs[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const long long r = r0 + q * step;
            dvs[q] = r < rows ? __ldg(dz + r * vpr + v) : make_uint4(0u, 0u, 0u, 0u);
            yvs[q] = r < rows ? __ldg(y + r * vpr + v) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const long long r = r0 + q * step;
            uint4 ov;
            const __nv_bfloat162* dh = reinterpret_cast<const __nv_bfloat162*>(&dvs[q]);
            const __nv_bfloat162* yh = reinterpret_cast<const __nv_bfloat162*>(&yvs[q]);
            __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&ov);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 d2 = __bfloat1622float2(dh[e]), y2 = __bfloat1622float2(yh[e]);
                float o[2];
                const float dd[2] = {d2.x, d2.y}, yy[2] = {y2.x, y2.y};
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int j = 2 * e + u;
                    float d = dd[u];
                    if (relu && !(fmaf(yy[u], sc[j], sh[j]) > 0.0f)) d = 0.f;
                    const float xhat = (yy[u] - mu[j]) * inv[j];
                    o[u] = k1[j] * (m * d - k0[j] - xhat * t1[j]);
                }
                oh[e] = __floats2bfloat162_rn(o[0], o[1]);
            }
            if (r < rows) dx[r * vpr + v] = ov;
        }
    }
}

// Vectorised statistics pass (bf16, spatial): thread t owns channel vector
// t % vpr, accumulates fp32 over its rows of the block's chunk, then the
// block reduces the rows in a fixed order (double) -> part[chunk][c][2].
// MODE 0: (sum x, sum x^2); MODE 1: (sum d, sum d*xhat), d = dy masked by
// y > 0 when relu (y = the BN output).
template <int MODE>
__global__ void __launch_bounds__(256) bn_partial_vec_kernel(
    const uint4* __restrict__ x, const uint4* __restrict__ y, const uint4* __restrict__ dy,
    long long rows, int c, int vpr, int chunks, const float* __restrict__ mean,
    const float* __restrict__ invstd, int relu, double* __restrict__ part) {
    __shared__ float red[16][257];
    const int t = threadIdx.x, v = t & (vpr - 1), rpb = 256 / vpr;
    const long long per = (rows + chunks - 1) / chunks;
    const long long r0 = blockIdx.x * per, r1 = min(rows, r0 + per);
    float a[8], b[8], mu[8], inv[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        a[e] = b[e] = 0.f;
        const int ch = v * 8 + e;
        mu[e] = (MODE == 1 && ch < c) ? mean[ch] : 0.f;
        inv[e] = (MODE == 1 && ch < c) ? invstd[ch] : 0.f;
    }
#pragma unroll 4
    for (long long r = r0 + t / vpr; r < r1; r += rpb) {
        const uint4 xv = __ldg(x + r * vpr + v);
        const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&xv);
        if (MODE == 0) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(xh[e]);
                a[2 * e] += f.x;
                b[2 * e] = fmaf(f.x, f.x, b[2 * e]);
                a[2 * e + 1] += f.y;
                b[2 * e + 1] = fmaf(f.y, f.y, b[2 * e + 1]);
            }
        } else {
            const uint4 dv = __ldg(dy + r * vpr + v);
            const __nv_bfloat162* dh = reinterpret_cast<const __nv_bfloat162*>(&dv);
            uint4 yv = make_uint4(0u, 0u, 0u, 0u);
            if (relu) yv = __ldg(y + r * vpr + v);
            const __nv_bfloat162* yh = reinterpret_cast<const __nv_bfloat162*>(&yv);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(xh[e]), d2 = __bfloat1622float2(dh[e]);
                const float2 y2 = __bfloat1622float2(yh[e]);
                const float d0 = (relu && !(y2.x > 0.f)) ? 0.f : d2.x;
                const float d1 = (relu && !(y2.y > 0.f)) ? 0.f : d2.y;
                a[2 * e] += d0;
                b[2 * e] = fmaf(d0, (f.x - mu[2 * e]) * inv[2 * e], b[2 * e]);
                a[2 * e + 1] += d1;
                b[2 * e + 1] = fmaf(d1, (f.y - mu[2 * e + 1]) * inv[2 * e + 1], b[2 * e + 1]);
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        red[e][t] = a[e];
        red[8 + e][t] = b[e];
    }
    __syncthreads();
    for (int o = t; o < vpr * 8; o += 256) {
        const int vv = o >> 3, e = o & 7, ch = vv * 8 + e;
        double sa = 0.0, sb = 0.0;
        for (int k = 0; k < rpb; ++k) {
            sa += red[e][vv + k * vpr];
            sb += red[8 + e][vv + k * vpr];
        }
        if (ch < c) {
            part[((size_t)blockIdx.x * c + ch) * 2 + 0] = sa;
            part[((size_t)blockIdx.x * c + ch) * 2 + 1] = sb;
        }
    }
}

inline int bn_vec_chunks(long long rows) {
    long long ch = rows / 64;
    if (ch > 148LL * 4) ch = 148LL * 4;
    return (int)(ch < 1 ? 1 : ch);
}

inline bool bn_vec_ok(int dtype, int pitch) {
    const int vpr = pitch / 8;
    return dtype == PK_BF16 && pitch % 8 == 0 && vpr >= 1 && vpr <= 256 && (vpr & (vpr - 1)) == 0;
}

inline unsigned bn_vec_blocks(long long rows, int vpr) {
    long long b = (rows * vpr + 255) / 256;
    if (b > 148LL * 8) b = 148LL * 8;
    return (unsigned)(b < 1 ? 1 : b);
}

// Single-launch persistent forms (bn_coop.cu); cudaErrorNotSupported when the
// layout does not qualify (then the multi-kernel path below runs).
size_t bn_coop_scratch_bytes(int c);
cudaError_t bn_coop_fwd(const void* x, void* y, long long rows, int c, int pitch, int dtype,
                        const float* gamma, const float* beta, float* running_mean,
                        float* running_var, float eps, float momentum, float* saved_mean,
                        float* saved_invstd, int relu, const float* ext, int ext_slots,
                        void* scratch, cudaStream_t st);
cudaError_t bn_coop_bwd(const void* x, const void* y, const void* dy, void* dx, long long rows,
                        int c, int pitch, int dtype, const float* gamma, const float* beta,
                        const float* mean, const float* invstd, float* dgamma, float* dbeta,
                        int relu, int round_bf16, const float* ext, int ext_slots, float* tot,
                        void* scratch, cudaStream_t st);

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
    if (bn_coop_fwd(x, y, rows, c, pitch, dtype, gamma, beta, running_mean, running_var, eps,
                    momentum, saved_mean, saved_invstd, relu, part, slots, nullptr,
                    st) == cudaSuccess)
        return cudaSuccess;
    cudaGetLastError();
    bn_finalize_partials_kernel<<<(c + 7) / 8, 256, 0, st>>>(
        part, slots, c, (double)rows, eps, momentum, running_mean, running_var, saved_mean,
        saved_invstd);
    if (bn_vec_ok(dtype, pitch)) {
        bn_apply_bf16x8_kernel<<<bn_vec_blocks(rows, pitch / 8), 256, 0, st>>>(
            (const uint4*)x, (uint4*)y, rows, c, pitch / 8, gamma, beta, saved_mean, saved_invstd,
            relu);
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
    if (!bn_vec_ok(dtype, pitch)) return cudaErrorNotSupported;
    const long long rows = (long long)n * hw;
    if (bn_coop_bwd(y, nullptr, dz, dx, rows, c, pitch, dtype, gamma, beta, mean, invstd, dgamma,
                    dbeta, relu, 1, part, slots, tot_scratch, nullptr, st) == cudaSuccess)
        return cudaSuccess;
    cudaGetLastError();
    bn_bwd_finalize_partials_kernel<<<(c + 7) / 8, 256, 0, st>>>(part, slots, c, 1, dgamma,
                                                                      dbeta, tot_scratch);
    bn_bwd_apply_bf16x8_kernel<<<bn_vec_blocks(rows, pitch / 8), 256, 0, st>>>(
        (const uint4*)dz, (const uint4*)y, (uint4*)dx, rows, c, pitch / 8, (float)rows, gamma, beta,
        mean, invstd, tot_scratch, relu);
    count_launch(2);
    return cudaGetLastError();
}

cudaError_t pk_cuda_bn_apply_stats(const void* x, void* y, int n, int c, int hw, int pitch,
                                   int dtype, const float* gamma, const float* beta,
                                   const float* mean, const float* invstd, int relu,
                                   cudaStream_t st) {
    const long long rows = (long long)n * hw;
    if (bn_vec_ok(dtype, pitch)) {
        bn_apply_bf16x8_kernel<<<bn_vec_blocks(rows, pitch / 8), 256, 0, st>>>(
            (const uint4*)x, (uint4*)y, rows, c, pitch / 8, gamma, beta, mean, invstd, relu);
    } else {
        PK_DISPATCH_DTYPE(dtype, T,
                          bn_apply_kernel<T><<<gsz(rows * pitch), 256, 0, st>>>(
                              (const T*)x, (T*)y, rows, c, hw, pitch, 0, gamma, beta, mean, invstd,
                              relu));
    }
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_bn_bwd_fold(const void* x, const void* dz, void* dx, int n, int c, int hw,
                                int pitch, int dtype, const float* gamma, const float* beta,
                                const float* mean, const float* invstd, int relu, float* dgamma,
                                float* dbeta, void* scratch, cudaStream_t st) {
    const long long rows = (long long)n * hw;
    float* tot = (float*)((char*)scratch + bn_coop_scratch_bytes(c) - (size_t)c * 2 * sizeof(float) - 256);
    return bn_coop_bwd(x, nullptr, dz, dx, rows, c, pitch, dtype, gamma, beta, mean, invstd,
                       dgamma, dbeta, relu, dtype == PK_BF16, nullptr, 0, tot, scratch, st);
}

size_t pk_bn_scratch_bytes(int n, int c, int hw, int per_act) {
    if (per_act) return (size_t)c * hw * 2 * sizeof(double);
    const int a = bn_chunks((long long)n * hw, c), b = bn_vec_chunks((long long)n * hw);
    const size_t legacy = (size_t)(a > b ? a : b) * c * 2 * sizeof(double);
    const size_t coop = bn_coop_scratch_bytes(c);
    return legacy > coop ? legacy : coop;
}

cudaError_t pk_cuda_bn_fwd_train(const void* x, void* y, int n, int c, int hw, int pitch,
                                 int dtype, int per_act, const float* gamma, const float* beta,
                                 float* running_mean, float* running_var, float eps,
                                 float momentum, float* saved_mean, float* saved_invstd,
                                 int relu, void* scratch, cudaStream_t st) {
    const long long rows = (long long)n * hw;
    if (!per_act && bn_coop_fwd(x, y, rows, c, pitch, dtype, gamma, beta, running_mean,
                                running_var, eps, momentum, saved_mean, saved_invstd, relu,
                                nullptr, 0, scratch, st) == cudaSuccess)
        return cudaSuccess;
    cudaGetLastError();
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
    } else if (bn_vec_ok(dtype, pitch)) {
        chunks = bn_vec_chunks(rows);
        bn_partial_vec_kernel<0><<<chunks, 256, 0, st>>>((const uint4*)x, nullptr, nullptr, rows, c,
                                                         pitch / 8, chunks, nullptr, nullptr, 0, part);
    } else {
        chunks = bn_chunks(rows, c);
        dim3 grid((c + 31) / 32, chunks);
        PK_DISPATCH_DTYPE(dtype, T,
                          bn_partial_kernel<T, 0><<<grid, 256, 0, st>>>(
                              (const T*)x, nullptr, nullptr, rows, c, pitch, chunks, nullptr,
                              nullptr, 0, part));
    }
    bn_finalize_fwd_kernel<<<(nstat + 7) / 8, 256, 0, st>>>(
        part, chunks, nstat, m, eps, momentum, running_mean, running_var, saved_mean,
        saved_invstd);
    if (!per_act && bn_vec_ok(dtype, pitch))
        bn_apply_bf16x8_kernel<<<bn_vec_blocks(rows, pitch / 8), 256, 0, st>>>(
            (const uint4*)x, (uint4*)y, rows, c, pitch / 8, gamma, beta, saved_mean, saved_invstd,
            relu);
    else
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
    if (!per_act) {
        // totals live behind the CTA partials in the scratch
        float* tot = (float*)((char*)scratch + bn_coop_scratch_bytes(c) - (size_t)c * 2 * sizeof(float) - 256);
        if (bn_coop_bwd(x, y, dy, dx, rows, c, pitch, dtype, gamma, nullptr, saved_mean,
                        saved_invstd, dgamma, dbeta, relu, round_params_bf16, nullptr, 0, tot,
                        scratch, st) == cudaSuccess)
            return cudaSuccess;
        cudaGetLastError();
    }
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
    } else if (bn_vec_ok(dtype, pitch)) {
        chunks = bn_vec_chunks(rows);
        bn_partial_vec_kernel<1><<<chunks, 256, 0, st>>>((const uint4*)x, (const uint4*)y,
                                                         (const uint4*)dy, rows, c, pitch / 8,
                                                         chunks, saved_mean, saved_invstd, relu,
                                                         part);
    } else {
        chunks = bn_chunks(rows, c);
        dim3 grid((c + 31) / 32, chunks);
        PK_DISPATCH_DTYPE(dtype, T,
                          bn_partial_kernel<T, 1><<<grid, 256, 0, st>>>(
                              (const T*)x, (const T*)y, (const T*)dy, rows, c, pitch, chunks,
                              saved_mean, saved_invstd, relu, part));
    }
    bn_finalize_bwd_kernel<<<(nstat + 7) / 8, 256, 0, st>>>(part, chunks, nstat, dgamma,
                                                                 dbeta, round_params_bf16);
    PK_DISPATCH_DTYPE(dtype, T,
                      bn_dx_kernel<T><<<gsz(rows * pitch), 256, 0, st>>>(
                          (const T*)x, (const T*)y, (const T*)dy, (T*)dx, rows, c, hw, pitch,
                          per_act, m, gamma, saved_mean, saved_invstd, part, relu));
    count_launch(3);
    return cudaGetLastError();
}

}  // extern "C"
