// Single-launch training batch-norm for bf16 NHWC (spatial mode): statistics,
// finalize and the elementwise pass in ONE persistent kernel with two grid
// barriers, so a BN layer costs one launch and no host round trip.
//
// Semantics are the reference's (proj/src/core/primitives.cpp:61-152) and
// bit-for-bit those of the multi-kernel path in bn.cu (same per-channel
// folding, same dx formula); only the reduction tree differs, and it is fixed
// for a given device (grid = resident CTAs), so results are deterministic.
//
//   phase 1  every CTA reduces a contiguous row range: fp32 sums over 8 rows
//            in flight per thread, folded into double accumulators, then a
//            fixed-order block reduction -> part[cta][c][2] (double)
//   barrier
//   phase 2  one warp per channel sums the CTAs' partials in fixed order
//            (lanes strided over CTAs, butterfly) -> mean/invstd + running
//            stats (forward) or dbeta/dgamma + totals (backward)
//   barrier
//   phase 3  the CTA's rows again, in REVERSE order, so the rows it read last
//            in phase 1 are still in L2 (for tensors below ~L2 size most of
//            the second read is an L2 hit)
//
// Modes: FWD (stats of x), FWD_EXT (fp32 partials from a conv epilogue),
// BWD (sums of d, d*xhat from x, dy[, y]), BWD_EXT (dgrad-epilogue partials).
#include <cstdlib>

#include "common.cuh"

namespace pk {
namespace {

enum BnCoopMode { FWD = 0, FWD_EXT = 1, BWD = 2, BWD_EXT = 3, BWD_FOLD = 4 };
constexpr int kThreads = 256;

struct BnCoopArgs {
    const uint4* x;    // BN input
    const uint4* y;    // BWD: BN output (ReLU mask) or null
    const uint4* dy;   // BWD/BWD_EXT: incoming gradient
    uint4* out;        // FWD*: y; BWD*: dx
    long long rows;
    int c, vpr;
    const float* gamma;
    const float* beta;
    float* running_mean;
    float* running_var;
    float eps, momentum;
    float* mean;       // FWD*: written; BWD*: read
    float* invstd;
    float* dgamma;
    float* dbeta;
    int relu, round_bf16;
    double* part;      // [nctas][c][2] own partials (FWD/BWD)
    const float* ext;  // [slots][c][2] epilogue partials (*_EXT)
    int ext_slots;
    float* tot;        // [c][2] backward totals (float), read back in phase 3
    unsigned* sync;    // [2] barrier arrivals / exits, zero at launch
};

__device__ __forceinline__ void grid_arrive_wait(unsigned* sync, unsigned target) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        atomicAdd(&sync[0], 1u);
        unsigned seen;
        do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(seen) : "l"(sync) : "memory");
            if (seen < target) __nanosleep(32);
        } while (seen < target);
    }
    __syncthreads();
}

__device__ __forceinline__ void unpack8(const uint4& v, float f[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float2 p = __bfloat1622float2(h[e]);
        f[2 * e] = p.x;
        f[2 * e + 1] = p.y;
    }
}

__device__ __forceinline__ uint4 pack8(const float f[8]) {
    uint4 v;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
    return v;
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 2) bn_coop_kernel(const BnCoopArgs a) {
    constexpr bool kStats = MODE == FWD || MODE == BWD || MODE == BWD_FOLD;
    constexpr bool kBwd = MODE == BWD || MODE == BWD_EXT || MODE == BWD_FOLD;
    // ReLU mask of the backward pass: from the given BN output y (BWD) or
    // recomputed from the BN input with the folded affine (BWD_EXT, BWD_FOLD)
    constexpr bool kFoldMask = MODE == BWD_EXT || MODE == BWD_FOLD;
    __shared__ double red[16][kThreads + 1];
    const int t = threadIdx.x, vpr = a.vpr, v = t & (vpr - 1), rsub = t / vpr, rpb = kThreads / vpr;
    const unsigned nctas = gridDim.x;
    const long long per = (a.rows + nctas - 1) / nctas;
    const long long r0 = (long long)blockIdx.x * per, r1 = min(a.rows, r0 + per);
    const int c = a.c;

    // ---- phase 1: this CTA's partial sums --------------------------------------
    if (kStats) {
        float mu[8], inv[8], fsc[8], fsh[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int ch = v * 8 + e;
            mu[e] = (kBwd && ch < c) ? a.mean[ch] : 0.f;
            inv[e] = (kBwd && ch < c) ? a.invstd[ch] : 0.f;
            fsc[e] = (kFoldMask && ch < c) ? a.gamma[ch] * inv[e] : 0.f;
            fsh[e] = (kFoldMask && ch < c) ? a.beta[ch] - mu[e] * fsc[e] : 0.f;
        }
        // double accumulators in shared memory (thread t owns column t), fp32
        // sums over the U rows in flight folded in once per iteration: keeps
        // the registers for loads in flight (the pass is latency-bound)
#pragma unroll
        for (int e = 0; e < 16; ++e) red[e][t] = 0.0;
        constexpr int U = kBwd ? 6 : 12;  // rows in flight per thread
        const bool use_y = MODE == BWD && a.relu && a.y;
        for (long long base = r0 + rsub; base < r1; base += (long long)rpb * U) {
            uint4 xv[U], dv[U], yv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long r = base + (long long)u * rpb;
                const bool ok = r < r1;
                xv[u] = ok ? __ldg(a.x + r * vpr + v) : make_uint4(0u, 0u, 0u, 0u);
                if (kBwd) {
                    dv[u] = ok ? __ldg(a.dy + r * vpr + v) : make_uint4(0u, 0u, 0u, 0u);
                    yv[u] = (ok && use_y) ? __ldg(a.y + r * vpr + v) : make_uint4(0u, 0u, 0u, 0u);
                }
            }
            float f0[8], f1[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) f0[e] = f1[e] = 0.f;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                float xf[8];
                unpack8(xv[u], xf);
                if (!kBwd) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        f0[e] += xf[e];
                        f1[e] = fmaf(xf[e], xf[e], f1[e]);
                    }
                } else {
                    float df[8], yf[8];
                    unpack8(dv[u], df);
                    unpack8(yv[u], yf);
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        float d = (use_y && !(yf[e] > 0.f)) ? 0.f : df[e];
                        if (kFoldMask && a.relu && !(fmaf(xf[e], fsc[e], fsh[e]) > 0.f)) d = 0.f;
                        f0[e] += d;
                        f1[e] = fmaf(d, (xf[e] - mu[e]) * inv[e], f1[e]);
                    }
                }
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                red[e][t] += (double)f0[e];
                red[8 + e][t] += (double)f1[e];
            }
        }
        __syncthreads();
        for (int o = t; o < vpr * 8; o += kThreads) {
            const int vv = o >> 3, e = o & 7, ch = vv * 8 + e;
            double sa = 0.0, sb = 0.0;
            for (int k = 0; k < rpb; ++k) {
                sa += red[e][vv + k * vpr];
                sb += red[8 + e][vv + k * vpr];
            }
            if (ch < c) {
                a.part[((size_t)blockIdx.x * c + ch) * 2 + 0] = sa;
                a.part[((size_t)blockIdx.x * c + ch) * 2 + 1] = sb;
            }
        }
        grid_arrive_wait(a.sync, nctas);
    }

    // ---- phase 2: finalize, one warp per channel ------------------------------
    {
        const int lane = t & 31;
        const int slots = kStats ? (int)nctas : a.ext_slots;
        const double m = (double)a.rows;
        for (int ch = blockIdx.x * (kThreads / 32) + (t >> 5); ch < c; ch += nctas * (kThreads / 32)) {
            double sa = 0.0, sb = 0.0;
            for (int k = lane; k < slots; k += 32) {
                if (kStats) {
                    const double2 p = __ldcg(reinterpret_cast<const double2*>(a.part) + (size_t)k * c + ch);
                    sa += p.x;
                    sb += p.y;
                } else {
                    const float2 p = __ldcg(reinterpret_cast<const float2*>(a.ext) + (size_t)k * c + ch);
                    sa += (double)p.x;
                    sb += (double)p.y;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                sa += __shfl_xor_sync(0xffffffffu, sa, o);
                sb += __shfl_xor_sync(0xffffffffu, sb, o);
            }
            if (lane == 0) {
                if (!kBwd) {
                    const double mu = sa / m;
                    const double var = fmax(0.0, sb / m - mu * mu);
                    a.mean[ch] = (float)mu;
                    a.invstd[ch] = (float)(1.0 / sqrt(var + (double)a.eps));
                    if (a.running_mean) {
                        a.running_mean[ch] = (1.0f - a.momentum) * a.running_mean[ch] + a.momentum * (float)mu;
                        a.running_var[ch] = (1.0f - a.momentum) * a.running_var[ch] + a.momentum * (float)var;
                    }
                } else {
                    float fs = (float)sa, ft = (float)sb;
                    a.tot[2 * ch] = fs;
                    a.tot[2 * ch + 1] = ft;
                    if (a.round_bf16) {
                        fs = __bfloat162float(__float2bfloat16_rn(fs));
                        ft = __bfloat162float(__float2bfloat16_rn(ft));
                    }
                    if (a.dbeta) a.dbeta[ch] = fs;
                    if (a.dgamma) a.dgamma[ch] = ft;
                }
            }
        }
    }
    grid_arrive_wait(a.sync, kStats ? 2 * nctas : nctas);

    // ---- phase 3: elementwise pass over the CTA's rows, last-read first --------
    float sc[8], sh[8], mu[8], inv[8], k1[8], t0[8], t1[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int ch = v * 8 + e;
        sc[e] = sh[e] = mu[e] = inv[e] = k1[e] = t0[e] = t1[e] = 0.f;
        if (ch < c) {
            // plain (L1-allocating) loads: every warp of every CTA reads the same
            // few lines here; through L1 only the first warp per SM goes to L2
            // (L2-only loads measured ~10 us of same-line contention). The lines
            // were written in phase 2 and never cached in this SM's L1 before.
            mu[e] = a.mean[ch];
            inv[e] = a.invstd[ch];
            sc[e] = a.gamma[ch] * inv[e];
            sh[e] = a.beta ? a.beta[ch] - mu[e] * sc[e] : 0.f;
            if (kBwd) {
                k1[e] = a.gamma[ch] * inv[e] / (float)a.rows;
                t0[e] = a.tot[2 * ch];
                t1[e] = a.tot[2 * ch + 1];
            }
        }
    }
    const float fm = (float)a.rows;
    // the CTA's rows from the top down (rows r1-1-j, j = rsub, rsub + rpb, ...)
    constexpr int U3 = MODE == BWD ? 3 : kBwd ? 4 : 8;  // rows in flight, phase 3
    const long long span = r1 - r0;
    for (long long j0 = rsub; j0 < span; j0 += (long long)rpb * U3) {
        uint4 xv[U3], dv[U3], yv[U3];
#pragma unroll
        for (int u = 0; u < U3; ++u) {
            const long long j = j0 + (long long)u * rpb;
            const long long r = r1 - 1 - j;
            const bool ok = j < span;
            xv[u] = ok ? __ldg(a.x + r * vpr + v) : make_uint4(0u, 0u, 0u, 0u);
            if (kBwd) {
                dv[u] = ok ? __ldg(a.dy + r * vpr + v) : make_uint4(0u, 0u, 0u, 0u);
                yv[u] = (ok && MODE == BWD && a.relu && a.y) ? __ldg(a.y + r * vpr + v)
                                                               : make_uint4(0u, 0u, 0u, 0u);
            }
        }
#pragma unroll
        for (int u = 0; u < U3; ++u) {
            const long long j = j0 + (long long)u * rpb;
            const long long r = r1 - 1 - j;
            float xf[8], o[8];
            unpack8(xv[u], xf);
            if (!kBwd) {
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    float val = fmaf(xf[e], sc[e], sh[e]);
                    if (a.relu) val = val > 0.f ? val : 0.f;
                    o[e] = val;
                }
            } else {
                float df[8], yf[8];
                unpack8(dv[u], df);
                unpack8(yv[u], yf);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    float d = df[e];
                    if (a.relu) {
                        // standalone: the given BN output; epilogue form: the mask
                        // recomputed from the BN input with the folded affine
                        const bool on = MODE == BWD ? (a.y ? yf[e] > 0.f : true)
                                                    : fmaf(xf[e], sc[e], sh[e]) > 0.f;
                        if (!on) d = 0.f;
                    }
                    const float xhat = (xf[e] - mu[e]) * inv[e];
                    o[e] = k1[e] * (fm * d - t0[e] - xhat * t1[e]);
                }
            }
            if (j < span) a.out[r * vpr + v] = pack8(o);
        }
    }

    // the last CTA out re-arms the barrier slot for the next launch
    __syncthreads();
    if (t == 0 && atomicAdd(&a.sync[1], 1u) == nctas - 1) {
        a.sync[0] = 0u;
        a.sync[1] = 0u;
        __threadfence();
    }
}

template <int MODE>
int coop_ctas() {
    // resident CTAs per SM for this instance, per device (co-residency is what
    // makes the spin barriers safe)
    static int cached[16] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 16) return 0;
    if (!cached[dev]) {
        int sms = 0, per = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bn_coop_kernel<MODE>, kThreads, 0);
        cached[dev] = sms * (per < 2 ? per : 2);
    }
    return cached[dev];
}

template <int MODE>
cudaError_t launch_coop(BnCoopArgs& a, cudaStream_t st) {
    int grid = coop_ctas<MODE>();
    if (grid <= 0) return cudaErrorNotSupported;
    // at least 16 rows per thread-row of a CTA keeps the partials small
    const long long rpb = kThreads / a.vpr;
    const long long want = (a.rows + rpb * 16 - 1) / (rpb * 16);
    if (want < grid) grid = (int)(want < 1 ? 1 : want);
    a.sync = splitk_sync_slot();
    if (!a.sync) return cudaErrorNotSupported;
    note_kernel(reinterpret_cast<const void*>(bn_coop_kernel<MODE>));
    bn_coop_kernel<MODE><<<grid, kThreads, 0, st>>>(a);
    count_launch();
    return cudaGetLastError();
}

bool coop_ok(int dtype, int pitch) {
    static const bool on = [] {
        const char* v = std::getenv("PK_BN_COOP");
        return !(v && v[0] == '0');
    }();
    const int vpr = pitch / 8;
    return on && dtype == PK_BF16 && pitch % 8 == 0 && vpr >= 1 && vpr <= kThreads &&
           (vpr & (vpr - 1)) == 0;
}

}  // namespace

size_t bn_coop_scratch_bytes(int c) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
        cudaGetLastError();
        sms = 148;
    }
    return (size_t)sms * 2 * c * 2 * sizeof(double) + (size_t)c * 2 * sizeof(float) + 256;
}

cudaError_t bn_coop_fwd(const void* x, void* y, long long rows, int c, int pitch, int dtype,
                        const float* gamma, const float* beta, float* running_mean,
                        float* running_var, float eps, float momentum, float* saved_mean,
                        float* saved_invstd, int relu, const float* ext, int ext_slots,
                        void* scratch, cudaStream_t st) {
    if (!coop_ok(dtype, pitch)) return cudaErrorNotSupported;
    BnCoopArgs a{};
    a.x = (const uint4*)x;
    a.out = (uint4*)y;
    a.rows = rows;
    a.c = c;
    a.vpr = pitch / 8;
    a.gamma = gamma;
    a.beta = beta;
    a.running_mean = running_mean;
    a.running_var = running_var;
    a.eps = eps;
    a.momentum = momentum;
    a.mean = saved_mean;
    a.invstd = saved_invstd;
    a.relu = relu;
    a.part = (double*)scratch;
    a.ext = ext;
    a.ext_slots = ext_slots;
    return ext ? launch_coop<FWD_EXT>(a, st) : launch_coop<FWD>(a, st);
}

cudaError_t bn_coop_bwd(const void* x, const void* y, const void* dy, void* dx, long long rows,
                        int c, int pitch, int dtype, const float* gamma, const float* beta,
                        const float* mean, const float* invstd, float* dgamma, float* dbeta,
                        int relu, int round_bf16, const float* ext, int ext_slots, float* tot,
                        void* scratch, cudaStream_t st) {
    if (!coop_ok(dtype, pitch)) return cudaErrorNotSupported;
    BnCoopArgs a{};
    a.x = (const uint4*)x;
    a.y = (const uint4*)y;
    a.dy = (const uint4*)dy;
    a.out = (uint4*)dx;
    a.rows = rows;
    a.c = c;
    a.vpr = pitch / 8;
    a.gamma = gamma;
    a.beta = beta;
    a.mean = const_cast<float*>(mean);
    a.invstd = const_cast<float*>(invstd);
    a.dgamma = dgamma;
    a.dbeta = dbeta;
    a.relu = relu;
    a.round_bf16 = round_bf16;
    a.part = (double*)scratch;
    a.ext = ext;
    a.ext_slots = ext_slots;
    a.tot = tot;
    if (ext) return launch_coop<BWD_EXT>(a, st);
    // ReLU without the BN output: mask from the BN input (needs beta)
    if (relu && !y) return beta ? launch_coop<BWD_FOLD>(a, st) : cudaErrorNotSupported;
    return launch_coop<BWD>(a, st);
}

}  // namespace pk
