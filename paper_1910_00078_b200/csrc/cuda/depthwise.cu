// Depthwise convolution (groups == C == K: one input and one output channel per
// group), NHWC, CUDA cores, f32 / bf16 storage with fp32 accumulation.
//
// Same products as the reference's Direct loops restricted to cg == kg == 1
// (proj/src/core/conv.cpp:99-133 forward, :716-756 backward data, :816-850
// backward weights), scheduled for HBM: a thread owns 8 consecutive channels
// of one pixel, so a warp's x / dY loads are contiguous 16-byte (bf16) or
// 32-byte (f32) vectors, and the CTA's filter taps sit in shared memory as
// [tap][channel] fp32 rows. The generic Direct kernels put lanes on pixels and
// read one channel per lane at a channel-pitch stride (~70x slower on these
// shapes). Forward and backward-data accumulate taps in (r, s) order like the
// reference; backward weights reduces per CTA chunk in a fixed order and sums
// the chunks in a second fixed-order pass, so every result is deterministic.
#include "common.cuh"

namespace pk {
namespace {

constexpr int kThreads = 256;
constexpr int kTapGroup = 9;  // wgrad taps accumulated in registers per pass

__device__ __forceinline__ void load8v(const float* p, float (&v)[8]) {
    const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void load8v(const __nv_bfloat16* p, float (&v)[8]) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h[i]);
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
    }
}
__device__ __forceinline__ void store8v(float* p, const float (&v)[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void store8v(__nv_bfloat16* p, const float (&v)[8]) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = u;
}

// Channel block per CTA (a multiple of 8 dividing the channel pitch).
__host__ __device__ inline int dw_block_channels(int pitch) {
    return pitch % 64 == 0 ? 64 : pitch % 32 == 0 ? 32 : pitch % 16 == 0 ? 16 : 8;
}

// Filter taps of channels [c0, c0 + cb) -> smem [tap][cb] (zero past K).
template <typename T>
__device__ __forceinline__ void stage_filter(const pk_conv_geom& g, const T* f, float* sw, int c0, int cb) {
    const int taps = g.r * g.s;
    for (int i = threadIdx.x; i < taps * cb; i += blockDim.x) {
        const int tap = i / cb, c = c0 + i % cb;
        sw[i] = c < g.k ? ld(f + ((size_t)c * taps + tap) * g.f_pitch) : 0.0f;
    }
}

// Forward (BWD = false): y[n,oh,ow,c] = sum_{r,s} x[n, oh*sh-ph+r*dh, ow*sw-pw+s*dw, c] w[c,r,s].
// Backward data (BWD = true): dx[n,ih,iw,c] = sum_{r,s} dy[n,oh,ow,c] w[c,r,s] over the (oh, ow)
// with oh*sh - ph + r*dh == ih (and likewise for w).
// K3: 3x3 filter known at compile time (taps unrolled, loads issued together).
template <typename T, bool BWD, bool K3>
__global__ void __launch_bounds__(kThreads) depthwise_kernel(pk_conv_geom g, const T* __restrict__ src,
                                                             const T* __restrict__ f,
                                                             T* __restrict__ dst, pk_epilogue e) {
    extern __shared__ float sw[];
    const int pitch = BWD ? g.x_pitch : g.y_pitch, src_pitch = BWD ? g.y_pitch : g.x_pitch;
    const int cb = dw_block_channels(pitch), cv = cb / 8, lanes_px = kThreads / cv;
    const int c0 = blockIdx.y * cb;
    stage_filter(g, f, sw, c0, cb);
    __syncthreads();
    const int cvi = threadIdx.x % cv, pl = threadIdx.x / cv;
    const int oh_n = BWD ? g.h : g.p, ow_n = BWD ? g.w : g.q;  // this pass's output grid
    const int ih_n = BWD ? g.p : g.h, iw_n = BWD ? g.q : g.w;  // and the grid it reads
    // work unit = (output row, segment of lanes_px pixels); the row split is
    // block-uniform 32-bit math, not a 64-bit divide per pixel
    const int segs = (ow_n + lanes_px - 1) / lanes_px;
    const unsigned units = (unsigned)g.n * oh_n * segs;
    const int cc = c0 + cvi * 8;
    const bool epi = !BWD && epilogue_active(&e);
    for (unsigned u = blockIdx.x; u < units; u += gridDim.x) {
        const unsigned row = u / segs;
        const int ow = (int)(u - row * segs) * lanes_px + pl;
        if (ow >= ow_n) continue;
        const int oh = (int)(row % oh_n), n = (int)(row / oh_n);
        const long long pix = (long long)row * ow_n + ow;
        const T* sn = src + (size_t)n * ih_n * iw_n * src_pitch + cc;
        float acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
        const int R = K3 ? 3 : g.r, S = K3 ? 3 : g.s;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            int ih;
            if (!BWD) {
                ih = oh * g.str_h - g.pad_h + r * g.dil_h;
                if (ih < 0 || ih >= ih_n) continue;
            } else {
                const int num = oh + g.pad_h - r * g.dil_h;
                if (num < 0 || num % g.str_h) continue;
                ih = num / g.str_h;
                if (ih >= ih_n) continue;
            }
#pragma unroll
            for (int s = 0; s < S; ++s) {
                int iw;
                if (!BWD) {
                    iw = ow * g.str_w - g.pad_w + s * g.dil_w;
                    if (iw < 0 || iw >= iw_n) continue;
                } else {
                    const int num = ow + g.pad_w - s * g.dil_w;
                    if (num < 0 || num % g.str_w) continue;
                    iw = num / g.str_w;
                    if (iw >= iw_n) continue;
                }
                float v[8];
                load8v(sn + ((size_t)ih * iw_n + iw) * src_pitch, v);
                const float4* wp = reinterpret_cast<const float4*>(sw + (r * S + s) * cb + cvi * 8);
                const float4 w0 = wp[0], w1 = wp[1];
                acc[0] += v[0] * w0.x; acc[1] += v[1] * w0.y; acc[2] += v[2] * w0.z; acc[3] += v[3] * w0.w;
                acc[4] += v[4] * w1.x; acc[5] += v[5] * w1.y; acc[6] += v[6] * w1.z; acc[7] += v[7] * w1.w;
            }
        }
        const int kmax = BWD ? g.c : g.k;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (cc + j >= kmax)
                acc[j] = 0.0f;  // pad lanes stay zero (layout contract)
            else if (epi)
                acc[j] = apply_epilogue(e, acc[j], cc + j, oh, ow, g.p, g.q);
        }
        store8v(dst + (size_t)pix * pitch + cc, acc);
    }
}

// 3x3, stride 1, dilation 1 (forward and backward data): a thread owns 8
// channels of 4 consecutive output pixels of one row, so each input row's 6
// vectors serve 12 taps from registers and the index math is per quad. The
// input column of tap s for output j is j + s (forward, pad subtracted) or
// j + 2 - s (backward data, the flipped correlation), relative to c_lo.
template <typename T, bool BWD>
__global__ void __launch_bounds__(kThreads) depthwise3_s1_kernel(pk_conv_geom g, const T* __restrict__ src,
                                                                 const T* __restrict__ f,
                                                                 T* __restrict__ dst, pk_epilogue e) {
    extern __shared__ float sw[];
    const int pitch = BWD ? g.x_pitch : g.y_pitch, src_pitch = BWD ? g.y_pitch : g.x_pitch;
    const int cb = dw_block_channels(pitch), cv = cb / 8, lanes_px = kThreads / cv;
    const int c0 = blockIdx.y * cb;
    stage_filter(g, f, sw, c0, cb);
    __syncthreads();
    const int cvi = threadIdx.x % cv, pl = threadIdx.x / cv, cc = c0 + cvi * 8;
    const int oh_n = BWD ? g.h : g.p, ow_n = BWD ? g.w : g.q;
    const int ih_n = BWD ? g.p : g.h, iw_n = BWD ? g.q : g.w;
    const int off_h = BWD ? g.pad_h - 2 : -g.pad_h, off_w = BWD ? g.pad_w - 2 : -g.pad_w;
    const int qpr = (ow_n + 3) / 4;
    const unsigned quads = (unsigned)g.n * oh_n * qpr;
    const int kmax = BWD ? g.c : g.k;
    const bool epi = !BWD && epilogue_active(&e);
    for (unsigned qi = blockIdx.x * lanes_px + pl; qi < quads; qi += gridDim.x * lanes_px) {
        const unsigned row = qi / qpr;
        const int ow0 = (int)(qi - row * qpr) * 4;
        const int oh = (int)(row % oh_n), n = (int)(row / oh_n);
        const T* sn = src + (size_t)n * ih_n * iw_n * src_pitch + cc;
        float acc[4][8];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[j][c] = 0.0f;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const int ih = oh + off_h + (BWD ? 2 - r : r);
            if (ih < 0 || ih >= ih_n) continue;
            float v[6][8];
            const int iw0 = ow0 + off_w;
            const T* rp = sn + (ih * iw_n + iw0) * src_pitch;  // 32-bit offsets within an image
            if (iw0 >= 0 && iw0 + 5 < iw_n) {  // interior quad: no column checks
#pragma unroll
                for (int i = 0; i < 6; ++i) load8v(rp + i * src_pitch, v[i]);
            } else {
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    if (iw0 + i >= 0 && iw0 + i < iw_n)
                        load8v(rp + i * src_pitch, v[i]);
                    else
#pragma unroll
                        for (int c = 0; c < 8; ++c) v[i][c] = 0.0f;
                }
            }
            float w[3][8];
#pragma unroll
            for (int s = 0; s < 3; ++s) {
                const float4* wp = reinterpret_cast<const float4*>(sw + (r * 3 + s) * cb + cvi * 8);
                const float4 w0 = wp[0], w1 = wp[1];
                w[s][0] = w0.x; w[s][1] = w0.y; w[s][2] = w0.z; w[s][3] = w0.w;
                w[s][4] = w1.x; w[s][5] = w1.y; w[s][6] = w1.z; w[s][7] = w1.w;
            }
            // taps in (r, s) order per output, as the reference accumulates
#pragma unroll
            for (int s = 0; s < 3; ++s)
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int c = 0; c < 8; ++c) acc[j][c] += v[BWD ? j + 2 - s : j + s][c] * w[s][c];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int ow = ow0 + j;
            if (ow >= ow_n) break;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                if (cc + c >= kmax)
                    acc[j][c] = 0.0f;
                else if (epi)
                    acc[j][c] = apply_epilogue(e, acc[j][c], cc + c, oh, ow, g.p, g.q);
            }
            store8v(dst + ((size_t)row * ow_n + ow) * pitch + cc, acc[j]);
        }
    }
}

// Backward weights, pass 1: CTA (chunk, channel block) sums dY * x over its
// slice of output pixels for a group of up to kTapGroup taps, lanes of equal
// channel vector combined by shuffles, warps in fixed order through smem;
// partial[chunk][tap][c] (fp32, channel pitch).
template <typename T, bool K3>
__global__ void __launch_bounds__(kThreads) depthwise_wgrad_kernel(pk_conv_geom g, const T* __restrict__ dy,
                                                                   const T* __restrict__ x,
                                                                   float* __restrict__ partial) {
    __shared__ float red[kThreads / 32][kTapGroup][64];
    const int cb = dw_block_channels(g.x_pitch), cv = cb / 8, lanes_px = kThreads / cv;
    const int c0 = blockIdx.y * cb, cvi = threadIdx.x % cv, pl = threadIdx.x / cv, cc = c0 + cvi * 8;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, taps = K3 ? 9 : g.r * g.s;
    // chunk = a contiguous range of output rows (n, oh)
    const int rows = g.n * g.p;
    const int per = (rows + gridDim.x - 1) / gridDim.x;
    const int r0 = blockIdx.x * per, r1 = r0 + per < rows ? r0 + per : rows;
    for (int t0 = 0; t0 < taps; t0 += kTapGroup) {
        float acc[kTapGroup][8];
#pragma unroll
        for (int t = 0; t < kTapGroup; ++t)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[t][j] = 0.0f;
        for (int row = r0; row < r1; ++row) {
          const int oh = row % g.p, n = row / g.p;
          for (int ow = pl; ow < g.q; ow += lanes_px) {
            const long long pix = (long long)row * g.q + ow;
            float d[8];
            load8v(dy + (size_t)pix * g.y_pitch + cc, d);
            const T* xn = x + (size_t)n * g.h * g.w * g.x_pitch + cc;
            if (K3) {
                const int ih0 = oh * g.str_h - g.pad_h, iw0 = ow * g.str_w - g.pad_w;
                const int lh = 2 * g.dil_h, lw = 2 * g.dil_w;
                if (ih0 >= 0 && ih0 + lh < g.h && iw0 >= 0 && iw0 + lw < g.w) {
                    // interior pixel: all 9 taps in range, 32-bit offsets from one base
                    const T* xb = xn + (ih0 * g.w + iw0) * g.x_pitch;
                    const int dr = g.dil_h * g.w * g.x_pitch, ds = g.dil_w * g.x_pitch;
                    float v[9][8];
#pragma unroll
                    for (int t = 0; t < 9; ++t) load8v(xb + (t / 3) * dr + (t % 3) * ds, v[t]);
#pragma unroll
                    for (int t = 0; t < 9; ++t)
#pragma unroll
                        for (int j = 0; j < 8; ++j) acc[t][j] += d[j] * v[t][j];
                    continue;
                }
            }
#pragma unroll
            for (int t = 0; t < kTapGroup; ++t) {
                const int tap = t0 + t;
                if (tap >= taps) break;
                const int gs = K3 ? 3 : g.s, r = tap / gs, s = tap - r * gs;
                const int ih = oh * g.str_h - g.pad_h + r * g.dil_h, iw = ow * g.str_w - g.pad_w + s * g.dil_w;
                if (ih < 0 || ih >= g.h || iw < 0 || iw >= g.w) continue;
                float v[8];
                load8v(xn + ((size_t)ih * g.w + iw) * g.x_pitch, v);
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[t][j] += d[j] * v[j];
            }
          }
        }
        // lanes cvi, cvi + cv, ... of a warp hold the same channels
#pragma unroll
        for (int t = 0; t < kTapGroup; ++t)
#pragma unroll
            for (int j = 0; j < 8; ++j)
                for (int o = cv; o < 32; o <<= 1) acc[t][j] += __shfl_xor_sync(0xffffffffu, acc[t][j], o);
        if (lane < cv)
#pragma unroll
            for (int t = 0; t < kTapGroup; ++t)
#pragma unroll
                for (int j = 0; j < 8; ++j) red[warp][t][lane * 8 + j] = acc[t][j];
        __syncthreads();
        for (int i = threadIdx.x; i < kTapGroup * cb; i += kThreads) {
            const int t = i / cb, c = i % cb;
            if (t0 + t < taps) {
                float sum = 0.0f;
#pragma unroll
                for (int w = 0; w < kThreads / 32; ++w) sum += red[w][t][c];
                partial[((size_t)blockIdx.x * taps + t0 + t) * g.x_pitch + c0 + c] = sum;
            }
        }
        __syncthreads();
    }
}

// Backward weights, pass 2: dw[c][tap][0] = sum over chunks in order; the
// filter's pad lanes (1 .. f_pitch-1) are written as zero.
template <typename T>
__global__ void depthwise_wgrad_sum_kernel(pk_conv_geom g, const float* __restrict__ partial, int chunks,
                                           T* __restrict__ dw) {
    const int taps = g.r * g.s;
    const long long total = (long long)taps * g.x_pitch;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % g.x_pitch), tap = (int)(i / g.x_pitch);
        if (c >= g.k) continue;
        float sum = 0.0f;
        for (int ch = 0; ch < chunks; ++ch) sum += partial[(size_t)ch * total + i];
        T* out = dw + ((size_t)c * taps + tap) * g.f_pitch;
        st(out, sum);
        for (int l = 1; l < g.f_pitch; ++l) st(out + l, 0.0f);
    }
}

int dw_chunks(const pk_conv_geom* g, int num_sms) {
    const int cblocks = g->x_pitch / dw_block_channels(g->x_pitch);
    const long long want = (2LL * num_sms + cblocks - 1) / cblocks;
    const long long rows = (long long)g->n * g->p;
    return (int)std::max(1LL, std::min(want, rows));  // chunks hold whole output rows
}

// Grouped forward / backward data (C/g and K/g multiples of 8). A thread owns
// 8 consecutive output channels (k forward, c backward data) of one pixel;
// the 32 lanes of a warp are 32 pixels with the same channel vector, so the
// filter rows in shared memory ([tap][j][64 channels], j = reduction index
// within the group) are broadcast reads, and each lane streams its pixel's
// group channels as 8-channel vectors. Reduction in (r, s, j) order.
template <typename T, bool BWD>
__global__ void __launch_bounds__(kThreads) grouped_kernel(pk_conv_geom g, const T* __restrict__ src,
                                                           const T* __restrict__ f, T* __restrict__ dst,
                                                           pk_epilogue e) {
    extern __shared__ float sw[];
    const int taps = g.r * g.s;
    const int red = BWD ? g.kg : g.cg;             // reduction channels per group
    const int och = BWD ? g.cg : g.kg;             // output channels per group
    const int nout = BWD ? g.c : g.k;
    const int pitch = BWD ? g.x_pitch : g.y_pitch, src_pitch = BWD ? g.y_pitch : g.x_pitch;
    const int o0 = blockIdx.y * 64;
    for (int i = threadIdx.x; i < taps * red * 64; i += blockDim.x) {
        const int oo = i % 64, j = (i / 64) % red, tap = i / (64 * red);
        const int o = o0 + oo;
        float v = 0.0f;
        if (o < nout) {
            const int grp = o / och;
            if (!BWD)
                v = ld(f + ((size_t)o * taps + tap) * g.f_pitch + j);
            else
                v = ld(f + ((size_t)(grp * g.kg + j) * taps + tap) * g.f_pitch + (o - grp * g.cg));
        }
        sw[i] = v;
    }
    __syncthreads();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int oc = o0 + warp * 8;  // this warp's 8 output channels
    if (oc >= nout) return;
    const int grp = oc / och;
    const int oh_n = BWD ? g.h : g.p, ow_n = BWD ? g.w : g.q;
    const int ih_n = BWD ? g.p : g.h, iw_n = BWD ? g.q : g.w;
    const long long npix = (long long)g.n * oh_n * ow_n;
    const bool epi = !BWD && epilogue_active(&e);
    for (long long pix = (long long)blockIdx.x * 32 + lane; pix < npix; pix += (long long)gridDim.x * 32) {
        const int ow = (int)(pix % ow_n);
        const long long t = pix / ow_n;
        const int oh = (int)(t % oh_n), n = (int)(t / oh_n);
        const T* sn = src + (size_t)n * ih_n * iw_n * src_pitch + grp * red;
        float acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
        for (int r = 0; r < g.r; ++r) {
            int ih;
            if (!BWD) {
                ih = oh * g.str_h - g.pad_h + r * g.dil_h;
                if (ih < 0 || ih >= ih_n) continue;
            } else {
                const int num = oh + g.pad_h - r * g.dil_h;
                if (num < 0 || num % g.str_h) continue;
                ih = num / g.str_h;
                if (ih >= ih_n) continue;
            }
            for (int s = 0; s < g.s; ++s) {
                int iw;
                if (!BWD) {
                    iw = ow * g.str_w - g.pad_w + s * g.dil_w;
                    if (iw < 0 || iw >= iw_n) continue;
                } else {
                    const int num = ow + g.pad_w - s * g.dil_w;
                    if (num < 0 || num % g.str_w) continue;
                    iw = num / g.str_w;
                    if (iw >= iw_n) continue;
                }
                const T* xp = sn + (size_t)(ih * iw_n + iw) * src_pitch;
                const float* wt = sw + (r * g.s + s) * red * 64 + warp * 8;
                for (int j0 = 0; j0 < red; j0 += 8) {
                    float v[8];
                    load8v(xp + j0, v);
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        const float4 w0 = *reinterpret_cast<const float4*>(wt + (j0 + jj) * 64);
                        const float4 w1 = *reinterpret_cast<const float4*>(wt + (j0 + jj) * 64 + 4);
                        acc[0] += v[jj] * w0.x; acc[1] += v[jj] * w0.y; acc[2] += v[jj] * w0.z;
                        acc[3] += v[jj] * w0.w; acc[4] += v[jj] * w1.x; acc[5] += v[jj] * w1.y;
                        acc[6] += v[jj] * w1.z; acc[7] += v[jj] * w1.w;
                    }
                }
            }
        }
        if (epi)
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = apply_epilogue(e, acc[q], oc + q, oh, ow, g.p, g.q);
        store8v(dst + (size_t)pix * pitch + oc, acc);
    }
}

// Grouped backward weights (1 < C/g <= 32, C/g % 8 == 0, 64-channel K blocks
// aligned to groups): dW[k][r][s][c] = sum_pix dY[pix][k] * x[pix(r,s)][grp*cg + c].
// A thread owns one output channel k and 8 input channels of its group and
// accumulates up to kTapGroup taps over its slice of output rows; lanes of a
// warp are consecutive k (coalesced dY, broadcast x vectors within a group).
// Each thread's partial goes to partial[slot][k][tap][c] (slot = chunk x pixel
// lane); the fixed-order slot sum makes the result deterministic.
template <typename T>
__global__ void __launch_bounds__(kThreads) grouped_wgrad_kernel(pk_conv_geom g, const T* __restrict__ dy,
                                                                 const T* __restrict__ x,
                                                                 float* __restrict__ partial) {
    const int cvs = g.cg / 8, lanes_px = kThreads / (64 * cvs);
    const int kk = threadIdx.x % 64, rest = threadIdx.x / 64, cvi = rest % cvs, pl = rest / cvs;
    const int k = blockIdx.y * 64 + kk, grp = k / g.kg, taps = g.r * g.s;
    const int rows = g.n * g.p;
    const int per = (rows + gridDim.x - 1) / gridDim.x;
    const int r0 = blockIdx.x * per, r1 = r0 + per < rows ? r0 + per : rows;
    const int slot = blockIdx.x * lanes_px + pl;
    for (int t0 = 0; t0 < taps; t0 += kTapGroup) {
        float acc[kTapGroup][8];
#pragma unroll
        for (int t = 0; t < kTapGroup; ++t)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[t][j] = 0.0f;
        for (int row = r0; row < r1; ++row) {
            const int oh = row % g.p, n = row / g.p;
            const T* xn = x + (size_t)n * g.h * g.w * g.x_pitch + grp * g.cg + cvi * 8;
            for (int ow = pl; ow < g.q; ow += lanes_px) {
                const float d = ld(dy + ((size_t)row * g.q + ow) * g.y_pitch + k);
                if (taps == 9 && g.s == 3) {
                    const int ih0 = oh * g.str_h - g.pad_h, iw0 = ow * g.str_w - g.pad_w;
                    if (ih0 >= 0 && ih0 + 2 * g.dil_h < g.h && iw0 >= 0 && iw0 + 2 * g.dil_w < g.w) {
                        // interior pixel of a 3x3 filter: 9 loads from one base, no checks
                        const T* xb = xn + (ih0 * g.w + iw0) * g.x_pitch;
                        const int dr = g.dil_h * g.w * g.x_pitch, ds = g.dil_w * g.x_pitch;
                        float v[9][8];
#pragma unroll
                        for (int t = 0; t < 9; ++t) load8v(xb + (t / 3) * dr + (t % 3) * ds, v[t]);
#pragma unroll
                        for (int t = 0; t < 9; ++t)
#pragma unroll
                            for (int j = 0; j < 8; ++j) acc[t][j] += d * v[t][j];
                        continue;
                    }
                }
#pragma unroll
                for (int t = 0; t < kTapGroup; ++t) {
                    const int tap = t0 + t;
                    if (tap >= taps) break;
                    const int r = tap / g.s, s = tap - r * g.s;
                    const int ih = oh * g.str_h - g.pad_h + r * g.dil_h, iw = ow * g.str_w - g.pad_w + s * g.dil_w;
                    if (ih < 0 || ih >= g.h || iw < 0 || iw >= g.w) continue;
                    float v[8];
                    load8v(xn + (ih * g.w + iw) * g.x_pitch, v);
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[t][j] += d * v[j];
                }
            }
        }
#pragma unroll
        for (int t = 0; t < kTapGroup; ++t) {
            if (t0 + t >= taps) break;
            float* out = partial + (((size_t)slot * g.k + k) * taps + t0 + t) * g.cg + cvi * 8;
            reinterpret_cast<float4*>(out)[0] = make_float4(acc[t][0], acc[t][1], acc[t][2], acc[t][3]);
            reinterpret_cast<float4*>(out)[1] = make_float4(acc[t][4], acc[t][5], acc[t][6], acc[t][7]);
        }
    }
}

template <typename T>
__global__ void grouped_wgrad_sum_kernel(pk_conv_geom g, const float* __restrict__ partial, int slots,
                                         T* __restrict__ dw) {
    const long long total = (long long)g.k * g.r * g.s * g.cg;  // f_pitch == cg here
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        float sum = 0.0f;
        for (int sl = 0; sl < slots; ++sl) sum += partial[(size_t)sl * total + i];
        st(dw + i, sum);
    }
}

int gw_chunks(const pk_conv_geom* g, int num_sms) {
    const int kblocks = g->k / 64;
    const long long want = (2LL * num_sms + kblocks - 1) / kblocks;
    return (int)std::max(1LL, std::min(want, (long long)g->n * g->p));
}

}  // namespace
}  // namespace pk

using namespace pk;

extern "C" {

int pk_depthwise_supported(const pk_conv_geom* g) {
    return g->groups == g->c && g->c == g->k && g->cg == 1 && g->kg == 1 && !g->transpose &&
           g->x_pitch == g->y_pitch && g->x_pitch % 8 == 0 &&
           (long long)g->r * g->s * dw_block_channels(g->x_pitch) * 4 <= 48 * 1024 &&
           (long long)g->n * std::max(g->h, g->p) * std::max(g->w, g->q) < (1LL << 31) &&  // 32-bit units
           (long long)std::max(g->h, g->p) * std::max(g->w, g->q) * g->x_pitch < (1LL << 31);
}

cudaError_t pk_cuda_depthwise_fwd(const pk_conv_geom* g, int dtype, const void* x, const void* f, void* y,
                                  const pk_epilogue* epi, int num_sms, cudaStream_t st) {
    pk_epilogue none{};
    none.act = -1;
    const pk_epilogue e = epi ? *epi : none;
    const int cb = dw_block_channels(g->y_pitch);
    const long long lanes = kThreads / (cb / 8);
    const long long units = (long long)g->n * g->p * ceil_div(g->q, lanes);
    const int cblocks = g->y_pitch / cb;
    const long long want = (long long)num_sms * 8 / cblocks + 1;
    dim3 grid((unsigned)std::max(1LL, std::min(units, want)), cblocks);
    const size_t smem = (size_t)g->r * g->s * cb * sizeof(float);
    const bool k3 = g->r == 3 && g->s == 3;
    if (k3 && g->str_h == 1 && g->str_w == 1 && g->dil_h == 1 && g->dil_w == 1) {
        const long long quads = (long long)g->n * g->p * ((g->q + 3) / 4);
        dim3 grid4((unsigned)std::max(1LL, std::min((long long)ceil_div(quads, lanes), want)), cblocks);
        PK_DISPATCH_DTYPE(dtype, T,
                          depthwise3_s1_kernel<T, false><<<grid4, kThreads, smem, st>>>(*g, (const T*)x,
                                                                                        (const T*)f, (T*)y, e));
        count_launch();
        return cudaGetLastError();
    }
    PK_DISPATCH_DTYPE(dtype, T, {
        if (k3)
            depthwise_kernel<T, false, true><<<grid, kThreads, smem, st>>>(*g, (const T*)x, (const T*)f, (T*)y, e);
        else
            depthwise_kernel<T, false, false><<<grid, kThreads, smem, st>>>(*g, (const T*)x, (const T*)f, (T*)y, e);
    });
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_depthwise_bwd_data(const pk_conv_geom* g, int dtype, const void* dy, const void* f,
                                       void* dx, int num_sms, cudaStream_t st) {
    pk_epilogue none{};
    none.act = -1;
    const int cb = dw_block_channels(g->x_pitch);
    const long long lanes = kThreads / (cb / 8);
    const long long units = (long long)g->n * g->h * ceil_div(g->w, lanes);
    const int cblocks = g->x_pitch / cb;
    const long long want = (long long)num_sms * 8 / cblocks + 1;
    dim3 grid((unsigned)std::max(1LL, std::min(units, want)), cblocks);
    const size_t smem = (size_t)g->r * g->s * cb * sizeof(float);
    const bool k3 = g->r == 3 && g->s == 3;
    if (k3 && g->str_h == 1 && g->str_w == 1 && g->dil_h == 1 && g->dil_w == 1) {
        const long long quads = (long long)g->n * g->h * ((g->w + 3) / 4);
        dim3 grid4((unsigned)std::max(1LL, std::min((long long)ceil_div(quads, lanes), want)), cblocks);
        PK_DISPATCH_DTYPE(dtype, T,
                          depthwise3_s1_kernel<T, true><<<grid4, kThreads, smem, st>>>(*g, (const T*)dy,
                                                                                       (const T*)f, (T*)dx, none));
        count_launch();
        return cudaGetLastError();
    }
    PK_DISPATCH_DTYPE(dtype, T, {
        if (k3)
            depthwise_kernel<T, true, true><<<grid, kThreads, smem, st>>>(*g, (const T*)dy, (const T*)f, (T*)dx, none);
        else
            depthwise_kernel<T, true, false><<<grid, kThreads, smem, st>>>(*g, (const T*)dy, (const T*)f, (T*)dx,
                                                                           none);
    });
    count_launch();
    return cudaGetLastError();
}

size_t pk_depthwise_wgrad_workspace(const pk_conv_geom* g, int num_sms) {
    return (size_t)dw_chunks(g, num_sms) * g->r * g->s * g->x_pitch * sizeof(float);
}

cudaError_t pk_cuda_depthwise_wgrad(const pk_conv_geom* g, int dtype, const void* dy, const void* x, void* dw,
                                    void* ws, size_t ws_bytes, int num_sms, cudaStream_t st) {
    const int chunks = dw_chunks(g, num_sms);
    if (ws_bytes < pk_depthwise_wgrad_workspace(g, num_sms)) return cudaErrorInvalidValue;
    const int cblocks = g->x_pitch / dw_block_channels(g->x_pitch);
    const long long total = (long long)g->r * g->s * g->x_pitch;
    PK_DISPATCH_DTYPE(dtype, T, {
        if (g->r == 3 && g->s == 3)
            depthwise_wgrad_kernel<T, true><<<dim3(chunks, cblocks), kThreads, 0, st>>>(*g, (const T*)dy,
                                                                                      (const T*)x, (float*)ws);
        else
            depthwise_wgrad_kernel<T, false><<<dim3(chunks, cblocks), kThreads, 0, st>>>(*g, (const T*)dy,
                                                                                       (const T*)x, (float*)ws);
        depthwise_wgrad_sum_kernel<T><<<(unsigned)std::max(1LL, std::min((long long)ceil_div(total, 256), 4LL * num_sms)),
                                        256, 0, st>>>(*g, (const float*)ws, chunks, (T*)dw);
    });
    count_launch(2);
    return cudaGetLastError();
}

}  // extern "C"

extern "C" {

int pk_grouped_wgrad_supported(const pk_conv_geom* g) {
    return g->groups > 1 && !g->transpose && (g->cg == 8 || g->cg == 16 || g->cg == 32) && g->k % 64 == 0 &&
           (64 % g->kg == 0 || g->kg % 64 == 0) && g->f_pitch == g->cg && g->x_pitch == g->c &&
           (long long)g->h * g->w * g->x_pitch < (1LL << 31) && (long long)g->n * g->p < (1LL << 31);
}

size_t pk_grouped_wgrad_workspace(const pk_conv_geom* g, int num_sms) {
    const int lanes_px = kThreads / (64 * (g->cg / 8));
    return (size_t)gw_chunks(g, num_sms) * lanes_px * g->k * g->r * g->s * g->cg * sizeof(float);
}

cudaError_t pk_cuda_grouped_wgrad(const pk_conv_geom* g, int dtype, const void* dy, const void* x, void* dw,
                                  void* ws, size_t ws_bytes, int num_sms, cudaStream_t st) {
    if (!pk_grouped_wgrad_supported(g) || ws_bytes < pk_grouped_wgrad_workspace(g, num_sms))
        return cudaErrorInvalidValue;
    const int chunks = gw_chunks(g, num_sms), lanes_px = kThreads / (64 * (g->cg / 8));
    const long long total = (long long)g->k * g->r * g->s * g->cg;
    PK_DISPATCH_DTYPE(dtype, T, {
        grouped_wgrad_kernel<T><<<dim3(chunks, g->k / 64), kThreads, 0, st>>>(*g, (const T*)dy, (const T*)x,
                                                                              (float*)ws);
        grouped_wgrad_sum_kernel<T><<<(unsigned)std::max(1LL, std::min((long long)ceil_div(total, 256),
                                                                       4LL * num_sms)),
                                      256, 0, st>>>(*g, (const float*)ws, chunks * lanes_px, (T*)dw);
    });
    count_launch(2);
    return cudaGetLastError();
}

}  // extern "C"

extern "C" {

int pk_grouped_supported(const pk_conv_geom* g) {
    return g->groups > 1 && !g->transpose && g->cg % 8 == 0 && g->kg % 8 == 0 && g->x_pitch == g->c &&
           g->y_pitch == g->k && g->f_pitch == g->cg &&
           (long long)g->r * g->s * std::max(g->cg, g->kg) * 64 * 4 <= 160 * 1024 &&
           (long long)std::max(g->h, g->p) * std::max(g->w, g->q) * std::max(g->x_pitch, g->y_pitch) < (1LL << 31);
}

static cudaError_t grouped_launch(const pk_conv_geom* g, int dtype, bool bwd, const void* src, const void* f,
                                  void* dst, const pk_epilogue& e, int num_sms, cudaStream_t st) {
    const int nout = bwd ? g->c : g->k, red = bwd ? g->kg : g->cg;
    const long long npix = (long long)g->n * (bwd ? (long long)g->h * g->w : (long long)g->p * g->q);
    const int oblocks = (nout + 63) / 64;
    const long long want = (long long)num_sms * 4 / oblocks + 1;
    dim3 grid((unsigned)std::max(1LL, std::min((long long)ceil_div(npix, 32), want)), oblocks);
    const size_t smem = (size_t)g->r * g->s * red * 64 * sizeof(float);
    PK_DISPATCH_DTYPE(dtype, T, {
        auto kern = bwd ? grouped_kernel<T, true> : grouped_kernel<T, false>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, kThreads, smem, st>>>(*g, (const T*)src, (const T*)f, (T*)dst, e);
    });
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_grouped_fwd(const pk_conv_geom* g, int dtype, const void* x, const void* f, void* y,
                                const pk_epilogue* epi, int num_sms, cudaStream_t st) {
    pk_epilogue none{};
    none.act = -1;
    return grouped_launch(g, dtype, false, x, f, y, epi ? *epi : none, num_sms, st);
}

cudaError_t pk_cuda_grouped_bwd_data(const pk_conv_geom* g, int dtype, const void* dy, const void* f, void* dx,
                                     int num_sms, cudaStream_t st) {
    pk_epilogue none{};
    none.act = -1;
    return grouped_launch(g, dtype, true, dy, f, dx, none, num_sms, st);
}

}  // extern "C"
