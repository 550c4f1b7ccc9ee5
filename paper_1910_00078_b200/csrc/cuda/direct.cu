// Direct convolution on CUDA cores (fp32 FMA), NHWC.
//
// Device counterpart of the reference's Direct algorithm
// (proj/src/core/conv.cpp:99-173 forward / transpose, :716-756 backward data,
// :816-850 backward weights). Same arithmetic (fp32 accumulate of x*w over
// (c, y, x) with zero padding, groups, dilation), different schedule: lanes of
// a warp own consecutive output pixels and share the filter taps, which are
// warp-uniform loads served from L1.
#include "common.cuh"

namespace pk {

// Forward / transpose-forward: thread = (output pixel, KT consecutive output
// channels of one group).
template <typename T, int KT>
__global__ void __launch_bounds__(128) direct_fwd_kernel(pk_conv_geom g, const T* __restrict__ x,
                                                         const T* __restrict__ f,
                                                         T* __restrict__ y, pk_epilogue e) {
    const long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long npix = (long long)g.n * g.p * g.q;
    const int k0 = blockIdx.y * KT;
    if (pix >= npix || k0 >= g.k) return;
    const int ow = (int)(pix % g.q);
    const int oh = (int)((pix / g.q) % g.p);
    const int n = (int)(pix / ((long long)g.q * g.p));
    const int grp = k0 / g.kg;
    float acc[KT];
#pragma unroll
    for (int j = 0; j < KT; ++j) acc[j] = 0.0f;
    const T* xn = x + (size_t)n * g.h * g.w * g.x_pitch + grp * g.cg;
    for (int r = 0; r < g.r; ++r) {
        int ih;
        if (!g.transpose) {
            ih = oh * g.str_h - g.pad_h + r * g.dil_h;
            if (ih < 0 || ih >= g.h) continue;
        } else {
            const int num = oh + g.pad_h - r;
            if (num < 0 || num % g.str_h) continue;
            ih = num / g.str_h;
            if (ih >= g.h) continue;
        }
        for (int s = 0; s < g.s; ++s) {
            int iw;
            if (!g.transpose) {
                iw = ow * g.str_w - g.pad_w + s * g.dil_w;
                if (iw < 0 || iw >= g.w) continue;
            } else {
                const int num = ow + g.pad_w - s;
                if (num < 0 || num % g.str_w) continue;
                iw = num / g.str_w;
                if (iw >= g.w) continue;
            }
            const T* xp = xn + ((size_t)ih * g.w + iw) * g.x_pitch;
            for (int c = 0; c < g.cg; ++c) {
                const float xv = ld(xp + c);
#pragma unroll
                for (int j = 0; j < KT; ++j) {
                    const int k = k0 + j;
                    if (k >= g.k) break;
                    size_t fi;
                    if (!g.transpose)
                        fi = (((size_t)k * g.r + r) * g.s + s) * g.f_pitch + c;
                    else  // transpose filter [C][R][S][pitch(kg)]
                        fi = ((((size_t)grp * g.cg + c) * g.r + r) * g.s + s) * g.f_pitch +
                             (k - grp * g.kg);
                    acc[j] += xv * ld(f + fi);
                }
            }
        }
    }
    T* yp = y + (size_t)pix * g.y_pitch;
    const bool epi = epilogue_active(&e);
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        const int k = k0 + j;
        if (k >= g.k) break;
        st(yp + k, epi ? apply_epilogue(e, acc[j], k, oh, ow, g.p, g.q) : acc[j]);
    }
}

// 8 consecutive channels as fp32 (one 32-byte f32 / 16-byte bf16 vector load).
__device__ __forceinline__ void load8(const float* p, float (&v)[8]) {
    const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&v)[8]) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 f = __bfloat1622float2(h[i]);
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
    }
}

// Forward, register-tiled (groups == 1, convolution mode): a CTA computes 64
// output pixels x 64 output channels; per filter tap and 16-channel chunk the
// zero-padded input slice [16 c][64 px] and the filter slice [16 c][64 k] are
// staged in shared memory and every thread accumulates an 8 px x 4 k block
// (32 FMA per 3 vector shared loads). Same products as the reference Direct
// loop (conv.cpp:99-133), summed tap-major in fp32. Channel pad lanes of the
// NHWC / filter pitch are zero by the layout contract, so 8-channel vectors
// never need a channel mask.
template <typename T>
__global__ void __launch_bounds__(128) direct_fwd_tiled_kernel(pk_conv_geom g,
                                                               const T* __restrict__ x,
                                                               const T* __restrict__ f,
                                                               T* __restrict__ y, pk_epilogue e) {
    constexpr int TP = 64, TK = 64, CC = 16, LD = TP + 4;
    __shared__ __align__(16) float As[CC][LD];  // [channel][pixel]
    __shared__ __align__(16) float Bs[CC][LD];  // [channel][output channel]
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const long long npix = (long long)g.n * g.p * g.q;
    const long long px0 = blockIdx.x * (long long)TP;
    const int k0 = blockIdx.y * TK;
    // loaders: thread -> (pixel / output channel tid & 63, channel half tid >> 6)
    const int lp = tid & 63, lh = tid >> 6;
    const long long pix = px0 + lp;
    const bool pv = pix < npix;
    int ln = 0, loh = 0, low = 0;
    if (pv) {
        low = (int)(pix % g.q);
        loh = (int)((pix / g.q) % g.p);
        ln = (int)(pix / ((long long)g.q * g.p));
    }
    const int bk = k0 + lp;
    const bool kv = bk < g.k;
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    for (int r = 0; r < g.r; ++r) {
        const int ih = loh * g.str_h - g.pad_h + r * g.dil_h;
        for (int s = 0; s < g.s; ++s) {
            const int iw = low * g.str_w - g.pad_w + s * g.dil_w;
            const bool ok = pv && ih >= 0 && ih < g.h && iw >= 0 && iw < g.w;
            const T* xp = x + (((size_t)ln * g.h + ih) * g.w + iw) * g.x_pitch;
            const T* fp = f + (((size_t)(kv ? bk : 0) * g.r + r) * g.s + s) * g.f_pitch;
            for (int c0 = 0; c0 < g.cg; c0 += CC) {
                const int cb = c0 + lh * 8;
                float av[8], bv[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) av[i] = bv[i] = 0.0f;
                if (ok && cb < g.x_pitch) load8(xp + cb, av);
                if (kv && cb < g.f_pitch) load8(fp + cb, bv);
                __syncthreads();  // the previous chunk is consumed
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    As[lh * 8 + i][lp] = av[i];
                    Bs[lh * 8 + i][lp] = bv[i];
                }
                __syncthreads();
#pragma unroll
                for (int c = 0; c < CC; ++c) {
                    const float4 a0 = *reinterpret_cast<const float4*>(&As[c][ty * 8]);
                    const float4 a1 = *reinterpret_cast<const float4*>(&As[c][ty * 8 + 4]);
                    const float4 b = *reinterpret_cast<const float4*>(&Bs[c][tx * 4]);
                    const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                    const float bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                    for (int i = 0; i < 8; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
                }
            }
        }
    }
    const bool epi = epilogue_active(&e);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const long long p = px0 + ty * 8 + i;
        if (p >= npix) break;
        const int ow = (int)(p % g.q), oh = (int)((p / g.q) % g.p);
        T* yp = y + (size_t)p * g.y_pitch;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int k = k0 + tx * 4 + j;
            if (k < g.k) st(yp + k, epi ? apply_epilogue(e, acc[i][j], k, oh, ow, g.p, g.q) : acc[i][j]);
        }
    }
}

// Backward data: thread = (input pixel, CT consecutive input channels of one
// group), gathering over the output positions that read it.
template <typename T, int CT>
__global__ void __launch_bounds__(128) direct_bwd_data_kernel(pk_conv_geom g,
                                                              const T* __restrict__ dy,
                                                              const T* __restrict__ f,
                                                              T* __restrict__ dx) {
    const long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long npix = (long long)g.n * g.h * g.w;
    const int c0 = blockIdx.y * CT;
    if (pix >= npix || c0 >= g.c) return;
    const int iw = (int)(pix % g.w);
    const int ih = (int)((pix / g.w) % g.h);
    const int n = (int)(pix / ((long long)g.w * g.h));
    const int grp = c0 / g.cg;
    const int cl0 = c0 - grp * g.cg;
    float acc[CT];
#pragma unroll
    for (int j = 0; j < CT; ++j) acc[j] = 0.0f;
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
            const T* dyp = dy + (((size_t)n * g.p + oh) * g.q + ow) * g.y_pitch + grp * g.kg;
            for (int kk = 0; kk < g.kg; ++kk) {
                const float dv = ld(dyp + kk);
                const T* fp = f + (((size_t)(grp * g.kg + kk) * g.r + r) * g.s + s) * g.f_pitch;
#pragma unroll
                for (int j = 0; j < CT; ++j)
                    if (cl0 + j < g.cg) acc[j] += dv * ld(fp + cl0 + j);
            }
        }
    }
    T* dxp = dx + (size_t)pix * g.x_pitch;
#pragma unroll
    for (int j = 0; j < CT; ++j)
        if (cl0 + j < g.cg) st(dxp + c0 + j, acc[j]);
}

// Backward weights: block = (k, r, s, 32-channel slice); 8 warps split the
// (n, p, q) reduction, lane = channel; fixed-order smem combine, so the result
// is deterministic.
template <typename T>
__global__ void __launch_bounds__(256) direct_bwd_weights_kernel(pk_conv_geom g,
                                                                 const T* __restrict__ dy,
                                                                 const T* __restrict__ x,
                                                                 T* __restrict__ dw) {
    __shared__ float part[8][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cslices = (g.cg + 31) / 32;
    int b = blockIdx.x;
    const int cs = b % cslices;
    b /= cslices;
    const int s = b % g.s;
    b /= g.s;
    const int r = b % g.r;
    const int k = b / g.r;
    const int grp = k / g.kg;
    const int c = cs * 32 + lane;
    float acc = 0.0f;
    const long long npq = (long long)g.n * g.p * g.q;
    if (c < g.cg) {
        for (long long i = warp; i < npq; i += 8) {
            const int ow = (int)(i % g.q);
            const int oh = (int)((i / g.q) % g.p);
            const int n = (int)(i / ((long long)g.q * g.p));
            const int ih = oh * g.str_h - g.pad_h + r * g.dil_h;
            const int iw = ow * g.str_w - g.pad_w + s * g.dil_w;
            if (ih < 0 || ih >= g.h || iw < 0 || iw >= g.w) continue;
            acc += ld(dy + (size_t)i * g.y_pitch + k) *
                   ld(x + (((size_t)n * g.h + ih) * g.w + iw) * g.x_pitch + grp * g.cg + c);
        }
    }
    part[warp][lane] = acc;
    __syncthreads();
    if (warp == 0) {
        float t = 0.0f;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += part[w][lane];
        T* out = dw + (((size_t)k * g.r + r) * g.s + s) * g.f_pitch;
        if (c < g.cg)
            st(out + c, t);
        else if (c < g.f_pitch)
            st(out + c, 0.0f);  // keep the zero pad lanes defined
    }
}

// Backward data, register-tiled (groups == 1, convolution mode): a CTA owns 64
// input pixels x 64 input channels; per filter tap and 16-channel k chunk the
// gathered dY slice [16 k][64 px] (zero where the tap does not land on an
// output position) and the filter rows [16 k][64 c] are staged in smem and
// each thread accumulates 8 px x 4 c. Taps in (r, s) order, k ascending.
template <typename T>
__global__ void __launch_bounds__(128) direct_dgrad_tiled_kernel(pk_conv_geom g, const T* __restrict__ dy,
                                                                 const T* __restrict__ f, T* __restrict__ dx) {
    constexpr int TP = 64, TC = 64, KC = 16, LD = TP + 4;
    __shared__ __align__(16) float As[KC][LD];  // [k][pixel]
    __shared__ __align__(16) float Bs[KC][LD];  // [k][channel]
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    // stride phases: a CTA's pixels share (ih mod str_h, iw mod str_w), so a tap
    // lands for all of them or for none, and missing taps are skipped whole
    const int ph_h = blockIdx.z / g.str_w, ph_w = blockIdx.z % g.str_w;
    const int hp = (g.h - ph_h + g.str_h - 1) / g.str_h, wp = (g.w - ph_w + g.str_w - 1) / g.str_w;
    const int npix = g.n * hp * wp;  // pixels of this phase
    const int px0 = blockIdx.x * TP, c0 = blockIdx.y * TC;
    if (px0 >= npix) return;
    const int lp = tid & 63, lh = tid >> 6;          // dY loader: pixel, k half
    const int bk = tid >> 3, bc = (tid & 7) * 8;     // filter loader: k row, 8-channel vector
    const int pix = px0 + lp;
    const bool pv = pix < npix;
    int ln = 0, lih = 0, liw = 0;
    if (pv) {
        liw = ph_w + (pix % wp) * g.str_w;
        const int t = pix / wp;
        lih = ph_h + (t % hp) * g.str_h;
        ln = t / hp;
    }
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    for (int r = 0; r < g.r; ++r) {
        if (g.str_h > 1 && ((ph_h + g.pad_h - r * g.dil_h) % g.str_h + g.str_h) % g.str_h)
            continue;  // tap misses the phase
        const int nh = lih + g.pad_h - r * g.dil_h;
        const int oh = nh / g.str_h;
        const bool hv = nh >= 0 && nh % g.str_h == 0 && oh < g.p;
        for (int s = 0; s < g.s; ++s) {
            if (g.str_w > 1 && ((ph_w + g.pad_w - s * g.dil_w) % g.str_w + g.str_w) % g.str_w) continue;
            const int nw = liw + g.pad_w - s * g.dil_w;
            const int ow = nw / g.str_w;
            const bool ok = pv && hv && nw >= 0 && nw % g.str_w == 0 && ow < g.q;
            const T* dyp = dy + (((size_t)ln * g.p + (ok ? oh : 0)) * g.q + (ok ? ow : 0)) * g.y_pitch;
            for (int kc = 0; kc < g.k; kc += KC) {
                const int kb = kc + lh * 8;
                float av[8], bv[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) av[i] = bv[i] = 0.0f;
                if (ok && kb < g.y_pitch) load8(dyp + kb, av);
                if (kc + bk < g.k && c0 + bc < g.f_pitch)
                    load8(f + (((size_t)(kc + bk) * g.r + r) * g.s + s) * g.f_pitch + c0 + bc, bv);
                __syncthreads();  // the previous chunk is consumed
#pragma unroll
                for (int i = 0; i < 8; ++i) As[lh * 8 + i][lp] = av[i];
                *reinterpret_cast<float4*>(&Bs[bk][bc]) = make_float4(bv[0], bv[1], bv[2], bv[3]);
                *reinterpret_cast<float4*>(&Bs[bk][bc + 4]) = make_float4(bv[4], bv[5], bv[6], bv[7]);
                __syncthreads();
#pragma unroll
                for (int q = 0; q < KC; ++q) {
                    const float4 a0 = *reinterpret_cast<const float4*>(&As[q][ty * 8]);
                    const float4 a1 = *reinterpret_cast<const float4*>(&As[q][ty * 8 + 4]);
                    const float4 b = *reinterpret_cast<const float4*>(&Bs[q][tx * 4]);
                    const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                    const float bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                    for (int i = 0; i < 8; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int pp = px0 + ty * 8 + i;
        if (pp >= npix) break;
        const int iw = ph_w + (pp % wp) * g.str_w, t = pp / wp;
        const int ih = ph_h + (t % hp) * g.str_h, n = t / hp;
        T* xp = dx + (((size_t)n * g.h + ih) * g.w + iw) * g.x_pitch;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = c0 + tx * 4 + j;
            if (c < g.x_pitch) st(xp + c, acc[i][j]);  // pad lanes: zero filter lanes give 0
        }
    }
}

// Backward weights, register-tiled (groups == 1, convolution mode): the GEMM
// dW[k][(tap, c)] = sum_pix dY[pix][k] * x[pix + tap][c]. A CTA owns 64 k x 64
// channels of one tap over a contiguous pixel range (split z); per 16-pixel
// step the dY slice [16 px][64 k] and the gathered input slice [16 px][64 c]
// are staged in smem and each thread accumulates 8 k x 4 c. Splits write fp32
// partials summed in split order by direct_wgrad_sum_kernel (deterministic).
template <typename T>
__global__ void __launch_bounds__(128) direct_wgrad_tiled_kernel(pk_conv_geom g, const T* __restrict__ dy,
                                                                 const T* __restrict__ x, float* __restrict__ out,
                                                                 int px_per_split) {
    constexpr int TK = 64, TC = 64, PP = 16, LD = 68;
    __shared__ __align__(16) float As[PP][LD];  // [pixel][k]
    __shared__ __align__(16) float Bs[PP][LD];  // [pixel][c]
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int k0 = blockIdx.x * TK;
    const int cblocks = (g.f_pitch + TC - 1) / TC;
    const int tap = blockIdx.y / cblocks, c0 = (blockIdx.y % cblocks) * TC;
    const int r = tap / g.s, s = tap % g.s;
    const int npix = g.n * g.p * g.q;
    const int p0 = blockIdx.z * px_per_split, p1 = min(npix, p0 + px_per_split);
    const int lpx = tid >> 3, lv = (tid & 7) * 8;  // loader: pixel, 8-channel vector
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    for (int pb = p0; pb < p1; pb += PP) {
        const int pix = pb + lpx;
        float av[8], bv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) av[i] = bv[i] = 0.0f;
        if (pix < p1) {
            const int ow = pix % g.q, t = pix / g.q, oh = t % g.p, n = t / g.p;
            if (k0 + lv < g.y_pitch) load8(dy + (size_t)pix * g.y_pitch + k0 + lv, av);
            const int ih = oh * g.str_h - g.pad_h + r * g.dil_h, iw = ow * g.str_w - g.pad_w + s * g.dil_w;
            if (ih >= 0 && ih < g.h && iw >= 0 && iw < g.w && c0 + lv < g.x_pitch)
                load8(x + (((size_t)n * g.h + ih) * g.w + iw) * g.x_pitch + c0 + lv, bv);
        }
        __syncthreads();  // the previous step is consumed
        *reinterpret_cast<float4*>(&As[lpx][lv]) = make_float4(av[0], av[1], av[2], av[3]);
        *reinterpret_cast<float4*>(&As[lpx][lv + 4]) = make_float4(av[4], av[5], av[6], av[7]);
        *reinterpret_cast<float4*>(&Bs[lpx][lv]) = make_float4(bv[0], bv[1], bv[2], bv[3]);
        *reinterpret_cast<float4*>(&Bs[lpx][lv + 4]) = make_float4(bv[4], bv[5], bv[6], bv[7]);
        __syncthreads();
#pragma unroll
        for (int q = 0; q < PP; ++q) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[q][ty * 8]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[q][ty * 8 + 4]);
            const float4 b = *reinterpret_cast<const float4*>(&Bs[q][tx * 4]);
            const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            const float bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
        }
    }
    const int taps = g.r * g.s;
    const size_t total = (size_t)g.k * taps * g.f_pitch;
    float* o = out + (size_t)blockIdx.z * total;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int k = k0 + ty * 8 + i;
        if (k >= g.k) break;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = c0 + tx * 4 + j;
            if (c < g.f_pitch) o[((size_t)k * taps + tap) * g.f_pitch + c] = acc[i][j];
        }
    }
}

template <typename T>
__global__ void direct_wgrad_sum_kernel(const float* __restrict__ partial, int splits, long long total,
                                        T* __restrict__ dw) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        float sum = 0.0f;
        for (int sp = 0; sp < splits; ++sp) sum += partial[(size_t)sp * total + i];
        st(dw + i, sum);
    }
}

}  // namespace pk

using namespace pk;

extern "C" {

cudaError_t pk_cuda_direct_fwd(const pk_conv_geom* g, int dtype, const void* x, const void* f,
                               void* y, const pk_epilogue* epi, cudaStream_t st) {
    pk_epilogue none{};
    none.act = -1;
    const pk_epilogue e = epi ? *epi : none;
    const long long npix = (long long)g->n * g->p * g->q;
    if (g->groups == 1 && !g->transpose && g->x_pitch % 8 == 0 && g->f_pitch == g->x_pitch) {
        dim3 grid(ceil_div(npix, 64), ceil_div(g->k, 64));
        PK_DISPATCH_DTYPE(dtype, T,
                          direct_fwd_tiled_kernel<T><<<grid, 128, 0, st>>>(*g, (const T*)x, (const T*)f,
                                                                           (T*)y, e));
        count_launch();
        return cudaGetLastError();
    }
    const bool wide = (g->kg % 8) == 0;
    const int kt = wide ? 8 : 1;
    dim3 grid(ceil_div(npix, 128), ceil_div(g->k, kt));
    PK_DISPATCH_DTYPE(dtype, T, {
        if (wide)
            direct_fwd_kernel<T, 8><<<grid, 128, 0, st>>>(*g, (const T*)x, (const T*)f, (T*)y, e);
        else
            direct_fwd_kernel<T, 1><<<grid, 128, 0, st>>>(*g, (const T*)x, (const T*)f, (T*)y, e);
    });
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_direct_bwd_data(const pk_conv_geom* g, int dtype, const void* dy,
                                    const void* f, void* dx, cudaStream_t st) {
    const long long npix = (long long)g->n * g->h * g->w;
    const bool wide = (g->cg % 8) == 0;
    const int ct = wide ? 8 : 1;
    dim3 grid(ceil_div(npix, 128), ceil_div(g->c, ct));
    PK_DISPATCH_DTYPE(dtype, T, {
        if (wide)
            direct_bwd_data_kernel<T, 8>
                <<<grid, 128, 0, st>>>(*g, (const T*)dy, (const T*)f, (T*)dx);
        else
            direct_bwd_data_kernel<T, 1>
                <<<grid, 128, 0, st>>>(*g, (const T*)dy, (const T*)f, (T*)dx);
    });
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_direct_bwd_weights(const pk_conv_geom* g, int dtype, const void* dy,
                                       const void* x, void* dw, cudaStream_t st) {
    const long long blocks = (long long)g->k * g->r * g->s * ((g->cg + 31) / 32);
    PK_DISPATCH_DTYPE(dtype, T,
                      direct_bwd_weights_kernel<T><<<(unsigned)blocks, 256, 0, st>>>(
                          *g, (const T*)dy, (const T*)x, (T*)dw));
    count_launch();
    return cudaGetLastError();
}

int pk_direct_dgrad_tiled_supported(const pk_conv_geom* g) {
    return g->groups == 1 && !g->transpose && g->x_pitch % 8 == 0 && g->f_pitch == g->x_pitch &&
           g->y_pitch % 8 == 0 && (long long)g->n * g->h * g->w < (1LL << 31);
}

cudaError_t pk_cuda_direct_dgrad_tiled(const pk_conv_geom* g, int dtype, const void* dy, const void* f, void* dx,
                                       cudaStream_t st) {
    if (!pk_direct_dgrad_tiled_supported(g)) return cudaErrorInvalidValue;
    // phases: grid.z = str_h * str_w; grid.x covers the largest phase (phase 0)
    const long long most = (long long)g->n * ceil_div(g->h, g->str_h) * ceil_div(g->w, g->str_w);
    dim3 grid(ceil_div(most, 64), ceil_div(g->x_pitch, 64), g->str_h * g->str_w);
    PK_DISPATCH_DTYPE(dtype, T,
                      direct_dgrad_tiled_kernel<T><<<grid, 128, 0, st>>>(*g, (const T*)dy, (const T*)f, (T*)dx));
    count_launch();
    return cudaGetLastError();
}

int pk_direct_wgrad_tiled_supported(const pk_conv_geom* g) {
    return g->groups == 1 && !g->transpose && g->x_pitch % 8 == 0 && g->f_pitch == g->x_pitch &&
           g->y_pitch % 8 == 0 && (long long)g->n * g->p * g->q < (1LL << 31);
}

static int direct_wgrad_splits(const pk_conv_geom* g, int num_sms) {
    const long long tiles = (long long)ceil_div(g->k, 64) * g->r * g->s * ceil_div(g->f_pitch, 64);
    const long long npix = (long long)g->n * g->p * g->q;
    long long splits = (4LL * num_sms + tiles - 1) / tiles;
    splits = std::min(splits, std::max(1LL, npix / 256));  // >= 256 pixels per split
    return (int)std::max(1LL, std::min(splits, 1024LL));
}

size_t pk_direct_wgrad_tiled_workspace(const pk_conv_geom* g, int num_sms) {
    return (size_t)direct_wgrad_splits(g, num_sms) * g->k * g->r * g->s * g->f_pitch * sizeof(float);
}

cudaError_t pk_cuda_direct_wgrad_tiled(const pk_conv_geom* g, int dtype, const void* dy, const void* x, void* dw,
                                       void* ws, size_t ws_bytes, int num_sms, cudaStream_t st) {
    if (!pk_direct_wgrad_tiled_supported(g) || ws_bytes < pk_direct_wgrad_tiled_workspace(g, num_sms))
        return cudaErrorInvalidValue;
    const int splits = direct_wgrad_splits(g, num_sms);
    const long long npix = (long long)g->n * g->p * g->q;
    const int per = (int)((ceil_div(npix, splits) + 15) / 16 * 16);
    const long long total = (long long)g->k * g->r * g->s * g->f_pitch;
    dim3 grid(ceil_div(g->k, 64), g->r * g->s * ceil_div(g->f_pitch, 64), ceil_div(npix, per));
    PK_DISPATCH_DTYPE(dtype, T, {
        direct_wgrad_tiled_kernel<T><<<grid, 128, 0, st>>>(*g, (const T*)dy, (const T*)x, (float*)ws, per);
        direct_wgrad_sum_kernel<T><<<(unsigned)std::max(1LL, std::min((long long)ceil_div(total, 256),
                                                                      4LL * num_sms)),
                                     256, 0, st>>>((const float*)ws, (int)grid.z, total, (T*)dw);
    });
    count_launch(2);
    return cudaGetLastError();
}

}  // extern "C"
