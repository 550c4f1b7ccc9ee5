// Dense-reduction packing for convolutions whose channel pitch is not a
// multiple of 64 (the 3-channel ResNet/VGG stem). The (r, s, c) reduction is
// packed densely (no per-tap channel padding) into a column matrix
// col[pixel][kc], kc = (r*S + s)*C + c, padded to a multiple of 64, so the
// tensor-core GEMMs run full 64-wide K blocks through the plain TMA path:
//   forward      y   = col . Wp^T        (Wp = packed filter [K][kc])
//   backward W   dWp = dY^T . col        -> unpacked to [K][R][S][pitch]
//   backward X   colg = dY . Wp          -> col2im gather-add into dX
// These are HBM-bound elementwise/gather passes (one read, one write each).
#include "common.cuh"

namespace pk {
namespace {

inline unsigned blocks_for(long long total) {
    long long b = (total + 255) / 256;
    if (b > 148LL * 64) b = 148LL * 64;
    return (unsigned)(b < 1 ? 1 : b);
}

// One thread per (pixel, 8-element chunk of kc): 8 gathered loads, one 16-byte
// store (rows of the column matrix are written contiguously by a warp).
__global__ void im2col_pack_kernel(pk_conv_geom g, const __nv_bfloat16* __restrict__ x,
                                   __nv_bfloat16* __restrict__ col, int kcp) {
    const int chunks = kcp / 8;
    const long long rows = (long long)g.n * g.p * g.q;
    const long long total = rows * chunks;
    const int rsc = g.r * g.s * g.c;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int ch = (int)(i % chunks);
        const long long m = i / chunks;
        const int ow = (int)(m % g.q);
        const int oh = (int)((m / g.q) % g.p);
        const int n = (int)(m / ((long long)g.q * g.p));
        const __nv_bfloat16* xn = x + (size_t)n * g.h * g.w * g.x_pitch;
        __align__(16) __nv_bfloat16 v[8];
        int kc = ch * 8;
        int c = kc % g.c, tap = kc / g.c;
        int r = tap / g.s, s = tap - r * g.s;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            __nv_bfloat16 val = __float2bfloat16_rn(0.0f);
            if (kc + e < rsc) {
                const int ih = oh * g.str_h - g.pad_h + r * g.dil_h;
                const int iw = ow * g.str_w - g.pad_w + s * g.dil_w;
                if (ih >= 0 && ih < g.h && iw >= 0 && iw < g.w)
                    val = xn[((size_t)ih * g.w + iw) * g.x_pitch + c];
            }
            v[e] = val;
            if (++c == g.c) {  // advance (r, s, c) without divisions
                c = 0;
                if (++s == g.s) {
                    s = 0;
                    ++r;
                }
            }
        }
        reinterpret_cast<uint4*>(col)[i] = *reinterpret_cast<const uint4*>(v);
    }
}

// fp[k][kc] (transposed = 0) or ft[kc][kp] (transposed = 1) from f[k][r][s][f_pitch]
__global__ void filter_pack_kernel(pk_conv_geom g, const __nv_bfloat16* __restrict__ f,
                                   __nv_bfloat16* __restrict__ dst, int kcp, int transposed) {
    const int kp = (g.k + 7) / 8 * 8;
    const long long total = transposed ? (long long)kcp * kp : (long long)g.k * kcp;
    const int rsc = g.r * g.s * g.c;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        int k, kc;
        if (transposed) {
            k = (int)(i % kp);
            kc = (int)(i / kp);
        } else {
            kc = (int)(i % kcp);
            k = (int)(i / kcp);
        }
        __nv_bfloat16 v = __float2bfloat16_rn(0.0f);
        if (kc < rsc && k < g.k) {
            const int c = kc % g.c, tap = kc / g.c;
            v = f[((size_t)k * g.r * g.s + tap) * g.f_pitch + c];
        }
        dst[i] = v;
    }
}

// dx[n][h][w][c] = sum over taps reaching (h, w) of colg[(n, oh, ow)][(r*S+s)*C + c];
// one thread per (pixel, 8-channel chunk), 16-byte store.
__global__ void col2im_pack_kernel(pk_conv_geom g, const __nv_bfloat16* __restrict__ colg,
                                   int kcp, __nv_bfloat16* __restrict__ dx) {
    const int chunks = g.x_pitch / 8;
    const long long total = (long long)g.n * g.h * g.w * chunks;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c0 = (int)(i % chunks) * 8;
        const long long pix = i / chunks;
        const int iw = (int)(pix % g.w);
        const int ih = (int)((pix / g.w) % g.h);
        const int n = (int)(pix / ((long long)g.w * g.h));
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const int cn = min(8, g.c - c0);
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
                const __nv_bfloat16* src =
                    colg + (((size_t)n * g.p + oh) * g.q + ow) * kcp + (r * g.s + s) * g.c + c0;
                for (int e = 0; e < cn; ++e) acc[e] += __bfloat162float(src[e]);
            }
        }
        __align__(16) __nv_bfloat16 v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = __float2bfloat16_rn(e < cn ? acc[e] : 0.0f);
        reinterpret_cast<uint4*>(dx)[i] = *reinterpret_cast<const uint4*>(v);
    }
}

// dw[k][r][s][c] = dwp[k][(r*S+s)*C + c] (pad lanes zero)
__global__ void wgrad_unpack_kernel(pk_conv_geom g, const __nv_bfloat16* __restrict__ dwp,
                                    int kcp, __nv_bfloat16* __restrict__ dw) {
    const long long total = (long long)g.k * g.r * g.s * g.f_pitch;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % g.f_pitch);
        const long long t = i / g.f_pitch;
        const int tap = (int)(t % (g.r * g.s));
        const int k = (int)(t / (g.r * g.s));
        dw[i] = c < g.c ? dwp[(size_t)k * kcp + tap * g.c + c] : __float2bfloat16_rn(0.0f);
    }
}

}  // namespace
}  // namespace pk

using namespace pk;

extern "C" {

int pk_stem_kc_pitch(const pk_conv_geom* g) { return (g->r * g->s * g->c + 7) / 8 * 8; }

cudaError_t pk_cuda_im2col_pack(const pk_conv_geom* g, const void* x, void* col, cudaStream_t st) {
    const int kcp = pk_stem_kc_pitch(g);
    im2col_pack_kernel<<<blocks_for((long long)g->n * g->p * g->q * (kcp / 8)), 256, 0, st>>>(
        *g, (const __nv_bfloat16*)x, (__nv_bfloat16*)col, kcp);
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_filter_pack(const pk_conv_geom* g, const void* f, void* dst, int transposed,
                                cudaStream_t st) {
    const int kcp = pk_stem_kc_pitch(g);
    const long long total = (long long)kcp * (transposed ? pk_pitch(g->k) : g->k);
    filter_pack_kernel<<<blocks_for(total), 256, 0, st>>>(*g, (const __nv_bfloat16*)f,
                                                           (__nv_bfloat16*)dst, kcp, transposed);
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_col2im_pack(const pk_conv_geom* g, const void* colg, void* dx,
                                cudaStream_t st) {
    col2im_pack_kernel<<<blocks_for((long long)g->n * g->h * g->w * (g->x_pitch / 8)), 256, 0, st>>>(
        *g, (const __nv_bfloat16*)colg, pk_stem_kc_pitch(g), (__nv_bfloat16*)dx);
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_wgrad_unpack(const pk_conv_geom* g, const void* dwp, void* dw,
                                 cudaStream_t st) {
    wgrad_unpack_kernel<<<blocks_for((long long)g->k * g->r * g->s * g->f_pitch), 256, 0, st>>>(
        *g, (const __nv_bfloat16*)dwp, pk_stem_kc_pitch(g), (__nv_bfloat16*)dw);
    count_launch();
    return cudaGetLastError();
}

}  // extern "C"
