// Dense-reduction packing for convolutions whose channel pitch is not a
// multiple of 64 (the 3-channel ResNet/VGG stem). The (r, s, c) reduction is
// packed into a column matrix col[pixel][kc] with kc = (r*S + s)*cs + c, where
// cs = 4 for C <= 4 (else the channel pitch): 49 taps x 4 = 196 columns for
// ResNet's conv1 instead of 49 x 64 with per-tap padding. The tensor-core GEMMs
// then run dense 64-wide K blocks through the plain TMA path:
//   forward      y   = col . Wp^T        (Wp = packed filter [K][kcp])
//   backward W   dWp = dY^T . col        -> unpacked to [K][R][S][pitch]
//   backward X   colg = dY . Wp          -> col2im gather-add into dX
// The packing passes are HBM-bound: one thread per (pixel, tap) moves cs
// channels with one aligned 8/16-byte load and store.
#include "common.cuh"

namespace pk {
namespace {

inline unsigned blocks_for(long long total) {
    long long b = (total + 255) / 256;
    if (b > 148LL * 64) b = 148LL * 64;
    return (unsigned)(b < 1 ? 1 : b);
}

__host__ __device__ inline int stem_cs(const pk_conv_geom& g) {
    return g.c <= 4 ? 4 : (g.c + 7) / 8 * 8;
}

__host__ __device__ inline int stem_kcp(const pk_conv_geom& g) {
    return (g.r * g.s * stem_cs(g) + 7) / 8 * 8;
}

// Copy `cs` bf16 lanes (cs = 4: 8 bytes, else multiples of 8: 16-byte chunks).
__device__ __forceinline__ void copy_lanes(__nv_bfloat16* dst, const __nv_bfloat16* src, int cs) {
    if (cs == 4) {
        *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(src);
    } else {
        for (int j = 0; j < cs; j += 8)
            *reinterpret_cast<uint4*>(dst + j) = *reinterpret_cast<const uint4*>(src + j);
    }
}
__device__ __forceinline__ void zero_lanes(__nv_bfloat16* dst, int cs) {
    if (cs == 4) {
        *reinterpret_cast<uint2*>(dst) = make_uint2(0u, 0u);
    } else {
        for (int j = 0; j < cs; j += 8) *reinterpret_cast<uint4*>(dst + j) = make_uint4(0, 0, 0, 0);
    }
}

// One warp per output pixel (pixel decode once per warp, 32-bit math); lane t
// moves tap t's cs channels, so a warp writes its column-matrix row
// contiguously. Tap index R*S zero-fills the row tail.
__global__ void __launch_bounds__(256) im2col_pack_kernel(pk_conv_geom g,
                                                          const __nv_bfloat16* __restrict__ x,
                                                          __nv_bfloat16* __restrict__ col) {
    const int cs = stem_cs(g), kcp = stem_kcp(g), taps = g.r * g.s;
    const int lane = threadIdx.x & 31;
    const long long rows = (long long)g.n * g.p * g.q;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    long long m0 = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
    if (cs == 4 && taps <= 64) {
        // fast path: 4 pixels x 2 tap slots per lane, all 8 loads in flight
        // before the stores (the pass is latency-bound otherwise)
        const int pq = g.p * g.q;
        for (; m0 < rows; m0 += 4 * warps) {
            uint2 v[4][2];
            long long mm[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                mm[u] = m0 + u * warps;
                int n = 0, oh = 0, ow = 0;
                const bool live = mm[u] < rows;
                if (live) {
                    n = (int)(mm[u] / pq);
                    const int rem = (int)(mm[u] - (long long)n * pq);
                    oh = rem / g.q;
                    ow = rem - oh * g.q;
                }
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int t = lane + 32 * j;
                    v[u][j] = make_uint2(0u, 0u);
                    if (live && t < taps) {
                        const int r = t / g.s, s = t - r * g.s;
                        const int ih = oh * g.str_h - g.pad_h + r * g.dil_h;
                        const int iw = ow * g.str_w - g.pad_w + s * g.dil_w;
                        if (ih >= 0 && ih < g.h && iw >= 0 && iw < g.w)
                            v[u][j] = __ldg(reinterpret_cast<const uint2*>(
                                x + (((size_t)n * g.h + ih) * g.w + iw) * g.x_pitch));
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (mm[u] >= rows) continue;
                __nv_bfloat16* dst = col + mm[u] * kcp;
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int t = lane + 32 * j;
                    if (t < taps) *reinterpret_cast<uint2*>(dst + t * 4) = v[u][j];
                    else if (t * 4 < kcp) *reinterpret_cast<uint2*>(dst + t * 4) = make_uint2(0u, 0u);
                }
            }
        }
        return;
    }
    for (long long m = m0; m < rows; m += warps) {
        const int pq = g.p * g.q;
        const int n = (int)(m / pq);
        const int rem = (int)(m - (long long)n * pq);
        const int oh = rem / g.q, ow = rem - oh * g.q;
        const int ih0 = oh * g.str_h - g.pad_h, iw0 = ow * g.str_w - g.pad_w;
        const __nv_bfloat16* xn = x + (size_t)n * g.h * g.w * g.x_pitch;
        __nv_bfloat16* dst = col + m * kcp;
        for (int t = lane; t <= taps; t += 32) {
            if (t == taps) {
                for (int j = taps * cs; j < kcp; ++j) dst[j] = __float2bfloat16_rn(0.0f);
                continue;
            }
            const int r = t / g.s, s = t - r * g.s;
            const int ih = ih0 + r * g.dil_h, iw = iw0 + s * g.dil_w;
            if (ih >= 0 && ih < g.h && iw >= 0 && iw < g.w)
                copy_lanes(dst + t * cs, xn + ((size_t)ih * g.w + iw) * g.x_pitch, cs);
            else
                zero_lanes(dst + t * cs, cs);
        }
    }
}

// fp[k][kc] (transposed = 0) or ft[kc][pitch(K)] (transposed = 1)
__global__ void filter_pack_kernel(pk_conv_geom g, const __nv_bfloat16* __restrict__ f,
                                   __nv_bfloat16* __restrict__ dst, int transposed) {
    const int cs = stem_cs(g), kcp = stem_kcp(g);
    const int kp = (g.k + 7) / 8 * 8;
    const long long total = transposed ? (long long)kcp * kp : (long long)g.k * kcp;
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
        const int tap = kc / cs, c = kc - tap * cs;
        __nv_bfloat16 v = __float2bfloat16_rn(0.0f);
        if (tap < g.r * g.s && c < g.c && k < g.k) v = f[((size_t)k * g.r * g.s + tap) * g.f_pitch + c];
        dst[i] = v;
    }
}

// thread = (input pixel, cs-lane group): dx = sum over the taps reaching it
__global__ void col2im_pack_kernel(pk_conv_geom g, const __nv_bfloat16* __restrict__ colg,
                                   __nv_bfloat16* __restrict__ dx) {
    const int cs = stem_cs(g), kcp = stem_kcp(g);
    const int groups_per_px = (g.x_pitch + 7) / 8;  // write whole 16-byte pitch chunks
    const long long total = (long long)g.n * g.h * g.w * groups_per_px;
    const int hw = g.h * g.w;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c0 = groups_per_px == 1 ? 0 : (int)(i % groups_per_px) * 8;
        const long long pix = groups_per_px == 1 ? i : i / groups_per_px;
        const int n = (int)(pix / hw);
        const int rem = (int)(pix - (long long)n * hw);
        const int ih = rem / g.w, iw = rem - ih * g.w;
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const int cn = min(8, min(cs, g.c) - c0);  // lanes of this chunk that carry data
        // only the taps whose (ih + pad - r*dil) is a multiple of the stride
        // reach this pixel (dilation 1 here: r steps by the stride)
        const bool unit_dil = g.dil_h == 1 && g.dil_w == 1;
        const int r_first = unit_dil ? (ih + g.pad_h) % g.str_h : 0;
        const int s_first = unit_dil ? (iw + g.pad_w) % g.str_w : 0;
        const int r_step = unit_dil ? g.str_h : 1, s_step = unit_dil ? g.str_w : 1;
        if (cn > 0) {
            for (int r = r_first; r < g.r; r += r_step) {
                const int nh = ih + g.pad_h - r * g.dil_h;
                if (nh < 0) break;
                if (nh % g.str_h) continue;
                const int oh = nh / g.str_h;
                if (oh >= g.p) continue;
                for (int s = s_first; s < g.s; s += s_step) {
                    const int nw = iw + g.pad_w - s * g.dil_w;
                    if (nw < 0) break;
                    if (nw % g.str_w) continue;
                    const int ow = nw / g.str_w;
                    if (ow >= g.q) continue;
                    const __nv_bfloat16* src = colg + (((size_t)n * g.p + oh) * g.q + ow) * kcp +
                                               (r * g.s + s) * cs + c0;
                    if (cs == 4) {
                        const uint2 v = *reinterpret_cast<const uint2*>(src);
                        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
                        const float2 f0 = __bfloat1622float2(b[0]), f1 = __bfloat1622float2(b[1]);
                        acc[0] += f0.x;
                        acc[1] += f0.y;
                        acc[2] += f1.x;
                        acc[3] += f1.y;
                    } else {
                        const uint4 v = *reinterpret_cast<const uint4*>(src);
                        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float2 f = __bfloat1622float2(b[e]);
                            acc[2 * e] += f.x;
                            acc[2 * e + 1] += f.y;
                        }
                    }
                }
            }
        }
        __align__(16) __nv_bfloat16 v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = __float2bfloat16_rn(e < cn ? acc[e] : 0.0f);
        *reinterpret_cast<uint4*>(dx + pix * g.x_pitch + c0) = *reinterpret_cast<const uint4*>(v);
    }
}

// dw[k][r][s][c] = dwp[k][(r*S+s)*cs + c] (pad lanes zero)
__global__ void wgrad_unpack_kernel(pk_conv_geom g, const __nv_bfloat16* __restrict__ dwp,
                                    __nv_bfloat16* __restrict__ dw) {
    const int cs = stem_cs(g), kcp = stem_kcp(g);
    const long long total = (long long)g.k * g.r * g.s * g.f_pitch;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % g.f_pitch);
        const long long t = i / g.f_pitch;
        const int tap = (int)(t % (g.r * g.s));
        const int k = (int)(t / (g.r * g.s));
        dw[i] = c < g.c ? dwp[(size_t)k * kcp + tap * cs + c] : __float2bfloat16_rn(0.0f);
    }
}

}  // namespace
}  // namespace pk

using namespace pk;

extern "C" {

int pk_stem_kc_pitch(const pk_conv_geom* g) { return stem_kcp(*g); }

cudaError_t pk_cuda_im2col_pack(const pk_conv_geom* g, const void* x, void* col, cudaStream_t st) {
    const long long total = (long long)g->n * g->p * g->q * (g->r * g->s + 1);
    im2col_pack_kernel<<<blocks_for(total), 256, 0, st>>>(*g, (const __nv_bfloat16*)x,
                                                           (__nv_bfloat16*)col);
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_filter_pack(const pk_conv_geom* g, const void* f, void* dst, int transposed,
                                cudaStream_t st) {
    const int kcp = stem_kcp(*g);
    const long long total = (long long)kcp * (transposed ? pk_pitch(g->k) : g->k);
    filter_pack_kernel<<<blocks_for(total), 256, 0, st>>>(*g, (const __nv_bfloat16*)f,
                                                           (__nv_bfloat16*)dst, transposed);
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_col2im_pack(const pk_conv_geom* g, const void* colg, void* dx,
                                cudaStream_t st) {
    const long long total = (long long)g->n * g->h * g->w * ((g->x_pitch + 7) / 8);
    col2im_pack_kernel<<<blocks_for(total), 256, 0, st>>>(*g, (const __nv_bfloat16*)colg,
                                                           (__nv_bfloat16*)dx);
    count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_wgrad_unpack(const pk_conv_geom* g, const void* dwp, void* dw,
                                 cudaStream_t st) {
    wgrad_unpack_kernel<<<blocks_for((long long)g->k * g->r * g->s * g->f_pitch), 256, 0, st>>>(
        *g, (const __nv_bfloat16*)dwp, (__nv_bfloat16*)dw);
    count_launch();
    return cudaGetLastError();
}

}  // extern "C"
