// Winograd F(2x2, 3x3) convolution, zero workspace (CUDA cores, fp32).
//
// Same algorithm as the reference winograd_forward
// (proj/src/core/conv.cpp:269-365): U = G g G^T, V = B^T d B, M = sum_c U.V
// (16 multiplies per (tile, channel, output channel)), Y = A^T M A, zero
// padded / cropped edge tiles. Schedule: a CTA owns 32 output tiles x 32
// output channels; the input transform of each (tile, channel) and the filter
// transform of each (output channel, channel) are computed ONCE per CTA into
// shared memory (the reference recomputes V for every k), then every thread
// accumulates the 16 transformed products for 4 (tile, k) pairs.
#include "common.cuh"

namespace pk {

constexpr int WT = 32;   // tiles per CTA
constexpr int WK = 32;   // output channels per CTA
constexpr int WC = 8;    // channels per smem slice

template <typename T>
__global__ void __launch_bounds__(256) winograd_f23_kernel(pk_conv_geom g, const T* __restrict__ x,
                                                           const T* __restrict__ f,
                                                           T* __restrict__ y, pk_epilogue e) {
    __shared__ float Vs[WC][16][WT + 1];
    __shared__ __align__(16) float Us[WC][16][WK + 4];  // rows 16-byte aligned for float4 reads
    const int th = (g.p + 1) / 2, tw = (g.q + 1) / 2;
    const long long ntiles = (long long)g.n * th * tw;
    const long long t0 = (long long)blockIdx.x * WT;
    const int k0 = blockIdx.y * WK;
    const int grp = k0 / g.kg;  // host guarantees kg % WK == 0 or groups == 1
    const int tid = threadIdx.x;
    const int tx = tid % 32, ty = tid / 32;  // tile lane, k group (4 consecutive k)

    float M[4][16];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int q = 0; q < 16; ++q) M[j][q] = 0.0f;

    for (int c0 = 0; c0 < g.cg; c0 += WC) {
        // Input transform: thread -> (tile tid / WC, channel tid % WC); the WC
        // lanes of a tile read consecutive channels of each pixel (coalesced).
        {
            const int cl = tid % WC, tl = tid / WC, c = c0 + cl;
            const long long t = t0 + tl;
            float d[4][4];
            if (c < g.cg && t < ntiles) {
                const int tj = (int)(t % tw);
                const int ti = (int)((t / tw) % th);
                const int n = (int)(t / ((long long)tw * th));
                const T* xp = x + (size_t)n * g.h * g.w * g.x_pitch + grp * g.cg + c;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int ih = 2 * ti - g.pad_h + i;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int iw = 2 * tj - g.pad_w + j;
                        d[i][j] = (ih >= 0 && ih < g.h && iw >= 0 && iw < g.w)
                                      ? ld(xp + ((size_t)ih * g.w + iw) * g.x_pitch)
                                      : 0.0f;
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) d[i][j] = 0.0f;
            }
            float tt[4][4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                tt[0][j] = d[0][j] - d[2][j];
                tt[1][j] = d[1][j] + d[2][j];
                tt[2][j] = d[2][j] - d[1][j];
                tt[3][j] = d[1][j] - d[3][j];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                Vs[cl][i * 4 + 0][tl] = tt[i][0] - tt[i][2];
                Vs[cl][i * 4 + 1][tl] = tt[i][1] + tt[i][2];
                Vs[cl][i * 4 + 2][tl] = tt[i][2] - tt[i][1];
                Vs[cl][i * 4 + 3][tl] = tt[i][1] - tt[i][3];
            }
        }
        // Filter transform: thread -> (output channel tx, channel ty).
        {
            const int cl = ty, c = c0 + cl, k = k0 + tx;
            float gg[3][3];
            if (c < g.cg && k < g.k) {
                const T* fp = f + (size_t)k * 9 * g.f_pitch + c;
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j) gg[i][j] = ld(fp + (i * 3 + j) * g.f_pitch);
            } else {
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j) gg[i][j] = 0.0f;
            }
            float tt[4][3];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                tt[0][j] = gg[0][j];
                tt[1][j] = 0.5f * (gg[0][j] + gg[1][j] + gg[2][j]);
                tt[2][j] = 0.5f * (gg[0][j] - gg[1][j] + gg[2][j]);
                tt[3][j] = gg[2][j];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                Us[cl][i * 4 + 0][tx] = tt[i][0];
                Us[cl][i * 4 + 1][tx] = 0.5f * (tt[i][0] + tt[i][1] + tt[i][2]);
                Us[cl][i * 4 + 2][tx] = 0.5f * (tt[i][0] - tt[i][1] + tt[i][2]);
                Us[cl][i * 4 + 3][tx] = tt[i][2];
            }
        }
        __syncthreads();
        const int cmax = min(WC, g.cg - c0);
        for (int cl = 0; cl < cmax; ++cl) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const float v = Vs[cl][q][tx];
                const float4 u = *reinterpret_cast<const float4*>(&Us[cl][q][ty * 4]);  // broadcast
                M[0][q] += u.x * v;
                M[1][q] += u.y * v;
                M[2][q] += u.z * v;
                M[3][q] += u.w * v;
            }
        }
        __syncthreads();
    }

    const long long t = t0 + tx;
    if (t >= ntiles) return;
    const int tj = (int)(t % tw);
    const int ti = (int)((t / tw) % th);
    const int n = (int)(t / ((long long)tw * th));
    const bool epi = epilogue_active(&e);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int k = k0 + ty * 4 + j;
        if (k >= g.k) continue;
        const float* m = M[j];
        float rr[2][4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            rr[0][c] = m[0 * 4 + c] + m[1 * 4 + c] + m[2 * 4 + c];
            rr[1][c] = m[1 * 4 + c] - m[2 * 4 + c] - m[3 * 4 + c];
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int oh = 2 * ti + i;
            if (oh >= g.p) continue;
            const float o0 = rr[i][0] + rr[i][1] + rr[i][2];
            const float o1 = rr[i][1] - rr[i][2] - rr[i][3];
            for (int jj = 0; jj < 2; ++jj) {
                const int ow = 2 * tj + jj;
                if (ow >= g.q) continue;
                float v = jj == 0 ? o0 : o1;
                if (epi) v = apply_epilogue(e, v, k, oh, ow, g.p, g.q);
                st(y + (((size_t)n * g.p + oh) * g.q + ow) * g.y_pitch + k, v);
            }
        }
    }
}

}  // namespace pk

using namespace pk;

extern "C" cudaError_t pk_cuda_winograd_f23(const pk_conv_geom* g, int dtype, const void* x,
                                            const void* f, void* y, const pk_epilogue* epi,
                                            cudaStream_t st) {
    if (g->r != 3 || g->s != 3 || g->str_h != 1 || g->str_w != 1 || g->dil_h != 1 ||
        g->dil_w != 1 || g->transpose)
        return cudaErrorInvalidValue;
    if (g->groups > 1 && g->kg % WK != 0) {
        // Grouped shapes whose groups do not align with the 32-channel CTA
        // tile run one launch per group on offset views.
        pk_conv_geom gg = *g;
        gg.groups = 1;
        gg.c = g->cg;
        gg.k = g->kg;
        const size_t esz = dtype == PK_BF16 ? 2 : 4;
        for (int grp = 0; grp < g->groups; ++grp) {
            pk_epilogue e = epi ? *epi : pk_epilogue{};
            if (!epi) e.act = -1;
            if (e.bias) e.bias += grp * g->kg;
            const long long bn_off = (long long)grp * g->kg * (e.bn_per_activation ? g->p * g->q : 1);
            if (e.bn_mean) {
                e.bn_mean += bn_off;
                e.bn_var += bn_off;
                e.bn_gamma += bn_off;
                e.bn_beta += bn_off;
            }
            // input channel offset is applied through x, filter rows through f,
            // output channels through y (pitches unchanged).
            const char* xg = (const char*)x + (size_t)grp * g->cg * esz;
            const char* fg = (const char*)f + (size_t)grp * g->kg * 9 * g->f_pitch * esz;
            char* yg = (char*)y + (size_t)grp * g->kg * esz;
            dim3 grid(ceil_div((long long)g->n * ((g->p + 1) / 2) * ((g->q + 1) / 2), WT),
                      ceil_div(gg.k, WK));
            PK_DISPATCH_DTYPE(dtype, T,
                              winograd_f23_kernel<T><<<grid, 256, 0, st>>>(
                                  gg, (const T*)xg, (const T*)fg, (T*)yg, e));
            count_launch();
        }
        return cudaGetLastError();
    }
    pk_epilogue none{};
    none.act = -1;
    const pk_epilogue e = epi ? *epi : none;
    const long long ntiles = (long long)g->n * ((g->p + 1) / 2) * ((g->q + 1) / 2);
    dim3 grid(ceil_div(ntiles, WT), ceil_div(g->k, WK));
    PK_DISPATCH_DTYPE(dtype, T,
                      winograd_f23_kernel<T><<<grid, 256, 0, st>>>(*g, (const T*)x, (const T*)f,
                                                                   (T*)y, e));
    count_launch();
    return cudaGetLastError();
}
