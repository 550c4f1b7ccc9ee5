/* primkit oracle — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference CPU algorithms on the convolution
 * hot path, used solely by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the checker. It is never linked into or called by the
 * product library (paper_1910_00078_b200/lib/libprimkit.so).
 *
 * Parity is pinned two ways (tests/test_oracle.py): against the golden
 * vectors the reference's own tests hold (tests/golden/), and against the
 * unmodified reference built from its sources into oracle/_ref/ where
 * available. Every function cites the reference routine it restates
 * (paths relative to /root/reference/proj).
 *
 * Layout: packed NCHW float arrays, bf16 tensors carry bf16-rounded values.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t n, c, h, w, k, y, x;
    int64_t pad_h, pad_w, str_h, str_w, dil_h, dil_w, groups;
} oc_conv;

/* src/core/tensor.cpp:44-54 — RNE to bf16, widened back to f32. */
float oc_round_bf16(float v) {
    uint32_t u;
    memcpy(&u, &v, 4);
    if (isnan(v)) {
        u = (u & 0xffff0000u) | 0x00410000u;
    } else {
        u += 0x7fffu + ((u >> 16) & 1u);
        u &= 0xffff0000u;
    }
    memcpy(&v, &u, 4);
    return v;
}

void oc_quantize(float* a, int64_t n, int bf16) {
    if (!bf16) return;
    for (int64_t i = 0; i < n; ++i) a[i] = oc_round_bf16(a[i]);
}

/* src/core/conv.cpp:54-60 — output extent (convolution mode). */
int64_t oc_out_extent(int64_t in, int64_t pad, int64_t dil, int64_t f, int64_t str) {
    const int64_t span = dil * (f - 1) + 1;
    if (in + 2 * pad < span) return 0;
    return (in + 2 * pad - span) / str + 1;
}

/* src/core/conv.cpp:99-133 — Direct forward, loop order (n,k,oh,ow,c,y,x),
 * f32 accumulator; y must hold n*k*oh*ow floats. */
void oc_conv_fwd(const oc_conv* p, const float* in, const float* flt, float* out, int bf16) {
    const int64_t oh_n = oc_out_extent(p->h, p->pad_h, p->dil_h, p->y, p->str_h);
    const int64_t ow_n = oc_out_extent(p->w, p->pad_w, p->dil_w, p->x, p->str_w);
    const int64_t cg = p->c / p->groups, kg = p->k / p->groups;
    for (int64_t n = 0; n < p->n; ++n)
        for (int64_t k = 0; k < p->k; ++k) {
            const int64_t g = k / kg;
            for (int64_t oh = 0; oh < oh_n; ++oh)
                for (int64_t ow = 0; ow < ow_n; ++ow) {
                    float acc = 0.0f;
                    for (int64_t c = 0; c < cg; ++c) {
                        const float* ip = in + ((n * p->c + g * cg + c) * p->h) * p->w;
                        const float* fp = flt + ((k * cg + c) * p->y) * p->x;
                        for (int64_t yy = 0; yy < p->y; ++yy) {
                            const int64_t ih = oh * p->str_h - p->pad_h + yy * p->dil_h;
                            if (ih < 0 || ih >= p->h) continue;
                            for (int64_t xx = 0; xx < p->x; ++xx) {
                                const int64_t iw = ow * p->str_w - p->pad_w + xx * p->dil_w;
                                if (iw < 0 || iw >= p->w) continue;
                                acc += ip[ih * p->w + iw] * fp[yy * p->x + xx];
                            }
                        }
                    }
                    out[((n * p->k + k) * oh_n + oh) * ow_n + ow] = acc;
                }
        }
    oc_quantize(out, p->n * p->k * oh_n * ow_n, bf16);
}

/* src/core/conv.cpp:716-756 — Direct backward data. */
void oc_conv_bwd_data(const oc_conv* p, const float* dout, const float* flt, float* din,
                      int bf16) {
    const int64_t oh_n = oc_out_extent(p->h, p->pad_h, p->dil_h, p->y, p->str_h);
    const int64_t ow_n = oc_out_extent(p->w, p->pad_w, p->dil_w, p->x, p->str_w);
    const int64_t cg = p->c / p->groups, kg = p->k / p->groups;
    for (int64_t n = 0; n < p->n; ++n)
        for (int64_t c = 0; c < p->c; ++c) {
            const int64_t g = c / cg, cl = c % cg;
            for (int64_t h = 0; h < p->h; ++h)
                for (int64_t w = 0; w < p->w; ++w) {
                    float acc = 0.0f;
                    for (int64_t kk = 0; kk < kg; ++kk) {
                        const int64_t k = g * kg + kk;
                        for (int64_t yy = 0; yy < p->y; ++yy) {
                            const int64_t nh = h + p->pad_h - yy * p->dil_h;
                            if (nh < 0 || nh % p->str_h) continue;
                            const int64_t oh = nh / p->str_h;
                            if (oh >= oh_n) continue;
                            for (int64_t xx = 0; xx < p->x; ++xx) {
                                const int64_t nw = w + p->pad_w - xx * p->dil_w;
                                if (nw < 0 || nw % p->str_w) continue;
                                const int64_t ow = nw / p->str_w;
                                if (ow >= ow_n) continue;
                                acc += dout[((n * p->k + k) * oh_n + oh) * ow_n + ow] *
                                       flt[((k * cg + cl) * p->y + yy) * p->x + xx];
                            }
                        }
                    }
                    din[((n * p->c + c) * p->h + h) * p->w + w] = acc;
                }
        }
    oc_quantize(din, p->n * p->c * p->h * p->w, bf16);
}

/* src/core/conv.cpp:816-850 — Direct backward weights. */
void oc_conv_bwd_weights(const oc_conv* p, const float* dout, const float* in, float* dflt,
                         int bf16) {
    const int64_t oh_n = oc_out_extent(p->h, p->pad_h, p->dil_h, p->y, p->str_h);
    const int64_t ow_n = oc_out_extent(p->w, p->pad_w, p->dil_w, p->x, p->str_w);
    const int64_t cg = p->c / p->groups, kg = p->k / p->groups;
    for (int64_t k = 0; k < p->k; ++k) {
        const int64_t g = k / kg;
        for (int64_t c = 0; c < cg; ++c)
            for (int64_t yy = 0; yy < p->y; ++yy)
                for (int64_t xx = 0; xx < p->x; ++xx) {
                    float acc = 0.0f;
                    for (int64_t n = 0; n < p->n; ++n) {
                        const float* ip = in + ((n * p->c + g * cg + c) * p->h) * p->w;
                        const float* op = dout + ((n * p->k + k) * oh_n) * ow_n;
                        for (int64_t oh = 0; oh < oh_n; ++oh) {
                            const int64_t ih = oh * p->str_h - p->pad_h + yy * p->dil_h;
                            if (ih < 0 || ih >= p->h) continue;
                            for (int64_t ow = 0; ow < ow_n; ++ow) {
                                const int64_t iw = ow * p->str_w - p->pad_w + xx * p->dil_w;
                                if (iw < 0 || iw >= p->w) continue;
                                acc += op[oh * ow_n + ow] * ip[ih * p->w + iw];
                            }
                        }
                    }
                    dflt[((k * cg + c) * p->y + yy) * p->x + xx] = acc;
                }
    }
    oc_quantize(dflt, p->k * cg * p->y * p->x, bf16);
}

/* src/core/conv.cpp:269-365 — Winograd F(2x2,3x3), stride 1, dilation 1. */
void oc_winograd_f23(const oc_conv* p, const float* in, const float* flt, float* out, int bf16) {
    const int64_t oh_n = p->h + 2 * p->pad_h - 2, ow_n = p->w + 2 * p->pad_w - 2;
    const int64_t cg = p->c / p->groups, kg = p->k / p->groups;
    float* U = (float*)malloc(sizeof(float) * (size_t)(p->k * cg * 16));
    for (int64_t k = 0; k < p->k; ++k)
        for (int64_t c = 0; c < cg; ++c) {
            const float* g = flt + ((k * cg + c) * 3) * 3;
            float t[4][3];
            for (int j = 0; j < 3; ++j) {
                t[0][j] = g[j];
                t[1][j] = 0.5f * (g[j] + g[3 + j] + g[6 + j]);
                t[2][j] = 0.5f * (g[j] - g[3 + j] + g[6 + j]);
                t[3][j] = g[6 + j];
            }
            float* u = U + (k * cg + c) * 16;
            for (int i = 0; i < 4; ++i) {
                u[i * 4 + 0] = t[i][0];
                u[i * 4 + 1] = 0.5f * (t[i][0] + t[i][1] + t[i][2]);
                u[i * 4 + 2] = 0.5f * (t[i][0] - t[i][1] + t[i][2]);
                u[i * 4 + 3] = t[i][2];
            }
        }
    const int64_t th = (oh_n + 1) / 2, tw = (ow_n + 1) / 2;
    for (int64_t n = 0; n < p->n; ++n)
        for (int64_t k = 0; k < p->k; ++k) {
            const int64_t g = k / kg;
            for (int64_t ti = 0; ti < th; ++ti)
                for (int64_t tj = 0; tj < tw; ++tj) {
                    float M[16] = {0};
                    for (int64_t c = 0; c < cg; ++c) {
                        const float* ip = in + ((n * p->c + g * cg + c) * p->h) * p->w;
                        float d[4][4], t[4][4], V[4][4];
                        for (int i = 0; i < 4; ++i)
                            for (int j = 0; j < 4; ++j) {
                                const int64_t ih = 2 * ti - p->pad_h + i, iw = 2 * tj - p->pad_w + j;
                                d[i][j] = (ih >= 0 && ih < p->h && iw >= 0 && iw < p->w)
                                              ? ip[ih * p->w + iw] : 0.0f;
                            }
                        for (int j = 0; j < 4; ++j) {
                            t[0][j] = d[0][j] - d[2][j];
                            t[1][j] = d[1][j] + d[2][j];
                            t[2][j] = d[2][j] - d[1][j];
                            t[3][j] = d[1][j] - d[3][j];
                        }
                        for (int i = 0; i < 4; ++i) {
                            V[i][0] = t[i][0] - t[i][2];
                            V[i][1] = t[i][1] + t[i][2];
                            V[i][2] = t[i][2] - t[i][1];
                            V[i][3] = t[i][1] - t[i][3];
                        }
                        const float* u = U + (k * cg + c) * 16;
                        for (int e = 0; e < 16; ++e) M[e] += u[e] * V[e / 4][e % 4];
                    }
                    float r[2][4];
                    for (int j = 0; j < 4; ++j) {
                        r[0][j] = M[j] + M[4 + j] + M[8 + j];
                        r[1][j] = M[4 + j] - M[8 + j] - M[12 + j];
                    }
                    for (int i = 0; i < 2; ++i) {
                        const int64_t oh = 2 * ti + i;
                        if (oh >= oh_n) continue;
                        const float y0 = r[i][0] + r[i][1] + r[i][2];
                        const float y1 = r[i][1] - r[i][2] - r[i][3];
                        for (int j = 0; j < 2; ++j) {
                            const int64_t ow = 2 * tj + j;
                            if (ow >= ow_n) continue;
                            out[((n * p->k + k) * oh_n + oh) * ow_n + ow] = j ? y1 : y0;
                        }
                    }
                }
        }
    free(U);
    oc_quantize(out, p->n * p->k * oh_n * ow_n, bf16);
}

/* src/core/primitives.cpp:154-164 */
float oc_activation(int kind, float alpha, float v) {
    switch (kind) {
        case 0: return v > 0.0f ? v : 0.0f;
        case 1: return v > 0.0f ? v : alpha * v;
        case 2: return 1.0f / (1.0f + expf(-v));
        default: return tanhf(v);
    }
}

/* src/core/primitives.cpp:181-198 (ReLU'(0) = 0) */
float oc_activation_grad(int kind, float alpha, float v) {
    switch (kind) {
        case 0: return v > 0.0f ? 1.0f : 0.0f;
        case 1: return v > 0.0f ? 1.0f : alpha;
        case 2: {
            const float s = 1.0f / (1.0f + expf(-v));
            return s * (1.0f - s);
        }
        default: {
            const float t = tanhf(v);
            return 1.0f - t * t;
        }
    }
}

/* src/core/primitives.cpp:61-96 — training-mode batch-norm. mode 0 =
 * per-activation (stats per (c,h,w) over n), 1 = spatial (per c over n,h,w).
 * Sums in double, biased variance clamped at 0. */
void oc_bn_forward_train(int mode, const int64_t d[4], const float* x, const float* gamma,
                         const float* beta, float* rmean, float* rvar, float eps, float momentum,
                         float* y, float* smean, float* sinv, int bf16) {
    const int64_t N = d[0], Cc = d[1], HW = d[2] * d[3];
    const int64_t ns = mode == 0 ? Cc * HW : Cc;
    double* sum = (double*)calloc((size_t)ns, sizeof(double));
    double* sq = (double*)calloc((size_t)ns, sizeof(double));
    for (int64_t n = 0; n < N; ++n)
        for (int64_t c = 0; c < Cc; ++c)
            for (int64_t i = 0; i < HW; ++i) {
                const double v = x[(n * Cc + c) * HW + i];
                const int64_t si = mode == 0 ? c * HW + i : c;
                sum[si] += v;
                sq[si] += v * v;
            }
    const double m = mode == 0 ? (double)N : (double)(N * HW);
    for (int64_t si = 0; si < ns; ++si) {
        const double mu = sum[si] / m;
        double var = sq[si] / m - mu * mu;
        if (var < 0.0) var = 0.0;
        smean[si] = (float)mu;
        sinv[si] = (float)(1.0 / sqrt(var + eps));
        rmean[si] = (1.0f - momentum) * rmean[si] + momentum * (float)mu;
        rvar[si] = (1.0f - momentum) * rvar[si] + momentum * (float)var;
    }
    for (int64_t n = 0; n < N; ++n)
        for (int64_t c = 0; c < Cc; ++c)
            for (int64_t i = 0; i < HW; ++i) {
                const int64_t lin = (n * Cc + c) * HW + i;
                const int64_t si = mode == 0 ? c * HW + i : c;
                y[lin] = gamma[si] * (x[lin] - smean[si]) * sinv[si] + beta[si];
            }
    oc_quantize(y, N * Cc * HW, bf16);
    free(sum);
    free(sq);
}

/* src/core/primitives.cpp:98-111 — inference-mode batch-norm. */
void oc_bn_forward_infer(int mode, const int64_t d[4], const float* x, const float* gamma,
                         const float* beta, const float* rmean, const float* rvar, float eps,
                         float* y, int bf16) {
    const int64_t N = d[0], Cc = d[1], HW = d[2] * d[3];
    for (int64_t n = 0; n < N; ++n)
        for (int64_t c = 0; c < Cc; ++c)
            for (int64_t i = 0; i < HW; ++i) {
                const int64_t lin = (n * Cc + c) * HW + i;
                const int64_t si = mode == 0 ? c * HW + i : c;
                const float inv = 1.0f / sqrtf(rvar[si] + eps);
                y[lin] = gamma[si] * (x[lin] - rmean[si]) * inv + beta[si];
            }
    oc_quantize(y, N * Cc * HW, bf16);
}

/* src/core/primitives.cpp:113-152 — batch-norm backward. */
void oc_bn_backward(int mode, const int64_t d[4], const float* x, const float* dy,
                    const float* gamma, const float* smean, const float* sinv, float* dx,
                    float* dgamma, float* dbeta, int bf16) {
    const int64_t N = d[0], Cc = d[1], HW = d[2] * d[3];
    const int64_t ns = mode == 0 ? Cc * HW : Cc;
    double* db = (double*)calloc((size_t)ns, sizeof(double));
    double* dg = (double*)calloc((size_t)ns, sizeof(double));
    for (int64_t n = 0; n < N; ++n)
        for (int64_t c = 0; c < Cc; ++c)
            for (int64_t i = 0; i < HW; ++i) {
                const int64_t lin = (n * Cc + c) * HW + i;
                const int64_t si = mode == 0 ? c * HW + i : c;
                const double xhat = (double)((x[lin] - smean[si]) * sinv[si]);
                db[si] += dy[lin];
                dg[si] += dy[lin] * xhat;
            }
    const double m = mode == 0 ? (double)N : (double)(N * HW);
    for (int64_t n = 0; n < N; ++n)
        for (int64_t c = 0; c < Cc; ++c)
            for (int64_t i = 0; i < HW; ++i) {
                const int64_t lin = (n * Cc + c) * HW + i;
                const int64_t si = mode == 0 ? c * HW + i : c;
                const double xhat = (double)((x[lin] - smean[si]) * sinv[si]);
                dx[lin] = (float)((gamma[si] * sinv[si] / m) * (m * dy[lin] - db[si] - xhat * dg[si]));
            }
    for (int64_t si = 0; si < ns; ++si) {
        dgamma[si] = (float)dg[si];
        dbeta[si] = (float)db[si];
    }
    oc_quantize(dx, N * Cc * HW, bf16);
    oc_quantize(dgamma, ns, bf16);
    oc_quantize(dbeta, ns, bf16);
    free(db);
    free(dg);
}

/* src/core/fusion.cpp:384-398 — fused epilogue on one accumulator:
 * bias, then BN inference in the fused form (acc-mu)/sqrt(var+eps)*g+b,
 * then activation. Flags select the stages present in the plan. */
float oc_fused_epilogue(float acc, int has_bias, float bias, int has_bn, float mu, float var,
                        float gamma, float beta, float eps, int act, float alpha) {
    if (has_bias) acc += bias;
    if (has_bn) acc = (acc - mu) / sqrtf(var + eps) * gamma + beta;
    if (act >= 0) acc = oc_activation(act, alpha, acc);
    return acc;
}

/* ---- sampled direct formulas on the DEVICE layout (full-size parity) -----
 *
 * At BASELINE sizes (ResNet-50 / VGG-16 at N=128-256) the full CPU oracle is
 * minutes per layer, so the GPU result is checked on sampled coordinates
 * (>= 4096 output coordinates with the direct formula). These
 * evaluate the same sums as the reference's Direct kernels
 * (src/core/conv.cpp:99-133 forward, 702-799 backward data, 801-873 backward
 * weights; groups = 1, convolution mode) in double, reading the operands in
 * the device layout the GPU consumed: NHWC with channel pitch, filters
 * [K][R][S][pitch], element type bf16 (raw 16-bit) or f32. */
typedef struct {
    int64_t n, c, h, w, k, r, s, p, q;
    int64_t pad_h, pad_w, str_h, str_w, dil_h, dil_w;
    int64_t xp, yp, fp; /* channel pitches of x, y and the filter rows */
    int64_t bf16;
} oc_dev;

static inline double oc_ld(const void* base, int64_t i, int bf16) {
    if (!bf16) return ((const float*)base)[i];
    uint32_t u = (uint32_t)((const uint16_t*)base)[i] << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* forward: idx = ns x (n, k, oh, ow) */
void oc_sample_fwd(const oc_dev* g, const void* x, const void* w, const int64_t* idx, int64_t ns,
                   double* ref) {
    const int b = (int)g->bf16;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < ns; ++i) {
        const int64_t n = idx[4 * i], k = idx[4 * i + 1], oh = idx[4 * i + 2], ow = idx[4 * i + 3];
        double acc = 0.0;
        for (int64_t r = 0; r < g->r; ++r) {
            const int64_t ih = oh * g->str_h - g->pad_h + r * g->dil_h;
            if (ih < 0 || ih >= g->h) continue;
            for (int64_t s = 0; s < g->s; ++s) {
                const int64_t iw = ow * g->str_w - g->pad_w + s * g->dil_w;
                if (iw < 0 || iw >= g->w) continue;
                const int64_t xo = ((n * g->h + ih) * g->w + iw) * g->xp;
                const int64_t wo = ((k * g->r + r) * g->s + s) * g->fp;
                for (int64_t c = 0; c < g->c; ++c) acc += oc_ld(x, xo + c, b) * oc_ld(w, wo + c, b);
            }
        }
        ref[i] = acc;
    }
}

/* backward data: idx = ns x (n, c, h, w); dX[n,c,h,w] = sum over (k, r, s)
 * with oh*str = h + pad - r*dil (exact division) of dY[n,k,oh,ow] W[k,c,r,s] */
void oc_sample_dgrad(const oc_dev* g, const void* dy, const void* w, const int64_t* idx, int64_t ns,
                     double* ref) {
    const int b = (int)g->bf16;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < ns; ++i) {
        const int64_t n = idx[4 * i], c = idx[4 * i + 1], h = idx[4 * i + 2], wq = idx[4 * i + 3];
        double acc = 0.0;
        for (int64_t r = 0; r < g->r; ++r) {
            const int64_t th = h + g->pad_h - r * g->dil_h;
            if (th < 0 || th % g->str_h) continue;
            const int64_t oh = th / g->str_h;
            if (oh >= g->p) continue;
            for (int64_t s = 0; s < g->s; ++s) {
                const int64_t tw = wq + g->pad_w - s * g->dil_w;
                if (tw < 0 || tw % g->str_w) continue;
                const int64_t ow = tw / g->str_w;
                if (ow >= g->q) continue;
                const int64_t yo = ((n * g->p + oh) * g->q + ow) * g->yp;
                for (int64_t k = 0; k < g->k; ++k)
                    acc += oc_ld(dy, yo + k, b) * oc_ld(w, ((k * g->r + r) * g->s + s) * g->fp + c, b);
            }
        }
        ref[i] = acc;
    }
}

/* backward weights on a (ks x taps) grid: ref[a * nt + t] = dW[ks[a], tap t]
 * with tap t = (r, s, c) = taps[3t..3t+2]; sums over every (n, oh, ow). */
void oc_sample_wgrad(const oc_dev* g, const void* dy, const void* x, const int64_t* ks, int64_t nk,
                     const int64_t* taps, int64_t nt, double* ref) {
    const int b = (int)g->bf16;
    memset(ref, 0, sizeof(double) * nk * nt);
#pragma omp parallel
    {
        double* acc = (double*)calloc((size_t)(nk * nt), sizeof(double));
        double* dv = (double*)malloc(sizeof(double) * nk);
        double* xv = (double*)malloc(sizeof(double) * nt);
#pragma omp for schedule(dynamic, 1)
        for (int64_t n = 0; n < g->n; ++n)
            for (int64_t oh = 0; oh < g->p; ++oh)
                for (int64_t ow = 0; ow < g->q; ++ow) {
                    const int64_t yo = ((n * g->p + oh) * g->q + ow) * g->yp;
                    for (int64_t a = 0; a < nk; ++a) dv[a] = oc_ld(dy, yo + ks[a], b);
                    for (int64_t t = 0; t < nt; ++t) {
                        const int64_t ih = oh * g->str_h - g->pad_h + taps[3 * t] * g->dil_h;
                        const int64_t iw = ow * g->str_w - g->pad_w + taps[3 * t + 1] * g->dil_w;
                        xv[t] = (ih < 0 || ih >= g->h || iw < 0 || iw >= g->w)
                                    ? 0.0
                                    : oc_ld(x, ((n * g->h + ih) * g->w + iw) * g->xp + taps[3 * t + 2], b);
                    }
                    for (int64_t a = 0; a < nk; ++a) {
                        const double d = dv[a];
                        double* row = acc + a * nt;
                        for (int64_t t = 0; t < nt; ++t) row[t] += d * xv[t];
                    }
                }
#pragma omp critical
        for (int64_t i = 0; i < nk * nt; ++i) ref[i] += acc[i];
        free(acc);
        free(dv);
        free(xv);
    }
}

/* src/core/primitives.cpp:61-96 statistics (spatial mode) of a tensor in the
 * device layout [rows][pitch] (rows = N*H*W): double sums per channel,
 * mean = sum/m, biased var = max(0, E[x^2] - mean^2), invstd =
 * float(1/sqrt(var + eps)). */
void oc_bn_stats_dev(const void* x, int64_t rows, int64_t c, int64_t pitch, int64_t bf16, float eps,
                     float* mean, float* invstd, double* var) {
    double* sum = (double*)calloc((size_t)c, sizeof(double));
    double* sq = (double*)calloc((size_t)c, sizeof(double));
#pragma omp parallel
    {
        double* ls = (double*)calloc((size_t)c, sizeof(double));
        double* lq = (double*)calloc((size_t)c, sizeof(double));
#pragma omp for schedule(static)
        for (int64_t r = 0; r < rows; ++r)
            for (int64_t ch = 0; ch < c; ++ch) {
                const double v = oc_ld(x, r * pitch + ch, (int)bf16);
                ls[ch] += v;
                lq[ch] += v * v;
            }
#pragma omp critical
        for (int64_t ch = 0; ch < c; ++ch) {
            sum[ch] += ls[ch];
            sq[ch] += lq[ch];
        }
        free(ls);
        free(lq);
    }
    for (int64_t ch = 0; ch < c; ++ch) {
        const double mu = sum[ch] / (double)rows;
        double v = sq[ch] / (double)rows - mu * mu;
        if (v < 0.0) v = 0.0;
        mean[ch] = (float)mu;
        invstd[ch] = (float)(1.0 / sqrt(v + eps));
        var[ch] = v;
    }
    free(sum);
    free(sq);
}

/* src/core/primitives.cpp:204-260 — pooling forward, NCHW. kind 0 = max
 * (first maximum in window scan order, strict >; linear input index), 1 =
 * average (double sum of the valid taps / their count). Empty windows give 0
 * and index -1. win/pad/str = {h, w}. */
void oc_pool_fwd(int kind, const int64_t d[4], const int64_t win[2], const int64_t pad[2],
                 const int64_t str[2], const float* x, float* y, int64_t* idx, int bf16) {
    const int64_t N = d[0], Cc = d[1], H = d[2], W = d[3];
    const int64_t OH = (H + 2 * pad[0] - win[0]) / str[0] + 1, OW = (W + 2 * pad[1] - win[1]) / str[1] + 1;
    for (int64_t n = 0; n < N; ++n)
        for (int64_t c = 0; c < Cc; ++c)
            for (int64_t i = 0; i < OH; ++i)
                for (int64_t j = 0; j < OW; ++j) {
                    float best = -INFINITY;
                    int64_t bi = -1, count = 0;
                    double sum = 0.0;
                    for (int64_t p = 0; p < win[0]; ++p) {
                        const int64_t ih = i * str[0] - pad[0] + p;
                        if (ih < 0 || ih >= H) continue;
                        for (int64_t q = 0; q < win[1]; ++q) {
                            const int64_t iw = j * str[1] - pad[1] + q;
                            if (iw < 0 || iw >= W) continue;
                            const int64_t lin = ((n * Cc + c) * H + ih) * W + iw;
                            const float v = x[lin];
                            sum += v;
                            ++count;
                            if (v > best) {
                                best = v;
                                bi = lin;
                            }
                        }
                    }
                    const int64_t o = ((n * Cc + c) * OH + i) * OW + j;
                    if (kind == 0) {
                        y[o] = count ? best : 0.0f;
                        idx[o] = bi;
                    } else {
                        y[o] = count ? (float)(sum / (double)count) : 0.0f;
                        idx[o] = -1;
                    }
                    if (bf16) y[o] = oc_round_bf16(y[o]);
                }
}

/* src/core/primitives.cpp:262-310 — pooling backward (scatter in output
 * order, one rounding store per addition). dx must be zeroed by the caller. */
void oc_pool_bwd(int kind, const int64_t d[4], const int64_t win[2], const int64_t pad[2],
                 const int64_t str[2], const float* dy, const int64_t* idx, float* dx, int bf16) {
    const int64_t N = d[0], Cc = d[1], H = d[2], W = d[3];
    const int64_t OH = (H + 2 * pad[0] - win[0]) / str[0] + 1, OW = (W + 2 * pad[1] - win[1]) / str[1] + 1;
    if (kind == 0) {
        for (int64_t o = 0; o < N * Cc * OH * OW; ++o)
            if (idx[o] >= 0) {
                dx[idx[o]] += dy[o];
                if (bf16) dx[idx[o]] = oc_round_bf16(dx[idx[o]]);
            }
        return;
    }
    for (int64_t n = 0; n < N; ++n)
        for (int64_t c = 0; c < Cc; ++c)
            for (int64_t i = 0; i < OH; ++i)
                for (int64_t j = 0; j < OW; ++j) {
                    int64_t count = 0;
                    for (int64_t p = 0; p < win[0]; ++p) {
                        const int64_t ih = i * str[0] - pad[0] + p;
                        if (ih < 0 || ih >= H) continue;
                        for (int64_t q = 0; q < win[1]; ++q) {
                            const int64_t iw = j * str[1] - pad[1] + q;
                            if (iw >= 0 && iw < W) ++count;
                        }
                    }
                    if (!count) continue;
                    const float g = dy[((n * Cc + c) * OH + i) * OW + j] / (float)count;
                    for (int64_t p = 0; p < win[0]; ++p) {
                        const int64_t ih = i * str[0] - pad[0] + p;
                        if (ih < 0 || ih >= H) continue;
                        for (int64_t q = 0; q < win[1]; ++q) {
                            const int64_t iw = j * str[1] - pad[1] + q;
                            if (iw < 0 || iw >= W) continue;
                            const int64_t lin = ((n * Cc + c) * H + ih) * W + iw;
                            dx[lin] += g;
                            if (bf16) dx[lin] = oc_round_bf16(dx[lin]);
                        }
                    }
                }
}

/* src/core/primitives.cpp:329-351 — softmax forward over [outer][axis][inner]. */
void oc_softmax_fwd(int64_t outer, int64_t axis, int64_t inner, const float* x, float* y, int bf16) {
    for (int64_t o = 0; o < outer; ++o)
        for (int64_t i = 0; i < inner; ++i) {
            const float* xc = x + o * axis * inner + i;
            float mx = xc[0];
            for (int64_t a = 1; a < axis; ++a) mx = xc[a * inner] > mx ? xc[a * inner] : mx;
            double den = 0.0;
            for (int64_t a = 0; a < axis; ++a) den += exp((double)(xc[a * inner] - mx));
            for (int64_t a = 0; a < axis; ++a) {
                float v = (float)(exp((double)(xc[a * inner] - mx)) / den);
                y[o * axis * inner + i + a * inner] = bf16 ? oc_round_bf16(v) : v;
            }
        }
}

/* src/core/primitives.cpp:353-370 — softmax backward. */
void oc_softmax_bwd(int64_t outer, int64_t axis, int64_t inner, const float* y, const float* dy, float* dx,
                    int bf16) {
    for (int64_t o = 0; o < outer; ++o)
        for (int64_t i = 0; i < inner; ++i) {
            const int64_t b = o * axis * inner + i;
            double dot = 0.0;
            for (int64_t a = 0; a < axis; ++a) dot += (double)dy[b + a * inner] * y[b + a * inner];
            for (int64_t a = 0; a < axis; ++a) {
                float v = (float)(y[b + a * inner] * ((double)dy[b + a * inner] - dot));
                dx[b + a * inner] = bf16 ? oc_round_bf16(v) : v;
            }
        }
}
