// ConvPlan execution: maps (direction, algorithm, element type, shape) onto
// the sm_100a kernel families and advances the op counters exactly as the
// reference's CPU kernels do (proj/src/core/conv.cpp and tensor.cpp:169-170).
//
//   direction  algo         f32 (SIMT fp32)              bf16 (tcgen05 when supported)
//   Forward    Direct       direct_fwd                   direct_fwd
//              Im2colGemm   im2col + SIMT GEMM / image   im2col + tcgen05 GEMM / image
//              Winograd     winograd_f23                 winograd_f23
//              FFT          fft (complex<float>, batched) fft
//              ImplicitGemm igemm_simt_tiled / _fwd      igemm_tc_fwd
//   (f32 Direct / ImplicitGemm forward, groups 1, pitch % 32 == 0: 3xTF32 tcgen05, tf32x3_tc_fwd)
//   BwdData    Direct       direct_bwd_data              direct_bwd_data
//              Im2colGemm   SIMT GEMM + col2im / image   igemm_tc_dgrad
//   BwdWeights Direct       direct_bwd_weights           direct_bwd_weights
//              Im2colGemm   im2col + SIMT GEMM / image   igemm_tc_wgrad (split-K)
#include <cstdlib>
#include <cstring>

#include "../cuda/kernels.h"
#include "handle.hpp"
#include "solver.hpp"

namespace primkit {

namespace {

int dtype_of(ElementType t) { return t == ElementType::BF16 ? PK_BF16 : PK_F32; }

pk_conv_geom make_geom(const ConvProblem& p) {
    const ConvShapes s = resolve_shapes(p.input_desc(), p.filter_desc(), p.conv_desc());
    pk_conv_geom g{};
    g.n = (int)s.n;
    g.c = (int)s.c;
    g.h = (int)s.h;
    g.w = (int)s.w;
    g.k = (int)s.k;
    g.r = (int)s.y;
    g.s = (int)s.x;
    g.p = (int)s.oh;
    g.q = (int)s.ow;
    g.pad_h = (int)p.pad_h;
    g.pad_w = (int)p.pad_w;
    g.str_h = (int)p.stride_h;
    g.str_w = (int)p.stride_w;
    g.dil_h = (int)p.dilation_h;
    g.dil_w = (int)p.dilation_w;
    g.groups = (int)s.groups;
    g.cg = (int)s.cg;
    g.kg = (int)s.kg;
    g.x_pitch = pk_pitch(g.c);
    g.y_pitch = pk_pitch(g.k);
    g.transpose = p.mode == ConvMode::Transpose ? 1 : 0;
    g.f_pitch = g.transpose ? pk_pitch(g.kg) : pk_pitch(g.cg);
    return g;
}

// Reference counter semantics per (direction, algorithm).
OpCounters counters_for(const ConvProblem& p, ConvAlgo algo) {
    const ConvShapes s = resolve_shapes(p.input_desc(), p.filter_desc(), p.conv_desc());
    using u64 = std::uint64_t;
    OpCounters c;
    c.buffer_roundtrips = 1;
    const u64 n = s.n, k = s.k, oh = s.oh, ow = s.ow, cg = s.cg, kg = s.kg, y = s.y, x = s.x,
              grp = s.groups, h = s.h, w = s.w, ch = s.c;
    switch (p.direction) {
        case ConvDirection::Forward:
            switch (algo) {
                case ConvAlgo::Direct:
                case ConvAlgo::ImplicitGemm: c.scalar_muls = n * k * oh * ow * cg * y * x; break;
                case ConvAlgo::Im2colGemm:
                    c.gemm_calls = n * grp;
                    if (p.mode == ConvMode::Transpose)
                        c.scalar_muls = n * grp * (kg * y * x) * (h * w) * cg;
                    else
                        c.scalar_muls = n * grp * kg * (oh * ow) * (cg * y * x);
                    break;
                case ConvAlgo::Winograd:
                    c.scalar_muls = n * k * ((oh + 1) / 2) * ((ow + 1) / 2) * cg * 16;
                    break;
                case ConvAlgo::FFT: break;
            }
            break;
        case ConvDirection::BackwardData:
            if (algo == ConvAlgo::Direct) {
                c.scalar_muls = n * ch * h * w * kg * y * x;
            } else {
                c.gemm_calls = n * grp;
                c.scalar_muls = n * grp * (cg * y * x) * (oh * ow) * kg;
            }
            break;
        case ConvDirection::BackwardWeights:
            if (algo == ConvAlgo::Direct) {
                c.scalar_muls = k * cg * y * x * n * oh * ow;
            } else {
                c.gemm_calls = n * grp;
                c.scalar_muls = n * grp * kg * (cg * y * x) * (oh * ow);
            }
            break;
    }
    return c;
}

const pk_tc_config kDefaultTc{};  // heuristics throughout

// Output tile of the bf16 tensor-core Winograd: F(2x2,3x3) as the reference
// (conv.cpp:269-365); PK_WINOGRAD_M=4 selects F(4x4,3x3).
int winograd_tile_m() {
    const char* v = std::getenv("PK_WINOGRAD_M");
    return v && std::atoi(v) == 4 ? 4 : 2;
}

// Workspace cap for the tensor-core Winograd (PK_WINOGRAD_WS bytes; tests use
// it to exercise the chunked path).
std::size_t winograd_ws(const pk_conv_geom& g, int m) {
    std::size_t wb = pk_winograd_tc_workspace(&g, m);
    if (const char* v = std::getenv("PK_WINOGRAD_WS")) {
        const std::size_t cap = std::strtoull(v, nullptr, 10);
        if (cap && cap < wb) wb = cap;
    }
    return wb;
}

std::size_t col_bytes(const pk_conv_geom& g, int dtype) {
    return (std::size_t)g.p * g.q * g.r * g.s * g.f_pitch * (dtype == PK_BF16 ? 2 : 4);
}

std::size_t align256(std::size_t v) { return (v + 255) / 256 * 256; }

// The per-image GEMM of the forward Im2colGemm path as a 1x1 "convolution"
// over the column matrix: pixels = P*Q, reduction = R*S*f_pitch.
pk_conv_geom gemm_as_1x1(const pk_conv_geom& g) {
    pk_conv_geom m{};
    m.n = 1;
    m.h = 1;
    m.w = g.p * g.q;
    m.p = 1;
    m.q = g.p * g.q;
    m.c = g.r * g.s * g.f_pitch;
    m.cg = m.c;
    m.k = g.kg;
    m.kg = g.kg;
    m.r = m.s = 1;
    m.str_h = m.str_w = m.dil_h = m.dil_w = 1;
    m.groups = 1;
    m.x_pitch = m.c;
    m.f_pitch = m.c;
    m.y_pitch = g.y_pitch;
    return m;
}

// ---- narrow-channel (stem) layers: dense (r,s,c) packing + plain TMA GEMMs --

bool stem_eligible(const pk_conv_geom& g, int dt, const pk_epilogue* epi) {
    return dt == PK_BF16 && g.groups == 1 && !g.transpose && g.x_pitch % 64 != 0 &&
           pk_tc_fwd_supported(&g) && !(epi && epi->bn_mean && epi->bn_per_activation);
}

// A plain GEMM [rows][kred] x [kout][kred]^T as a 1x1 convolution geometry.
pk_conv_geom gemm_geom(long long rows, int kred, int kout) {
    pk_conv_geom m{};
    m.n = 1;
    m.h = m.p = 1;
    m.w = m.q = static_cast<int>(rows);
    m.c = m.cg = kred;
    m.k = m.kg = kout;
    m.r = m.s = 1;
    m.str_h = m.str_w = m.dil_h = m.dil_w = 1;
    m.groups = 1;
    m.x_pitch = m.f_pitch = kred;
    m.y_pitch = pk_pitch(kout);
    return m;
}

// Fused stem kernels (halo staged in smem, operand expanded on chip):
// forward and backward-weights. PK_STEM_FUSED=0 selects the packing path.
bool stem_fused(const pk_conv_geom& g, ConvDirection dir) {
    static const bool enabled = [] {
        const char* v = std::getenv("PK_STEM_FUSED");
        return !(v && v[0] == '0');
    }();
    if (!enabled) return false;
    return dir == ConvDirection::BackwardData ? pk_cuda_stem_fused_dgrad_supported(&g) != 0
                                              : pk_cuda_stem_fused_supported(&g) != 0;
}

std::size_t stem_workspace(const pk_conv_geom& g, ConvDirection dir, int num_sms) {
    if (stem_fused(g, dir))
        return dir == ConvDirection::BackwardWeights ? pk_cuda_stem_fused_wgrad_workspace(&g, num_sms) : 0;
    const std::size_t kcp = pk_stem_kc_pitch(&g);
    const std::size_t rows = (std::size_t)g.n * g.p * g.q;
    const std::size_t col = align256(rows * kcp * 2);
    switch (dir) {
        case ConvDirection::Forward: return col + align256((std::size_t)g.k * kcp * 2);
        case ConvDirection::BackwardData: return col + align256(kcp * pk_pitch(g.k) * 2);
        default: {
            const pk_conv_geom wg = gemm_geom((long long)rows, (int)kcp, g.k);
            return col + align256((std::size_t)g.k * kcp * 2) + pk_tc_wgrad_workspace(&wg, num_sms, &kDefaultTc);
        }
    }
}

void run_stem(const pk_conv_geom& g, ConvDirection dir, const void* a, const void* b, void* out,
              void* ws, const pk_epilogue* epi, int num_sms, cudaStream_t st) {
    auto ck = [](cudaError_t e, const char* what) { check_cuda(e, what); };
    const int kcp = pk_stem_kc_pitch(&g);
    const long long rows = (long long)g.n * g.p * g.q;
    char* col = static_cast<char*>(ws);
    char* aux = col + align256((std::size_t)rows * kcp * 2);
    if (stem_fused(g, dir)) {
        if (dir == ConvDirection::Forward)
            ck(pk_cuda_stem_fused_fprop(&g, a, b, out, epi, st), "stem_fused_fprop");
        else if (dir == ConvDirection::BackwardData)
            ck(pk_cuda_stem_fused_dgrad(&g, a, b, out, st), "stem_fused_dgrad");
        else
            ck(pk_cuda_stem_fused_wgrad(&g, a, b, out, ws, num_sms, st), "stem_fused_wgrad");
        return;
    }
    if (dir == ConvDirection::Forward) {
        // y = col . Wp^T
        ck(pk_cuda_im2col_pack(&g, a, col, st), "im2col_pack");
        ck(pk_cuda_filter_pack(&g, b, aux, 0, st), "filter_pack");
        pk_conv_geom m = gemm_geom(rows, kcp, g.k);
        ck(pk_cuda_igemm_tc_fwd(&m, col, aux, out, epi, &kDefaultTc, st), "stem_gemm");
    } else if (dir == ConvDirection::BackwardData) {
        // colg = dY . Wp (B = Wp^T as [kcp][pitch K]); dX = col2im(colg)
        ck(pk_cuda_filter_pack(&g, b, aux, 1, st), "filter_pack_t");
        pk_conv_geom m = gemm_geom(rows, pk_pitch(g.k), kcp);
        ck(pk_cuda_igemm_tc_fwd(&m, a, aux, col, nullptr, &kDefaultTc, st), "stem_dgrad_gemm");
        ck(pk_cuda_col2im_pack(&g, col, out, st), "col2im_pack");
    } else {
        // dWp = dY^T . col, then unpack to the filter layout
        ck(pk_cuda_im2col_pack(&g, b, col, st), "im2col_pack");
        pk_conv_geom wg = gemm_geom(rows, kcp, g.k);
        wg.y_pitch = g.y_pitch;
        char* wtmp = aux + align256((std::size_t)g.k * kcp * 2);
        ck(pk_cuda_igemm_tc_wgrad(&wg, a, col, aux, wtmp, num_sms, &kDefaultTc, st), "stem_wgrad");
        ck(pk_cuda_wgrad_unpack(&g, aux, out, st), "wgrad_unpack");
    }
}

}  // namespace

OpCounters conv_counters(const ConvProblem& p, ConvAlgo algo) { return counters_for(p, algo); }

bool ConvPlan::fuses_stats() const {
    const pk_conv_geom g = make_geom(problem_);
    if (problem_.etype != ElementType::BF16 || g.transpose || g.groups != 1) return false;
    if (problem_.direction == ConvDirection::Forward)
        return algo_ == ConvAlgo::ImplicitGemm && pk_tc_fwd_supported(&g);
    if (problem_.direction == ConvDirection::BackwardData)
        return algo_ == ConvAlgo::Im2colGemm && !stem_eligible(g, PK_BF16, nullptr) &&
               pk_tc_dgrad_supported(&g);
    return false;
}

// fp32 forward convolutions (Direct / ImplicitGemm, groups 1) run as 3xTF32 tensor-core
// GEMMs when the channel pitch allows (fp32-level accuracy; PK_TF32X3=0: SIMT kernels).
bool tf32x3_eligible(const pk_conv_geom& g, int dt) {
    static const bool off = [] {
        const char* v = std::getenv("PK_TF32X3");
        return v && v[0] == '0';
    }();
    return !off && dt == PK_F32 && !pk_depthwise_supported(&g) && !pk_grouped_supported(&g) &&
           pk_tf32x3_fwd_supported(&g);
}

std::size_t ConvPlan::device_workspace_bytes(int num_sms) const {
    // Every device buffer run() touches besides its operands comes out of the
    // caller's workspace, so this mirrors run()'s dispatch exactly. Split-K
    // partial counts scale with the SM count, hence the handle's num_sms.
    const pk_conv_geom g = make_geom(problem_);
    const int dt = dtype_of(problem_.etype);
    const std::size_t acc_rows = (std::size_t)g.p * g.q;
    const bool tc_algo = problem_.direction == ConvDirection::Forward
                             ? algo_ == ConvAlgo::ImplicitGemm
                             : algo_ == ConvAlgo::Im2colGemm;
    if (tc_algo && stem_eligible(g, dt, nullptr)) return stem_workspace(g, problem_.direction, num_sms);
    switch (problem_.direction) {
        case ConvDirection::Forward:
            if ((algo_ == ConvAlgo::Direct || algo_ == ConvAlgo::ImplicitGemm ||
                 (algo_ == ConvAlgo::Im2colGemm && !g.transpose)) &&
                tf32x3_eligible(g, dt))
                return pk_tf32x3_fwd_workspace(&g);
            if (algo_ == ConvAlgo::FFT) return pk_cuda_fft_scratch_bytes(&g);
            if (algo_ == ConvAlgo::Winograd && dt == PK_BF16 && pk_winograd_tc_supported(&g))
                return winograd_ws(g, winograd_tile_m());
            if (algo_ == ConvAlgo::Im2colGemm) {
                if (pk_depthwise_supported(&g) || pk_grouped_supported(&g)) return 0;
                if (g.transpose)  // fp32 column matrix [(r,s,kk)][h*w]
                    return (std::size_t)g.r * g.s * g.f_pitch * g.h * g.w * 4;
                return align256(col_bytes(g, dt)) + acc_rows * g.kg * 4;
            }
            return 0;
        case ConvDirection::BackwardData:
            if (algo_ == ConvAlgo::Im2colGemm) {
                if (pk_depthwise_supported(&g) || pk_grouped_supported(&g)) return 0;
                if (dt == PK_BF16 && pk_tc_dgrad_supported(&g)) return pk_tc_dgrad_workspace(&g);
                return (std::size_t)g.p * g.q * g.r * g.s * g.f_pitch * 4;
            }
            return 0;
        case ConvDirection::BackwardWeights:
            if (pk_depthwise_supported(&g)) return pk_depthwise_wgrad_workspace(&g, num_sms);
            if (pk_grouped_wgrad_supported(&g)) return pk_grouped_wgrad_workspace(&g, num_sms);
            if (algo_ == ConvAlgo::Direct)
                return pk_direct_wgrad_tiled_supported(&g) ? pk_direct_wgrad_tiled_workspace(&g, num_sms)
                                                           : 0;
            if (algo_ == ConvAlgo::Im2colGemm) {
                if (dt == PK_BF16 && pk_tc_wgrad_supported(&g))
                    return pk_tc_wgrad_workspace(&g, num_sms, &kcfg_);
                return align256(col_bytes(g, dt)) + (std::size_t)g.k * g.r * g.s * g.f_pitch * 4;
            }
            return 0;
    }
    return 0;
}

void ConvPlan::run(Handle& h, const void* a, const void* b, void* out, void* ws,
                   std::size_t ws_bytes, const pk_epilogue* epi) const {
    static const char* const kRange[3] = {"primkit conv forward", "primkit conv backward-data",
                                          "primkit conv backward-weights"};
    const NvtxRange range(kRange[static_cast<int>(problem_.direction)]);
    h.activate();
    const pk_conv_geom g = make_geom(problem_);
    const int dt = dtype_of(problem_.etype);
    const std::size_t esz = dt == PK_BF16 ? 2 : 4;
    cudaStream_t st = h.stream();
    if (ws_bytes < device_workspace_bytes(h.num_sms()))
        throw_error(ErrorCode::WorkspaceTooSmall, "workspace below requested size");
    auto ck = [](cudaError_t e, const char* what) { check_cuda(e, what); };

    const ConvDirection dir = problem_.direction;
    // Output channels beyond K (pitch padding) must hold zeros for the next
    // consumer; only non-multiple-of-8 channel counts have such lanes.
    if (dir == ConvDirection::Forward && g.y_pitch != g.k)
        ck(cudaMemsetAsync(out, 0, (std::size_t)g.n * g.p * g.q * g.y_pitch * esz, st), "memset");
    if (dir == ConvDirection::BackwardData && g.x_pitch != g.c)
        ck(cudaMemsetAsync(out, 0, (std::size_t)g.n * g.h * g.w * g.x_pitch * esz, st), "memset");

    const char* kernel = "?";
    pk_cuda_variant_reset();
    if (dir == ConvDirection::Forward) {
        switch (algo_) {
            case ConvAlgo::Direct:
                if (pk_depthwise_supported(&g)) {
                    kernel = "depthwise_simt";
                    ck(pk_cuda_depthwise_fwd(&g, dt, a, b, out, epi, h.num_sms(), st), "depthwise_fwd");
                    break;
                }
                if (pk_grouped_supported(&g)) {
                    kernel = "grouped_simt";
                    ck(pk_cuda_grouped_fwd(&g, dt, a, b, out, epi, h.num_sms(), st), "grouped_fwd");
                    break;
                }
                if (g.transpose && g.groups == 1 && g.dil_h == 1 && g.dil_w == 1 && !epi) {
                    // transpose-mode forward = backward data of the convolution whose
                    // output grid is x: swap the roles of (c, h, w) and (k, p, q); the
                    // transpose filter [C][R][S][pitch(K)] is that convolution's filter
                    pk_conv_geom d = g;
                    d.c = g.k; d.h = g.p; d.w = g.q;
                    d.k = g.c; d.p = g.h; d.q = g.w;
                    d.cg = g.kg; d.kg = g.cg;
                    d.x_pitch = g.y_pitch; d.y_pitch = g.x_pitch;
                    d.transpose = 0;
                    if (pk_direct_dgrad_tiled_supported(&d)) {
                        kernel = "direct_simt_tiled_transpose";
                        ck(pk_cuda_direct_dgrad_tiled(&d, dt, a, b, out, st), "direct_transpose_tiled");
                        break;
                    }
                }
                if (tf32x3_eligible(g, dt)) {
                    kernel = "tf32x3_tc_fwd";
                    ck(pk_cuda_tf32x3_fwd(&g, a, b, out, epi, ws, ws_bytes, st), "tf32x3_fwd");
                    break;
                }
                kernel = "direct_simt";
                ck(pk_cuda_direct_fwd(&g, dt, a, b, out, epi, st), "direct_fwd");
                break;
            case ConvAlgo::Winograd:
                if (dt == PK_BF16 && pk_winograd_tc_supported(&g)) {
                    // tensor-core Winograd: transforms + alpha^2 batched tcgen05 GEMMs
                    const int m = winograd_tile_m();
                    kernel = m == 4 ? "winograd_tc_f43" : "winograd_tc_f23";
                    const std::size_t wb = winograd_ws(g, m);
                    ck(pk_cuda_winograd_tc(&g, m, a, b, out, epi, ws, wb, st),
                       "winograd_tc");
                } else {
                    kernel = "winograd_f23";
                    ck(pk_cuda_winograd_f23(&g, dt, a, b, out, epi, st), "winograd_f23");
                }
                break;
            case ConvAlgo::FFT:
                kernel = "fft";
                ck(pk_cuda_fft_fwd(&g, dt, a, b, out, ws, st), "fft_fwd");
                break;
            case ConvAlgo::ImplicitGemm: {
                // Narrow-channel stems: dense (r,s,c) packing + plain GEMM
                // measured faster (1.28 ms) than 16-byte-row TMA boxes
                // (1.69 ms) for ResNet conv1 at N=256.
                if (stem_eligible(g, dt, epi)) {
                    kernel = stem_fused(g, dir) ? "stem_fused_tc" : "stem_pack+gemm_tc";
                    run_stem(g, dir, a, b, out, ws, epi, h.num_sms(), st);
                } else if (dt == PK_BF16 && pk_tc_fwd_supported(&g)) {
                    kernel = "igemm_tc_fwd";
                    ck(pk_cuda_igemm_tc_fwd(&g, a, b, out, epi, &kcfg_, st), "igemm_tc_fwd");
                } else if (pk_depthwise_supported(&g)) {
                    kernel = "depthwise_simt";
                    ck(pk_cuda_depthwise_fwd(&g, dt, a, b, out, epi, h.num_sms(), st), "depthwise_fwd");
                } else if (pk_grouped_supported(&g)) {
                    kernel = "grouped_simt";
                    ck(pk_cuda_grouped_fwd(&g, dt, a, b, out, epi, h.num_sms(), st), "grouped_fwd");
                } else if (tf32x3_eligible(g, dt)) {
                    kernel = "tf32x3_tc_fwd";
                    ck(pk_cuda_tf32x3_fwd(&g, a, b, out, epi, ws, ws_bytes, st), "tf32x3_fwd");
                } else {
                    if (g.groups == 1 && !g.transpose && g.x_pitch % 8 == 0 && g.f_pitch == g.x_pitch) {
                        // register-tiled implicit GEMM on CUDA cores (64 px x 64 k per CTA,
                        // smem-staged taps): 2.2x the column-gather SIMT kernel on cfg1
                        kernel = "igemm_simt_tiled";
                        ck(pk_cuda_direct_fwd(&g, dt, a, b, out, epi, st), "igemm_simt_tiled");
                    } else {
                        kernel = "igemm_simt_fwd";
                        ck(pk_cuda_igemm_simt_fwd(&g, dt, a, b, out, epi, st), "igemm_simt_fwd");
                    }
                }
                break;
            }
            case ConvAlgo::Im2colGemm: {
                // Depthwise / grouped: the per-(image, group) GEMMs degenerate to one
                // or a few rows, so the channel-vector kernels compute the same sums.
                if (pk_depthwise_supported(&g)) {
                    kernel = "depthwise_simt";
                    ck(pk_cuda_depthwise_fwd(&g, dt, a, b, out, epi, h.num_sms(), st), "depthwise_fwd");
                    break;
                }
                if (pk_grouped_supported(&g)) {
                    kernel = "grouped_simt";
                    ck(pk_cuda_grouped_fwd(&g, dt, a, b, out, epi, h.num_sms(), st), "grouped_fwd");
                    break;
                }
                if (g.transpose) {
                    // col[(r,s,kk)][hw] = W_g^T X_g ; then gather into the output
                    kernel = "im2col_gemm_transpose";
                    float* col = static_cast<float*>(ws);
                    const long long rows = (long long)g.r * g.s * g.f_pitch, hw = (long long)g.h * g.w;
                    for (int n = 0; n < g.n; ++n)
                        for (int grp = 0; grp < g.groups; ++grp) {
                            const char* wg = (const char*)b + (size_t)grp * g.cg * rows * esz;
                            const char* xg = (const char*)a +
                                             ((size_t)n * hw * g.x_pitch + (size_t)grp * g.cg) * esz;
                            ck(pk_cuda_gemm_simt((int)rows, (int)hw, g.cg, dt, wg, 1, rows, xg, 1,
                                                 g.x_pitch, col, hw, 0, st),
                               "gemm_simt");
                            ck(pk_cuda_col2im_transpose(&g, dt, col, n, grp, out, st), "col2im_t");
                        }
                    break;
                }
                if (tf32x3_eligible(g, dt)) {
                    // fp32: the column matrix formed on the fly by TMA (implicit im2col)
                    // and one 3xTF32 tensor-core GEMM instead of the per-image SIMT GEMMs
                    kernel = "tf32x3_tc_fwd";
                    ck(pk_cuda_tf32x3_fwd(&g, a, b, out, epi, ws, ws_bytes, st), "tf32x3_fwd");
                    break;
                }
                const bool tc = dt == PK_BF16 && pk_tc_fwd_supported(&g);
                kernel = tc ? "im2col+gemm_tc" : "im2col+gemm_simt";
                void* col = ws;
                float* acc = reinterpret_cast<float*>(static_cast<char*>(ws) + align256(col_bytes(g, dt)));
                const pk_conv_geom m = gemm_as_1x1(g);
                const long long kred = (long long)g.r * g.s * g.f_pitch;
                for (int n = 0; n < g.n; ++n)
                    for (int grp = 0; grp < g.groups; ++grp) {
                        ck(pk_cuda_im2col(&g, dt, a, n, grp, col, st), "im2col");
                        char* yg = (char*)out + ((size_t)n * g.p * g.q * g.y_pitch + (size_t)grp * g.kg) * esz;
                        const char* wg = (const char*)b + (size_t)grp * g.kg * kred * esz;
                        if (tc) {
                            pk_epilogue e{};
                            e.act = -1;
                            if (epi) {
                                e = *epi;
                                if (e.bias) e.bias += grp * g.kg;
                            }
                            ck(pk_cuda_igemm_tc_fwd(&m, col, wg, yg, epi ? &e : nullptr, &kDefaultTc, st),
                               "gemm_tc");
                        } else {
                            ck(pk_cuda_gemm_simt(g.p * g.q, g.kg, (int)kred, dt, col, kred, 1, wg, 1,
                                                 kred, acc, g.kg, 0, st),
                               "gemm_simt");
                            pk_epilogue e{};
                            e.act = -1;
                            if (epi) e = *epi;
                            ck(pk_cuda_store_rows(acc, g.p * g.q, g.kg, g.kg, yg, g.y_pitch, dt,
                                                  epi ? &e : nullptr, grp * g.kg, st),
                               "store_rows");
                        }
                    }
                break;
            }
        }
    } else if (dir == ConvDirection::BackwardData) {
        if (algo_ != ConvAlgo::Winograd && algo_ != ConvAlgo::FFT && pk_depthwise_supported(&g)) {
            kernel = "depthwise_simt_bwd_data";
            ck(pk_cuda_depthwise_bwd_data(&g, dt, a, b, out, h.num_sms(), st), "depthwise_bwd_data");
        } else if (algo_ != ConvAlgo::Winograd && algo_ != ConvAlgo::FFT && pk_grouped_supported(&g)) {
            kernel = "grouped_simt_bwd_data";
            ck(pk_cuda_grouped_bwd_data(&g, dt, a, b, out, h.num_sms(), st), "grouped_bwd_data");
        } else if (algo_ == ConvAlgo::Direct && pk_direct_dgrad_tiled_supported(&g)) {
            kernel = "direct_simt_tiled_bwd_data";
            ck(pk_cuda_direct_dgrad_tiled(&g, dt, a, b, out, st), "direct_dgrad_tiled");
        } else if (algo_ == ConvAlgo::Direct) {
            kernel = "direct_simt_bwd_data";
            ck(pk_cuda_direct_bwd_data(&g, dt, a, b, out, st), "direct_bwd_data");
        } else if (stem_eligible(g, dt, nullptr)) {
            kernel = stem_fused(g, dir) ? "stem_fused_dgrad_tc" : "stem_gemm_tc+col2im";
            run_stem(g, dir, a, b, out, ws, nullptr, h.num_sms(), st);
        } else if (dt == PK_BF16 && pk_tc_dgrad_supported(&g)) {
            kernel = "igemm_tc_dgrad";
            ck(pk_cuda_igemm_tc_dgrad(&g, a, b, out, ws, &kcfg_, st,
                                      (epi && epi->stats) ? epi : nullptr),
               "igemm_tc_dgrad");
        } else {
            kernel = "gemm_simt+col2im";
            float* col = static_cast<float*>(ws);
            const long long rowp = (long long)g.r * g.s * g.f_pitch;
            for (int n = 0; n < g.n; ++n)
                for (int grp = 0; grp < g.groups; ++grp) {
                    const char* dyg = (const char*)a +
                                      ((size_t)n * g.p * g.q * g.y_pitch + (size_t)grp * g.kg) * esz;
                    const char* wg = (const char*)b + (size_t)grp * g.kg * rowp * esz;
                    ck(pk_cuda_gemm_simt(g.p * g.q, (int)rowp, g.kg, dt, dyg, g.y_pitch, 1, wg,
                                         rowp, 1, col, rowp, 0, st),
                       "gemm_simt");
                    ck(pk_cuda_col2im(&g, dt, col, n, grp, out, st), "col2im");
                }
        }
    } else {
        if (algo_ != ConvAlgo::Winograd && algo_ != ConvAlgo::FFT && pk_depthwise_supported(&g)) {
            kernel = "depthwise_simt_bwd_weights";
            const std::size_t wb = pk_depthwise_wgrad_workspace(&g, h.num_sms());
            ck(pk_cuda_depthwise_wgrad(&g, dt, a, b, out, ws, wb, h.num_sms(), st),
               "depthwise_wgrad");
        } else if (algo_ != ConvAlgo::Winograd && algo_ != ConvAlgo::FFT && pk_grouped_wgrad_supported(&g)) {
            kernel = "grouped_simt_bwd_weights";
            const std::size_t wb = pk_grouped_wgrad_workspace(&g, h.num_sms());
            ck(pk_cuda_grouped_wgrad(&g, dt, a, b, out, ws, wb, h.num_sms(), st),
               "grouped_wgrad");
        } else if (algo_ == ConvAlgo::Direct && pk_direct_wgrad_tiled_supported(&g)) {
            kernel = "direct_simt_tiled_bwd_weights";
            const std::size_t wb = pk_direct_wgrad_tiled_workspace(&g, h.num_sms());
            ck(pk_cuda_direct_wgrad_tiled(&g, dt, a, b, out, ws, wb, h.num_sms(), st),
               "direct_wgrad_tiled");
        } else if (algo_ == ConvAlgo::Direct) {
            kernel = "direct_simt_bwd_weights";
            ck(pk_cuda_direct_bwd_weights(&g, dt, a, b, out, st), "direct_bwd_weights");
        } else if (stem_eligible(g, dt, nullptr)) {
            kernel = stem_fused(g, dir) ? "stem_fused_wgrad_tc" : "stem_pack+wgrad_tc";
            run_stem(g, dir, a, b, out, ws, nullptr, h.num_sms(), st);
        } else if (dt == PK_BF16 && pk_tc_wgrad_supported(&g)) {
            kernel = "igemm_tc_wgrad";
            ck(pk_cuda_igemm_tc_wgrad(&g, a, b, out, ws, h.num_sms(), &kcfg_, st),
               "igemm_tc_wgrad");
        } else {
            kernel = "im2col+gemm_simt_wgrad";
            void* col = ws;
            float* acc = reinterpret_cast<float*>(static_cast<char*>(ws) + align256(col_bytes(g, dt)));
            const long long rowp = (long long)g.r * g.s * g.f_pitch;
            for (int n = 0; n < g.n; ++n)
                for (int grp = 0; grp < g.groups; ++grp) {
                    ck(pk_cuda_im2col(&g, dt, b, n, grp, col, st), "im2col");
                    const char* dyg = (const char*)a +
                                      ((size_t)n * g.p * g.q * g.y_pitch + (size_t)grp * g.kg) * esz;
                    ck(pk_cuda_gemm_simt(g.kg, (int)rowp, g.p * g.q, dt, dyg, 1, g.y_pitch, col,
                                         rowp, 1, acc + (size_t)grp * g.kg * rowp, rowp, n > 0, st),
                       "gemm_simt");
                }
            ck(pk_cuda_store_rows(acc, g.k, (int)rowp, rowp, out, rowp, dt, nullptr, 0, st),
               "store_rows");
        }
    }
    h.last_kernel = kernel;
    h.last_variant = pk_cuda_variant();
    h.counters() += counters_for(problem_, algo_);
}

OpCounters ConvPlan::op_counters() const { return counters_for(problem_, algo_); }

}  // namespace primkit
