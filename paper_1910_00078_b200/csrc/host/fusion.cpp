#include "fusion.hpp"

#include <cmath>

#include "../cuda/kernels.h"

namespace primkit {

FusionOp FusionOp::conv_forward(ConvDescriptor conv, TensorDescriptor filter, ConvAlgo algo) {
    FusionOp op;
    op.kind = Kind::ConvForward;
    op.conv = conv;
    op.filter_desc = std::move(filter);
    op.algo = algo;
    return op;
}

FusionOp FusionOp::bias(std::int64_t channels) {
    FusionOp op;
    op.kind = Kind::Bias;
    op.bias_channels = channels;
    return op;
}

FusionOp FusionOp::batchnorm_inference(BatchNormMode mode) {
    FusionOp op;
    op.kind = Kind::BatchNormInference;
    op.bn_mode = mode;
    return op;
}

FusionOp FusionOp::activation(ActivationKind kind) {
    FusionOp op;
    op.kind = Kind::Activation;
    op.act = kind;
    return op;
}

struct FusionPlan::DeviceArgs {
    const Handle* owner = nullptr;
    bool valid = false;
    DeviceBuffer filter, bias, gamma, beta, mean, var;
    // bias and spatial BN folded into a per-channel affine for the tensor-core
    // epilogue: acc * scale[k] + shift[k] (padded to a multiple of 64 + 64)
    DeviceBuffer scale, shift;
    bool folded = false;
};

FusionPlan::FusionPlan(TensorDescriptor input_desc)
    : input_desc_(input_desc), cur_desc_(std::move(input_desc)) {
    if (input_desc_.rank() != 4) throw_error(ErrorCode::InvalidShape, "fusion input must be NCHW");
}

FusionPlan::~FusionPlan() = default;
FusionPlan::FusionPlan(FusionPlan&&) noexcept = default;

void FusionPlan::add_op(FusionOp op) {
    if (compiled_) throw_error(ErrorCode::AlreadyCompiled, "cannot add ops to a compiled plan");
    if (op.kind == FusionOp::Kind::ConvForward) {
        if (op.conv.mode != ConvMode::Convolution)
            throw_error(ErrorCode::InvalidValue, "fusion supports convolution mode only");
        cur_desc_ = output_dims(cur_desc_, op.filter_desc, op.conv);
    } else if (op.kind == FusionOp::Kind::Bias && op.bias_channels != cur_desc_.dims[1]) {
        throw_error(ErrorCode::ShapeMismatch, "bias channel count " +
                                                  std::to_string(op.bias_channels) +
                                                  " does not match " +
                                                  std::to_string(cur_desc_.dims[1]));
    }
    ops_.push_back(std::move(op));
}

void FusionPlan::set_args(FusionArgs args) {
    args_ = std::move(args);
    if (dev_) dev_->valid = false;
}

std::string FusionPlan::signature() const {
    std::string s = "fusion v1\n";
    for (std::int64_t d : input_desc_.dims) s += std::to_string(d) + ' ';
    s += element_type_name(input_desc_.etype);
    s += '\n';
    for (const FusionOp& op : ops_) {
        switch (op.kind) {
            case FusionOp::Kind::ConvForward:
                s += "conv ";
                s += conv_algo_name(op.algo);
                for (std::int64_t d : op.filter_desc.dims) s += ' ' + std::to_string(d);
                s += " p" + std::to_string(op.conv.pad_h) + ',' + std::to_string(op.conv.pad_w);
                s += " s" + std::to_string(op.conv.stride_h) + ',' + std::to_string(op.conv.stride_w);
                s += " d" + std::to_string(op.conv.dilation_h) + ',' +
                     std::to_string(op.conv.dilation_w);
                s += " g" + std::to_string(op.conv.group_count);
                break;
            case FusionOp::Kind::Bias: s += "bias " + std::to_string(op.bias_channels); break;
            case FusionOp::Kind::BatchNormInference:
                s += op.bn_mode == BatchNormMode::Spatial ? "bn spatial" : "bn peract";
                break;
            case FusionOp::Kind::Activation:
                s += "act " + std::to_string(static_cast<int>(op.act.tag));
                break;
        }
        s += '\n';
    }
    return s;
}

// ---- metadata graph (Tables I / II of the paper) --------

namespace {

enum Node : int { kStart, kConv, kConvBias, kConvBiasBn, kCba, kCbna, kNorm, kNa };

const FusionOp* conv_op(const FusionPlan& plan) {
    for (const FusionOp& op : plan.ops())
        if (op.kind == FusionOp::Kind::ConvForward) return &op;
    return nullptr;
}

using Verdict = std::optional<std::string>;

Verdict square(const FusionOp& conv, std::int64_t* f) {
    if (conv.filter_desc.dims[2] != conv.filter_desc.dims[3])
        return "fused convolutions require square filters";
    *f = conv.filter_desc.dims[2];
    return std::nullopt;
}

Verdict conv_entry(const FusionPlan& plan, std::size_t i) {
    const FusionOp& op = plan.ops()[i];
    if (op.conv.dilation_h != 1 || op.conv.dilation_w != 1)
        return "fused convolutions do not support dilation";
    if (op.algo != ConvAlgo::Direct && op.algo != ConvAlgo::Winograd)
        return std::string("algorithm ") + conv_algo_name(op.algo) + " has no fused variant";
    return std::nullopt;
}

// Winograd rows of Table I: minimum channel counts per filter size/stride.
Verdict winograd_row(std::int64_t f, std::int64_t stride, std::int64_t c) {
    if (stride == 1) {
        if (f <= 2) return c < 18 ? Verdict("filters up to 2x2 require c >= 18") : std::nullopt;
        if (f == 3)
            return (c < 18 || c % 2) ? Verdict("3x3 filters require c >= 18 and c even")
                                     : std::nullopt;
        if (f <= 6) return 4 * c < 18 ? Verdict("4x4 to 6x6 filters require 4c >= 18") : std::nullopt;
        if (f <= 9) return 12 * c < 18 ? Verdict("7x7 to 9x9 filters require 12c >= 18") : std::nullopt;
        if (f <= 12)
            return 16 * c < 18 ? Verdict("10x10 to 12x12 filters require 16c >= 18") : std::nullopt;
        return std::nullopt;
    }
    if (f == 1) return 2 * c < 18 ? Verdict("1x1 filters require 2c >= 18") : std::nullopt;
    if (f <= 6) return 4 * c < 18 ? Verdict("2x2 to 6x6 filters require 4c >= 18") : std::nullopt;
    if (f == 7) return 12 * c < 18 ? Verdict("7x7 filters require 12c >= 18") : std::nullopt;
    if (f <= 12) return 16 * c < 18 ? Verdict("8x8 to 12x12 filters require 16c >= 18") : std::nullopt;
    return std::nullopt;
}

Verdict cba_activation(const FusionPlan& plan, std::size_t i) {
    const FusionOp& act = plan.ops()[i];
    const FusionOp* conv = conv_op(plan);
    const std::int64_t c = plan.input_desc().dims[1] / conv->conv.group_count;
    std::int64_t f = 0;
    if (auto v = square(*conv, &f)) return v;
    if (conv->conv.stride_h != conv->conv.stride_w) return "fused convolutions require equal strides";
    const std::int64_t stride = conv->conv.stride_h;
    if (conv->algo == ConvAlgo::Direct) {
        if (f != 1) return "direct conv-bias-activation requires a 1x1 filter";
        if (stride != 1) return "direct conv-bias-activation does not support stride";
        if (conv->conv.pad_h != 0 || conv->conv.pad_w != 0)
            return "direct conv-bias-activation does not support padding";
        return std::nullopt;
    }
    if (plan.input_desc().etype == ElementType::BF16)
        return "bf16 conv-bias-activation supports the direct 1x1 row only";
    if (act.act.tag != ActivationKind::Tag::ReLU && act.act.tag != ActivationKind::Tag::LeakyReLU)
        return "winograd fusion supports ReLU and LeakyReLU activations only";
    if (stride != 1 && stride != 2) return "winograd fusion requires stride 1 or 2";
    return winograd_row(f, stride, c);
}

Verdict cbna_norm(const FusionPlan& plan, std::size_t) {
    const FusionOp* conv = conv_op(plan);
    if (conv->algo != ConvAlgo::Direct) return "conv-bias-norm-activation requires the direct algorithm";
    std::int64_t f = 0;
    if (auto v = square(*conv, &f)) return v;
    if (f != 3 && f != 5 && f != 7 && f != 9 && f != 11)
        return "conv-bias-norm-activation requires filter in {3x3,5x5,7x7,9x9,11x11}";
    const auto& cv = conv->conv;
    if (cv.stride_h != cv.stride_w || cv.stride_h < 1 || cv.stride_h > 2)
        return "conv-bias-norm-activation requires stride in {1,2}";
    if (cv.pad_h != cv.pad_w || cv.pad_h < 1 || cv.pad_h > 2)
        return "conv-bias-norm-activation requires padding in {1,2}";
    return std::nullopt;
}

Verdict na_norm(const FusionPlan& plan, std::size_t) {
    if (plan.input_desc().etype == ElementType::BF16) return "norm-activation fusion supports f32 only";
    return std::nullopt;  // host tensors are always packed
}

Verdict always(const FusionPlan&, std::size_t) { return std::nullopt; }

}  // namespace

MetadataGraph::MetadataGraph() {
    using K = FusionOp::Kind;
    edges_ = {
        {kStart, kConv, K::ConvForward, conv_entry},
        {kConv, kConvBias, K::Bias, always},
        {kConvBias, kCba, K::Activation, cba_activation},
        {kConvBias, kConvBiasBn, K::BatchNormInference, cbna_norm},
        {kConvBiasBn, kCbna, K::Activation, always},
        {kStart, kNorm, K::BatchNormInference, na_norm},
        {kNorm, kNa, K::Activation, always},
    };
    accepting_ = {kCba, kCbna, kNa};
}

std::optional<std::string> MetadataGraph::check(const FusionPlan& plan) const {
    if (plan.ops().empty()) return "empty fusion plan";
    int node = kStart;
    for (std::size_t i = 0; i < plan.ops().size(); ++i) {
        const Edge* edge = nullptr;
        for (const Edge& e : edges_)
            if (e.from == node && e.kind == plan.ops()[i].kind) {
                edge = &e;
                break;
            }
        if (!edge) return "op sequence not in the supported fusion table";
        if (auto v = edge->check(plan, i)) return v;
        node = edge->to;
    }
    for (int a : accepting_)
        if (a == node) return std::nullopt;
    return "op sequence is a prefix of a supported fusion, not a complete one";
}

const MetadataGraph& fusion_metadata_graph() {
    static const MetadataGraph graph;
    return graph;
}

void fusion_compile(Handle& handle, FusionPlan& plan) {
    if (plan.compiled_) return;
    if (auto violated = fusion_metadata_graph().check(plan))
        throw_error(ErrorCode::FusionNotSupported, *violated);
    const std::string sig = plan.signature();
    const std::string key = PlanCache::hash_key(sig, "fused", "");
    handle.plan_cache().get_or_build(
        key, sig, [&]() -> std::shared_ptr<void> { return std::make_shared<std::string>(sig); },
        [&](const std::string& body) -> std::shared_ptr<void> {
            return std::make_shared<std::string>(body);
        });
    plan.compiled_ = true;
}

// ---- execution -------------------------------------------------------------

namespace {

void require_args(const FusionPlan& plan) {
    const FusionArgs& a = plan.args();
    for (const FusionOp& op : plan.ops()) {
        switch (op.kind) {
            case FusionOp::Kind::ConvForward:
                if (!a.filter) throw_error(ErrorCode::MissingArgs, "filter not bound");
                if (a.filter->desc.dims != op.filter_desc.dims)
                    throw_error(ErrorCode::ShapeMismatch, "bound filter shape mismatch");
                break;
            case FusionOp::Kind::Bias:
                if (!a.bias) throw_error(ErrorCode::MissingArgs, "bias not bound");
                if (static_cast<std::int64_t>(a.bias->data.size()) != op.bias_channels)
                    throw_error(ErrorCode::ShapeMismatch, "bound bias length mismatch");
                break;
            case FusionOp::Kind::BatchNormInference:
                if (!a.bn_gamma || !a.bn_beta || !a.bn_mean || !a.bn_var)
                    throw_error(ErrorCode::MissingArgs, "batchnorm parameters not bound");
                break;
            case FusionOp::Kind::Activation: break;
        }
    }
}

void upload_vec(Handle& h, DeviceBuffer& buf, const std::optional<HostTensor>& t) {
    if (!t) return;
    buf.ensure(t->data.size() * 4);
    check_cuda(cudaMemcpyAsync(buf.get(), t->data.data(), t->data.size() * 4,
                               cudaMemcpyHostToDevice, h.stream()),
               "cudaMemcpyAsync");
}

int act_code(const FusionPlan& plan, const FusionOp& op, float* alpha) {
    *alpha = plan.args().act_alpha ? *plan.args().act_alpha : op.act.alpha;
    return static_cast<int>(op.act.tag);
}

pk_conv_geom fused_geom(const FusionPlan& plan, const FusionOp& conv) {
    const ConvShapes s = resolve_shapes(plan.input_desc(), conv.filter_desc, conv.conv);
    pk_conv_geom g{};
    g.n = (int)s.n; g.c = (int)s.c; g.h = (int)s.h; g.w = (int)s.w;
    g.k = (int)s.k; g.r = (int)s.y; g.s = (int)s.x; g.p = (int)s.oh; g.q = (int)s.ow;
    g.pad_h = (int)conv.conv.pad_h; g.pad_w = (int)conv.conv.pad_w;
    g.str_h = (int)conv.conv.stride_h; g.str_w = (int)conv.conv.stride_w;
    g.dil_h = (int)conv.conv.dilation_h; g.dil_w = (int)conv.conv.dilation_w;
    g.groups = (int)s.groups; g.cg = (int)s.cg; g.kg = (int)s.kg;
    g.x_pitch = pk_pitch(g.c); g.y_pitch = pk_pitch(g.k); g.f_pitch = pk_pitch(g.cg);
    return g;
}

// In-bounds multiply count of the reference fused loop (fusion.cpp:370-381
// counts one per valid tap): separable over rows and columns.
std::uint64_t fused_mults(const pk_conv_geom& g) {
    auto valid = [](int out, int in, int f, int stride, int pad) {
        std::uint64_t t = 0;
        for (int o = 0; o < out; ++o)
            for (int y = 0; y < f; ++y) {
                const int i = o * stride - pad + y;
                t += (i >= 0 && i < in) ? 1 : 0;
            }
        return t;
    };
    return (std::uint64_t)g.n * g.k * g.cg * valid(g.p, g.h, g.r, g.str_h, g.pad_h) *
           valid(g.q, g.w, g.s, g.str_w, g.pad_w);
}

}  // namespace

FusionPlan::DeviceArgs& FusionPlan::device_args(Handle& h) {
    if (!dev_) dev_ = std::make_unique<DeviceArgs>();
    if (dev_->valid && dev_->owner == &h) return *dev_;
    h.activate();
    if (args_.filter) {
        dev_->filter.ensure(device_bytes(args_.filter->desc));
        upload_nchw(h, args_.filter->desc, args_.filter->data.data(), dev_->filter.get());
    }
    upload_vec(h, dev_->bias, args_.bias);
    upload_vec(h, dev_->gamma, args_.bn_gamma);
    upload_vec(h, dev_->beta, args_.bn_beta);
    upload_vec(h, dev_->mean, args_.bn_mean);
    upload_vec(h, dev_->var, args_.bn_var);
    // Folded affine for the tensor-core epilogues (no per-activation BN):
    //   ((acc + b) - mu) / sqrt(var + eps) * g + beta = acc * s + t,
    //   s = g / sqrt(var + eps), t = (b - mu) * s + beta
    dev_->folded = false;
    const FusionOp* conv = conv_op(*this);
    bool per_act = false;
    for (const FusionOp& op : ops_)
        if (op.kind == FusionOp::Kind::BatchNormInference && op.bn_mode == BatchNormMode::PerActivation)
            per_act = true;
    // (also the fp32 3xTF32 path: its epilogue reads the affine as float4 vectors)
    if (conv && !per_act) {
        const std::int64_t k = cur_desc_.dims[1];
        const std::size_t padded = static_cast<std::size_t>((k + 63) / 64 * 64 + 64);
        std::vector<float> s(padded, 0.0f), t(padded, 0.0f);
        for (std::int64_t i = 0; i < k; ++i) {
            double sc = 1.0, sh = args_.bias ? args_.bias->data[i] : 0.0;
            if (args_.bn_gamma && args_.bn_var && args_.bn_mean && args_.bn_beta) {
                const double inv = args_.bn_gamma->data[i] /
                                   std::sqrt(static_cast<double>(args_.bn_var->data[i]) +
                                             static_cast<double>(args_.bn_epsilon));
                sh = (sh - args_.bn_mean->data[i]) * inv + args_.bn_beta->data[i];
                sc = inv;
            }
            s[i] = static_cast<float>(sc);
            t[i] = static_cast<float>(sh);
        }
        dev_->scale.ensure(padded * 4);
        dev_->shift.ensure(padded * 4);
        check_cuda(cudaMemcpyAsync(dev_->scale.get(), s.data(), padded * 4, cudaMemcpyHostToDevice,
                                   h.stream()),
                   "cudaMemcpyAsync");
        check_cuda(cudaMemcpyAsync(dev_->shift.get(), t.data(), padded * 4, cudaMemcpyHostToDevice,
                                   h.stream()),
                   "cudaMemcpyAsync");
        h.sync();  // host staging vectors go out of scope
        dev_->folded = true;
    }
    dev_->owner = &h;
    dev_->valid = true;
    return *dev_;
}

void fusion_execute(Handle& h, FusionPlan& plan, const void* input, void* output) {
    const NvtxRange range("primkit fusion execute");
    if (!plan.compiled()) throw_error(ErrorCode::NotCompiled, "fusion plan is not compiled");
    require_args(plan);
    auto& d = plan.device_args(h);
    const int dt = plan.input_desc().etype == ElementType::BF16 ? PK_BF16 : PK_F32;

    pk_epilogue e{};
    e.act = -1;
    for (const FusionOp& op : plan.ops()) {
        if (op.kind == FusionOp::Kind::Bias) e.bias = static_cast<const float*>(d.bias.get());
        if (op.kind == FusionOp::Kind::BatchNormInference) {
            e.bn_mean = static_cast<const float*>(d.mean.get());
            e.bn_var = static_cast<const float*>(d.var.get());
            e.bn_gamma = static_cast<const float*>(d.gamma.get());
            e.bn_beta = static_cast<const float*>(d.beta.get());
            e.bn_per_activation = op.bn_mode == BatchNormMode::PerActivation;
            e.bn_eps = plan.args().bn_epsilon;
        }
        if (op.kind == FusionOp::Kind::Activation) e.act = act_code(plan, op, &e.act_alpha);
    }
    const FusionOp* conv = conv_op(plan);
    cudaStream_t st = h.stream();
    if (conv) {
        const pk_conv_geom g = fused_geom(plan, *conv);
        if (g.y_pitch != g.k)
            check_cuda(cudaMemsetAsync(output, 0,
                                       (std::size_t)g.n * g.p * g.q * g.y_pitch * (dt == PK_BF16 ? 2 : 4),
                                       st),
                       "memset");
        const bool wino = conv->algo == ConvAlgo::Winograd && g.r == 3 && g.s == 3 && g.str_h == 1 &&
                          g.str_w == 1;
        if (dt == PK_BF16 && pk_tc_fwd_supported(&g)) {
            const pk_tc_config cfg{256, 4, 1};
            h.last_kernel = "igemm_tc_fwd+epilogue";
            pk_epilogue tce = e;
            if (d.folded) {
                tce.bias = nullptr;
                tce.bn_mean = tce.bn_var = tce.bn_gamma = tce.bn_beta = nullptr;
                tce.ch_scale = static_cast<const float*>(d.scale.get());
                tce.ch_shift = static_cast<const float*>(d.shift.get());
            }
            check_cuda(pk_cuda_igemm_tc_fwd(&g, input, d.filter.get(), output, &tce, &cfg, st),
                       "igemm_tc_fwd");
        } else if (wino) {
            h.last_kernel = "winograd_f23+epilogue";
            check_cuda(pk_cuda_winograd_f23(&g, dt, input, d.filter.get(), output, &e, st),
                       "winograd_f23");
        } else if (dt == PK_F32 && tf32x3_eligible(g, dt)) {
            // fp32 Direct row: 3xTF32 tensor-core GEMM (fp32-level accuracy), the
            // epilogue's exact formula applied before the fp32 store
            const std::size_t wsb = pk_tf32x3_fwd_workspace(&g);
            h.last_kernel = "tf32x3_tc_fwd+epilogue";
            pk_epilogue tce = e;
            if (d.folded) {
                tce.bias = nullptr;
                tce.bn_mean = tce.bn_var = tce.bn_gamma = tce.bn_beta = nullptr;
                tce.ch_scale = static_cast<const float*>(d.scale.get());
                tce.ch_shift = static_cast<const float*>(d.shift.get());
            }
            check_cuda(pk_cuda_tf32x3_fwd(&g, input, d.filter.get(), output, &tce, h.scratch(11, wsb), wsb, st),
                       "tf32x3_fwd");
        } else {
            h.last_kernel = "direct_simt+epilogue";
            check_cuda(pk_cuda_direct_fwd(&g, dt, input, d.filter.get(), output, &e, st),
                       "direct_fwd");
        }
        h.counters().scalar_muls += fused_mults(g);
    } else {
        const auto& in = plan.input_desc().dims;
        h.last_kernel = "pointwise_bn_act";
        check_cuda(pk_cuda_pointwise(input, output, (int)in[0], (int)in[1], (int)(in[2] * in[3]),
                                     pk_pitch((int)in[1]), dt, &e, st),
                   "pointwise");
    }
    h.counters().buffer_roundtrips += 1;
}

void fusion_execute_unfused(Handle& h, FusionPlan& plan, const void* input, void* output) {
    const NvtxRange range("primkit fusion execute (unfused)");
    if (!plan.compiled()) throw_error(ErrorCode::NotCompiled, "fusion plan is not compiled");
    require_args(plan);
    auto& d = plan.device_args(h);
    const ElementType et = plan.input_desc().etype;
    const int dt = et == ElementType::BF16 ? PK_BF16 : PK_F32;
    cudaStream_t st = h.stream();

    // Ping-pong through two intermediate buffers; the last op writes `output`.
    TensorDescriptor cur = plan.input_desc();
    const void* src = input;
    const std::size_t n_ops = plan.ops().size();
    for (std::size_t i = 0; i < n_ops; ++i) {
        const FusionOp& op = plan.ops()[i];
        TensorDescriptor next = cur;
        if (op.kind == FusionOp::Kind::ConvForward) next = output_dims(cur, op.filter_desc, op.conv);
        void* dst = (i + 1 == n_ops) ? output : h.scratch(20 + (int)(i % 2), device_bytes(next));
        const auto& nd = next.dims;
        const int n = (int)nd[0], c = (int)nd[1], hw = (int)(nd[2] * nd[3]);
        switch (op.kind) {
            case FusionOp::Kind::ConvForward: {
                ConvAlgo algo = op.algo;
                if (algo == ConvAlgo::Winograd &&
                    (op.filter_desc.dims[2] != 3 || op.filter_desc.dims[3] != 3 ||
                     op.conv.stride_h != 1 || op.conv.stride_w != 1))
                    algo = ConvAlgo::Direct;  // fusion.cpp:443-450
                ConvProblem p;
                p.n = cur.dims[0]; p.c = cur.dims[1]; p.h = cur.dims[2]; p.w = cur.dims[3];
                p.k = op.filter_desc.dims[0]; p.y = op.filter_desc.dims[2]; p.x = op.filter_desc.dims[3];
                p.pad_h = op.conv.pad_h; p.pad_w = op.conv.pad_w;
                p.stride_h = op.conv.stride_h; p.stride_w = op.conv.stride_w;
                p.dilation_h = op.conv.dilation_h; p.dilation_w = op.conv.dilation_w;
                p.groups = op.conv.group_count;
                p.etype = et;
                const pk_conv_geom g = fused_geom(plan, op);
                if (dt == PK_BF16 && pk_tc_fwd_supported(&g)) {
                    // Same tensor-core convolution as the fused path, without
                    // the epilogue: the two executors differ only in where
                    // bias/BN/activation run (and the extra round trips).
                    const pk_tc_config cfg{256, 4, 1};
                    check_cuda(pk_cuda_igemm_tc_fwd(&g, src, d.filter.get(), dst, nullptr, &cfg, st),
                               "igemm_tc_fwd");
                    h.counters() += conv_counters(p, algo);
                } else {
                    const ConvPlan cp(p, algo, {});
                    const std::size_t dws = cp.device_workspace_bytes(h.num_sms());
                    cp.run(h, src, d.filter.get(), dst, h.scratch(0, dws), dws);
                }
                break;
            }
            case FusionOp::Kind::Bias:
            case FusionOp::Kind::BatchNormInference:
            case FusionOp::Kind::Activation: {
                pk_epilogue e{};
                e.act = -1;
                if (op.kind == FusionOp::Kind::Bias) e.bias = static_cast<const float*>(d.bias.get());
                if (op.kind == FusionOp::Kind::BatchNormInference) {
                    if (plan.args().bn_epsilon <= 0.0f)
                        throw_error(ErrorCode::InvalidEpsilon, "epsilon must be positive");
                    e.bn_mean = static_cast<const float*>(d.mean.get());
                    e.bn_var = static_cast<const float*>(d.var.get());
                    e.bn_gamma = static_cast<const float*>(d.gamma.get());
                    e.bn_beta = static_cast<const float*>(d.beta.get());
                    e.bn_per_activation = op.bn_mode == BatchNormMode::PerActivation;
                    e.bn_standalone = 1;  // batchnorm_forward_infer formula
                    e.bn_eps = plan.args().bn_epsilon;
                }
                if (op.kind == FusionOp::Kind::Activation) {
                    e.act = act_code(plan, op, &e.act_alpha);
                    if (op.act.tag == ActivationKind::Tag::LeakyReLU && e.act_alpha < 0.0f)
                        throw_error(ErrorCode::InvalidValue, "LeakyReLU alpha must be >= 0");
                }
                check_cuda(pk_cuda_pointwise(src, dst, n, c, hw, pk_pitch(c), dt, &e, st),
                           "pointwise");
                h.counters().buffer_roundtrips += 1;
                break;
            }
        }
        src = dst;
        cur = next;
    }
    h.last_kernel = "unfused";
}

}  // namespace primkit
