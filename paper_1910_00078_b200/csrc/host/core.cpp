#include "core.hpp"

#include <bit>
#include <cmath>
#include <cuda_runtime.h>

namespace primkit {

void throw_error(ErrorCode code, const std::string& what) { throw Error(code, what); }

void check_cuda(int err, const char* what) {
    if (err != cudaSuccess)
        throw std::runtime_error(std::string("CUDA error in ") + what + ": " +
                                 cudaGetErrorString(static_cast<cudaError_t>(err)));
}

const char* element_type_name(ElementType t) { return t == ElementType::BF16 ? "bf16" : "f32"; }

// Round-to-nearest-even to bfloat16, widened back to f32; NaN becomes a quiet
// NaN that survives truncation (same contract as tensor.cpp:44-54).
float round_bf16(float x) {
    std::uint32_t bits = std::bit_cast<std::uint32_t>(x);
    if (std::isnan(x)) return std::bit_cast<float>((bits & 0xffff0000u) | 0x00410000u);
    bits += 0x7fffu + ((bits >> 16) & 1u);
    return std::bit_cast<float>(bits & 0xffff0000u);
}

TensorDescriptor TensorDescriptor::packed(std::vector<std::int64_t> d, ElementType t) {
    for (auto v : d)
        if (v < 1) throw_error(ErrorCode::InvalidShape, "dims must be >= 1");
    TensorDescriptor out;
    out.dims = std::move(d);
    out.etype = t;
    return out;
}

std::int64_t TensorDescriptor::elem_count() const {
    std::int64_t n = 1;
    for (auto v : dims) n *= v;
    return n;
}

const char* conv_algo_name(ConvAlgo a) {
    switch (a) {
        case ConvAlgo::Im2colGemm: return "Im2colGemm";
        case ConvAlgo::Direct: return "Direct";
        case ConvAlgo::Winograd: return "Winograd";
        case ConvAlgo::FFT: return "FFT";
        case ConvAlgo::ImplicitGemm: return "ImplicitGemm";
    }
    return "?";
}

ConvShapes resolve_shapes(const TensorDescriptor& in, const TensorDescriptor& flt,
                          const ConvDescriptor& cv) {
    if (in.rank() != 4 || flt.rank() != 4)
        throw_error(ErrorCode::InvalidShape, "convolution expects 4-D tensors");
    if (cv.stride_h < 1 || cv.stride_w < 1 || cv.dilation_h < 1 || cv.dilation_w < 1 ||
        cv.pad_h < 0 || cv.pad_w < 0 || cv.group_count < 1)
        throw_error(ErrorCode::InvalidValue, "bad convolution descriptor");
    if (cv.mode == ConvMode::Transpose && (cv.dilation_h != 1 || cv.dilation_w != 1))
        throw_error(ErrorCode::InvalidValue, "transpose mode requires dilation 1");

    ConvShapes s{};
    s.n = in.dims[0];
    s.c = in.dims[1];
    s.h = in.dims[2];
    s.w = in.dims[3];
    s.groups = cv.group_count;
    s.y = flt.dims[2];
    s.x = flt.dims[3];
    if (cv.mode == ConvMode::Convolution) {
        s.k = flt.dims[0];
        if (s.c % s.groups != 0 || s.k % s.groups != 0)
            throw_error(ErrorCode::GroupMismatch,
                        "group count must divide input and output channels");
        if (flt.dims[1] != s.c / s.groups)
            throw_error(ErrorCode::ShapeMismatch,
                        "filter channel extent does not match input/groups");
        const std::int64_t span_h = cv.dilation_h * (s.y - 1) + 1;
        const std::int64_t span_w = cv.dilation_w * (s.x - 1) + 1;
        const std::int64_t eh = s.h + 2 * cv.pad_h, ew = s.w + 2 * cv.pad_w;
        // An empty window (padded extent shorter than the dilated filter) is
        // an invalid shape even where C's truncating division would round the
        // negative quotient up to a positive extent.
        s.oh = eh < span_h ? 0 : (eh - span_h) / cv.stride_h + 1;
        s.ow = ew < span_w ? 0 : (ew - span_w) / cv.stride_w + 1;
    } else {
        if (flt.dims[0] != s.c)
            throw_error(ErrorCode::ShapeMismatch,
                        "transpose filter leading extent must match input channels");
        s.k = flt.dims[1] * s.groups;
        if (s.c % s.groups != 0)
            throw_error(ErrorCode::GroupMismatch, "group count must divide input channels");
        s.oh = cv.stride_h * (s.h - 1) + s.y - 2 * cv.pad_h;
        s.ow = cv.stride_w * (s.w - 1) + s.x - 2 * cv.pad_w;
    }
    if (s.oh < 1 || s.ow < 1) throw_error(ErrorCode::InvalidShape, "output extent below 1");
    s.cg = s.c / s.groups;
    s.kg = s.k / s.groups;
    return s;
}

TensorDescriptor output_dims(const TensorDescriptor& in, const TensorDescriptor& flt,
                             const ConvDescriptor& cv) {
    const ConvShapes s = resolve_shapes(in, flt, cv);
    return TensorDescriptor::packed({s.n, s.k, s.oh, s.ow}, in.etype);
}

namespace {
std::int64_t pow2_at_least(std::int64_t v) {
    std::int64_t p = 1;
    while (p < v) p <<= 1;
    return p;
}
}  // namespace

std::size_t conv_workspace_bytes(ConvAlgo algo, const TensorDescriptor& in,
                                 const TensorDescriptor& flt, const ConvDescriptor& cv,
                                 const ImplicitGemmTiles& t) {
    const ConvShapes s = resolve_shapes(in, flt, cv);
    switch (algo) {
        case ConvAlgo::Direct:
        case ConvAlgo::Winograd: return 0;
        case ConvAlgo::Im2colGemm:
            // one (image, group) column matrix of f32
            if (cv.mode == ConvMode::Transpose)
                return static_cast<std::size_t>(s.kg * s.y * s.x * s.h * s.w) * 4u;
            return static_cast<std::size_t>(s.cg * s.y * s.x * s.oh * s.ow) * 4u;
        case ConvAlgo::FFT: {
            // complex<double> spectra: cg input planes, kg*cg filter planes,
            // one accumulator plane, plus 16 bytes of alignment slack
            const std::int64_t plane = pow2_at_least(s.h + 2 * cv.pad_h + s.y - 1) *
                                       pow2_at_least(s.w + 2 * cv.pad_w + s.x - 1);
            const std::int64_t planes = s.cg + s.kg * s.cg + 1;
            return static_cast<std::size_t>(planes * plane) * 16u + 16u;
        }
        case ConvAlgo::ImplicitGemm: {
            const std::int64_t a = t.tile_m * t.tile_k * s.y * s.x;
            const std::int64_t b = t.tile_k * t.tile_n * s.y * s.x;
            return static_cast<std::size_t>(a + b + t.tile_m * t.tile_n) * 4u;
        }
    }
    return 0;
}

std::string ConvProblem::key() const {
    std::string out;
    for (std::int64_t v : {n, c, h, w, k, y, x, pad_h, pad_w, stride_h, stride_w, dilation_h,
                           dilation_w, groups}) {
        out += std::to_string(v);
        out += '-';
    }
    out += direction == ConvDirection::Forward        ? "F"
           : direction == ConvDirection::BackwardData ? "BD"
                                                      : "BW";
    out += mode == ConvMode::Convolution ? "-C-" : "-T-";
    out += element_type_name(etype);
    return out;
}

ConvDescriptor ConvProblem::conv_desc() const {
    ConvDescriptor d;
    d.pad_h = pad_h;
    d.pad_w = pad_w;
    d.stride_h = stride_h;
    d.stride_w = stride_w;
    d.dilation_h = dilation_h;
    d.dilation_w = dilation_w;
    d.mode = mode;
    d.group_count = groups;
    return d;
}

TensorDescriptor ConvProblem::input_desc() const {
    return TensorDescriptor::packed({n, c, h, w}, etype);
}

TensorDescriptor ConvProblem::filter_desc() const {
    if (mode == ConvMode::Transpose) return TensorDescriptor::packed({c, k / groups, y, x}, etype);
    return TensorDescriptor::packed({k, c / groups, y, x}, etype);
}

TensorDescriptor ConvProblem::output_desc() const {
    return output_dims(input_desc(), filter_desc(), conv_desc());
}

}  // namespace primkit
