// primkit-b200 host core: error model, element types, descriptors, the
// convolution shape algebra and the canonical problem key.
//
// Behaviour mirrors the reference C++ API (names, argument meaning, error
// codes and messages that tests match on):
//   errors        proj/src/core/errors.hpp:8-46
//   descriptors   proj/src/core/tensor.hpp:29-49, tensor.cpp:58-92
//   round_bf16    proj/src/core/tensor.cpp:44-54
//   shapes        proj/src/core/conv.cpp:21-78, 615-620
//   problem key   proj/src/core/problem.cpp:7-48
//   workspace     proj/src/core/conv.cpp:423-429, 507-514, 633-654
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

namespace primkit {

// NVTX range for profilers (nsys / ncu --nvtx): header-only NVTX3, a no-op
// unless a tool is attached (SURVEY §5 tracing).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

enum class ErrorCode {
    Ok = 0,
    ShapeMismatch,
    InvalidShape,
    GroupMismatch,
    AlgoNotApplicable,
    WorkspaceTooSmall,
    DuplicateSolver,
    NoApplicableSolver,
    NotTunable,
    NoValidConfig,
    IoError,
    ParseError,
    LayoutNotDescending,
    InvalidEpsilon,
    InvalidAxis,
    FusionNotSupported,
    AlreadyCompiled,
    NotCompiled,
    MissingArgs,
    InvalidValue,
};

class Error : public std::runtime_error {
public:
    Error(ErrorCode code, const std::string& what) : std::runtime_error(what), code_(code) {}
    ErrorCode code() const { return code_; }

private:
    ErrorCode code_;
};

[[noreturn]] void throw_error(ErrorCode code, const std::string& what);
// CUDA failures surface as std::runtime_error -> PRIMKIT_STATUS_INTERNAL.
void check_cuda(int cuda_error, const char* what);

enum class ElementType { F32, BF16 };
const char* element_type_name(ElementType t);

float round_bf16(float x);

struct OpCounters {
    std::uint64_t gemm_calls = 0;
    std::uint64_t scalar_muls = 0;
    std::uint64_t buffer_roundtrips = 0;
    void reset() { *this = OpCounters{}; }
    OpCounters& operator+=(const OpCounters& o) {
        gemm_calls += o.gemm_calls;
        scalar_muls += o.scalar_muls;
        buffer_roundtrips += o.buffer_roundtrips;
        return *this;
    }
};

// Packed (row-major, NCHW for rank 4) descriptor; strided host tensors never
// cross the C ABI, so only the packed form exists here.
struct TensorDescriptor {
    std::vector<std::int64_t> dims;
    ElementType etype = ElementType::F32;

    static TensorDescriptor packed(std::vector<std::int64_t> d, ElementType t = ElementType::F32);
    std::int64_t rank() const { return static_cast<std::int64_t>(dims.size()); }
    std::int64_t elem_count() const;
    bool operator==(const TensorDescriptor&) const = default;
};

enum class ConvMode { Convolution, Transpose };
enum class ConvAlgo { Im2colGemm, Direct, Winograd, FFT, ImplicitGemm };
enum class ConvDirection { Forward, BackwardData, BackwardWeights };
const char* conv_algo_name(ConvAlgo a);

struct ConvDescriptor {
    std::int64_t pad_h = 0, pad_w = 0;
    std::int64_t stride_h = 1, stride_w = 1;
    std::int64_t dilation_h = 1, dilation_w = 1;
    ConvMode mode = ConvMode::Convolution;
    std::int64_t group_count = 1;
};

// tile_m blocks output channels, tile_n output pixels, tile_k input channels
// (proj/src/core/conv.hpp:25-32). On B200 the same three values select the
// tcgen05 tile configuration (see solver.cpp).
struct ImplicitGemmTiles {
    std::int64_t tile_m = 1, tile_n = 1, tile_k = 1;
};

struct ConvShapes {
    std::int64_t n, c, h, w;
    std::int64_t k, y, x;
    std::int64_t oh, ow;
    std::int64_t cg, kg;
    std::int64_t groups;
};

ConvShapes resolve_shapes(const TensorDescriptor& input, const TensorDescriptor& filter,
                          const ConvDescriptor& conv);
TensorDescriptor output_dims(const TensorDescriptor& input, const TensorDescriptor& filter,
                             const ConvDescriptor& conv);
std::size_t conv_workspace_bytes(ConvAlgo algo, const TensorDescriptor& input,
                                 const TensorDescriptor& filter, const ConvDescriptor& conv,
                                 const ImplicitGemmTiles& tiles = {});

struct ConvProblem {
    std::int64_t n = 1, c = 1, h = 1, w = 1;
    std::int64_t k = 1, y = 1, x = 1;
    std::int64_t pad_h = 0, pad_w = 0;
    std::int64_t stride_h = 1, stride_w = 1;
    std::int64_t dilation_h = 1, dilation_w = 1;
    std::int64_t groups = 1;
    ConvDirection direction = ConvDirection::Forward;
    ConvMode mode = ConvMode::Convolution;
    ElementType etype = ElementType::F32;

    bool operator==(const ConvProblem&) const = default;
    std::string key() const;
    ConvDescriptor conv_desc() const;
    TensorDescriptor input_desc() const;
    TensorDescriptor filter_desc() const;
    TensorDescriptor output_desc() const;
};

}  // namespace primkit
