// TEST INFRASTRUCTURE ONLY (see oracle/Makefile.ref).
//
// extern "C" wrappers over the reference's C++-only entry points so the
// parity tests can drive them through ctypes. The reference C ABI
// (proj/include/primkit/primkit.h) exposes batch-norm only as a fusion op
// (primkit.h:195-196); training-mode forward and backward live in the C++ API
// (proj/src/core/primitives.hpp:29-46). Nothing here computes anything itself:
// every call forwards to the unmodified reference routine.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "core/primitives.hpp"
#include "core/tensor.hpp"

using namespace primkit;

namespace {

thread_local std::string g_shim_error;

Tensor make(const std::vector<std::int64_t>& dims, ElementType et,
            const float* src) {
    Tensor t(TensorDescriptor::packed(dims, et));
    if (src) std::memcpy(t.data(), src, sizeof(float) * t.size());
    t.quantize();
    return t;
}

std::vector<std::int64_t> param_dims(int mode, const std::int64_t* d) {
    if (mode == 0) return {1, d[1], d[2], d[3]};  // PerActivation
    return {1, d[1], 1, 1};                        // Spatial
}

template <typename Fn>
int guard(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const Error& e) {
        g_shim_error = e.what();
        return static_cast<int>(e.code());
    } catch (const std::exception& e) {
        g_shim_error = e.what();
        return 20;
    }
}

BatchNormParams params(int mode, const std::int64_t* dims, int etype,
                       const float* gamma, const float* beta,
                       const float* rmean, const float* rvar, float eps,
                       float momentum) {
    const auto pd = param_dims(mode, dims);
    BatchNormParams p;
    // Parameters are F32 tensors in the reference's own fusion binding
    // (proj/src/capi/primkit_c.cpp:459-471); keep that convention.
    (void)etype;
    p.gamma = make(pd, ElementType::F32, gamma);
    p.beta = make(pd, ElementType::F32, beta);
    p.running_mean = make(pd, ElementType::F32, rmean);
    p.running_var = make(pd, ElementType::F32, rvar);
    p.epsilon = eps;
    p.momentum = momentum;
    return p;
}

}  // namespace

extern "C" {

const char* ref_shim_last_error() { return g_shim_error.c_str(); }

int ref_bn_forward_train(int mode, const std::int64_t dims[4], int etype,
                         const float* x, const float* gamma, const float* beta,
                         float* running_mean, float* running_var, float eps,
                         float momentum, float* y, float* saved_mean,
                         float* saved_invstd) {
    return guard([&] {
        const std::vector<std::int64_t> d(dims, dims + 4);
        const auto et = static_cast<ElementType>(etype);
        BatchNormParams p = params(mode, dims, etype, gamma, beta,
                                   running_mean, running_var, eps, momentum);
        const Tensor tx = make(d, et, x);
        BatchNormForwardResult r = batchnorm_forward_train(
            static_cast<BatchNormMode>(mode == 0 ? 0 : 1), tx, p);
        std::memcpy(y, r.y.data(), sizeof(float) * r.y.size());
        std::memcpy(saved_mean, r.saved_mean.data(),
                    sizeof(float) * r.saved_mean.size());
        std::memcpy(saved_invstd, r.saved_invstd.data(),
                    sizeof(float) * r.saved_invstd.size());
        std::memcpy(running_mean, p.running_mean.data(),
                    sizeof(float) * p.running_mean.size());
        std::memcpy(running_var, p.running_var.data(),
                    sizeof(float) * p.running_var.size());
    });
}

int ref_bn_forward_infer(int mode, const std::int64_t dims[4], int etype,
                         const float* x, const float* gamma, const float* beta,
                         const float* running_mean, const float* running_var,
                         float eps, float* y) {
    return guard([&] {
        const std::vector<std::int64_t> d(dims, dims + 4);
        BatchNormParams p = params(mode, dims, etype, gamma, beta,
                                   running_mean, running_var, eps, 0.1f);
        const Tensor tx = make(d, static_cast<ElementType>(etype), x);
        const Tensor r = batchnorm_forward_infer(
            static_cast<BatchNormMode>(mode == 0 ? 0 : 1), tx, p);
        std::memcpy(y, r.data(), sizeof(float) * r.size());
    });
}

int ref_bn_backward(int mode, const std::int64_t dims[4], int etype,
                    const float* x, const float* dy, const float* gamma,
                    const float* beta, const float* saved_mean,
                    const float* saved_invstd, float eps, float* dx,
                    float* dgamma, float* dbeta) {
    return guard([&] {
        const std::vector<std::int64_t> d(dims, dims + 4);
        const auto et = static_cast<ElementType>(etype);
        const auto pd = param_dims(mode, dims);
        std::vector<float> zeros(static_cast<std::size_t>(pd[1] * pd[2] * pd[3]), 0.0f);
        std::vector<float> ones(zeros.size(), 1.0f);
        BatchNormParams p = params(mode, dims, etype, gamma, beta, zeros.data(),
                                   ones.data(), eps, 0.1f);
        std::int64_t stat = 1;
        for (std::size_t i = 1; i < pd.size(); ++i) stat *= pd[i];
        const Tensor tx = make(d, et, x);
        const Tensor tdy = make(d, et, dy);
        const Tensor sm = make({stat}, ElementType::F32, saved_mean);
        const Tensor si = make({stat}, ElementType::F32, saved_invstd);
        BatchNormBackwardResult r = batchnorm_backward(
            static_cast<BatchNormMode>(mode == 0 ? 0 : 1), tx, tdy, p, sm, si);
        std::memcpy(dx, r.dx.data(), sizeof(float) * r.dx.size());
        std::memcpy(dgamma, r.dgamma.data(), sizeof(float) * r.dgamma.size());
        std::memcpy(dbeta, r.dbeta.data(), sizeof(float) * r.dbeta.size());
    });
}

int ref_activation_forward(int kind, float alpha, const std::int64_t dims[4],
                           int etype, const float* x, float* y) {
    return guard([&] {
        const std::vector<std::int64_t> d(dims, dims + 4);
        ActivationKind k{static_cast<ActivationKind::Tag>(kind), alpha};
        const Tensor r =
            activation_forward(k, make(d, static_cast<ElementType>(etype), x));
        std::memcpy(y, r.data(), sizeof(float) * r.size());
    });
}

int ref_activation_backward(int kind, float alpha, const std::int64_t dims[4],
                            int etype, const float* x, const float* dy,
                            float* dx) {
    return guard([&] {
        const std::vector<std::int64_t> d(dims, dims + 4);
        const auto et = static_cast<ElementType>(etype);
        ActivationKind k{static_cast<ActivationKind::Tag>(kind), alpha};
        const Tensor r = activation_backward(k, make(d, et, x), make(d, et, dy));
        std::memcpy(dx, r.data(), sizeof(float) * r.size());
    });
}

float ref_round_bf16(float v) { return round_bf16(v); }

}  // extern "C"

// ---- pooling / softmax (C++-only in the reference: primitives.hpp:65-91) ----
extern "C" {

int ref_pooling_forward(int kind, const std::int64_t win[2], const std::int64_t pad[2],
                        const std::int64_t str[2], const std::int64_t dims[4], int etype,
                        const float* x, float* y, std::int64_t* indices) {
    return guard([&] {
        PoolingDescriptor pd;
        pd.window_h = win[0];
        pd.window_w = win[1];
        pd.pad_h = pad[0];
        pd.pad_w = pad[1];
        pd.stride_h = str[0];
        pd.stride_w = str[1];
        const std::vector<std::int64_t> d(dims, dims + 4);
        PoolingForwardResult r = pooling_forward(static_cast<PoolingKind>(kind), pd,
                                                 make(d, static_cast<ElementType>(etype), x));
        std::memcpy(y, r.y.data(), sizeof(float) * r.y.size());
        std::memcpy(indices, r.indices.data(), sizeof(std::int64_t) * r.indices.size());
    });
}

int ref_pooling_backward(int kind, const std::int64_t win[2], const std::int64_t pad[2],
                         const std::int64_t str[2], const std::int64_t dims[4], int etype,
                         const float* dy, const std::int64_t* indices, float* dx) {
    return guard([&] {
        PoolingDescriptor pd;
        pd.window_h = win[0];
        pd.window_w = win[1];
        pd.pad_h = pad[0];
        pd.pad_w = pad[1];
        pd.stride_h = str[0];
        pd.stride_w = str[1];
        const auto et = static_cast<ElementType>(etype);
        const std::int64_t oh = (dims[2] + 2 * pad[0] - win[0]) / str[0] + 1;
        const std::int64_t ow = (dims[3] + 2 * pad[1] - win[1]) / str[1] + 1;
        const Tensor tdy = make({dims[0], dims[1], oh, ow}, et, dy);
        std::vector<std::int64_t> idx(indices, indices + tdy.size());
        const Tensor r = pooling_backward(static_cast<PoolingKind>(kind), pd,
                                          TensorDescriptor::packed({dims[0], dims[1], dims[2], dims[3]}, et),
                                          tdy, idx);
        std::memcpy(dx, r.data(), sizeof(float) * r.size());
    });
}

int ref_softmax_forward(int rank, const std::int64_t* dims, int etype, std::int64_t axis, const float* x,
                        float* y) {
    return guard([&] {
        const std::vector<std::int64_t> d(dims, dims + rank);
        const Tensor r = softmax_forward(make(d, static_cast<ElementType>(etype), x), axis);
        std::memcpy(y, r.data(), sizeof(float) * r.size());
    });
}

int ref_softmax_backward(int rank, const std::int64_t* dims, int etype, std::int64_t axis, const float* y,
                         const float* dy, float* dx) {
    return guard([&] {
        const std::vector<std::int64_t> d(dims, dims + rank);
        const auto et = static_cast<ElementType>(etype);
        const Tensor r = softmax_backward(make(d, et, y), make(d, et, dy), axis);
        std::memcpy(dx, r.data(), sizeof(float) * r.size());
    });
}

}  // extern "C"
