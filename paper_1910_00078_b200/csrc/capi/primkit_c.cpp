// C ABI of primkit-b200 (include/primkit/primkit.h).
//
// Section 1 functions are drop-in replacements for the reference's
// proj/src/capi/primkit_c.cpp:154-496: same validation order, same status
// mapping (no exception crosses the boundary; a thread-local message records
// the last failure), same operand conventions. The compute behind them runs
// on the GPU: host NCHW buffers are staged into the device layout, the
// selected sm_100a kernel runs on the handle's stream, results come back.
#include "primkit/primkit.h"

#include <cuda_runtime.h>

#include <cstring>
#include <algorithm>
#include <exception>
#include <vector>
#include <memory>
#include <string>

#include "../cuda/kernels.h"
#include "../host/dp.hpp"
#include "../host/fusion.hpp"
#include "../host/handle.hpp"

namespace {

thread_local std::string g_last_error;

primkit_status fail(primkit_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

template <typename Fn>
primkit_status guarded(Fn&& fn) {
    try {
        fn();
        return PRIMKIT_STATUS_OK;
    } catch (const primkit::Error& e) {
        return fail(static_cast<primkit_status>(e.code()), e.what());
    } catch (const std::exception& e) {
        return fail(PRIMKIT_STATUS_INTERNAL, e.what());
    } catch (...) {
        return fail(PRIMKIT_STATUS_INTERNAL, "unknown error");
    }
}

template <typename T>
T* need(T* p, const char* what) {
    if (!p) primkit::throw_error(primkit::ErrorCode::InvalidValue, std::string("null ") + what);
    return p;
}

primkit::ConvProblem to_problem(const primkit_conv_problem* pp) {
    const primkit_conv_problem& p = *need(pp, "problem");
    primkit::ConvProblem o;
    o.n = p.n; o.c = p.c; o.h = p.h; o.w = p.w;
    o.k = p.k; o.y = p.y; o.x = p.x;
    o.pad_h = p.pad_h; o.pad_w = p.pad_w;
    o.stride_h = p.stride_h; o.stride_w = p.stride_w;
    o.dilation_h = p.dilation_h; o.dilation_w = p.dilation_w;
    o.groups = p.groups;
    o.direction = static_cast<primkit::ConvDirection>(p.direction);
    o.mode = static_cast<primkit::ConvMode>(p.mode);
    o.etype = static_cast<primkit::ElementType>(p.etype);
    return o;
}

// Data operands per direction: Forward (input, filter), BackwardData
// (dOutput, filter), BackwardWeights (dOutput, input).
std::pair<primkit::TensorDescriptor, primkit::TensorDescriptor> operand_descs(
    const primkit::ConvProblem& p) {
    using D = primkit::ConvDirection;
    if (p.direction == D::Forward) return {p.input_desc(), p.filter_desc()};
    if (p.direction == D::BackwardData) return {p.output_desc(), p.filter_desc()};
    return {p.output_desc(), p.input_desc()};
}

primkit::TensorDescriptor result_desc(const primkit::ConvProblem& p) {
    using D = primkit::ConvDirection;
    if (p.direction == D::Forward) return p.output_desc();
    if (p.direction == D::BackwardData) return p.input_desc();
    return p.filter_desc();
}

// ---- overlapped host-buffer path ------------------------------------------
// primkit_conv_run with PINNED host buffers and a forward / backward-data
// problem: the batch is processed in image chunks so that the host->device
// copy of chunk j+1, the compute of chunk j and the device->host copy of
// chunk j-1 run concurrently (PCIe is full duplex; the copies dominate this
// ABI). Results are identical to the single-shot path (per-image kernels);
// the op counters advance once for the whole problem, as in the reference.
bool is_pinned(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

int host_chunk_images(const primkit::ConvProblem& p, const float* a, const float* out) {
    using D = primkit::ConvDirection;
    if (p.direction == D::BackwardWeights || p.n < 2) return 0;
    const auto da = operand_descs(p).first;
    const auto dr = result_desc(p);
    const double per_img = 4.0 * std::max(da.elem_count() / p.n, dr.elem_count() / p.n);
    double target = 16.0 * 1024 * 1024;  // bytes per chunk transfer (measured best of 8-48 MB)
    if (const char* v = std::getenv("PK_HOST_CHUNK_KB")) target = std::atof(v) * 1024;
    if (target <= 0) return 0;
    const long long nc = std::max<long long>(1, (long long)(target / per_img));
    if (nc * 2 > p.n) return 0;  // fewer than two chunks: nothing to overlap
    if (!is_pinned(a) || !is_pinned(out)) return 0;
    return (int)nc;
}

void conv_run_chunked(primkit::Handle& hd, const primkit::ConvProblem& p,
                      const primkit::Solver& solver, const primkit::PerfConfig& cfg, const float* a,
                      const float* b, float* out, int nc) {
    const auto [da, db] = operand_descs(p);
    const primkit::TensorDescriptor dr = result_desc(p);
    const int dt = p.etype == primkit::ElementType::BF16 ? PK_BF16 : PK_F32;
    const size_t esz = p.etype == primkit::ElementType::BF16 ? 2 : 4;
    const int ca = (int)da.dims[1], co = (int)dr.dims[1];
    const long long hwa = da.dims[2] * da.dims[3], hwo = dr.dims[2] * dr.dims[3];
    const size_t img_a_host = (size_t)ca * hwa, img_o_host = (size_t)co * hwo;  // floats
    const size_t img_a_dev = (size_t)hwa * pk_pitch(ca) * esz, img_o_dev = (size_t)hwo * pk_pitch(co) * esz;
    char* dva = static_cast<char*>(hd.scratch(1, primkit::device_bytes(da)));
    void* dvb = hd.scratch(2, primkit::device_bytes(db));
    char* dvo = static_cast<char*>(hd.scratch(3, primkit::device_bytes(dr)));
    float* in_stage[2] = {static_cast<float*>(hd.scratch(30, img_a_host * nc * 4)),
                          static_cast<float*>(hd.scratch(31, img_a_host * nc * 4))};
    float* out_stage[2] = {static_cast<float*>(hd.scratch(32, img_o_host * nc * 4)),
                           static_cast<float*>(hd.scratch(33, img_o_host * nc * 4))};
    cudaStream_t cs = hd.stream(), up = hd.copy_stream(0), down = hd.copy_stream(1);
    auto ck = [](cudaError_t e, const char* w) { primkit::check_cuda(e, w); };
    // the filter goes first, on the compute stream (small)
    primkit::upload_nchw(hd, db, need(b, "operand b"), dvb);
    // copy streams start after everything already queued on the compute stream
    cudaEvent_t start = hd.event(0);
    ck(cudaEventRecord(start, cs), "cudaEventRecord");
    ck(cudaStreamWaitEvent(up, start, 0), "cudaStreamWaitEvent");
    ck(cudaStreamWaitEvent(down, start, 0), "cudaStreamWaitEvent");
    const primkit::OpCounters saved = hd.counters();
    std::string kernel, variant;
    std::unique_ptr<primkit::ConvPlan> chunk_plan;
    cudaEvent_t t0 = hd.timing_event(0), t1 = hd.timing_event(1);
    ck(cudaEventRecord(t0, cs), "cudaEventRecord");
    const int chunks = (int)((p.n + nc - 1) / nc);
    for (int j = 0; j < chunks; ++j) {
        const int s = j & 1;
        const int n0 = j * nc, nj = (int)std::min<long long>(nc, p.n - n0);
        cudaEvent_t h2d = hd.event(1 + s), consumed = hd.event(3 + s), conv_out = hd.event(5 + s),
                    d2h = hd.event(7 + s);
        if (j >= 2) ck(cudaStreamWaitEvent(up, consumed, 0), "cudaStreamWaitEvent");
        ck(cudaMemcpyAsync(in_stage[s], a + (size_t)n0 * img_a_host, (size_t)nj * img_a_host * 4,
                           cudaMemcpyHostToDevice, up),
           "cudaMemcpyAsync");
        ck(cudaEventRecord(h2d, up), "cudaEventRecord");
        ck(cudaStreamWaitEvent(cs, h2d, 0), "cudaStreamWaitEvent");
        ck(pk_cuda_nchw_to_nhwc(in_stage[s], dva + (size_t)n0 * img_a_dev, nj, ca, (int)hwa,
                                pk_pitch(ca), dt, cs),
           "nchw_to_nhwc");
        ck(cudaEventRecord(consumed, cs), "cudaEventRecord");
        // chunk plans stay out of the plan cache: the reference makes exactly
        // one cached_build per conv_run (below, for the whole problem)
        primkit::ConvProblem pj = p;
        pj.n = nj;
        if (nj != nc || !chunk_plan) chunk_plan = std::make_unique<primkit::ConvPlan>(solver.build_plan(pj, &cfg));
        const size_t dws = chunk_plan->device_workspace_bytes(hd.num_sms());
        void* ws = hd.scratch(0, dws);
        chunk_plan->run(hd, dva + (size_t)n0 * img_a_dev, dvb, dvo + (size_t)n0 * img_o_dev, ws, dws);
        kernel = hd.last_kernel;
        variant = hd.last_variant;
        if (j >= 2) ck(cudaStreamWaitEvent(cs, d2h, 0), "cudaStreamWaitEvent");
        ck(pk_cuda_nhwc_to_nchw(dvo + (size_t)n0 * img_o_dev, out_stage[s], nj, co, (int)hwo,
                                pk_pitch(co), dt, cs),
           "nhwc_to_nchw");
        ck(cudaEventRecord(conv_out, cs), "cudaEventRecord");
        ck(cudaStreamWaitEvent(down, conv_out, 0), "cudaStreamWaitEvent");
        ck(cudaMemcpyAsync(out + (size_t)n0 * img_o_host, out_stage[s], (size_t)nj * img_o_host * 4,
                           cudaMemcpyDeviceToHost, down),
           "cudaMemcpyAsync");
        ck(cudaEventRecord(d2h, down), "cudaEventRecord");
    }
    // the compute stream (and so later work on it) waits for the last copies
    cudaEvent_t done = hd.event(9);
    ck(cudaEventRecord(done, down), "cudaEventRecord");
    ck(cudaStreamWaitEvent(cs, done, 0), "cudaStreamWaitEvent");
    ck(cudaEventRecord(t1, cs), "cudaEventRecord");
    ck(cudaStreamSynchronize(down), "cudaStreamSynchronize");
    ck(cudaEventSynchronize(t1), "cudaEventSynchronize");
    float ms = 0.0f;  // copies + conversions + convolutions of the whole call
    ck(cudaEventElapsedTime(&ms, t0, t1), "cudaEventElapsedTime");
    hd.record_device_ms(ms);
    hd.counters() = saved;
    hd.counters() += hd.cached_build(p, solver, &cfg)->op_counters();
    hd.last_kernel = kernel;
    hd.last_variant = variant;
}

void copy_name(char* buf, size_t len, const std::string& name) {
    if (!buf || len == 0) primkit::throw_error(primkit::ErrorCode::InvalidValue, "null output buffer");
    if (name.size() + 1 > len)
        primkit::throw_error(primkit::ErrorCode::InvalidValue, "output buffer too small");
    std::memcpy(buf, name.c_str(), name.size() + 1);
}

// Host copy quantized to the element type (tensor_from in the reference).
primkit::HostTensor host_tensor(const primkit::TensorDescriptor& d, const float* data) {
    primkit::HostTensor t{d, std::vector<float>(data, data + d.elem_count())};
    if (d.etype == primkit::ElementType::BF16)
        for (float& v : t.data) v = primkit::round_bf16(v);
    return t;
}

}  // namespace

struct primkit_handle {
    primkit::Handle impl;
    primkit_handle() = default;
    primkit_handle(cudaStream_t s, int dev) : impl(s, dev) {}
};

struct primkit_fusion_plan {
    primkit::FusionPlan impl;
};

struct primkit_dp {
    primkit::DataParallel* impl = nullptr;
    ~primkit_dp() { primkit::dp_destroy(impl); }
};

namespace {

primkit::Handle& H(primkit_handle* h) { return need(h, "handle")->impl; }
primkit::FusionPlan& P(primkit_fusion_plan* p) { return need(p, "fusion plan")->impl; }

const primkit::Solver& solver_named(primkit_handle* h, const char* name) {
    const primkit::Solver* s = H(h).find_solver(name ? name : "");
    if (!s)
        primkit::throw_error(primkit::ErrorCode::InvalidValue,
                             std::string("unknown solver '") + (name ? name : "") + "'");
    return *s;
}

// Solver selection shared by the host and device run entry points
// (primkit_c.cpp:296-312 of the reference).
const primkit::Solver& select_solver(primkit_handle* h, const primkit::ConvProblem& p,
                                     const char* name) {
    if (name) {
        const primkit::Solver& s = solver_named(h, name);
        if (!s.is_applicable(p))
            primkit::throw_error(primkit::ErrorCode::AlgoNotApplicable,
                                 s.name() + " is not applicable to " + p.key());
        return s;
    }
    for (const auto& s : H(h).solvers())
        if (s->is_applicable(p)) return *s;
    primkit::throw_error(primkit::ErrorCode::NoApplicableSolver, "no applicable solver for " + p.key());
}

primkit::TensorDescriptor dims4(const int64_t d[4], primkit_element_type et) {
    need(d, "dims");
    return primkit::TensorDescriptor::packed({d[0], d[1], d[2], d[3]},
                                             static_cast<primkit::ElementType>(et));
}

std::int64_t bn_stat_count(primkit_batchnorm_mode mode, const int64_t d[4]) {
    return mode == PRIMKIT_BN_PER_ACTIVATION ? d[1] * d[2] * d[3] : d[1];
}

}  // namespace

extern "C" {

const char* primkit_last_error(void) { return g_last_error.c_str(); }

primkit_status primkit_handle_create(primkit_handle** out) {
    return guarded([&] {
        need(out, "handle output");
        *out = new primkit_handle();
    });
}

void primkit_handle_destroy(primkit_handle* handle) { delete handle; }

primkit_status primkit_handle_use_fake_clock(primkit_handle* h) {
    return guarded([&] { H(h).use_fake_clock(); });
}

primkit_status primkit_handle_now_ms(primkit_handle* h, double* out) {
    return guarded([&] { *need(out, "output") = H(h).now_ms(); });
}

primkit_status primkit_handle_set_cache_dir(primkit_handle* h, const char* dir) {
    return guarded([&] { H(h).set_cache_dir(need(dir, "directory")); });
}

primkit_status primkit_handle_counters(primkit_handle* h, primkit_counters* out) {
    return guarded([&] {
        const primkit::OpCounters& c = H(h).counters();
        need(out, "output");
        out->gemm_calls = c.gemm_calls;
        out->scalar_muls = c.scalar_muls;
        out->buffer_roundtrips = c.buffer_roundtrips;
    });
}

primkit_status primkit_handle_reset_counters(primkit_handle* h) {
    return guarded([&] { H(h).counters().reset(); });
}

primkit_status primkit_handle_set_seed(primkit_handle* h, uint64_t seed) {
    return guarded([&] { H(h).rng_seed = seed; });
}

primkit_status primkit_problem_key(const primkit_conv_problem* p, char* buf, size_t len) {
    return guarded([&] { copy_name(buf, len, to_problem(p).key()); });
}

primkit_status primkit_conv_output_dims(const primkit_conv_problem* p, int64_t dims[4]) {
    return guarded([&] {
        const primkit::TensorDescriptor d = result_desc(to_problem(p));
        for (int i = 0; i < 4; ++i) dims[i] = d.dims[static_cast<size_t>(i)];
    });
}

primkit_status primkit_solver_count(primkit_handle* h, int* out) {
    return guarded([&] { *need(out, "output") = static_cast<int>(H(h).solvers().size()); });
}

primkit_status primkit_solver_name(primkit_handle* h, int index, char* buf, size_t len) {
    return guarded([&] {
        const auto& s = H(h).solvers();
        if (index < 0 || index >= static_cast<int>(s.size()))
            primkit::throw_error(primkit::ErrorCode::InvalidValue, "solver index out of range");
        copy_name(buf, len, s[static_cast<size_t>(index)]->name());
    });
}

primkit_status primkit_solver_is_applicable(primkit_handle* h, const char* name,
                                            const primkit_conv_problem* p, int* out) {
    return guarded([&] { *out = solver_named(h, name).is_applicable(to_problem(p)) ? 1 : 0; });
}

primkit_status primkit_solver_is_tunable(primkit_handle* h, const char* name, int* out) {
    return guarded([&] { *out = solver_named(h, name).is_tunable() ? 1 : 0; });
}

primkit_status primkit_solver_workspace_bytes(primkit_handle* h, const char* name,
                                              const primkit_conv_problem* pp, uint64_t* out) {
    return guarded([&] {
        const primkit::Solver& s = solver_named(h, name);
        const primkit::ConvProblem p = to_problem(pp);
        const primkit::PerfConfig cfg = H(h).resolve_config(p, s);
        *out = s.workspace_bytes(p, &cfg);
    });
}

primkit_status primkit_find_convolution(primkit_handle* h, const primkit_conv_problem* pp,
                                        const float* a, const float* b, size_t ws_bytes,
                                        primkit_algo_perf* results, int capacity, int* out_count) {
    return guarded([&] {
        const primkit::ConvProblem p = to_problem(pp);
        const auto [da, db] = operand_descs(p);
        primkit::Handle& hd = H(h);
        void* dva = hd.scratch(1, primkit::device_bytes(da));
        void* dvb = hd.scratch(2, primkit::device_bytes(db));
        primkit::upload_nchw(hd, da, need(a, "operand a"), dva);
        primkit::upload_nchw(hd, db, need(b, "operand b"), dvb);
        const auto perf = hd.find_convolution(p, dva, dvb, ws_bytes);
        *out_count = static_cast<int>(perf.size());
        const int n = std::min(capacity, *out_count);
        for (int i = 0; i < n; ++i) {
            const auto& src = perf[static_cast<size_t>(i)];
            copy_name(results[i].solver_name, sizeof(results[i].solver_name), src.solver_name);
            results[i].algo = static_cast<primkit_conv_algo>(src.algo);
            results[i].time_ms = src.time_ms;
            results[i].workspace_bytes = src.workspace_bytes;
        }
    });
}

primkit_status primkit_conv_run(primkit_handle* h, const primkit_conv_problem* pp,
                                const char* solver_name, const float* a, const float* b,
                                float* output, size_t ws_bytes) {
    return guarded([&] {
        const primkit::ConvProblem p = to_problem(pp);
        const primkit::Solver& solver = select_solver(h, p, solver_name);
        primkit::Handle& hd = H(h);
        const primkit::PerfConfig cfg = hd.resolve_config(p, solver);
        if (solver.workspace_bytes(p, &cfg) > ws_bytes)
            primkit::throw_error(primkit::ErrorCode::WorkspaceTooSmall,
                                 "workspace too small for " + solver.name());
        if (const int nc = host_chunk_images(p, need(a, "operand a"), need(output, "output"))) {
            conv_run_chunked(hd, p, solver, cfg, a, b, output, nc);
            return;
        }
        const auto [da, db] = operand_descs(p);
        const primkit::TensorDescriptor dr = result_desc(p);
        void* dva = hd.scratch(1, primkit::device_bytes(da));
        void* dvb = hd.scratch(2, primkit::device_bytes(db));
        void* dvo = hd.scratch(3, primkit::device_bytes(dr));
        primkit::upload_nchw(hd, da, need(a, "operand a"), dva);
        primkit::upload_nchw(hd, db, need(b, "operand b"), dvb);
        auto plan = hd.cached_build(p, solver, &cfg);
        const size_t dws = plan->device_workspace_bytes(hd.num_sms());
        void* ws = hd.scratch(0, dws);
        if (hd.device_timing())
            hd.record_device_ms(hd.time_ms([&] { plan->run(hd, dva, dvb, dvo, ws, dws); }));
        else
            plan->run(hd, dva, dvb, dvo, ws, dws);
        primkit::download_nchw(hd, dr, dvo, need(output, "output"));
    });
}

primkit_status primkit_tune(primkit_handle* h, const primkit_conv_problem* pp,
                            const char* solver_name, int64_t budget, int exhaustive,
                            int64_t* evals) {
    return guarded([&] {
        const primkit::ConvProblem p = to_problem(pp);
        const primkit::Solver& s = solver_named(h, solver_name);
        if (budget <= 0) budget = primkit::default_tune_budget(s, p);
        const primkit::TuneResult r = primkit::tune(H(h), s, p, budget, exhaustive != 0);
        if (evals) *evals = r.evaluations;
    });
}

primkit_status primkit_perfdb_save(primkit_handle* h, const char* path) {
    return guarded([&] { H(h).perfdb().save(need(path, "path")); });
}

primkit_status primkit_perfdb_load(primkit_handle* h, const char* path) {
    return guarded([&] { H(h).perfdb() = primkit::PerfDb::load(need(path, "path")); });
}

primkit_status primkit_fusion_plan_create(const int64_t dims[4], primkit_element_type et,
                                          primkit_fusion_plan** out) {
    return guarded([&] {
        need(out, "plan output");
        *out = new primkit_fusion_plan{primkit::FusionPlan(dims4(dims, et))};
    });
}

void primkit_fusion_plan_destroy(primkit_fusion_plan* plan) { delete plan; }

primkit_status primkit_fusion_add_conv(primkit_fusion_plan* plan, const int64_t fd[4],
                                       int64_t pad_h, int64_t pad_w, int64_t stride_h,
                                       int64_t stride_w, int64_t groups, primkit_conv_algo algo) {
    return guarded([&] {
        primkit::ConvDescriptor cv;
        cv.pad_h = pad_h;
        cv.pad_w = pad_w;
        cv.stride_h = stride_h;
        cv.stride_w = stride_w;
        cv.group_count = groups;
        primkit::FusionPlan& pl = P(plan);
        pl.add_op(primkit::FusionOp::conv_forward(
            cv, dims4(fd, static_cast<primkit_element_type>(pl.input_desc().etype)),
            static_cast<primkit::ConvAlgo>(algo)));
    });
}

primkit_status primkit_fusion_add_bias(primkit_fusion_plan* plan, int64_t channels) {
    return guarded([&] { P(plan).add_op(primkit::FusionOp::bias(channels)); });
}

primkit_status primkit_fusion_add_batchnorm(primkit_fusion_plan* plan, primkit_batchnorm_mode m) {
    return guarded([&] {
        P(plan).add_op(primkit::FusionOp::batchnorm_inference(
            m == PRIMKIT_BN_PER_ACTIVATION ? primkit::BatchNormMode::PerActivation
                                           : primkit::BatchNormMode::Spatial));
    });
}

primkit_status primkit_fusion_add_activation(primkit_fusion_plan* plan, primkit_activation kind,
                                             float alpha) {
    return guarded([&] {
        primkit::ActivationKind act;
        switch (kind) {
            case PRIMKIT_ACT_RELU: act = {primkit::ActivationKind::Tag::ReLU, 0.0f}; break;
            case PRIMKIT_ACT_LEAKY_RELU: act = {primkit::ActivationKind::Tag::LeakyReLU, alpha}; break;
            case PRIMKIT_ACT_SIGMOID: act = {primkit::ActivationKind::Tag::Sigmoid, 0.0f}; break;
            case PRIMKIT_ACT_TANH: act = {primkit::ActivationKind::Tag::Tanh, 0.0f}; break;
            default: primkit::throw_error(primkit::ErrorCode::InvalidValue, "unknown activation kind");
        }
        P(plan).add_op(primkit::FusionOp::activation(act));
    });
}

primkit_status primkit_fusion_compile(primkit_handle* h, primkit_fusion_plan* plan) {
    return guarded([&] { primkit::fusion_compile(H(h), P(plan)); });
}

primkit_status primkit_fusion_output_dims(primkit_fusion_plan* plan, int64_t dims[4]) {
    return guarded([&] {
        const auto& d = P(plan).output_desc().dims;
        for (int i = 0; i < 4; ++i) dims[i] = d[static_cast<size_t>(i)];
    });
}

primkit_status primkit_fusion_set_args(primkit_fusion_plan* plan, const float* filter,
                                       const float* bias, const float* g, const float* b,
                                       const float* mean, const float* var, float eps,
                                       const float* act_alpha) {
    return guarded([&] {
        primkit::FusionPlan& pl = P(plan);
        primkit::FusionArgs args;
        primkit::TensorDescriptor cur = pl.input_desc();
        using K = primkit::FusionOp::Kind;
        for (const primkit::FusionOp& op : pl.ops()) {
            switch (op.kind) {
                case K::ConvForward:
                    if (filter) args.filter = host_tensor(op.filter_desc, filter);
                    cur = primkit::output_dims(cur, op.filter_desc, op.conv);
                    break;
                case K::Bias:
                    if (bias) args.bias = host_tensor(primkit::TensorDescriptor::packed({op.bias_channels}), bias);
                    break;
                case K::BatchNormInference: {
                    const primkit::TensorDescriptor shape =
                        op.bn_mode == primkit::BatchNormMode::Spatial
                            ? primkit::TensorDescriptor::packed({1, cur.dims[1], 1, 1})
                            : primkit::TensorDescriptor::packed({1, cur.dims[1], cur.dims[2], cur.dims[3]});
                    // flat f32 parameter vectors
                    const auto flat = primkit::TensorDescriptor::packed({shape.elem_count()});
                    if (g) args.bn_gamma = host_tensor(flat, g);
                    if (b) args.bn_beta = host_tensor(flat, b);
                    if (mean) args.bn_mean = host_tensor(flat, mean);
                    if (var) args.bn_var = host_tensor(flat, var);
                    args.bn_epsilon = eps;
                    break;
                }
                case K::Activation: break;
            }
        }
        if (act_alpha) args.act_alpha = *act_alpha;
        pl.set_args(std::move(args));
    });
}

primkit_status primkit_fusion_execute(primkit_handle* h, primkit_fusion_plan* plan,
                                      const float* input, float* output, int unfused) {
    return guarded([&] {
        primkit::FusionPlan& pl = P(plan);
        primkit::Handle& hd = H(h);
        if (!pl.compiled())
            primkit::throw_error(primkit::ErrorCode::NotCompiled, "fusion plan is not compiled");
        // bindings are validated before any device work (MissingArgs is a
        // host-side error in the reference too)
        {
            const auto& a = pl.args();
            for (const auto& op : pl.ops()) {
                using K = primkit::FusionOp::Kind;
                if (op.kind == K::ConvForward && !a.filter)
                    primkit::throw_error(primkit::ErrorCode::MissingArgs, "filter not bound");
                if (op.kind == K::Bias && !a.bias)
                    primkit::throw_error(primkit::ErrorCode::MissingArgs, "bias not bound");
                if (op.kind == K::BatchNormInference &&
                    (!a.bn_gamma || !a.bn_beta || !a.bn_mean || !a.bn_var))
                    primkit::throw_error(primkit::ErrorCode::MissingArgs,
                                         "batchnorm parameters not bound");
            }
        }
        const primkit::TensorDescriptor& din = pl.input_desc();
        const primkit::TensorDescriptor dout = primkit::TensorDescriptor::packed(
            pl.output_desc().dims, din.etype);
        void* dvi = hd.scratch(1, primkit::device_bytes(din));
        void* dvo = hd.scratch(2, primkit::device_bytes(dout));
        primkit::upload_nchw(hd, din, need(input, "input"), dvi);
        auto run = [&] {
            if (unfused)
                primkit::fusion_execute_unfused(hd, pl, dvi, dvo);
            else
                primkit::fusion_execute(hd, pl, dvi, dvo);
        };
        if (hd.device_timing())
            hd.record_device_ms(hd.time_ms(run));
        else
            run();
        primkit::download_nchw(hd, dout, dvo, need(output, "output"));
    });
}

// ---- section 2 --------------------------------------------------------------

primkit_status primkit_handle_create_with_stream(void* stream, int device, primkit_handle** out) {
    return guarded([&] {
        need(out, "handle output");
        *out = new primkit_handle(static_cast<cudaStream_t>(stream), device);
    });
}

primkit_status primkit_handle_set_stream(primkit_handle* h, void* stream) {
    return guarded([&] { H(h).set_stream(static_cast<cudaStream_t>(stream)); });
}

int64_t primkit_channel_pitch(int64_t c) { return (c + 7) / 8 * 8; }

primkit_status primkit_conv_device_workspace(primkit_handle* h, const primkit_conv_problem* pp,
                                             const char* solver_name, uint64_t* out) {
    return guarded([&] {
        const primkit::ConvProblem p = to_problem(pp);
        const primkit::Solver& s = select_solver(h, p, solver_name);
        auto plan = H(h).cached_build(p, s, nullptr);
        *need(out, "output") = plan->device_workspace_bytes(H(h).num_sms());
    });
}

primkit_status primkit_conv_run_device(primkit_handle* h, const primkit_conv_problem* pp,
                                       const char* solver_name, const void* a, const void* b,
                                       void* output, void* workspace, size_t ws_bytes) {
    return guarded([&] {
        const primkit::ConvProblem p = to_problem(pp);
        const primkit::Solver& s = select_solver(h, p, solver_name);
        auto plan = H(h).cached_build(p, s, nullptr);
        plan->run(H(h), need(a, "operand a"), need(b, "operand b"), need(output, "output"),
                  workspace, ws_bytes);
    });
}

// Per-CTA fp32 partials (+ 2 x C finalize scratch) over the channels of the
// convolution OUTPUT (K forward, C backward data), then the standalone BN's
// scratch (its per-CTA double partials): all of it from the caller's workspace.
static std::size_t conv_bn_part_bytes(const primkit::ConvProblem& p) {
    const std::size_t ch = p.direction == primkit::ConvDirection::BackwardData ? p.c : p.k;
    return (((std::size_t)pk_stats_slots() + 1) * ch * 2 * sizeof(float) + 255) / 256 * 256;
}

static std::size_t conv_bn_stats_bytes(const primkit::ConvProblem& p) {
    const primkit::ConvShapes sh = primkit::resolve_shapes(p.input_desc(), p.filter_desc(),
                                                            p.conv_desc());
    const bool bwd = p.direction == primkit::ConvDirection::BackwardData;
    const int ch = (int)(bwd ? sh.c : sh.k), hw = (int)(bwd ? sh.h * sh.w : sh.oh * sh.ow);
    return conv_bn_part_bytes(p) + pk_bn_scratch_bytes((int)sh.n, ch, hw, 0);
}

primkit_status primkit_conv_bn_workspace(primkit_handle* h, const primkit_conv_problem* pp,
                                         const char* solver_name, uint64_t* out) {
    return guarded([&] {
        const primkit::ConvProblem p = to_problem(pp);
        const primkit::Solver& s = select_solver(h, p, solver_name);
        auto plan = H(h).cached_build(p, s, nullptr);
        const std::size_t conv = (plan->device_workspace_bytes(H(h).num_sms()) + 255) / 256 * 256;
        *need(out, "output") = conv + conv_bn_stats_bytes(p);
    });
}

// Statistics in the conv epilogue pay off only when the convolution leaves
// the epilogue slack: spatial filters, or 1x1 layers of high arithmetic
// intensity. On HBM-bound 1x1 layers the epilogue is the critical path and the
// per-channel reductions there cost more than the separate statistics read
// they save (measured, ResNet-50 N=256: conv2_1c 0.388 ms fused vs 0.348 ms
// conv + standalone BN; conv4_2a 0.080 vs 0.090). PK_CBN_FUSE=1 / 0 forces.
// Statistics in the conv epilogue save the BN statistics pass's read of the conv
// output. Measured per layer on all 53 ResNet-50 convs at N=256 (tools/bench_configs.py
// cfg4, profiles/r02_cfg4_layers.json) against conv + the single-launch BN
// (bn_coop.cu), whose two passes over the output are L2 hits for every layer whose
// output fits the 126 MB L2: the epilogue form was slower or equal on 51 of 53
// layers (its atomics and the partial-buffer reset cost more than an L2 re-read), so
// it is opt-in (PK_CBN_FUSE=1). The saving that remains is the normalised output's
// HBM round trip, which needs the NEXT convolution to apply BN + ReLU while loading
// its A operand.
bool stats_epilogue_pays(const primkit::ConvProblem&, const primkit::ConvShapes&) {
    if (const char* v = std::getenv("PK_CBN_FUSE")) return v[0] != '0';
    return false;
}

primkit_status primkit_conv_bn_forward_train_device(
    primkit_handle* h, const primkit_conv_problem* pp, const char* solver_name, const void* x,
    const void* w, const float* gamma, const float* beta, float* running_mean, float* running_var,
    float eps, float momentum, void* conv_out, void* y, float* saved_mean, float* saved_invstd,
    int relu, void* workspace, size_t ws_bytes) {
    return guarded([&] {
        if (eps <= 0.0f)
            primkit::throw_error(primkit::ErrorCode::InvalidEpsilon, "epsilon must be positive");
        const primkit::ConvProblem p = to_problem(pp);
        if (p.direction != primkit::ConvDirection::Forward || p.mode != primkit::ConvMode::Convolution)
            primkit::throw_error(primkit::ErrorCode::InvalidValue,
                                 "conv+BN fusion needs a forward convolution");
        const primkit::Solver& s = select_solver(h, p, solver_name);
        auto plan = H(h).cached_build(p, s, nullptr);
        primkit::Handle& hd = H(h);
        hd.activate();
        const std::size_t conv = (plan->device_workspace_bytes(hd.num_sms()) + 255) / 256 * 256;
        if (ws_bytes < conv + conv_bn_stats_bytes(p))
            primkit::throw_error(primkit::ErrorCode::WorkspaceTooSmall, "workspace below requested size");
        const primkit::ConvShapes sh = primkit::resolve_shapes(p.input_desc(), p.filter_desc(),
                                                                p.conv_desc());
        const int n = (int)sh.n, k = (int)sh.k, hw = (int)(sh.oh * sh.ow);
        const int dt = p.etype == primkit::ElementType::BF16 ? PK_BF16 : PK_F32;
        float* part = reinterpret_cast<float*>(static_cast<char*>(workspace) + conv);
        const bool fused = dt == PK_BF16 && plan->fuses_stats() && stats_epilogue_pays(p, sh);
        cudaStream_t st = hd.stream();
        if (fused) {
            primkit::check_cuda(cudaMemsetAsync(part, 0, conv_bn_part_bytes(p), st), "memset");
            pk_epilogue e{};
            e.act = -1;
            e.stats = part;
            plan->run(hd, need(x, "x"), need(w, "w"), need(conv_out, "conv_out"), workspace, conv, &e);
            primkit::check_cuda(pk_cuda_bn_finalize_apply(part, pk_stats_slots(), conv_out, need(y, "y"),
                                                          n, k, hw, pk_pitch(k), dt, gamma, beta,
                                                          running_mean, running_var, eps, momentum,
                                                          saved_mean, saved_invstd, relu, st),
                                "bn_finalize_apply");
            hd.last_kernel = hd.last_kernel + "+bn_stats_epilogue";
        } else {
            plan->run(hd, need(x, "x"), need(w, "w"), need(conv_out, "conv_out"), workspace, conv);
            void* scratch = static_cast<char*>(workspace) + conv + conv_bn_part_bytes(p);
            primkit::check_cuda(pk_cuda_bn_fwd_train(conv_out, need(y, "y"), n, k, hw, pk_pitch(k), dt,
                                                     0, gamma, beta, running_mean, running_var, eps,
                                                     momentum, saved_mean, saved_invstd, relu,
                                                     scratch, st),
                                "bn_fwd_train");
        }
    });
}

primkit_status primkit_conv_backward_data_bn_device(
    primkit_handle* h, const primkit_conv_problem* pp, const char* solver_name, const void* dy,
    const void* w, void* dz, const void* bn_x, const float* gamma, const float* beta,
    const float* saved_mean, const float* saved_invstd, int relu, void* bn_dx, float* dgamma,
    float* dbeta, void* workspace, size_t ws_bytes) {
    return guarded([&] {
        const primkit::ConvProblem p = to_problem(pp);
        if (p.direction != primkit::ConvDirection::BackwardData ||
            p.mode != primkit::ConvMode::Convolution)
            primkit::throw_error(primkit::ErrorCode::InvalidValue,
                                 "dgrad+BN fusion needs a backward-data convolution");
        const primkit::Solver& s = select_solver(h, p, solver_name);
        auto plan = H(h).cached_build(p, s, nullptr);
        primkit::Handle& hd = H(h);
        hd.activate();
        const std::size_t conv = (plan->device_workspace_bytes(hd.num_sms()) + 255) / 256 * 256;
        if (ws_bytes < conv + conv_bn_stats_bytes(p))
            primkit::throw_error(primkit::ErrorCode::WorkspaceTooSmall, "workspace below requested size");
        const int n = (int)p.n, c = (int)p.c, hw = (int)(p.h * p.w);
        const int dt = p.etype == primkit::ElementType::BF16 ? PK_BF16 : PK_F32;
        float* part = reinterpret_cast<float*>(static_cast<char*>(workspace) + conv);
        float* tot = part + (std::size_t)pk_stats_slots() * c * 2;
        cudaStream_t st = hd.stream();
        void* scratch = static_cast<char*>(workspace) + conv + conv_bn_part_bytes(p);
        // BN statistics in the dgrad epilogue (PK_CBN_BWD_EPI=1) re-read the BN
        // input inside the epilogue on the MMA pipeline's critical path; measured
        // slower (ResNet-50 N=256: 13.5 ms vs 10.2 ms for all layers) than the
        // plain dgrad + ONE persistent BN-backward launch that recomputes the ReLU
        // mask from the BN input (no BN output read, no y rebuild).
        const char* epi_env = std::getenv("PK_CBN_BWD_EPI");
        const bool epi_stats = epi_env && epi_env[0] == '1';
        if (dt == PK_BF16 && epi_stats && plan->fuses_stats()) {
            primkit::check_cuda(cudaMemsetAsync(part, 0, (std::size_t)pk_stats_slots() * c * 2 * 4, st),
                                "memset");
            pk_epilogue e{};
            e.act = -1;
            e.stats = part;
            e.bnb_y = need(bn_x, "bn_x");
            e.bnb_gamma = gamma;
            e.bnb_beta = beta;
            e.bnb_mean = saved_mean;
            e.bnb_invstd = saved_invstd;
            e.bnb_relu = relu;
            plan->run(hd, need(dy, "dy"), need(w, "w"), need(dz, "dz"), workspace, conv, &e);
            primkit::check_cuda(pk_cuda_bn_bwd_finalize_apply(part, pk_stats_slots(), dz, bn_x,
                                                              need(bn_dx, "bn_dx"), n, c, hw,
                                                              pk_pitch(c), dt, gamma, beta,
                                                              saved_mean, saved_invstd, relu,
                                                              dgamma, dbeta, tot, st),
                                "bn_bwd_finalize_apply");
            hd.last_kernel = hd.last_kernel + "+bn_bwd_stats_epilogue";
            return;
        }
        plan->run(hd, need(dy, "dy"), need(w, "w"), need(dz, "dz"), workspace, conv);
        const cudaError_t fe = pk_cuda_bn_bwd_fold(need(bn_x, "bn_x"), dz, need(bn_dx, "bn_dx"), n, c, hw,
                                                   pk_pitch(c), dt, gamma, beta, saved_mean,
                                                   saved_invstd, relu, dgamma, dbeta, scratch, st);
        if (fe == cudaSuccess) {
            hd.last_kernel = hd.last_kernel + "+bn_bwd_fold";
            return;
        }
        if (fe != cudaErrorNotSupported) primkit::check_cuda(fe, "bn_bwd_fold");
        cudaGetLastError();
        // other layouts (f32): rebuild the BN output for the ReLU mask, then the
        // standalone backward
        void* ybuf = hd.scratch(8, (std::size_t)n * hw * pk_pitch(c) * (dt == PK_BF16 ? 2 : 4));
        primkit::check_cuda(pk_cuda_bn_apply_stats(bn_x, ybuf, n, c, hw, pk_pitch(c), dt, gamma,
                                                   beta, saved_mean, saved_invstd, relu, st),
                            "bn_apply");
        primkit::check_cuda(pk_cuda_bn_bwd(bn_x, ybuf, dz, bn_dx, n, c, hw, pk_pitch(c), dt, 0, gamma,
                                           saved_mean, saved_invstd, dgamma, dbeta, relu,
                                           dt == PK_BF16, scratch, st),
                            "bn_bwd");
    });
}

primkit_status primkit_fusion_execute_device(primkit_handle* h, primkit_fusion_plan* plan,
                                             const void* input, void* output, int unfused) {
    return guarded([&] {
        if (unfused)
            primkit::fusion_execute_unfused(H(h), P(plan), need(input, "input"), need(output, "output"));
        else
            primkit::fusion_execute(H(h), P(plan), need(input, "input"), need(output, "output"));
    });
}

primkit_status primkit_batchnorm_forward_train(primkit_handle* h, primkit_batchnorm_mode mode,
                                               const int64_t dims[4], primkit_element_type et,
                                               const float* x, const float* gamma,
                                               const float* beta, float* running_mean,
                                               float* running_var, float eps, float momentum,
                                               float* y, float* saved_mean, float* saved_invstd) {
    return guarded([&] {
        if (eps <= 0.0f)
            primkit::throw_error(primkit::ErrorCode::InvalidEpsilon, "epsilon must be positive");
        const primkit::TensorDescriptor d = dims4(dims, et);
        primkit::Handle& hd = H(h);
        const std::int64_t ns = bn_stat_count(mode, dims);
        const int per_act = mode == PRIMKIT_BN_PER_ACTIVATION;
        const int n = (int)dims[0], c = (int)dims[1], hw = (int)(dims[2] * dims[3]);
        void* dx = hd.scratch(1, primkit::device_bytes(d));
        void* dy = hd.scratch(2, primkit::device_bytes(d));
        float* par = static_cast<float*>(hd.scratch(6, (size_t)ns * 6 * 4));
        void* scratch = hd.scratch(7, pk_bn_scratch_bytes(n, c, hw, per_act));
        primkit::upload_nchw(hd, d, need(x, "x"), dx);
        const size_t vb = (size_t)ns * 4;
        auto up = [&](float* dst, const float* src) {
            primkit::check_cuda(cudaMemcpyAsync(dst, need(src, "parameter"), vb,
                                                cudaMemcpyHostToDevice, hd.stream()),
                                "cudaMemcpyAsync");
        };
        up(par, gamma);
        up(par + ns, beta);
        up(par + 2 * ns, running_mean);
        up(par + 3 * ns, running_var);
        primkit::check_cuda(
            pk_cuda_bn_fwd_train(dx, dy, n, c, hw, pk_pitch(c),
                                 et == PRIMKIT_BF16 ? PK_BF16 : PK_F32, per_act, par, par + ns,
                                 par + 2 * ns, par + 3 * ns, eps, momentum, par + 4 * ns,
                                 par + 5 * ns, 0, scratch, hd.stream()),
            "bn_fwd_train");
        primkit::download_nchw(hd, d, dy, need(y, "y"));
        auto down = [&](float* dst, const float* src) {
            primkit::check_cuda(cudaMemcpyAsync(need(dst, "output"), src, vb,
                                                cudaMemcpyDeviceToHost, hd.stream()),
                                "cudaMemcpyAsync");
        };
        down(running_mean, par + 2 * ns);
        down(running_var, par + 3 * ns);
        down(saved_mean, par + 4 * ns);
        down(saved_invstd, par + 5 * ns);
        hd.sync();
    });
}

primkit_status primkit_batchnorm_forward_infer(primkit_handle* h, primkit_batchnorm_mode mode,
                                               const int64_t dims[4], primkit_element_type et,
                                               const float* x, const float* gamma,
                                               const float* beta, const float* running_mean,
                                               const float* running_var, float eps, float* y) {
    return guarded([&] {
        if (eps <= 0.0f)
            primkit::throw_error(primkit::ErrorCode::InvalidEpsilon, "epsilon must be positive");
        const primkit::TensorDescriptor d = dims4(dims, et);
        primkit::Handle& hd = H(h);
        const std::int64_t ns = bn_stat_count(mode, dims);
        const int n = (int)dims[0], c = (int)dims[1], hw = (int)(dims[2] * dims[3]);
        void* dx = hd.scratch(1, primkit::device_bytes(d));
        void* dy = hd.scratch(2, primkit::device_bytes(d));
        float* par = static_cast<float*>(hd.scratch(6, (size_t)ns * 4 * 4));
        primkit::upload_nchw(hd, d, need(x, "x"), dx);
        const float* src[4] = {gamma, beta, running_mean, running_var};
        for (int i = 0; i < 4; ++i)
            primkit::check_cuda(cudaMemcpyAsync(par + i * ns, need(src[i], "parameter"),
                                                (size_t)ns * 4, cudaMemcpyHostToDevice,
                                                hd.stream()),
                                "cudaMemcpyAsync");
        pk_epilogue e{};
        e.act = -1;
        e.bn_gamma = par;
        e.bn_beta = par + ns;
        e.bn_mean = par + 2 * ns;
        e.bn_var = par + 3 * ns;
        e.bn_per_activation = mode == PRIMKIT_BN_PER_ACTIVATION;
        e.bn_standalone = 1;
        e.bn_eps = eps;
        primkit::check_cuda(pk_cuda_pointwise(dx, dy, n, c, hw, pk_pitch(c),
                                              et == PRIMKIT_BF16 ? PK_BF16 : PK_F32, &e,
                                              hd.stream()),
                            "pointwise");
        primkit::download_nchw(hd, d, dy, need(y, "y"));
    });
}

primkit_status primkit_batchnorm_backward(primkit_handle* h, primkit_batchnorm_mode mode,
                                          const int64_t dims[4], primkit_element_type et,
                                          const float* x, const float* dy, const float* gamma,
                                          const float* saved_mean, const float* saved_invstd,
                                          float* dx, float* dgamma, float* dbeta) {
    return guarded([&] {
        const primkit::TensorDescriptor d = dims4(dims, et);
        primkit::Handle& hd = H(h);
        const std::int64_t ns = bn_stat_count(mode, dims);
        const int per_act = mode == PRIMKIT_BN_PER_ACTIVATION;
        const int n = (int)dims[0], c = (int)dims[1], hw = (int)(dims[2] * dims[3]);
        void* dvx = hd.scratch(1, primkit::device_bytes(d));
        void* dvdy = hd.scratch(2, primkit::device_bytes(d));
        void* dvdx = hd.scratch(3, primkit::device_bytes(d));
        float* par = static_cast<float*>(hd.scratch(6, (size_t)ns * 5 * 4));
        void* scratch = hd.scratch(7, pk_bn_scratch_bytes(n, c, hw, per_act));
        primkit::upload_nchw(hd, d, need(x, "x"), dvx);
        primkit::upload_nchw(hd, d, need(dy, "dy"), dvdy);
        const float* src[3] = {gamma, saved_mean, saved_invstd};
        for (int i = 0; i < 3; ++i)
            primkit::check_cuda(cudaMemcpyAsync(par + i * ns, need(src[i], "parameter"),
                                                (size_t)ns * 4, cudaMemcpyHostToDevice,
                                                hd.stream()),
                                "cudaMemcpyAsync");
        primkit::check_cuda(
            pk_cuda_bn_bwd(dvx, nullptr, dvdy, dvdx, n, c, hw, pk_pitch(c),
                           et == PRIMKIT_BF16 ? PK_BF16 : PK_F32, per_act, par, par + ns,
                           par + 2 * ns, par + 3 * ns, par + 4 * ns, 0, et == PRIMKIT_BF16,
                           scratch, hd.stream()),
            "bn_bwd");
        primkit::download_nchw(hd, d, dvdx, need(dx, "dx"));
        primkit::check_cuda(cudaMemcpyAsync(need(dgamma, "dgamma"), par + 3 * ns, (size_t)ns * 4,
                                            cudaMemcpyDeviceToHost, hd.stream()),
                            "cudaMemcpyAsync");
        primkit::check_cuda(cudaMemcpyAsync(need(dbeta, "dbeta"), par + 4 * ns, (size_t)ns * 4,
                                            cudaMemcpyDeviceToHost, hd.stream()),
                            "cudaMemcpyAsync");
        hd.sync();
    });
}

primkit_status primkit_batchnorm_forward_train_device(
    primkit_handle* h, const int64_t dims[4], primkit_element_type et, const void* x,
    const float* gamma, const float* beta, float* running_mean, float* running_var, float eps,
    float momentum, void* y, float* saved_mean, float* saved_invstd, int relu) {
    return guarded([&] {
        if (eps <= 0.0f)
            primkit::throw_error(primkit::ErrorCode::InvalidEpsilon, "epsilon must be positive");
        primkit::Handle& hd = H(h);
        hd.activate();
        const int n = (int)dims[0], c = (int)dims[1], hw = (int)(dims[2] * dims[3]);
        void* scratch = hd.scratch(7, pk_bn_scratch_bytes(n, c, hw, 0));
        primkit::check_cuda(pk_cuda_bn_fwd_train(x, y, n, c, hw, pk_pitch(c),
                                                 et == PRIMKIT_BF16 ? PK_BF16 : PK_F32, 0, gamma,
                                                 beta, running_mean, running_var, eps, momentum,
                                                 saved_mean, saved_invstd, relu, scratch,
                                                 hd.stream()),
                            "bn_fwd_train");
    });
}

primkit_status primkit_batchnorm_backward_device(
    primkit_handle* h, const int64_t dims[4], primkit_element_type et, const void* x,
    const void* y, const void* dy, const float* gamma, const float* beta,
    const float* saved_mean, const float* saved_invstd, void* dx, float* dgamma, float* dbeta,
    int relu) {
    (void)beta;
    return guarded([&] {
        primkit::Handle& hd = H(h);
        hd.activate();
        const int n = (int)dims[0], c = (int)dims[1], hw = (int)(dims[2] * dims[3]);
        void* scratch = hd.scratch(7, pk_bn_scratch_bytes(n, c, hw, 0));
        primkit::check_cuda(pk_cuda_bn_bwd(x, y, dy, dx, n, c, hw, pk_pitch(c),
                                           et == PRIMKIT_BF16 ? PK_BF16 : PK_F32, 0, gamma,
                                           saved_mean, saved_invstd, dgamma, dbeta, relu, 0,
                                           scratch, hd.stream()),
                            "bn_bwd");
    });
}

primkit_status primkit_activation_forward(primkit_handle* h, primkit_activation kind, float alpha,
                                          const int64_t dims[4], primkit_element_type et,
                                          const float* x, float* y) {
    return guarded([&] {
        if (kind == PRIMKIT_ACT_LEAKY_RELU && alpha < 0.0f)
            primkit::throw_error(primkit::ErrorCode::InvalidValue, "LeakyReLU alpha must be >= 0");
        const primkit::TensorDescriptor d = dims4(dims, et);
        primkit::Handle& hd = H(h);
        void* dx = hd.scratch(1, primkit::device_bytes(d));
        void* dy = hd.scratch(2, primkit::device_bytes(d));
        primkit::upload_nchw(hd, d, need(x, "x"), dx);
        pk_epilogue e{};
        e.act = static_cast<int>(kind);
        e.act_alpha = alpha;
        const int c = (int)dims[1];
        primkit::check_cuda(pk_cuda_pointwise(dx, dy, (int)dims[0], c, (int)(dims[2] * dims[3]),
                                              pk_pitch(c), et == PRIMKIT_BF16 ? PK_BF16 : PK_F32,
                                              &e, hd.stream()),
                            "pointwise");
        primkit::download_nchw(hd, d, dy, need(y, "y"));
    });
}

primkit_status primkit_activation_backward(primkit_handle* h, primkit_activation kind,
                                           float alpha, const int64_t dims[4],
                                           primkit_element_type et, const float* x,
                                           const float* dy, float* dx) {
    return guarded([&] {
        const primkit::TensorDescriptor d = dims4(dims, et);
        primkit::Handle& hd = H(h);
        void* dvx = hd.scratch(1, primkit::device_bytes(d));
        void* dvdy = hd.scratch(2, primkit::device_bytes(d));
        void* dvdx = hd.scratch(3, primkit::device_bytes(d));
        primkit::upload_nchw(hd, d, need(x, "x"), dvx);
        primkit::upload_nchw(hd, d, need(dy, "dy"), dvdy);
        const int c = (int)dims[1];
        primkit::check_cuda(pk_cuda_activation_bwd(dvx, dvdy, dvdx, (int)dims[0], c,
                                                   (int)(dims[2] * dims[3]), pk_pitch(c),
                                                   et == PRIMKIT_BF16 ? PK_BF16 : PK_F32,
                                                   static_cast<int>(kind), alpha, hd.stream()),
                            "activation_bwd");
        primkit::download_nchw(hd, d, dvdx, need(dx, "dx"));
    });
}

primkit_status primkit_nchw_to_device(primkit_handle* h, const int64_t dims[4],
                                      primkit_element_type et, const float* src, void* dst) {
    return guarded([&] {
        primkit::Handle& hd = H(h);
        hd.activate();
        const int c = (int)dims[1];
        primkit::check_cuda(pk_cuda_nchw_to_nhwc(src, dst, (int)dims[0], c,
                                                 (int)(dims[2] * dims[3]), pk_pitch(c),
                                                 et == PRIMKIT_BF16 ? PK_BF16 : PK_F32,
                                                 hd.stream()),
                            "nchw_to_nhwc");
    });
}

primkit_status primkit_device_to_nchw(primkit_handle* h, const int64_t dims[4],
                                      primkit_element_type et, const void* src, float* dst) {
    return guarded([&] {
        primkit::Handle& hd = H(h);
        hd.activate();
        const int c = (int)dims[1];
        primkit::check_cuda(pk_cuda_nhwc_to_nchw(src, dst, (int)dims[0], c,
                                                 (int)(dims[2] * dims[3]), pk_pitch(c),
                                                 et == PRIMKIT_BF16 ? PK_BF16 : PK_F32,
                                                 hd.stream()),
                            "nhwc_to_nchw");
    });
}

primkit_status primkit_handle_kernel_launches(primkit_handle* h, uint64_t* out) {
    return guarded([&] {
        (void)H(h);
        *need(out, "output") = pk_cuda_launch_count();
    });
}

primkit_status primkit_handle_last_device_ms(primkit_handle* h, double* out) {
    return guarded([&] { *need(out, "output") = H(h).last_device_ms(); });
}

primkit_status primkit_handle_last_kernel(primkit_handle* h, char* buf, size_t len) {
    return guarded([&] { copy_name(buf, len, H(h).last_kernel); });
}

primkit_status primkit_handle_last_variant(primkit_handle* h, char* buf, size_t len) {
    return guarded([&] { copy_name(buf, len, H(h).last_variant); });
}

primkit_status primkit_tune_kernels(primkit_handle* h, const primkit_conv_problem* pp,
                                    const char* solver_name, int64_t budget, char* best_values,
                                    size_t buf_len, double* default_ms, double* best_ms) {
    return guarded([&] {
        const primkit::ConvProblem p = to_problem(pp);
        const primkit::Solver& s = solver_named(h, solver_name);
        if (budget <= 0) budget = 256;
        const primkit::KernelTuneResult r = primkit::tune_kernels(H(h), s, p, budget);
        if (best_values) copy_name(best_values, buf_len, primkit::serialize_kernel_config(r.best));
        if (default_ms) *default_ms = r.default_ms;
        if (best_ms) *best_ms = r.best_ms;
    });
}

primkit_status primkit_plan_kernel_config(primkit_handle* h, const primkit_conv_problem* pp,
                                          const char* solver_name, char* buf, size_t buf_len) {
    return guarded([&] {
        const primkit::ConvProblem p = to_problem(pp);
        const primkit::Solver& s = solver_named(h, solver_name);
        auto plan = H(h).cached_build(p, s, nullptr);
        copy_name(buf, buf_len, primkit::serialize_kernel_config(plan->kernel_config()));
    });
}

primkit_status primkit_handle_load_system_db(primkit_handle* h, const char* path) {
    return guarded([&] { H(h).load_system_db(path ? path : ""); });
}

primkit_status primkit_handle_system_db(primkit_handle* h, char* buf, size_t buf_len,
                                        uint64_t* records) {
    return guarded([&] {
        if (buf) copy_name(buf, buf_len, H(h).system_db_path());
        if (records) *records = H(h).system_db().size();
    });
}

// ---- pooling / softmax (reference primitives.cpp:204-370) -------------------

namespace {

pk_pool_geom pool_geom(const int64_t win[2], const int64_t pad[2], const int64_t str[2],
                       const int64_t d[4]) {
    need(win, "window");
    need(pad, "pad");
    need(str, "stride");
    need(d, "dims");
    // primitives.cpp:207-220: validation order and messages
    if (win[0] < 1 || win[1] < 1 || str[0] < 1 || str[1] < 1 || pad[0] < 0 || pad[1] < 0)
        primkit::throw_error(primkit::ErrorCode::InvalidValue, "bad pooling descriptor");
    for (int i = 0; i < 4; ++i)
        if (d[i] < 0) primkit::throw_error(primkit::ErrorCode::InvalidShape, "negative dimension");
    const int64_t oh = (d[2] + 2 * pad[0] - win[0]) / str[0] + 1;
    const int64_t ow = (d[3] + 2 * pad[1] - win[1]) / str[1] + 1;
    if (oh < 1 || ow < 1)
        primkit::throw_error(primkit::ErrorCode::InvalidShape, "pooling output extent below 1");
    pk_pool_geom g{};
    g.n = (int)d[0]; g.c = (int)d[1]; g.h = (int)d[2]; g.w = (int)d[3];
    g.oh = (int)oh; g.ow = (int)ow;
    g.win_h = (int)win[0]; g.win_w = (int)win[1];
    g.str_h = (int)str[0]; g.str_w = (int)str[1];
    g.pad_h = (int)pad[0]; g.pad_w = (int)pad[1];
    g.pitch = pk_pitch(g.c);
    return g;
}

struct AxisSplit {
    long long outer = 1, axis = 1, inner = 1;
};

// primitives.cpp:312-324
AxisSplit split_axis(int rank, const int64_t* dims, int64_t axis) {
    if (rank < 1 || !dims) primkit::throw_error(primkit::ErrorCode::InvalidShape, "softmax needs a tensor");
    if (axis < 0 || axis >= rank) primkit::throw_error(primkit::ErrorCode::InvalidAxis, "softmax axis out of range");
    AxisSplit s;
    s.axis = dims[axis];
    for (int64_t i = 0; i < axis; ++i) s.outer *= dims[i];
    for (int64_t i = axis + 1; i < rank; ++i) s.inner *= dims[i];
    return s;
}

int dtype_of(primkit_element_type et) { return et == PRIMKIT_BF16 ? PK_BF16 : PK_F32; }

// Packed host floats <-> device elements of `et` (bf16: RNE, the reference's quantize-on-entry).
void* upload_packed(primkit::Handle& hd, int slot, const float* src, size_t count, primkit_element_type et) {
    void* dev = hd.scratch(slot, count * (et == PRIMKIT_BF16 ? 2 : 4));
    if (et == PRIMKIT_BF16) {
        std::vector<uint16_t> bits(count);
        for (size_t i = 0; i < count; ++i) {
            const float v = primkit::round_bf16(src[i]);
            uint32_t u;
            std::memcpy(&u, &v, 4);
            bits[i] = (uint16_t)(u >> 16);
        }
        primkit::check_cuda(cudaMemcpyAsync(dev, bits.data(), count * 2, cudaMemcpyHostToDevice, hd.stream()),
                            "cudaMemcpyAsync");
        hd.sync();  // bits is a stack vector
    } else {
        primkit::check_cuda(cudaMemcpyAsync(dev, src, count * 4, cudaMemcpyHostToDevice, hd.stream()),
                            "cudaMemcpyAsync");
    }
    return dev;
}

void download_packed(primkit::Handle& hd, const void* dev, float* dst, size_t count, primkit_element_type et) {
    if (et == PRIMKIT_BF16) {
        std::vector<uint16_t> bits(count);
        primkit::check_cuda(cudaMemcpyAsync(bits.data(), dev, count * 2, cudaMemcpyDeviceToHost, hd.stream()),
                            "cudaMemcpyAsync");
        hd.sync();
        for (size_t i = 0; i < count; ++i) {
            const uint32_t u = (uint32_t)bits[i] << 16;
            std::memcpy(dst + i, &u, 4);
        }
    } else {
        primkit::check_cuda(cudaMemcpyAsync(dst, dev, count * 4, cudaMemcpyDeviceToHost, hd.stream()),
                            "cudaMemcpyAsync");
        hd.sync();
    }
}

}  // namespace

primkit_status primkit_pooling_output_dims(const int64_t window[2], const int64_t pad[2],
                                           const int64_t stride[2], const int64_t dims[4],
                                           int64_t out_dims[4]) {
    return guarded([&] {
        const pk_pool_geom g = pool_geom(window, pad, stride, dims);
        need(out_dims, "output");
        out_dims[0] = g.n; out_dims[1] = g.c; out_dims[2] = g.oh; out_dims[3] = g.ow;
    });
}

primkit_status primkit_pooling_forward_device(primkit_handle* h, primkit_pooling_kind kind,
                                              const int64_t window[2], const int64_t pad[2],
                                              const int64_t stride[2], const int64_t dims[4],
                                              primkit_element_type et, const void* x, void* y,
                                              int64_t* indices) {
    return guarded([&] {
        const pk_pool_geom g = pool_geom(window, pad, stride, dims);
        primkit::Handle& hd = H(h);
        hd.activate();
        primkit::check_cuda(pk_cuda_pool_fwd(&g, dtype_of(et), kind == PRIMKIT_POOL_MAX, need(x, "x"),
                                             need(y, "y"), reinterpret_cast<long long*>(indices), hd.stream()),
                            "pool_fwd");
        hd.last_kernel = kind == PRIMKIT_POOL_MAX ? "pool_max_fwd" : "pool_avg_fwd";
    });
}

primkit_status primkit_pooling_backward_device(primkit_handle* h, primkit_pooling_kind kind,
                                               const int64_t window[2], const int64_t pad[2],
                                               const int64_t stride[2], const int64_t dims[4],
                                               primkit_element_type et, const void* dy,
                                               const int64_t* indices, void* dx) {
    return guarded([&] {
        const pk_pool_geom g = pool_geom(window, pad, stride, dims);
        if (kind == PRIMKIT_POOL_MAX) need(indices, "indices");
        primkit::Handle& hd = H(h);
        hd.activate();
        primkit::check_cuda(pk_cuda_pool_bwd(&g, dtype_of(et), kind == PRIMKIT_POOL_MAX, need(dy, "dy"),
                                             reinterpret_cast<const long long*>(indices), need(dx, "dx"),
                                             hd.stream()),
                            "pool_bwd");
        hd.last_kernel = kind == PRIMKIT_POOL_MAX ? "pool_max_bwd" : "pool_avg_bwd";
    });
}

primkit_status primkit_pooling_forward(primkit_handle* h, primkit_pooling_kind kind,
                                       const int64_t window[2], const int64_t pad[2],
                                       const int64_t stride[2], const int64_t dims[4],
                                       primkit_element_type et, const float* x, float* y,
                                       int64_t* indices) {
    return guarded([&] {
        const pk_pool_geom g = pool_geom(window, pad, stride, dims);
        primkit::Handle& hd = H(h);
        const primkit::TensorDescriptor din = dims4(dims, et);
        const int64_t od[4] = {g.n, g.c, g.oh, g.ow};
        const primkit::TensorDescriptor dout = dims4(od, et);
        void* dvx = hd.scratch(1, primkit::device_bytes(din));
        void* dvy = hd.scratch(2, primkit::device_bytes(dout));
        const size_t nidx = (size_t)g.n * g.c * g.oh * g.ow;
        long long* dvi = kind == PRIMKIT_POOL_MAX ? static_cast<long long*>(hd.scratch(4, nidx * 8)) : nullptr;
        primkit::upload_nchw(hd, din, need(x, "x"), dvx);
        primkit::check_cuda(pk_cuda_pool_fwd(&g, dtype_of(et), kind == PRIMKIT_POOL_MAX, dvx, dvy, dvi,
                                             hd.stream()),
                            "pool_fwd");
        primkit::download_nchw(hd, dout, dvy, need(y, "y"));
        if (dvi && indices) {  // device order [n][oh][ow][c] -> reference order [n][c][oh][ow]
            std::vector<int64_t> tmp(nidx);
            primkit::check_cuda(cudaMemcpyAsync(tmp.data(), dvi, nidx * 8, cudaMemcpyDeviceToHost, hd.stream()),
                                "cudaMemcpyAsync");
            hd.sync();
            const size_t hw = (size_t)g.oh * g.ow;
            for (size_t n = 0; n < (size_t)g.n; ++n)
                for (size_t p = 0; p < hw; ++p)
                    for (size_t c = 0; c < (size_t)g.c; ++c)
                        indices[(n * g.c + c) * hw + p] = tmp[(n * hw + p) * g.c + c];
        } else if (indices) {
            std::fill(indices, indices + nidx, (int64_t)-1);  // average pooling: no argmax (reference: -1)
        }
    });
}

primkit_status primkit_pooling_backward(primkit_handle* h, primkit_pooling_kind kind,
                                        const int64_t window[2], const int64_t pad[2],
                                        const int64_t stride[2], const int64_t dims[4],
                                        primkit_element_type et, const float* dy,
                                        const int64_t* indices, float* dx) {
    return guarded([&] {
        const pk_pool_geom g = pool_geom(window, pad, stride, dims);
        if (kind == PRIMKIT_POOL_MAX) need(indices, "indices");
        primkit::Handle& hd = H(h);
        const primkit::TensorDescriptor din = dims4(dims, et);
        const int64_t od[4] = {g.n, g.c, g.oh, g.ow};
        const primkit::TensorDescriptor dout = dims4(od, et);
        void* dvdy = hd.scratch(1, primkit::device_bytes(dout));
        void* dvdx = hd.scratch(2, primkit::device_bytes(din));
        const size_t nidx = (size_t)g.n * g.c * g.oh * g.ow;
        long long* dvi = nullptr;
        primkit::upload_nchw(hd, dout, need(dy, "dy"), dvdy);
        if (kind == PRIMKIT_POOL_MAX) {
            const size_t hw = (size_t)g.oh * g.ow;
            std::vector<int64_t> tmp(nidx);
            for (size_t n = 0; n < (size_t)g.n; ++n)
                for (size_t p = 0; p < hw; ++p)
                    for (size_t c = 0; c < (size_t)g.c; ++c)
                        tmp[(n * hw + p) * g.c + c] = indices[(n * g.c + c) * hw + p];
            dvi = static_cast<long long*>(hd.scratch(4, nidx * 8));
            primkit::check_cuda(cudaMemcpyAsync(dvi, tmp.data(), nidx * 8, cudaMemcpyHostToDevice, hd.stream()),
                                "cudaMemcpyAsync");
            hd.sync();
        }
        primkit::check_cuda(pk_cuda_pool_bwd(&g, dtype_of(et), kind == PRIMKIT_POOL_MAX, dvdy, dvi, dvdx,
                                             hd.stream()),
                            "pool_bwd");
        primkit::download_nchw(hd, din, dvdx, need(dx, "dx"));
    });
}

primkit_status primkit_softmax_forward_device(primkit_handle* h, int rank, const int64_t* dims,
                                              primkit_element_type et, int64_t axis, const void* x,
                                              void* y) {
    return guarded([&] {
        const AxisSplit s = split_axis(rank, dims, axis);
        primkit::Handle& hd = H(h);
        hd.activate();
        primkit::check_cuda(pk_cuda_softmax_fwd(dtype_of(et), need(x, "x"), need(y, "y"), s.outer, (int)s.axis,
                                                s.inner, hd.stream()),
                            "softmax_fwd");
    });
}

primkit_status primkit_softmax_backward_device(primkit_handle* h, int rank, const int64_t* dims,
                                               primkit_element_type et, int64_t axis, const void* y,
                                               const void* dy, void* dx) {
    return guarded([&] {
        const AxisSplit s = split_axis(rank, dims, axis);
        primkit::Handle& hd = H(h);
        hd.activate();
        primkit::check_cuda(pk_cuda_softmax_bwd(dtype_of(et), need(y, "y"), need(dy, "dy"), need(dx, "dx"),
                                                s.outer, (int)s.axis, s.inner, hd.stream()),
                            "softmax_bwd");
    });
}

primkit_status primkit_softmax_forward(primkit_handle* h, int rank, const int64_t* dims,
                                       primkit_element_type et, int64_t axis, const float* x, float* y) {
    return guarded([&] {
        const AxisSplit s = split_axis(rank, dims, axis);
        primkit::Handle& hd = H(h);
        hd.activate();
        const size_t count = (size_t)(s.outer * s.axis * s.inner);
        void* dx = upload_packed(hd, 1, need(x, "x"), count, et);
        void* dy = hd.scratch(2, count * (et == PRIMKIT_BF16 ? 2 : 4));
        primkit::check_cuda(pk_cuda_softmax_fwd(dtype_of(et), dx, dy, s.outer, (int)s.axis, s.inner, hd.stream()),
                            "softmax_fwd");
        download_packed(hd, dy, need(y, "y"), count, et);
    });
}

primkit_status primkit_softmax_backward(primkit_handle* h, int rank, const int64_t* dims,
                                        primkit_element_type et, int64_t axis, const float* y,
                                        const float* dy, float* dx) {
    return guarded([&] {
        const AxisSplit s = split_axis(rank, dims, axis);
        primkit::Handle& hd = H(h);
        hd.activate();
        const size_t count = (size_t)(s.outer * s.axis * s.inner);
        void* dvy = upload_packed(hd, 1, need(y, "y"), count, et);
        void* dvdy = upload_packed(hd, 2, need(dy, "dy"), count, et);
        void* dvdx = hd.scratch(3, count * (et == PRIMKIT_BF16 ? 2 : 4));
        primkit::check_cuda(pk_cuda_softmax_bwd(dtype_of(et), dvy, dvdy, dvdx, s.outer, (int)s.axis, s.inner,
                                                hd.stream()),
                            "softmax_bwd");
        download_packed(hd, dvdx, need(dx, "dx"), count, et);
    });
}

primkit_status primkit_handle_plan_cache_stats(primkit_handle* h, uint64_t* builds,
                                              uint64_t* memory_hits, uint64_t* disk_hits) {
    return guarded([&] {
        const auto st = H(h).plan_cache().stats();
        *need(builds, "output") = st.builds;
        *need(memory_hits, "output") = st.memory_hits;
        *need(disk_hits, "output") = st.disk_hits;
    });
}

// ---- section 3: data-parallel gradient all-reduce ---------------------------

static primkit::DataParallel& DP(primkit_dp* d) {
    if (!d || !d->impl) primkit::throw_error(primkit::ErrorCode::InvalidValue, "null dp context");
    return *d->impl;
}

primkit_status primkit_dp_unique_id(uint8_t id[PRIMKIT_DP_UNIQUE_ID_BYTES]) {
    return guarded([&] { primkit::dp_unique_id(need(id, "id")); });
}

primkit_status primkit_dp_create(primkit_handle* h, const uint8_t id[PRIMKIT_DP_UNIQUE_ID_BYTES],
                                 int nranks, int rank, int average, primkit_dp** out) {
    return guarded([&] {
        need(out, "dp output");
        auto d = std::make_unique<primkit_dp>();
        d->impl = primkit::dp_create(H(h), need(id, "id"), nranks, rank, average != 0);
        *out = d.release();
    });
}

void primkit_dp_destroy(primkit_dp* dp) { delete dp; }

primkit_status primkit_dp_set_bucket_bytes(primkit_dp* dp, uint64_t bytes) {
    return guarded([&] { primkit::dp_set_bucket_bytes(DP(dp), bytes); });
}

primkit_status primkit_dp_register(primkit_dp* dp, void* grad, uint64_t elems,
                                   primkit_element_type etype, int* out_index) {
    return guarded([&] {
        const int i = primkit::dp_add(DP(dp), grad, elems, static_cast<primkit::ElementType>(etype));
        if (out_index) *out_index = i;
    });
}

primkit_status primkit_dp_grad_ready(primkit_dp* dp, int index) {
    return guarded([&] { primkit::dp_ready(DP(dp), index); });
}

primkit_status primkit_dp_finish(primkit_dp* dp) {
    return guarded([&] { primkit::dp_finish(DP(dp)); });
}

primkit_status primkit_dp_check(primkit_dp* dp) {
    return guarded([&] { primkit::dp_check(DP(dp)); });
}

primkit_status primkit_dp_buckets(primkit_dp* dp, int* out_count) {
    return guarded([&] { *need(out_count, "output") = primkit::dp_bucket_count(DP(dp)); });
}

primkit_status primkit_dp_bucket_of(primkit_dp* dp, int index, int* out_bucket) {
    return guarded([&] { *need(out_bucket, "output") = primkit::dp_bucket_of(DP(dp), index); });
}

}  // extern "C"
