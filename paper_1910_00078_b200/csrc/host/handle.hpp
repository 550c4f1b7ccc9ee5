// Library context (proj/src/core/handle.hpp:24-80, re-designed for a GPU).
//
// A Handle owns: the CUDA device + stream it enqueues on (MIOpen's
// stream-created handle), a grow-only device scratch pool,
// CUDA events for device timing, the op counters, the solver registry, the
// perf-db, the plan cache and an injectable clock. Find and tune time
// solvers with CUDA events on the handle's stream (1 warm-up + 5 timed runs,
// median), unless a fake/injected clock is installed, in which case the
// reference's clock protocol (read before and after each run) is used so
// tests stay deterministic.
#pragma once

#include <cuda_runtime.h>

#include <filesystem>
#include <functional>
#include <map>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "core.hpp"
#include "perfdb.hpp"
#include "solver.hpp"

namespace primkit {

struct ConvAlgoPerf {
    ConvAlgo algo;
    std::string solver_name;
    double time_ms;
    std::size_t workspace_bytes;
};

enum class FindEnforce { None, Search };

// Grow-only device allocation.
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(std::size_t bytes) { ensure(bytes); }
    ~DeviceBuffer();
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : ptr_(o.ptr_), bytes_(o.bytes_) {
        o.ptr_ = nullptr;
        o.bytes_ = 0;
    }
    void* ensure(std::size_t bytes);
    void* get() const { return ptr_; }
    std::size_t bytes() const { return bytes_; }

private:
    void* ptr_ = nullptr;
    std::size_t bytes_ = 0;
};

class Handle {
public:
    Handle();
    Handle(cudaStream_t stream, int device);
    ~Handle();
    Handle(const Handle&) = delete;
    Handle& operator=(const Handle&) = delete;

    OpCounters& counters() { return counters_; }
    PerfDb& perfdb() { return perfdb_; }
    PlanCache& plan_cache() { return *plan_cache_; }
    std::uint64_t rng_seed = 0x5eed;

    double now_ms() const { return clock_(); }
    void set_clock(std::function<double()> clock) {
        clock_ = std::move(clock);
        device_timing_ = false;
    }
    void use_fake_clock();
    bool device_timing() const { return device_timing_; }

    void set_cache_dir(const std::filesystem::path& dir);
    FindEnforce find_enforce() const { return find_enforce_; }
    void set_find_enforce(FindEnforce e) { find_enforce_ = e; }

    void register_solver(std::shared_ptr<const Solver> solver);
    const std::vector<std::shared_ptr<const Solver>>& solvers() const { return solvers_; }
    const Solver* find_solver(const std::string& name) const;

    // a/b: device operands in the device layout; `workspace_bytes` is the
    // caller's workspace budget (gates solvers by the reference formula).
    std::vector<ConvAlgoPerf> find_convolution(const ConvProblem& problem, const void* a,
                                               const void* b, std::size_t workspace_bytes);
    std::shared_ptr<const ConvPlan> cached_build(const ConvProblem& problem, const Solver& solver,
                                                 const PerfConfig* config);
    PerfConfig resolve_config(const ConvProblem& problem, const Solver& solver) const;

    // Shipped ("system") perf-db, consulted after the user perf-db by
    // resolve_config and kernel_record: tuned configs and kernel records for
    // the ResNet-50 / VGG-16 benchmark shapes (MIOpen ships tuned parameters,
    // PAPER.md:69). Loaded at handle creation from $PRIMKIT_SYSTEM_DB, else
    // <library dir>/../db/sm100_b200.pkdb; an empty path disables it.
    void load_system_db(const std::string& path);
    const PerfDb& system_db() const { return system_db_; }
    const std::string& system_db_path() const { return system_db_path_; }
    // The "<solver>#sm100" kernel record for the problem (user db, then system
    // db), if any.
    bool kernel_record(const ConvProblem& problem, const Solver& solver, pk_tc_config* out) const;

    // Device context.
    int device() const { return device_; }
    cudaStream_t stream() const { return stream_; }
    void set_stream(cudaStream_t s) { stream_ = s; }
    void activate() const;  // cudaSetDevice(device_)
    int num_sms() const { return num_sms_; }
    // Scratch slots are independent grow-only buffers (slot 0: plan
    // workspace, 1..: staging for host-ABI operands).
    void* scratch(int slot, std::size_t bytes);
    void sync() const;
    // Non-blocking copy streams (0: host->device, 1: device->host) and a pool
    // of timing-free events for the overlapped host-buffer path; lazily made.
    cudaStream_t copy_stream(int i);
    cudaEvent_t event(int i);
    // The two timing-enabled events time_ms() uses (0: start, 1: stop).
    cudaEvent_t timing_event(int i) {
        activate();
        return i ? ev1_ : ev0_;
    }

    // Times `fn` (one enqueue of device work) in ms: CUDA events on the
    // handle's stream, or the injected clock.
    double time_ms(const std::function<void()>& fn);
    void record_device_ms(double ms) { last_device_ms_ = ms; }
    double last_device_ms() const { return last_device_ms_; }
    std::string last_kernel;
    // Template instances of the kernels the last conv run launched, in launch
    // order ("conv_tma_fprop_kernel<256, 6, false, false, 1, true>+...").
    std::string last_variant;

    static constexpr int kWarmupRuns = 1;
    static constexpr int kTimedRuns = 5;

private:
    void init_device(int device);

    OpCounters counters_;
    PerfDb perfdb_;
    PerfDb system_db_;
    std::string system_db_path_;
    std::shared_ptr<PlanCache> plan_cache_;
    std::vector<std::shared_ptr<const Solver>> solvers_;
    std::function<double()> clock_;
    bool device_timing_ = true;
    FindEnforce find_enforce_ = FindEnforce::None;
    std::map<std::string, std::vector<ConvAlgoPerf>> find_memo_;

    int device_ = 0;
    int num_sms_ = 148;
    cudaStream_t stream_ = nullptr;
    cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
    cudaStream_t copy_streams_[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> events_;
    std::map<int, DeviceBuffer> scratch_;
    double last_device_ms_ = 0.0;
    bool flush_init_ = false;
};

struct TuneResult {
    PerfConfig best;
    std::int64_t evaluations = 0;
};

TuneResult tune(Handle& handle, const Solver& solver, const ConvProblem& problem,
                std::int64_t budget, bool exhaustive = false);

// Device-timed search over the tcgen05 kernel choices (pk_tc_config) for a
// problem under any solver whose plan runs the tensor-core families, every
// direction (the reference's tune covers only the ImplicitGemm forward grid).
// Candidates that launch the same kernel instances are timed once. The best
// is recorded in the perf-db as "<solver>#sm100" and used by later builds.
struct KernelTuneResult {
    pk_tc_config best{};
    double best_ms = 0.0;
    double default_ms = 0.0;
    std::int64_t evaluations = 0;
    std::string best_variant;
};
KernelTuneResult tune_kernels(Handle& handle, const Solver& solver, const ConvProblem& problem,
                              std::int64_t budget);
std::int64_t default_tune_budget(const Solver& solver, const ConvProblem& problem);

// ---- host <-> device operand staging (the host-buffer ABI) ----
std::size_t etype_bytes(ElementType t);
// Bytes of a device-layout activation tensor [n][h][w][pitch(c)].
std::size_t device_act_bytes(std::int64_t n, std::int64_t c, std::int64_t h, std::int64_t w,
                             ElementType t);
// Device layout bytes of the reference-order tensor `desc` (activation or
// filter; filters [K][C'][R][S] become [K][R][S][pitch(C')]).
std::size_t device_bytes(const TensorDescriptor& desc);
// Upload packed NCHW floats (bf16 tensors: values are rounded to bf16 on the
// way, as the reference quantizes on entry) into the device layout.
void upload_nchw(Handle& h, const TensorDescriptor& desc, const float* host, void* dev);
void download_nchw(Handle& h, const TensorDescriptor& desc, const void* dev, float* host);

}  // namespace primkit
