/* primkit-b200 — B200-native convolution / fusion / batch-norm primitives
 * behind the primkit C ABI.
 *
 * Drop-in boundary. Every declaration in section 1 replaces the reference
 * declaration of the same name in /root/reference/proj/include/primkit/primkit.h
 * with an identical signature, identical enum values and identical struct
 * layouts (reference lines cited per group). Host buffers are packed NCHW
 * `float` arrays exactly as in the reference (bf16 tensors carry bf16-rounded
 * values widened to f32); internally every buffer is uploaded to the GPU,
 * converted to the device layout and processed by sm_100a kernels. There is
 * no CPU compute path: a call that cannot reach a CUDA device fails with
 * PRIMKIT_STATUS_INTERNAL.
 *
 * Section 2 is additive (B200 only): stream-bound handles, device-pointer
 * entry points that skip the host round trip, training-mode batch-norm and
 * activation (C++-only in the reference, primitives.hpp:29-46), and launch
 * statistics.
 */
#ifndef PRIMKIT_H
#define PRIMKIT_H

#include <stddef.h>
#include <stdint.h>

#if defined(_WIN32)
#define PRIMKIT_API __declspec(dllexport)
#else
#define PRIMKIT_API __attribute__((visibility("default")))
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- 1. Reference ABI --------------------------------------------------- */

/* Values mirror primkit::ErrorCode (ref primkit.h:25-47, errors.hpp:8-29). */
typedef enum primkit_status {
    PRIMKIT_STATUS_OK = 0,
    PRIMKIT_STATUS_SHAPE_MISMATCH = 1,
    PRIMKIT_STATUS_INVALID_SHAPE = 2,
    PRIMKIT_STATUS_GROUP_MISMATCH = 3,
    PRIMKIT_STATUS_ALGO_NOT_APPLICABLE = 4,
    PRIMKIT_STATUS_WORKSPACE_TOO_SMALL = 5,
    PRIMKIT_STATUS_DUPLICATE_SOLVER = 6,
    PRIMKIT_STATUS_NO_APPLICABLE_SOLVER = 7,
    PRIMKIT_STATUS_NOT_TUNABLE = 8,
    PRIMKIT_STATUS_NO_VALID_CONFIG = 9,
    PRIMKIT_STATUS_IO_ERROR = 10,
    PRIMKIT_STATUS_PARSE_ERROR = 11,
    PRIMKIT_STATUS_LAYOUT_NOT_DESCENDING = 12,
    PRIMKIT_STATUS_INVALID_EPSILON = 13,
    PRIMKIT_STATUS_INVALID_AXIS = 14,
    PRIMKIT_STATUS_FUSION_NOT_SUPPORTED = 15,
    PRIMKIT_STATUS_ALREADY_COMPILED = 16,
    PRIMKIT_STATUS_NOT_COMPILED = 17,
    PRIMKIT_STATUS_MISSING_ARGS = 18,
    PRIMKIT_STATUS_INVALID_VALUE = 19,
    PRIMKIT_STATUS_INTERNAL = 20
} primkit_status;

/* ref primkit.h:49-83 */
typedef enum primkit_element_type { PRIMKIT_F32 = 0, PRIMKIT_BF16 = 1 } primkit_element_type;
typedef enum primkit_conv_mode { PRIMKIT_CONV_CONVOLUTION = 0, PRIMKIT_CONV_TRANSPOSE = 1 } primkit_conv_mode;
typedef enum primkit_conv_direction {
    PRIMKIT_DIR_FORWARD = 0,
    PRIMKIT_DIR_BACKWARD_DATA = 1,
    PRIMKIT_DIR_BACKWARD_WEIGHTS = 2
} primkit_conv_direction;
typedef enum primkit_conv_algo {
    PRIMKIT_ALGO_IM2COL_GEMM = 0,
    PRIMKIT_ALGO_DIRECT = 1,
    PRIMKIT_ALGO_WINOGRAD = 2,
    PRIMKIT_ALGO_FFT = 3,
    PRIMKIT_ALGO_IMPLICIT_GEMM = 4
} primkit_conv_algo;
typedef enum primkit_activation {
    PRIMKIT_ACT_RELU = 0,
    PRIMKIT_ACT_LEAKY_RELU = 1,
    PRIMKIT_ACT_SIGMOID = 2,
    PRIMKIT_ACT_TANH = 3
} primkit_activation;
typedef enum primkit_batchnorm_mode {
    PRIMKIT_BN_PER_ACTIVATION = 0,
    PRIMKIT_BN_SPATIAL = 1
} primkit_batchnorm_mode;

typedef struct primkit_handle primkit_handle;
typedef struct primkit_fusion_plan primkit_fusion_plan;

/* ref primkit.h:88-111 (layouts are part of the ABI) */
typedef struct primkit_conv_problem {
    int64_t n, c, h, w;
    int64_t k, y, x;
    int64_t pad_h, pad_w;
    int64_t stride_h, stride_w;
    int64_t dilation_h, dilation_w;
    int64_t groups;
    primkit_conv_direction direction;
    primkit_conv_mode mode;
    primkit_element_type etype;
} primkit_conv_problem;

typedef struct primkit_algo_perf {
    char solver_name[64];
    primkit_conv_algo algo;
    double time_ms;
    uint64_t workspace_bytes;
} primkit_algo_perf;

typedef struct primkit_counters {
    uint64_t gemm_calls;
    uint64_t scalar_muls;
    uint64_t buffer_roundtrips;
} primkit_counters;

/* Error reporting and handle lifecycle (ref primkit.h:113-128). */
PRIMKIT_API const char* primkit_last_error(void);
PRIMKIT_API primkit_status primkit_handle_create(primkit_handle** out);
PRIMKIT_API void primkit_handle_destroy(primkit_handle* handle);
PRIMKIT_API primkit_status primkit_handle_use_fake_clock(primkit_handle* handle);
PRIMKIT_API primkit_status primkit_handle_now_ms(primkit_handle* handle, double* out_ms);
PRIMKIT_API primkit_status primkit_handle_set_cache_dir(primkit_handle* handle, const char* dir);
PRIMKIT_API primkit_status primkit_handle_counters(primkit_handle* handle, primkit_counters* out);
PRIMKIT_API primkit_status primkit_handle_reset_counters(primkit_handle* handle);
PRIMKIT_API primkit_status primkit_handle_set_seed(primkit_handle* handle, uint64_t seed);

/* Problem and solver queries (ref primkit.h:130-151). */
PRIMKIT_API primkit_status primkit_problem_key(const primkit_conv_problem* problem, char* buf,
                                               size_t buf_len);
PRIMKIT_API primkit_status primkit_conv_output_dims(const primkit_conv_problem* problem,
                                                    int64_t dims[4]);
PRIMKIT_API primkit_status primkit_solver_count(primkit_handle* handle, int* out_count);
PRIMKIT_API primkit_status primkit_solver_name(primkit_handle* handle, int index, char* buf,
                                               size_t buf_len);
PRIMKIT_API primkit_status primkit_solver_is_applicable(primkit_handle* handle,
                                                        const char* solver_name,
                                                        const primkit_conv_problem* problem,
                                                        int* out_applicable);
PRIMKIT_API primkit_status primkit_solver_is_tunable(primkit_handle* handle,
                                                     const char* solver_name, int* out_tunable);
PRIMKIT_API primkit_status primkit_solver_workspace_bytes(primkit_handle* handle,
                                                          const char* solver_name,
                                                          const primkit_conv_problem* problem,
                                                          uint64_t* out_bytes);

/* Find: device-timed (CUDA events) benchmark of every applicable solver,
 * sorted by (time, name) (ref primkit.h:153-160). */
PRIMKIT_API primkit_status primkit_find_convolution(primkit_handle* handle,
                                                    const primkit_conv_problem* problem,
                                                    const float* a, const float* b,
                                                    size_t workspace_bytes,
                                                    primkit_algo_perf* results, int capacity,
                                                    int* out_count);

/* Run one solver; a null name takes the first applicable solver in registry
 * order, as the reference implementation does (ref primkit_c.cpp:303-311). */
PRIMKIT_API primkit_status primkit_conv_run(primkit_handle* handle,
                                            const primkit_conv_problem* problem,
                                            const char* solver_name, const float* a,
                                            const float* b, float* output,
                                            size_t workspace_bytes);

/* Tuning and perf-db (ref primkit.h:171-182). */
PRIMKIT_API primkit_status primkit_tune(primkit_handle* handle,
                                        const primkit_conv_problem* problem,
                                        const char* solver_name, int64_t budget, int exhaustive,
                                        int64_t* out_evaluations);
PRIMKIT_API primkit_status primkit_perfdb_save(primkit_handle* handle, const char* path);
PRIMKIT_API primkit_status primkit_perfdb_load(primkit_handle* handle, const char* path);

/* Fusion plans (ref primkit.h:184-217). */
PRIMKIT_API primkit_status primkit_fusion_plan_create(const int64_t input_dims[4],
                                                      primkit_element_type etype,
                                                      primkit_fusion_plan** out);
PRIMKIT_API void primkit_fusion_plan_destroy(primkit_fusion_plan* plan);
PRIMKIT_API primkit_status primkit_fusion_add_conv(primkit_fusion_plan* plan,
                                                   const int64_t filter_dims[4], int64_t pad_h,
                                                   int64_t pad_w, int64_t stride_h,
                                                   int64_t stride_w, int64_t groups,
                                                   primkit_conv_algo algo);
PRIMKIT_API primkit_status primkit_fusion_add_bias(primkit_fusion_plan* plan, int64_t channels);
PRIMKIT_API primkit_status primkit_fusion_add_batchnorm(primkit_fusion_plan* plan,
                                                        primkit_batchnorm_mode mode);
PRIMKIT_API primkit_status primkit_fusion_add_activation(primkit_fusion_plan* plan,
                                                         primkit_activation kind, float alpha);
PRIMKIT_API primkit_status primkit_fusion_compile(primkit_handle* handle,
                                                  primkit_fusion_plan* plan);
PRIMKIT_API primkit_status primkit_fusion_output_dims(primkit_fusion_plan* plan,
                                                      int64_t dims[4]);
PRIMKIT_API primkit_status primkit_fusion_set_args(primkit_fusion_plan* plan, const float* filter,
                                                   const float* bias, const float* bn_gamma,
                                                   const float* bn_beta, const float* bn_mean,
                                                   const float* bn_var, float bn_epsilon,
                                                   const float* act_alpha);
PRIMKIT_API primkit_status primkit_fusion_execute(primkit_handle* handle,
                                                  primkit_fusion_plan* plan, const float* input,
                                                  float* output, int unfused);

/* ---- 2. B200 additions -------------------------------------------------- */

/* MIOpen-style handle bound to a caller stream. `stream` is
 * a cudaStream_t (0 = legacy default stream); `device` a CUDA ordinal. */
PRIMKIT_API primkit_status primkit_handle_create_with_stream(void* stream, int device,
                                                             primkit_handle** out);
PRIMKIT_API primkit_status primkit_handle_set_stream(primkit_handle* handle, void* stream);

/* Device layout. Activations are NHWC with the channel dimension padded to
 * primkit_channel_pitch(C) elements (pad lanes hold zeros); filters are
 * [K][Y][X][pitch(C/groups)] (transpose mode: [C][Y][X][pitch(K/groups)]);
 * backward-weights results are produced in the filter layout. Element type
 * is f32 or bf16 (raw 16-bit) per problem.etype. */
PRIMKIT_API int64_t primkit_channel_pitch(int64_t channels);

/* Device-resident convolution: a/b/output follow the operand order of
 * primkit_conv_run; workspace is caller-provided device memory of
 * primkit_conv_device_workspace() bytes. Enqueued on the handle's stream, no
 * host synchronisation. */
PRIMKIT_API primkit_status primkit_conv_device_workspace(primkit_handle* handle,
                                                         const primkit_conv_problem* problem,
                                                         const char* solver_name,
                                                         uint64_t* out_bytes);
PRIMKIT_API primkit_status primkit_conv_run_device(primkit_handle* handle,
                                                   const primkit_conv_problem* problem,
                                                   const char* solver_name, const void* a,
                                                   const void* b, void* output, void* workspace,
                                                   size_t workspace_bytes);

/* Fused (unfused=0) or per-op (unfused=1) execution on device tensors in the
 * device layout; arguments come from primkit_fusion_set_args. */
PRIMKIT_API primkit_status primkit_fusion_execute_device(primkit_handle* handle,
                                                         primkit_fusion_plan* plan,
                                                         const void* input, void* output,
                                                         int unfused);

/* Batch-norm (C++-only in the reference: primitives.hpp:29-46). Host NCHW
 * float buffers; parameters are f32 [C] (spatial) or [C*H*W] (per
 * activation); running statistics are updated in place; saved_mean /
 * saved_invstd receive the batch statistics (1-D, reference layout). */
PRIMKIT_API primkit_status primkit_batchnorm_forward_train(
    primkit_handle* handle, primkit_batchnorm_mode mode, const int64_t dims[4],
    primkit_element_type etype, const float* x, const float* gamma, const float* beta,
    float* running_mean, float* running_var, float epsilon, float momentum, float* y,
    float* saved_mean, float* saved_invstd);
PRIMKIT_API primkit_status primkit_batchnorm_forward_infer(
    primkit_handle* handle, primkit_batchnorm_mode mode, const int64_t dims[4],
    primkit_element_type etype, const float* x, const float* gamma, const float* beta,
    const float* running_mean, const float* running_var, float epsilon, float* y);
PRIMKIT_API primkit_status primkit_batchnorm_backward(
    primkit_handle* handle, primkit_batchnorm_mode mode, const int64_t dims[4],
    primkit_element_type etype, const float* x, const float* dy, const float* gamma,
    const float* saved_mean, const float* saved_invstd, float* dx, float* dgamma,
    float* dbeta);

/* Device-resident spatial batch-norm on NHWC tensors (channel pitch as
 * above). Statistics/parameter vectors are f32 device arrays of length C.
 * `relu` != 0 fuses a ReLU after the normalisation (forward) or the ReLU mask
 * (backward, evaluated on y). */
PRIMKIT_API primkit_status primkit_batchnorm_forward_train_device(
    primkit_handle* handle, const int64_t dims[4], primkit_element_type etype, const void* x,
    const float* gamma, const float* beta, float* running_mean, float* running_var,
    float epsilon, float momentum, void* y, float* saved_mean, float* saved_invstd, int relu);
PRIMKIT_API primkit_status primkit_batchnorm_backward_device(
    primkit_handle* handle, const int64_t dims[4], primkit_element_type etype, const void* x,
    const void* y, const void* dy, const float* gamma, const float* beta,
    const float* saved_mean, const float* saved_invstd, void* dx, float* dgamma, float* dbeta,
    int relu);

/* Convolution forward fused with training-mode spatial batch-norm (+ReLU)
 * (BASELINE cfg4): the convolution epilogue stores the bf16 conv output
 * `conv_out` (kept for the backward pass) and accumulates the per-channel
 * batch statistics of exactly those stored values, so the BN statistics need
 * no extra read of conv_out; one vectorised pass then writes
 * y = gamma*(conv_out-mean)*invstd+beta (ReLU if relu != 0). Semantics of the
 * statistics / running update: primitives.cpp:61-96. Device NHWC tensors;
 * gamma/beta/running/saved vectors are f32 [K]. workspace >=
 * primkit_conv_bn_workspace() bytes. Tensor-core (bf16) convolutions fuse;
 * other element types / kernels run conv then the standalone BN. */
PRIMKIT_API primkit_status primkit_conv_bn_workspace(primkit_handle* handle,
                                                     const primkit_conv_problem* problem,
                                                     const char* solver_name, uint64_t* out_bytes);
PRIMKIT_API primkit_status primkit_conv_bn_forward_train_device(
    primkit_handle* handle, const primkit_conv_problem* problem, const char* solver_name,
    const void* x, const void* w, const float* gamma, const float* beta, float* running_mean,
    float* running_var, float epsilon, float momentum, void* conv_out, void* y,
    float* saved_mean, float* saved_invstd, int relu, void* workspace, size_t workspace_bytes);

/* Backward counterpart (cfg4 bwd): a backward-data convolution whose output
 * dz is the gradient w.r.t. the output of a preceding training BN (+ReLU)
 * layer, with that BN's backward reductions (sum d, sum d*xhat, d = dz*mask)
 * accumulated in the convolution epilogue from the stored dz and the BN input
 * `bn_x`; one vectorised pass then writes bn_dx = dL/d(bn_x) and dgamma /
 * dbeta (primitives.cpp:113-152 semantics; ReLU mask recomputed from bn_x).
 * problem: the BackwardData convolution (operands dy, w as in
 * primkit_conv_run); bn_* vectors f32 [C]. workspace >=
 * primkit_conv_bn_workspace(problem) bytes. bf16 tensor-core dgrad fuses;
 * otherwise dgrad then the standalone BN backward. */
PRIMKIT_API primkit_status primkit_conv_backward_data_bn_device(
    primkit_handle* handle, const primkit_conv_problem* problem, const char* solver_name,
    const void* dy, const void* w, void* dz, const void* bn_x, const float* gamma,
    const float* beta, const float* saved_mean, const float* saved_invstd, int relu, void* bn_dx,
    float* dgamma, float* dbeta, void* workspace, size_t workspace_bytes);

/* Pointwise activation (ref primitives.hpp:55-60), host NCHW buffers. */
PRIMKIT_API primkit_status primkit_activation_forward(primkit_handle* handle,
                                                      primkit_activation kind, float alpha,
                                                      const int64_t dims[4],
                                                      primkit_element_type etype,
                                                      const float* x, float* y);
PRIMKIT_API primkit_status primkit_activation_backward(primkit_handle* handle,
                                                       primkit_activation kind, float alpha,
                                                       const int64_t dims[4],
                                                       primkit_element_type etype,
                                                       const float* x, const float* dy,
                                                       float* dx);

/* Pooling (reference primitives.hpp:65-86, primitives.cpp:204-310). window,
 * pad, stride are {h, w}; dims the NCHW input. Max keeps the first maximum in
 * window scan order; indices receive its linear NCHW input offset (-1 for an
 * empty window, and everywhere for average pooling); average divides by the
 * number of valid (unpadded) taps. Host variants take packed NCHW floats and
 * indices in NCHW output order; device variants take the device layout
 * (NHWC, channel pitch) with indices [N][OH][OW][C]. Backward is computed as
 * a deterministic gather that reproduces the reference's accumulation order. */
typedef enum { PRIMKIT_POOL_MAX = 0, PRIMKIT_POOL_AVG = 1 } primkit_pooling_kind;
PRIMKIT_API primkit_status primkit_pooling_output_dims(const int64_t window[2], const int64_t pad[2],
                                                       const int64_t stride[2], const int64_t dims[4],
                                                       int64_t out_dims[4]);
PRIMKIT_API primkit_status primkit_pooling_forward(primkit_handle* handle, primkit_pooling_kind kind,
                                                   const int64_t window[2], const int64_t pad[2],
                                                   const int64_t stride[2], const int64_t dims[4],
                                                   primkit_element_type etype, const float* x, float* y,
                                                   int64_t* indices);
PRIMKIT_API primkit_status primkit_pooling_backward(primkit_handle* handle, primkit_pooling_kind kind,
                                                    const int64_t window[2], const int64_t pad[2],
                                                    const int64_t stride[2], const int64_t dims[4],
                                                    primkit_element_type etype, const float* dy,
                                                    const int64_t* indices, float* dx);
PRIMKIT_API primkit_status primkit_pooling_forward_device(
    primkit_handle* handle, primkit_pooling_kind kind, const int64_t window[2], const int64_t pad[2],
    const int64_t stride[2], const int64_t dims[4], primkit_element_type etype, const void* x, void* y,
    int64_t* indices);
PRIMKIT_API primkit_status primkit_pooling_backward_device(
    primkit_handle* handle, primkit_pooling_kind kind, const int64_t window[2], const int64_t pad[2],
    const int64_t stride[2], const int64_t dims[4], primkit_element_type etype, const void* dy,
    const int64_t* indices, void* dx);

/* Softmax along `axis` of a packed rank-`rank` tensor (reference
 * primitives.hpp:88-91, primitives.cpp:312-370): max-stabilised, denominator
 * and backward dot product in double. INVALID_AXIS for an axis out of range. */
PRIMKIT_API primkit_status primkit_softmax_forward(primkit_handle* handle, int rank, const int64_t* dims,
                                                   primkit_element_type etype, int64_t axis,
                                                   const float* x, float* y);
PRIMKIT_API primkit_status primkit_softmax_backward(primkit_handle* handle, int rank, const int64_t* dims,
                                                    primkit_element_type etype, int64_t axis,
                                                    const float* y, const float* dy, float* dx);
PRIMKIT_API primkit_status primkit_softmax_forward_device(primkit_handle* handle, int rank,
                                                          const int64_t* dims, primkit_element_type etype,
                                                          int64_t axis, const void* x, void* y);
PRIMKIT_API primkit_status primkit_softmax_backward_device(primkit_handle* handle, int rank,
                                                           const int64_t* dims, primkit_element_type etype,
                                                           int64_t axis, const void* y, const void* dy,
                                                           void* dx);

/* Layout converters used by the host ABI, exposed for device callers:
 * packed NCHW f32 (device memory) <-> device NHWC layout of `etype`. */
PRIMKIT_API primkit_status primkit_nchw_to_device(primkit_handle* handle, const int64_t dims[4],
                                                  primkit_element_type etype, const float* src,
                                                  void* dst);
PRIMKIT_API primkit_status primkit_device_to_nchw(primkit_handle* handle, const int64_t dims[4],
                                                  primkit_element_type etype, const void* src,
                                                  float* dst);

/* Launch statistics: number of primkit CUDA kernels launched by this handle
 * and the device time (ms, CUDA events) of the most recent conv/fusion run. */
PRIMKIT_API primkit_status primkit_handle_kernel_launches(primkit_handle* handle,
                                                         uint64_t* out_launches);
PRIMKIT_API primkit_status primkit_handle_last_device_ms(primkit_handle* handle,
                                                         double* out_ms);
/* Name of the device kernel family the last conv run dispatched to
 * (e.g. "igemm_tc_fwd", "direct_simt"). */
PRIMKIT_API primkit_status primkit_handle_last_kernel(primkit_handle* handle, char* buf,
                                                     size_t buf_len);
/* Plan-cache counters of the handle (reference PlanCache::Stats,
 * proj/src/core/plan_cache.hpp): plans built, memory hits, disk hits. */
PRIMKIT_API primkit_status primkit_handle_plan_cache_stats(primkit_handle* handle, uint64_t* builds,
                                                          uint64_t* memory_hits,
                                                          uint64_t* disk_hits);
/* Template instances of the tensor-core kernels the last conv run launched,
 * in launch order, joined by '+' (e.g.
 * "conv_tma_fprop_kernel<256, 6, false, false, 1, true>"); empty for the
 * CUDA-core families, which last_kernel names completely. */
PRIMKIT_API primkit_status primkit_handle_last_variant(primkit_handle* handle, char* buf,
                                                      size_t buf_len);

/* ---- auto-tuning of the B200 kernel choice (handle.cpp tune_kernels) ----
 * The reference tunes only the ImplicitGemm forward grid (primkit_tune,
 * handle.cpp:167-226 of the reference). Here every solver whose plan runs the
 * tcgen05 families, in every direction, has a kernel choice
 * "<block_n>,<family>,<pair>,<mt>,<split>" (0 = heuristic; see pk_tc_config):
 * primkit_tune_kernels times the candidates on device tensors (U(-1,1), the
 * handle's seed), drops any whose output differs from the heuristic choice's
 * beyond the dtype tolerance, stores the fastest in the perf-db under
 * "<solver>#sm100" and returns its values plus the heuristic and best medians. */
PRIMKIT_API primkit_status primkit_tune_kernels(primkit_handle* handle,
                                               const primkit_conv_problem* problem,
                                               const char* solver_name, int64_t budget,
                                               char* best_values, size_t buf_len,
                                               double* default_ms, double* best_ms);
/* The kernel choice a plan for (problem, solver) would run with after the
 * perf-db lookups (user db, then the shipped system db). */
PRIMKIT_API primkit_status primkit_plan_kernel_config(primkit_handle* handle,
                                                     const primkit_conv_problem* problem,
                                                     const char* solver_name, char* buf,
                                                     size_t buf_len);
/* Replace the handle's shipped ("system") perf-db, consulted after the user
 * perf-db: NULL or "" disables it. At creation it is loaded from
 * $PRIMKIT_SYSTEM_DB, else <libprimkit dir>/../db/sm100_b200.pkdb. */
PRIMKIT_API primkit_status primkit_handle_load_system_db(primkit_handle* handle, const char* path);
/* Path of the loaded system perf-db ("" when none) and its record count. */
PRIMKIT_API primkit_status primkit_handle_system_db(primkit_handle* handle, char* buf,
                                                   size_t buf_len, uint64_t* records);

/* ---- 3. data-parallel weight-gradient all-reduce (north_star) ----
 * One process per GPU, the batch sharded over them. Backward-weights results
 * are registered in the order the backward pass produces them (reverse layer
 * order) and grouped into fp32 buckets; when the last gradient of a bucket is
 * marked ready, the bucket is all-reduced with NCCL (sum, optional 1/world
 * average) on an internal comm stream gated by an event on the handle's
 * stream, so it overlaps the remaining backward kernels. finish() makes the
 * handle's stream wait for all buckets. All work is stream-ordered and can be
 * captured into a CUDA graph. While a dp context exists, grid-wide barriers
 * inside the convolution kernels are disabled (the collective occupies SMs).
 * NCCL is loaded at run time (libnccl.so.2). No reference counterpart: the
 * reference is a single-process CPU library. */
#define PRIMKIT_DP_UNIQUE_ID_BYTES 128
typedef struct primkit_dp primkit_dp;

PRIMKIT_API primkit_status primkit_dp_unique_id(uint8_t id[PRIMKIT_DP_UNIQUE_ID_BYTES]);
PRIMKIT_API primkit_status primkit_dp_create(primkit_handle* handle,
                                             const uint8_t id[PRIMKIT_DP_UNIQUE_ID_BYTES],
                                             int nranks, int rank, int average, primkit_dp** out);
PRIMKIT_API void primkit_dp_destroy(primkit_dp* dp);
/* Target fp32 bytes per bucket (default 25 MiB); before the first grad_ready. */
PRIMKIT_API primkit_status primkit_dp_set_bucket_bytes(primkit_dp* dp, uint64_t bytes);
PRIMKIT_API primkit_status primkit_dp_register(primkit_dp* dp, void* grad, uint64_t elems,
                                               primkit_element_type etype, int* out_index);
PRIMKIT_API primkit_status primkit_dp_grad_ready(primkit_dp* dp, int index);
PRIMKIT_API primkit_status primkit_dp_finish(primkit_dp* dp);
/* Polls NCCL for an asynchronous error; on one, aborts the communicator and
 * returns PRIMKIT_STATUS_INTERNAL with the NCCL message. */
PRIMKIT_API primkit_status primkit_dp_check(primkit_dp* dp);
PRIMKIT_API primkit_status primkit_dp_buckets(primkit_dp* dp, int* out_count);
PRIMKIT_API primkit_status primkit_dp_bucket_of(primkit_dp* dp, int index, int* out_bucket);

#ifdef __cplusplus
}
#endif

#endif /* PRIMKIT_H */
