// Internal host -> device boundary of primkit-b200.
//
// The C++ host layer only ever calls the extern "C" pk_cuda_* launchers
// declared here: POD argument structs, raw device pointers and a
// cudaStream_t, returning cudaError_t. No C++ or torch types cross this line.
//
// Device layout:
//   activations  NHWC, channel pitch = pk_pitch(C) (zero padded lanes)
//   filters      [K][R][S][pitch(C/groups)]   (transpose: [C][R][S][pitch(K/groups)])
//   element type f32 or bf16 storage; arithmetic is always fp32 (SIMT FMA or
//                tcgen05 with an fp32 TMEM accumulator).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum pk_dtype { PK_F32 = 0, PK_BF16 = 1 };

static inline int pk_pitch(int c) { return (c + 7) / 8 * 8; }

// One convolution instance in device terms (shapes are those of the forward
// convolution even for the backward passes).
typedef struct pk_conv_geom {
    int n, c, h, w;          // input image
    int k, r, s;             // filter: output channels, rows (y), cols (x)
    int p, q;                // output image
    int pad_h, pad_w, str_h, str_w, dil_h, dil_w;
    int groups, cg, kg;      // channels per group
    int x_pitch;             // channel pitch of the input activations
    int y_pitch;             // channel pitch of the output activations
    int f_pitch;             // innermost filter pitch
    int transpose;           // 1 = transpose-mode forward
} pk_conv_geom;

// Epilogue applied to the fp32 accumulator before the single store:
// bias -> batch-norm inference -> activation (reference order,
// proj/src/core/fusion.cpp:384-398). Null pointers / act < 0 disable a stage.
typedef struct pk_epilogue {
    const float* bias;       // [K]
    const float* bn_mean;    // [K] (spatial) or [K*P*Q] (per activation)
    const float* bn_var;
    const float* bn_gamma;
    const float* bn_beta;
    int bn_per_activation;
    int bn_standalone;       // 1: gamma*(x-mu)*(1/sqrt(var+eps))+beta (primitives.cpp:105-108)
                             // 0: (x-mu)/sqrt(var+eps)*gamma+beta    (fusion.cpp:390-394)
    float bn_eps;
    int act;                 // -1 none, 0 ReLU, 1 LeakyReLU, 2 Sigmoid, 3 Tanh
    float act_alpha;
    // Optional folded per-channel affine (bias and spatial BN folded on the
    // host): acc * ch_scale[k] + ch_shift[k], then the activation. Used by the
    // tensor-core epilogues (bf16 outputs) in place of bias/bn_* when set.
    const float* ch_scale;
    const float* ch_shift;
    // Optional batch-norm (training) statistics of the STORED outputs: when
    // set, every CTA adds per-channel sum and sum of squares of its
    // bf16-rounded outputs into stats[blockIdx.x][channel][2] (fp32, zeroed by
    // the caller; pk_stats_slots() slices). Spatial mode only.
    float* stats;
    // Backward variant (a dgrad producing dz = dL/d(BN output) of a preceding
    // training BN): with bnb_y = that BN's input (same NHWC layout as this
    // output), the epilogue instead accumulates per channel
    //   stats[cta][ch][0] += d,  stats[cta][ch][1] += d * xhat,
    //   d = dz * mask (mask = bnb_relu ? BN(y) > 0 : 1), xhat = (y - mean) * invstd.
    const void* bnb_y;
    const float* bnb_gamma;
    const float* bnb_beta;
    const float* bnb_mean;
    const float* bnb_invstd;
    int bnb_relu;
} pk_epilogue;

// Per-CTA slices of pk_epilogue.stats (persistent conv grids use <= this many CTAs).
static inline int pk_stats_slots(void) { return 148; }

// ---- layout conversion ------------------------------------------------------
// NCHW f32 [n][c][hw] <-> NHWC [n][hw][pitch] of dtype (RNE on bf16 stores).
cudaError_t pk_cuda_nchw_to_nhwc(const float* src, void* dst, int n, int c, int hw, int pitch,
                                 int dtype, cudaStream_t st);
cudaError_t pk_cuda_nhwc_to_nchw(const void* src, float* dst, int n, int c, int hw, int pitch,
                                 int dtype, cudaStream_t st);
// Filter [K][R][S][f_pitch] -> dgrad operand [C][R][S][pitch(K)] (same dtype).
cudaError_t pk_cuda_filter_to_dgrad(const pk_conv_geom* g, int dtype, const void* f, void* dst,
                                    cudaStream_t st);

// ---- Direct (SIMT fp32) -------------------------------------------------------
cudaError_t pk_cuda_direct_fwd(const pk_conv_geom* g, int dtype, const void* x, const void* f,
                               void* y, const pk_epilogue* epi, cudaStream_t st);
cudaError_t pk_cuda_direct_bwd_data(const pk_conv_geom* g, int dtype, const void* dy,
                                    const void* f, void* dx, cudaStream_t st);
// Depthwise (groups == C == K), depthwise.cu: channel-vector lanes, filter taps
// in shared memory; wgrad = per-chunk partials + a fixed-order chunk sum.
int pk_depthwise_supported(const pk_conv_geom* g);
cudaError_t pk_cuda_depthwise_fwd(const pk_conv_geom* g, int dtype, const void* x, const void* f, void* y,
                                  const pk_epilogue* epi, int num_sms, cudaStream_t st);
cudaError_t pk_cuda_depthwise_bwd_data(const pk_conv_geom* g, int dtype, const void* dy, const void* f,
                                       void* dx, int num_sms, cudaStream_t st);
size_t pk_depthwise_wgrad_workspace(const pk_conv_geom* g, int num_sms);
cudaError_t pk_cuda_depthwise_wgrad(const pk_conv_geom* g, int dtype, const void* dy, const void* x, void* dw,
                                    void* ws, size_t ws_bytes, int num_sms, cudaStream_t st);
// Grouped forward / backward data, C/g and K/g multiples of 8 (depthwise.cu).
int pk_grouped_supported(const pk_conv_geom* g);
cudaError_t pk_cuda_grouped_fwd(const pk_conv_geom* g, int dtype, const void* x, const void* f, void* y,
                                const pk_epilogue* epi, int num_sms, cudaStream_t st);
cudaError_t pk_cuda_grouped_bwd_data(const pk_conv_geom* g, int dtype, const void* dy, const void* f, void* dx,
                                     int num_sms, cudaStream_t st);
// Grouped backward weights for C/g in {8, 16, 32} (depthwise.cu).
int pk_grouped_wgrad_supported(const pk_conv_geom* g);
size_t pk_grouped_wgrad_workspace(const pk_conv_geom* g, int num_sms);
cudaError_t pk_cuda_grouped_wgrad(const pk_conv_geom* g, int dtype, const void* dy, const void* x, void* dw,
                                  void* ws, size_t ws_bytes, int num_sms, cudaStream_t st);
// Register-tiled SIMT backward data (groups 1), direct.cu.
int pk_direct_dgrad_tiled_supported(const pk_conv_geom* g);
cudaError_t pk_cuda_direct_dgrad_tiled(const pk_conv_geom* g, int dtype, const void* dy, const void* f, void* dx,
                                       cudaStream_t st);
// Register-tiled SIMT backward weights (groups 1), split over pixels + fixed-order sum (direct.cu).
int pk_direct_wgrad_tiled_supported(const pk_conv_geom* g);
size_t pk_direct_wgrad_tiled_workspace(const pk_conv_geom* g, int num_sms);
cudaError_t pk_cuda_direct_wgrad_tiled(const pk_conv_geom* g, int dtype, const void* dy, const void* x, void* dw,
                                       void* ws, size_t ws_bytes, int num_sms, cudaStream_t st);
cudaError_t pk_cuda_direct_bwd_weights(const pk_conv_geom* g, int dtype, const void* dy,
                                       const void* x, void* dw, cudaStream_t st);

// ---- im2col / col2im + GEMM (Im2colGemm solver) ------------------------------
// col[(p,q)][(r,s,c)] for one (image, group); row pitch = r*s*f_pitch
// (zero in padded lanes), element type dtype.
cudaError_t pk_cuda_im2col(const pk_conv_geom* g, int dtype, const void* x, int image, int group,
                           void* col, cudaStream_t st);
// dx[image][:, group channels] = col2im(col), col fp32 [(p,q)][(r,s,c)] with
// row pitch r*s*f_pitch (gather formulation: no atomics, overwrites dx).
cudaError_t pk_cuda_col2im(const pk_conv_geom* g, int dtype, const float* col, int image,
                           int group, void* dx, cudaStream_t st);
// Transpose mode: out[image][oh][ow][group*kg + kk] = sum over taps of
// col[((r*S + s)*f_pitch + kk) * (H*W) + h*W + w] with oh = h*str - pad + r.
cudaError_t pk_cuda_col2im_transpose(const pk_conv_geom* g, int dtype, const float* col,
                                     int image, int group, void* out, cudaStream_t st);
// Strided SIMT GEMM, fp32 arithmetic:
//   C[i*ldc + j] (+)= sum_l A[i*sam + l*sak] * B[l*sbk + j*sbn]
// A/B element type dtype_ab; C is fp32 (accumulate != 0 adds to C).
cudaError_t pk_cuda_gemm_simt(int m, int n, int k, int dtype_ab, const void* a, long long sam,
                              long long sak, const void* b, long long sbk, long long sbn,
                              float* c, long long ldc, int accumulate, cudaStream_t st);
// dst[i*dst_pitch + j] = (dtype) src[i*ld + j] for i<rows, j<cols, with the
// epilogue applied per column (column = output channel).
cudaError_t pk_cuda_store_rows(const float* src, int rows, int cols, long long ld, void* dst,
                               long long dst_pitch, int dtype, const pk_epilogue* epi,
                               int chan_offset, cudaStream_t st);

// ---- SIMT implicit GEMM forward (fp32 arithmetic, any shape/groups/dilation)
cudaError_t pk_cuda_igemm_simt_fwd(const pk_conv_geom* g, int dtype, const void* x, const void* f,
                                   void* y, const pk_epilogue* epi, cudaStream_t st);

// ---- Winograd F(2x2,3x3) (SIMT, zero workspace) -------------------------------
cudaError_t pk_cuda_winograd_f23(const pk_conv_geom* g, int dtype, const void* x, const void* f,
                                 void* y, const pk_epilogue* epi, cudaStream_t st);

// ---- Winograd F(m x m, 3x3) on the tensor cores (bf16, m = 2 or 4) ----------
// Filter/input transforms in registers, alpha^2 batched tcgen05 GEMMs, output
// transform + epilogue; V/M staged in ws (chunked over tiles).
int pk_winograd_tc_supported(const pk_conv_geom* g);
size_t pk_winograd_tc_workspace(const pk_conv_geom* g, int m);
cudaError_t pk_cuda_winograd_tc(const pk_conv_geom* g, int m, const void* x, const void* f,
                                void* y, const pk_epilogue* epi, void* ws, size_t ws_bytes,
                                cudaStream_t st);
// Batched plain tcgen05 GEMM: Y[b][i][j] = sum_l A[b][i][l] * B[b][j][l] (bf16 in,
// fp32 accumulate, bf16 out). A/Y rows per batch must be a multiple of 128.
cudaError_t pk_cuda_gemm_tc_batched(const void* a, const void* b, void* y, int batch,
                                    int rows_per_batch, int kdim, int n_out, int b_rows_per_batch,
                                    int out_pitch, cudaStream_t st, int f16);

// ---- FFT convolution (complex<double>, radix-2, pow2 planes) -----------------
size_t pk_cuda_fft_scratch_bytes(const pk_conv_geom* g);
cudaError_t pk_cuda_fft_fwd(const pk_conv_geom* g, int dtype, const void* x, const void* f,
                            void* y, void* scratch, cudaStream_t st);

// ---- tcgen05 implicit GEMM (bf16 in, fp32 TMEM accumulate) -------------------
// Kernel choice of the tcgen05 convolution families (the auto-tuner's design
// space, solver.cpp / handle.cpp tune). Every field: 0 = the built-in
// heuristic; a value the geometry cannot honour falls back to the heuristic.
typedef struct pk_tc_config {
    int block_n;  // output-channel (fwd/dgrad) or filter-position (wgrad) tile: 64/128/256
    int family;   // 1: no halo-reuse kernels; 2: no halo, no TMA rectangles (cp.async gather)
    int pair;     // 1: never CTA pairs (cta_group::2); 2: CTA pairs wherever supported
    int mt;       // 1: one M=128 tile per CTA; 2: two (256-pixel rectangles, M=256 wgrad)
    int split;    // wgrad split-K: splits = max(1, one_wave_splits * split / 4)
} pk_tc_config;
// 1 if the tensor-core path supports this geometry (groups == 1, bf16, ...).
int pk_tc_fwd_supported(const pk_conv_geom* g);
int pk_tc_dgrad_supported(const pk_conv_geom* g);
int pk_tc_wgrad_supported(const pk_conv_geom* g);
size_t pk_tc_dgrad_workspace(const pk_conv_geom* g);
// Streams `bytes` of `buf` through L2 (reads only): evicts the previous working
// set before a timed run (Find / tune device timing).
cudaError_t pk_cuda_l2_flush(const void* buf, size_t bytes, cudaStream_t st);
// sums[0] = sum (a-b)^2, sums[1] = sum b^2 (device doubles) over n elements
cudaError_t pk_cuda_sq_diff(const void* a, const void* b, long long n, int dtype, double* sums,
                            cudaStream_t st);
// split-K partials of pk_cuda_igemm_tc_wgrad under the same config
size_t pk_tc_wgrad_workspace(const pk_conv_geom* g, int num_sms, const pk_tc_config* cfg);
// fp32 forward convolution on the tensor cores at fp32 accuracy (3xTF32: hi/lo
// operand split into the workspace, one tf32 GEMM over the concatenation, fp32 out;
// groups 1, channel pitch multiple of 32). cudaErrorNotSupported: not eligible.
int pk_tf32x3_fwd_supported(const pk_conv_geom* g);
size_t pk_tf32x3_fwd_workspace(const pk_conv_geom* g);
cudaError_t pk_cuda_tf32x3_fwd(const pk_conv_geom* g, const void* x, const void* w, void* y,
                               const pk_epilogue* epi, void* workspace, size_t ws_bytes, cudaStream_t st);
cudaError_t pk_cuda_igemm_tc_fwd(const pk_conv_geom* g, const void* x, const void* f, void* y,
                                 const pk_epilogue* epi, const pk_tc_config* cfg,
                                 cudaStream_t st);
cudaError_t pk_cuda_igemm_tc_dgrad(const pk_conv_geom* g, const void* dy, const void* f, void* dx,
                                   void* workspace, const pk_tc_config* cfg, cudaStream_t st,
                                   const pk_epilogue* stats_epi);
cudaError_t pk_cuda_igemm_tc_wgrad(const pk_conv_geom* g, const void* dy, const void* x, void* dw,
                                   void* workspace, int num_sms, const pk_tc_config* cfg,
                                   cudaStream_t st);

// ---- dense-reduction packing for narrow-channel (stem) layers, bf16 ---------
int pk_stem_kc_pitch(const pk_conv_geom* g);  // roundup(R*S*C, 8)
cudaError_t pk_cuda_im2col_pack(const pk_conv_geom* g, const void* x, void* col, cudaStream_t st);
// transposed = 0: [K][kc_pitch]; 1: [kc_pitch][pitch(K)]
cudaError_t pk_cuda_filter_pack(const pk_conv_geom* g, const void* f, void* dst, int transposed,
                                cudaStream_t st);
cudaError_t pk_cuda_col2im_pack(const pk_conv_geom* g, const void* colg, void* dx, cudaStream_t st);
cudaError_t pk_cuda_wgrad_unpack(const pk_conv_geom* g, const void* dwp, void* dw, cudaStream_t st);

// ---- fused narrow-channel (stem, C <= 4) tcgen05 convolutions, bf16 ---------
// Input halo staged in smem and expanded into the tap-packed operand on chip
// (no column matrix in HBM). K (output channels) in {64, 128}, y pitch == K.
int pk_cuda_stem_fused_supported(const pk_conv_geom* g);
cudaError_t pk_cuda_stem_fused_fprop(const pk_conv_geom* g, const void* x, const void* w, void* y,
                                     const pk_epilogue* epi, cudaStream_t st);
size_t pk_cuda_stem_fused_wgrad_workspace(const pk_conv_geom* g, int num_sms);
// backward data (gather formulation; dY channels K == 64): no workspace
int pk_cuda_stem_fused_dgrad_supported(const pk_conv_geom* g);
cudaError_t pk_cuda_stem_fused_dgrad(const pk_conv_geom* g, const void* dy, const void* w, void* dx,
                                     cudaStream_t st);
cudaError_t pk_cuda_stem_fused_wgrad(const pk_conv_geom* g, const void* dy, const void* x,
                                     void* dw, void* workspace, int num_sms, cudaStream_t st);

// ---- pointwise / batch-norm ----------------------------------------------------
// y = epilogue(x + 0) elementwise over NHWC (bias/bn/act all optional).
cudaError_t pk_cuda_pointwise(const void* x, void* y, int n, int c, int hw, int pitch, int dtype,
                              const pk_epilogue* epi, cudaStream_t st);
cudaError_t pk_cuda_activation_bwd(const void* x, const void* dy, void* dx, int n, int c, int hw,
                                   int pitch, int dtype, int act, float alpha, cudaStream_t st);
// Training-mode batch-norm over NHWC. Spatial mode reduces over n*hw per
// channel; per-activation mode (per_act=1) reduces over n per (c, hw).
// scratch: pk_bn_scratch_bytes(); stats are reduced deterministically.
size_t pk_bn_scratch_bytes(int n, int c, int hw, int per_act);
cudaError_t pk_cuda_bn_fwd_train(const void* x, void* y, int n, int c, int hw, int pitch,
                                 int dtype, int per_act, const float* gamma, const float* beta,
                                 float* running_mean, float* running_var, float eps,
                                 float momentum, float* saved_mean, float* saved_invstd,
                                 int relu, void* scratch, cudaStream_t st);
// Finalize training BN from per-CTA fp32 partials [slots][c][2] (sum, sumsq)
// of m values per channel: reference semantics (double, biased var clamped,
// running stats update), then y = BN(x) (+ReLU) with 16-byte vector accesses.
cudaError_t pk_cuda_bn_finalize_apply(const float* part, int slots, const void* x, void* y, int n,
                                      int c, int hw, int pitch, int dtype, const float* gamma,
                                      const float* beta, float* running_mean, float* running_var,
                                      float eps, float momentum, float* saved_mean,
                                      float* saved_invstd, int relu, cudaStream_t st);
// y = gamma*(x-mean)*invstd+beta (+ReLU) with given batch statistics.
cudaError_t pk_cuda_bn_apply_stats(const void* x, void* y, int n, int c, int hw, int pitch,
                                   int dtype, const float* gamma, const float* beta,
                                   const float* mean, const float* invstd, int relu,
                                   cudaStream_t st);
// BN backward from per-CTA fp32 partials [slots][c][2] (sum d, sum d*xhat)
// of a dgrad epilogue: dgamma/dbeta (rounded to bf16 when dtype is bf16, the
// reference's etype rule) and dx = gamma*invstd/m * (m*d - dbeta - xhat*dgamma)
// with d = dz * mask, vectorised over bf16 NHWC.
cudaError_t pk_cuda_bn_bwd_finalize_apply(const float* part, int slots, const void* dz,
                                          const void* y, void* dx, int n, int c, int hw, int pitch,
                                          int dtype, const float* gamma, const float* beta,
                                          const float* mean, const float* invstd, int relu,
                                          float* dgamma, float* dbeta, float* tot_scratch,
                                          cudaStream_t st);
// BN backward (+ReLU with the mask recomputed from the BN input x through the
// folded affine, so the BN output is not needed) in one launch: statistics of
// d = dz * mask, then dx; bf16 NHWC only (cudaErrorNotSupported otherwise).
cudaError_t pk_cuda_bn_bwd_fold(const void* x, const void* dz, void* dx, int n, int c, int hw,
                                int pitch, int dtype, const float* gamma, const float* beta,
                                const float* mean, const float* invstd, int relu, float* dgamma,
                                float* dbeta, void* scratch, cudaStream_t st);
cudaError_t pk_cuda_bn_bwd(const void* x, const void* y, const void* dy, void* dx, int n, int c,
                           int hw, int pitch, int dtype, int per_act, const float* gamma,
                           const float* saved_mean, const float* saved_invstd, float* dgamma,
                           float* dbeta, int relu, int round_params_bf16, void* scratch,
                           cudaStream_t st);

// ---- pooling / softmax (pool.cu; reference primitives.cpp:204-370) -------------
typedef struct pk_pool_geom {
    int n, c, h, w, oh, ow;
    int win_h, win_w, str_h, str_w, pad_h, pad_w;
    int pitch;  // channel pitch of x / y / dx / dy (NHWC device layout)
} pk_pool_geom;
int pk_pool_supported(const pk_pool_geom* g);
// y [n][oh][ow][pitch]; indices (max only, nullable) [n][oh][ow][c] int64 =
// linear NCHW input offset of the first maximum (-1 for an empty window).
cudaError_t pk_cuda_pool_fwd(const pk_pool_geom* g, int dtype, int is_max, const void* x, void* y,
                             long long* indices, cudaStream_t st);
cudaError_t pk_cuda_pool_bwd(const pk_pool_geom* g, int dtype, int is_max, const void* dy,
                             const long long* indices, void* dx, cudaStream_t st);
// packed tensor viewed as [outer][axis][inner]
cudaError_t pk_cuda_softmax_fwd(int dtype, const void* x, void* y, long long outer, int axis,
                                long long inner, cudaStream_t st);
cudaError_t pk_cuda_softmax_bwd(int dtype, const void* y, const void* dy, void* dx, long long outer,
                                int axis, long long inner, cudaStream_t st);

// ---- data-parallel gradient buckets (dp.cu) -----------------------------------
// One gradient tensor inside an fp32 bucket: device pointer, element count,
// element type (pk_dtype) and its element offset in the bucket.
typedef struct pk_dp_seg {
    void* ptr;
    long long elems;
    long long offset;
    int dtype;
    int pad_;
} pk_dp_seg;
// bucket[seg.offset + i] = float(seg.ptr[i]) for every segment (segs in device memory).
cudaError_t pk_cuda_dp_pack(const pk_dp_seg* segs_dev, int nseg, long long max_elems, float* bucket,
                            cudaStream_t st);
// seg.ptr[i] = dtype(bucket[seg.offset + i] * scale) (RNE for bf16).
cudaError_t pk_cuda_dp_unpack(const pk_dp_seg* segs_dev, int nseg, long long max_elems,
                              const float* bucket, float scale, cudaStream_t st);
// Grid-wide barriers (the in-kernel split-K finish) need every CTA of a grid
// co-resident; with a collective running concurrently on other SMs that no
// longer holds, so the data-parallel layer turns them off (process-wide).
void pk_cuda_allow_grid_barriers(int on);

// Launch accounting: number of kernels this library launched (process-wide).
uint64_t pk_cuda_launch_count(void);
// Kernel-variant log of the calling thread: the demangled template instance of
// every kernel launched through pk_launch since the last reset, joined by '+'.
void pk_cuda_variant_reset(void);
const char* pk_cuda_variant(void);

#ifdef __cplusplus
}
#endif
