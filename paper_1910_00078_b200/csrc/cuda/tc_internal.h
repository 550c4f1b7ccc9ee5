// Internal entry points shared between the tcgen05 kernel translation units
// (not part of the pk_cuda_* host boundary).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include "kernels.h"

// TMA rectangle-tile path (conv_tma.cu). cudaErrorNotSupported = geometry
// not eligible (nothing launched); callers then use the cp.async gather path.
// filt_mn (backward data): filt is the ORIGINAL filter W[K][R][S][pitch], read as an
// MN-major B operand (no transposed copy); otherwise the transposed [C][R][S][pitch K].
cudaError_t pk_tma_conv(const pk_conv_geom* g, bool dgrad, const void* src, const void* filt,
                        void* out, const pk_epilogue* epi, int bn_want, cudaStream_t st,
                        bool filt_mn = false);
bool pk_tma_wgrad_supported(const pk_conv_geom* g);
size_t pk_tma_wgrad_workspace(const pk_conv_geom* g, int num_sms);
cudaError_t pk_tma_wgrad(const pk_conv_geom* g, const void* dy, const void* x, void* dw,
                         void* workspace, int num_sms, cudaStream_t st);

// Halo-reuse path for stride-1 spatial filters (conv_halo.cu): forward, or
// backward data (filt = transposed filter [C][R][S][pitch K]) when dgrad.
cudaError_t pk_halo_conv(const pk_conv_geom* g, bool dgrad, const void* src, const void* filt,
                         void* out, const pk_epilogue* epi, cudaStream_t st, bool filt_mn = false);

// CTA-pair (cta_group::2) plain GEMM for 1x1 layers whose filter slice cannot
// stay resident (conv_tc2.cu): y[M][out_pitch] = a[M][kdim] . b[n_out][kdim]^T.
int pk_gemm_pair_eligible(int M, int kdim, int n_out, int out_pitch);
// b_mn_pitch > 0: b is MN-major ([kdim rows][b_mn_pitch], e.g. the filter itself for
// backward data) instead of K-major [n_out][kdim].
cudaError_t pk_gemm_pair(const void* a, const void* b, void* y, int M, int kdim, int n_out,
                         int out_pitch, int P, int Q, const pk_epilogue* epi, cudaStream_t st,
                         int b_mn_pitch = 0);

// Padded-grid halo backward weights for stride-1 spatial filters on 64-channel
// tensors (wgrad_halo.cu): fp32 partials [splits][K][R*S*64]; splits = 0 when
// the geometry is not eligible.
int pk_halo_wgrad_splits(const pk_conv_geom* g, int num_sms);
// dw/sync: when sync is non-null the kernel finishes the split-K sum itself
// (grid barrier, fixed split order) and writes bf16 dW.
cudaError_t pk_halo_wgrad(const pk_conv_geom* g, const void* dy, const void* x, float* partial,
                          int splits, cudaStream_t st, void* dw, unsigned int* sync);
