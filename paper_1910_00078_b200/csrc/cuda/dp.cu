// Gradient bucket pack / unpack for the data-parallel all-reduce (dp.cpp).
//
// A bucket is a contiguous fp32 buffer holding several weight-gradient
// tensors back to back. pack widens bf16 (or copies f32) gradients into it
// before the NCCL sum; unpack scales the reduced sums and stores them back in
// the gradients' element type (RNE for bf16). One launch per bucket covers all
// of its tensors: blockIdx.y selects the tensor, the x blocks stride over it
// with 16-byte vectors. HBM-bound (2 + 4 bytes per bf16 element each way).
#include "common.cuh"

namespace pk {
namespace {

__global__ void __launch_bounds__(256) dp_pack_kernel(const pk_dp_seg* __restrict__ segs,
                                                      float* __restrict__ bucket) {
    const pk_dp_seg sg = segs[blockIdx.y];
    float* dst = bucket + sg.offset;
    const long long n = sg.elems;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (sg.dtype == PK_BF16) {
        const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(sg.ptr);
        const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
        long long done = 0;
        if (vec) {
            const long long n8 = n / 8;
            for (long long i = t0; i < n8; i += stride) {
                const uint4 v = reinterpret_cast<const uint4*>(src)[i];
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
                float4 a, b;
                float2 f0 = __bfloat1622float2(h[0]), f1 = __bfloat1622float2(h[1]);
                float2 f2 = __bfloat1622float2(h[2]), f3 = __bfloat1622float2(h[3]);
                a = make_float4(f0.x, f0.y, f1.x, f1.y);
                b = make_float4(f2.x, f2.y, f3.x, f3.y);
                reinterpret_cast<float4*>(dst)[2 * i] = a;
                reinterpret_cast<float4*>(dst)[2 * i + 1] = b;
            }
            done = n8 * 8;
        }
        for (long long i = done + t0; i < n; i += stride) dst[i] = __bfloat162float(src[i]);
    } else {
        const float* src = static_cast<const float*>(sg.ptr);
        for (long long i = t0; i < n; i += stride) dst[i] = src[i];
    }
}

__global__ void __launch_bounds__(256) dp_unpack_kernel(const pk_dp_seg* __restrict__ segs,
                                                        const float* __restrict__ bucket,
                                                        float scale) {
    const pk_dp_seg sg = segs[blockIdx.y];
    const float* src = bucket + sg.offset;
    const long long n = sg.elems;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (sg.dtype == PK_BF16) {
        __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(sg.ptr);
        const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
        long long done = 0;
        if (vec) {
            const long long n8 = n / 8;
            for (long long i = t0; i < n8; i += stride) {
                const float4 a = reinterpret_cast<const float4*>(src)[2 * i];
                const float4 b = reinterpret_cast<const float4*>(src)[2 * i + 1];
                __nv_bfloat162 h[4] = {__floats2bfloat162_rn(a.x * scale, a.y * scale),
                                       __floats2bfloat162_rn(a.z * scale, a.w * scale),
                                       __floats2bfloat162_rn(b.x * scale, b.y * scale),
                                       __floats2bfloat162_rn(b.z * scale, b.w * scale)};
                reinterpret_cast<uint4*>(dst)[i] = *reinterpret_cast<const uint4*>(h);
            }
            done = n8 * 8;
        }
        for (long long i = done + t0; i < n; i += stride) dst[i] = __float2bfloat16_rn(src[i] * scale);
    } else {
        float* dst = static_cast<float*>(sg.ptr);
        for (long long i = t0; i < n; i += stride) dst[i] = src[i] * scale;
    }
}

unsigned dp_blocks(long long max_elems) {
    long long b = (max_elems / 8 + 255) / 256;
    if (b < 1) b = 1;
    if (b > 148 * 4) b = 148 * 4;  // a few waves per tensor; the tensors share the grid
    return (unsigned)b;
}

}  // namespace
}  // namespace pk

extern "C" {

cudaError_t pk_cuda_dp_pack(const pk_dp_seg* segs_dev, int nseg, long long max_elems, float* bucket,
                            cudaStream_t st) {
    if (nseg <= 0) return cudaSuccess;
    pk::dp_pack_kernel<<<dim3(pk::dp_blocks(max_elems), nseg), 256, 0, st>>>(segs_dev, bucket);
    pk::count_launch();
    return cudaGetLastError();
}

cudaError_t pk_cuda_dp_unpack(const pk_dp_seg* segs_dev, int nseg, long long max_elems,
                              const float* bucket, float scale, cudaStream_t st) {
    if (nseg <= 0) return cudaSuccess;
    pk::dp_unpack_kernel<<<dim3(pk::dp_blocks(max_elems), nseg), 256, 0, st>>>(segs_dev, bucket, scale);
    pk::count_launch();
    return cudaGetLastError();
}

}  // extern "C"
