// Host-side helpers shared by the tcgen05 kernels: TMA descriptor encoding
// through the driver entry point (no libcuda link dependency).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>

namespace pk::tc {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
        else
            cudaGetLastError();
    });
    return fn;
}

// 2-D bf16 row-major [rows][cols] (row stride in elements), 128-byte swizzle,
// box {64 cols, box_rows}, zero fill out of bounds.
inline bool make_map_2d(CUtensorMap* map, const void* base, long long rows, long long cols,
                        long long row_stride, int box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)row_stride * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 4-D bf16 NHWC tensor [n][h][w][pitch] viewed as dims {pitch, w, h, n};
// box {64, bw, bh, bn} with traversal strides {1, sw, sh, 1}; the box extent
// passed to the driver is the number of elements traversed (bw*sw), so a
// strided box still delivers bw x bh x bn rows of 128 bytes.
inline bool make_map_nhwc(CUtensorMap* map, const void* base, int n, int h, int w, int pitch,
                          int bw, int bh, int bn, int sw = 1, int sh = 1, int box_c = 64) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    if (bw * sw > 256 || bh * sh > 256 || bn > 256) return false;
    cuuint64_t dims[4] = {(cuuint64_t)pitch, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
    cuuint64_t strides[3] = {(cuuint64_t)pitch * 2, (cuuint64_t)w * pitch * 2,
                             (cuuint64_t)h * w * pitch * 2};
    cuuint32_t box[4] = {(cuuint32_t)box_c, (cuuint32_t)(bw * sw), (cuuint32_t)(bh * sh),
                         (cuuint32_t)bn};
    cuuint32_t estr[4] = {1, (cuuint32_t)sw, (cuuint32_t)sh, 1};
    // 64-channel (128-byte) boxes use the 128B swizzle; 8-channel (16-byte)
    // boxes land as plain 16-byte rows (UMMA "interleaved" core matrices)
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              box_c == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 4-D bf16 view with explicit element strides per dimension (w, h, n): a
// sub-pixel phase of an NHWC tensor for TMA stores (box {64, bw, bh, bn}).
inline bool make_map_nhwc_strided(CUtensorMap* map, const void* base, int n, int h, int w,
                                  int pitch, long long w_stride, long long h_stride,
                                  long long n_stride, int bw, int bh, int bn) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[4] = {(cuuint64_t)pitch, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
    cuuint64_t strides[3] = {(cuuint64_t)w_stride * 2, (cuuint64_t)h_stride * 2,
                             (cuuint64_t)n_stride * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bn};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The filter W[K][taps][pitch] as an MN-major B operand for backward data:
// 3-D view (channel, tap, output channel), box {64 channels, 1 tap, 64 k} = one
// 8 KB SW128 atom (64 k rows of 64 channels).
inline bool make_map_filter_mn(CUtensorMap* map, const void* w, int k, int taps, int pitch) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)taps, (cuuint64_t)k};
    cuuint64_t strides[2] = {(cuuint64_t)pitch * 2, (cuuint64_t)taps * pitch * 2};
    cuuint32_t box[3] = {64, 1, 64};
    cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(w), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D bf16 view of an NHWC tensor as rows of pixels: dims {w*pitch, h, n},
// box {box_elems, box_rows, 1}, no swizzle (plain rows of box_elems*2 bytes).
// Used for narrow-channel halos, where a per-pixel (16-byte) inner box
// dimension would make the TMA engine move 16 bytes per element.
inline bool make_map_pixel_rows(CUtensorMap* map, const void* base, int n, int h, int w, int pitch,
                                int box_elems, int box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || box_elems > 256 || box_rows > 256 || (box_elems * 2) % 16) return false;
    cuuint64_t dims[3] = {(cuuint64_t)w * pitch, (cuuint64_t)h, (cuuint64_t)n};
    cuuint64_t strides[2] = {(cuuint64_t)w * pitch * 2, (cuuint64_t)h * w * pitch * 2};
    cuuint32_t box[3] = {(cuuint32_t)box_elems, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Rectangular tile (bw x bh x bn pixels, product `rows`, powers of two) that
// covers an (n, h, w) output volume with the least padding.
struct RectTile {
    int bw, bh, bn;
};
inline RectTile best_rect(int n, int h, int w, int rows) {
    RectTile best{rows, 1, 1};
    long long best_vol = -1;
    for (int bw = 1; bw <= rows && bw <= 128; bw *= 2)
        for (int bh = 1; bw * bh <= rows && bh <= 128; bh *= 2) {
            const int bn = rows / (bw * bh);
            if (bn < 1 || bn > 256 || bw * bh * bn != rows) continue;
            const long long vol = (long long)((w + bw - 1) / bw) * bw * ((h + bh - 1) / bh) * bh *
                                  ((n + bn - 1) / bn) * bn;
            // least padding; ties -> wider rows (longer contiguous runs)
            if (best_vol < 0 || vol < best_vol || (vol == best_vol && bw > best.bw)) {
                best_vol = vol;
                best = {bw, bh, bn};
            }
        }
    return best;
}

inline int num_sms_of_current_device() {
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 148;
    }
    return cached[dev];
}

}  // namespace pk::tc
