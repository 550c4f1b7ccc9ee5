// Probe: per-SM TMA load throughput vs box shape. One CTA per SM streams a
// [rows_total][K] bf16 matrix (its own slice) into a ring of smem buffers with
// SW128 boxes of {64, R} (2-D) or {64, R, C} (3-D view: C 64-wide k-chunks per
// box), `inflight` boxes outstanding, and reports aggregate GB/s.
//   nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a tma_box_probe.cu -lcuda -o tma_box_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <string>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void stream_kernel(const __grid_constant__ CUtensorMap map, int dims3, int box_rows, int box_chunks,
                              int boxes_per_cta, int inflight, int box_bytes, int rows_per_cta, int kchunks) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    uint64_t* bars = (uint64_t*)(sm + inflight * box_bytes);
    if (threadIdx.x == 0) {
        for (int i = 0; i < inflight; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const int row0 = blockIdx.x * rows_per_cta;
    const int per_row_block = kchunks / box_chunks;
    auto issue = [&](int b, int slot) {
        const int rb = b / per_row_block, cb = b % per_row_block;
        const uint32_t dst = su32(sm + slot * box_bytes), bar = su32(&bars[slot]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(box_bytes) : "memory");
        if (dims3)
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
                "l"((uint64_t)&map), "r"(0), "r"(row0 + rb * box_rows), "r"(cb * box_chunks), "r"(bar) : "memory");
        else
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
                "l"((uint64_t)&map), "r"(cb * 64), "r"(row0 + rb * box_rows), "r"(bar) : "memory");
    };
    for (int b = 0; b < inflight && b < boxes_per_cta; ++b) issue(b, b);
    for (int b = 0; b < boxes_per_cta; ++b) {
        const int slot = b % inflight;
        const uint32_t ph = (b / inflight) & 1;
        uint32_t done = 0;
        do {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                         : "=r"(done) : "r"(su32(&bars[slot])), "r"(ph) : "memory");
        } while (!done);
        if (b + inflight < boxes_per_cta) issue(b + inflight, slot);
    }
}

__global__ void halo4_kernel(const __grid_constant__ CUtensorMap map, int tx, int ty, int sx, int sy, int oob,
                             int total, int inflight, int bytes, int stride) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    uint64_t* bars = (uint64_t*)(sm + inflight * stride);
    if (threadIdx.x == 0) {
        for (int i = 0; i < inflight; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    auto issue = [&](int t, int slot) {
        const int x = t % tx, y = (t / tx) % ty, n = t / (tx * ty);
        const uint32_t dst = su32(sm + slot * stride), bar = su32(&bars[slot]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
            "l"((uint64_t)&map), "r"(0), "r"(x * sx - oob), "r"(y * sy - oob), "r"(n), "r"(bar) : "memory");
    };
    int mine = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) ++mine;
    for (int i = 0; i < inflight && i < mine; ++i) issue(blockIdx.x + i * gridDim.x, i);
    for (int i = 0; i < mine; ++i) {
        const int slot = i % inflight;
        const uint32_t ph = (i / inflight) & 1;
        uint32_t done = 0;
        do {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                         : "=r"(done) : "r"(su32(&bars[slot])), "r"(ph) : "memory");
        } while (!done);
        if (i + inflight < mine) issue(blockIdx.x + (i + inflight) * gridDim.x, slot);
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int K = 512, kchunks = K / 64;
    const long long rows_per_cta = 4096;  // 4096 x 512 x 2 B = 4 MB per SM
    const long long rows = rows_per_cta * sms;
    void* buf;
    cudaMalloc(&buf, rows * K * 2);
    cudaMemset(buf, 1, rows * K * 2);
    struct Cfg { int dims3, box_rows, box_chunks, inflight; };
    std::vector<Cfg> cfgs = {{0, 32, 1, 8}, {0, 64, 1, 8}, {0, 128, 1, 4}, {0, 128, 1, 8}, {0, 256, 1, 4},
                             {1, 128, 2, 4}, {1, 128, 4, 2}, {1, 128, 4, 3}, {1, 64, 8, 3}, {1, 256, 2, 3}};
    for (const auto& c : cfgs) {
        CUtensorMap map;
        CUresult r;
        if (c.dims3) {
            cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)kchunks};
            cuuint64_t strides[2] = {(cuuint64_t)K * 2, 128};
            cuuint32_t box[3] = {64, (cuuint32_t)c.box_rows, (cuuint32_t)c.box_chunks};
            cuuint32_t es[3] = {1, 1, 1};
            r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
            cuuint64_t strides[1] = {(cuuint64_t)K * 2};
            cuuint32_t box[2] = {64, (cuuint32_t)c.box_rows};
            cuuint32_t es[2] = {1, 1};
            r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
        const int box_bytes = 64 * 2 * c.box_rows * c.box_chunks;
        const int boxes = (int)(rows_per_cta / c.box_rows) * (kchunks / c.box_chunks);
        const int smem = c.inflight * box_bytes + 1024 + 256;
        cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            stream_kernel<<<sms, 32, smem>>>(map, c.dims3, c.box_rows, c.box_chunks, boxes, c.inflight, box_bytes,
                                             (int)rows_per_cta, kchunks);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double gb = (double)rows * K * 2 / 1e9;
        printf("%s box {64,%d%s} %6d B, %d in flight: %7.1f GB/s (%.3f us per box per SM) err=%s\n",
               c.dims3 ? "3d" : "2d", c.box_rows, c.dims3 ? (",x" + std::to_string(c.box_chunks)).c_str() : "",
               box_bytes, c.inflight, gb / (ms / 1e3), ms * 1e3 / boxes, cudaGetErrorString(cudaGetLastError()));
    }
    // 4-D halo boxes over an NHWC [n][112][112][64] tensor (the stem dgrad dY):
    // box {64, bw, bh, 1} at tile origins on a (bw-2) x (bh-2) grid (overlapping
    // halos), with and without out-of-bounds borders.
    {
        const int n = 256;
        struct H4 { int bw, bh, oob, inflight, H, W; };
        // the last six: ResNet conv2_x (56x56x64) halo rows as the halo kernel loads them
        // (58-wide boxes at x = -1, i.e. OOB left/right borders) vs in-bounds boxes of the same bytes on a 58-wide tensor
        std::vector<H4> hc = {{11, 11, 1, 3, 112, 112}, {11, 11, 0, 3, 112, 112}, {11, 11, 1, 6, 112, 112},
                              {19, 11, 1, 3, 112, 112}, {34, 6, 1, 3, 112, 112}, {58, 6, 0, 3, 112, 112},
                              {58, 8, 1, 2, 56, 56},     {58, 8, 1, 3, 56, 56},   {58, 8, 0, 2, 56, 58},
                              {58, 8, 0, 3, 56, 58},     {58, 4, 1, 4, 56, 56},   {58, 4, 0, 4, 56, 58}};
        for (const auto& c : hc) {
            const int H = c.H, W = c.W;
            CUtensorMap map;
            cuuint64_t dims[4] = {64, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)n};
            cuuint64_t strides[3] = {128, (cuuint64_t)W * 128, (cuuint64_t)H * W * 128};
            cuuint32_t box[4] = {64, (cuuint32_t)c.bw, (cuuint32_t)c.bh, 1};
            cuuint32_t es[4] = {1, 1, 1, 1};
            if (cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, strides, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
                printf("4d encode failed\n");
                continue;
            }
            const int sx = (c.bw >= W) ? W : c.bw - 2, sy = c.bh - 2;  // tile step (halo overlap of 2)
            const int tx = W / sx, ty = H / sy;
            const int box_bytes = (c.bw * c.bh * 128 + 1023) / 1024 * 1024;
            const int smem = c.inflight * box_bytes + 1024 + 256;
            cudaFuncSetAttribute(halo4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            const int total = n * tx * ty;
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                halo4_kernel<<<sms, 32, smem>>>(map, tx, ty, sx, sy, c.oob, total, c.inflight, c.bw * c.bh * 128, box_bytes);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double gb = (double)total * c.bw * c.bh * 128 / 1e9;
            printf("4d halo box {64,%d,%d} %s, %d in flight: %7.1f GB/s of box bytes (%.3f us per box per SM) err=%s\n",
                   c.bw, c.bh, c.oob ? "origin -1 (OOB borders)" : "in bounds", c.inflight, gb / (ms / 1e3),
                   ms * 1e3 / ((double)total / sms), cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
