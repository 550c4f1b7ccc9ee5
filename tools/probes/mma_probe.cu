// Micro-probe: tcgen05.mma (kind::f16, M=128, K=16) issue-to-completion time
// per instruction vs N, with A from shared memory (SS) or tensor memory (TS).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_probe.cu -o mma_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
    uint64_t d = (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32);
    d |= 1ull << 46; d |= 2ull << 61; return d;
}
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <int N, bool TS, int MODE>
__global__ void probe(unsigned long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x)
        ((uint32_t*)smem)[i] = (MODE & 1) ? (0x3f803f80u ^ (i * 2654435761u & 0x00ff00ffu)) : 0u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = slot;
    __shared__ uint64_t spin_bar;
    __shared__ volatile int stop;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&spin_bar)));
        stop = 0;
    }
    __syncthreads();
    if ((MODE & 8) && threadIdx.x >= 32 && (threadIdx.x & 31) == 0 + ((MODE & 16) ? 0 : 0)) {
        // spin like a waiting pipeline role: try_wait on a barrier that completes at the end
        uint32_t done = 0;
        while (!done) {
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}"
                         : "=r"(done) : "r"(su32(&spin_bar)));
        }
    }
    if (threadIdx.x == 0) {
        const uint32_t a = su32(smem), b = su32(smem + 65536 + 32768);
        constexpr uint32_t id = idesc(128, N);
        long long t0 = clock64();
        uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            const int nk = (MODE & 2) ? 13 : 4;
            for (int k = 0; k < nk; ++k) {
                const uint32_t ao = (MODE & 2) ? (k >> 2) * 16384 + (k & 3) * 32 : k * 32;
                const uint32_t bo = (MODE & 2) ? (k >> 2) * (N * 128) + (k & 3) * 32 : k * 32;
                if (TS) {
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}"
                                 :: "r"(tm), "r"(tm + 256 + (k & 3) * 8), "l"(desc_sw128(b + bo)), "r"(id));
                } else {
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\n"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                                 :: "r"(tm), "l"(desc_sw128(a + ao)), "l"(desc_sw128(b + bo)), "r"(id));
                }
            }
            if (MODE & 4) {  // latency-exposed groups: commit + wait after each group
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&bar)));
                uint32_t done = 0;
                while (!done)
                    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                                 : "=r"(done) : "r"(su32(&bar)), "r"(ph));
                ph ^= 1;
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&bar)));
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                         : "=r"(done) : "r"(su32(&bar)), "r"(ph));
        long long t1 = clock64();
        out[blockIdx.x] = (unsigned long long)(t1 - t0);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(&spin_bar)));
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tm));
}

template <int N, bool TS, int MODE>
void run(int grid) {
    unsigned long long* d; cudaMalloc(&d, 8 * 148);
    auto k = probe<N, TS, MODE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    const int iters = 600;
    const int thr = (MODE & 8) ? 416 : 128;
    k<<<grid, thr, 160 * 1024>>>(d, 10);
    k<<<grid, thr, 160 * 1024>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148]; cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
    double cyc = (double)h[0] / (iters * ((MODE & 2) ? 13 : 4));
    printf("N=%3d %s mode=%d (rand=%d 64KB-A=%d grouped=%d) grid=%3d: %.1f clk per MMA -> %.0f FLOP/clk/SM  %s\n",
           N, TS ? "TS" : "SS", MODE, MODE & 1, (MODE >> 1) & 1, (MODE >> 2) & 1,
           grid, cyc, 2.0 * 128 * N * 16 / cyc, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    const int grid = 148;
    run<64, false, 3>(grid); run<64, false, 11>(grid); run<64, false, 7>(grid); run<64, false, 15>(grid);
    run<128, false, 3>(grid); run<128, false, 11>(grid);
    run<64, true, 1>(grid); run<64, true, 9>(grid);
    return 0;
}
