// Probe: latency of the intra-CTA handshakes the persistent tcgen05 kernels
// chain per tile: (1) mbarrier ping-pong between two warps (arrive -> try_wait
// wake-up), (2) tcgen05.commit -> mbarrier with no MMA outstanding, (3) the
// same after one M=128 N=64 K=16 MMA, (4) named barrier ping-pong.
//   nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a handshake_probe.cu -o handshake_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
    uint32_t done = 0;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(done) : "r"(su32(b)), "r"(ph) : "memory");
    } while (!done);
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}

constexpr int kIters = 1000;

__global__ void probe(long long* out) {
    __shared__ uint64_t bars[4];
    __shared__ uint32_t tslot;
    __shared__ __align__(1024) uint8_t opnd[32768];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) bar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(opnd)[i] = 0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    // (1) mbarrier ping-pong between warp 0 and warp 1
    long long t0 = clock64();
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < kIters; ++i) {
            bar_arrive(&bars[0]);
            bar_wait(&bars[1], i & 1);
        }
    } else if (warp == 1 && lane == 0) {
        for (int i = 0; i < kIters; ++i) {
            bar_wait(&bars[0], i & 1);
            bar_arrive(&bars[1]);
        }
    }
    __syncthreads();
    long long t1 = clock64();
    // (2) commit with nothing outstanding -> wait
    if (warp == 0) {
        for (int i = 0; i < kIters; ++i) {
            asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bars[2])) : "memory");
            bar_wait(&bars[2], i & 1);
        }
    }
    __syncthreads();
    long long t2 = clock64();
    // (3) one M=128 N=64 K=16 MMA then commit -> wait
    if (warp == 0) {
        const uint32_t a = su32(opnd), b = su32(opnd + 16384);
        auto desc = [](uint32_t addr) {
            uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32);
            return d | (1ull << 46) | (2ull << 61);
        };
        const uint64_t ad = desc(a), bd = desc(b);
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
        for (int i = 0; i < kIters; ++i) {
            asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;\n\t}"
                         ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc) : "memory");
            asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bars[3])) : "memory");
            bar_wait(&bars[3], i & 1);
        }
    }
    __syncthreads();
    long long t3 = clock64();
    // (4) named barrier ping-pong (2 warps, 64 threads)
    if (warp < 2)
        for (int i = 0; i < kIters; ++i) asm volatile("bar.sync 1, 64;" ::: "memory");
    __syncthreads();
    long long t4 = clock64();
    if (threadIdx.x == 0) {
        out[0] = (t1 - t0) / kIters;
        out[1] = (t2 - t1) / kIters;
        out[2] = (t3 - t2) / kIters;
        out[3] = (t4 - t3) / kIters;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

int main() {
    long long* d;
    cudaMalloc(&d, 4 * sizeof(long long));
    probe<<<1, 128>>>(d);
    long long h[4];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("mbarrier ping-pong round trip: %lld clk\n", h[0]);
    printf("tcgen05.commit (nothing outstanding) -> wait: %lld clk\n", h[1]);
    printf("1 MMA (M128 N64 K16) + commit -> wait: %lld clk\n", h[2]);
    printf("named barrier (2 warps): %lld clk\n", h[3]);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
