// Probe: 2-CTA (cta_group::2) tcgen05 GEMM on a CTA pair, M = 256 per pair,
// N = 256, K = 64 * KB, bf16 in, fp32 out. Each CTA TMA-loads its 128 rows of
// A and its 128-row half of B (cta_group::2 loads signal the leader's
// barrier); the leader issues M=256 MMAs; commits are multicast to both CTAs;
// both epilogues drain their own TMEM half and signal the leader remotely.
// Checks against a host fp32 reference and times it. Build:
//   nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a cta2_probe.cu -lcuda -o cta2_probe
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e = (x);                                                         \
        if (e != cudaSuccess) {                                                      \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                 \
        }                                                                            \
    } while (0)

constexpr int KB = 4;        // k-blocks of 64
constexpr int STAGES = 2;
constexpr int kA = 128 * 64 * 2, kB = 128 * 64 * 2, kStage = kA + kB;

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
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
    uint64_t d = (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(16 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32);
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
}
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    gemm2(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap, float* C,
          int N) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    uint64_t* full = (uint64_t*)(sm + STAGES * kStage);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 1;
    uint32_t* tslot = (uint32_t*)(tempty + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cta_rank();
    const int pair = blockIdx.x >> 1;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) {
            bar_init(&full[i], 1);
            bar_init(&empty[i], 1);
        }
        bar_init(tfull, 1);
        bar_init(tempty, 8);  // 4 epilogue warps x 2 CTAs (only the leader's is used)
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = *tslot;

    if (warp == 0 && lane == 0) {
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % STAGES;
            bar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
            const uint32_t fb = su32(&full[s]) & 0xFEFFFFFFu;  // leader's barrier
            if (rank == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])),
                             "r"(2 * kStage) : "memory");
            uint8_t* sa = sm + s * kStage;
            asm volatile(
                "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(sa)),
                "l"((uint64_t)&amap), "r"(kb * 64), "r"(pair * 256 + (int)rank * 128), "r"(fb) : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(sa + kA)),
                "l"((uint64_t)&bmap), "r"(kb * 64), "r"((int)rank * 128), "r"(fb) : "memory");
        }
    } else if (warp == 1 && rank == 0) {
        bar_wait(tempty, 1);  // fresh barrier: parity 1 passes
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % STAGES;
            bar_wait(&full[s], (kb / STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint64_t ad = desc_sw128(su32(sm + s * kStage)), bd = desc_sw128(su32(sm + s * kStage + kA));
            for (int k = 0; k < 4; ++k) {
                const uint32_t acc = (kb | k) != 0;
                asm volatile(
                    "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                    "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase),
                    "l"(ad + 2 * k), "l"(bd + 2 * k), "r"(idesc(256, 256)), "r"(acc) : "memory");
            }
            asm volatile(
                "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(su32(&empty[s])),
                "h"((uint16_t)3) : "memory");
        }
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(su32(tfull)),
            "h"((uint16_t)3) : "memory");
    } else if (warp >= 2) {
        const int q = warp & 3;
        bar_wait(tfull, 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int row = pair * 256 + (int)rank * 128 + q * 32 + lane;
        for (int c0 = 0; c0 < 256; c0 += 16) {
            uint32_t v[16];
            const uint32_t ta = tbase + c0 + ((uint32_t)(q * 32) << 16);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int e = 0; e < 16; ++e) C[(size_t)row * N + c0 + e] = __uint_as_float(v[e]);
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) {
            uint32_t remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(su32(tempty)));
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(256));
    }
}

static bool make_map(CUtensorMap* m, void* base, int rows, int cols) {
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    return cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int main() {
    const int P = 2, M = 256 * P, N = 256, K = 64 * KB;
    std::vector<__nv_bfloat16> A(M * K), B(N * K);
    std::vector<float> Af(M * K), Bf(N * K);
    std::mt19937 rng(1);
    std::uniform_real_distribution<float> d(-1, 1);
    for (int i = 0; i < M * K; ++i) { A[i] = __float2bfloat16(d(rng)); Af[i] = __bfloat162float(A[i]); }
    for (int i = 0; i < N * K; ++i) { B[i] = __float2bfloat16(d(rng)); Bf[i] = __bfloat162float(B[i]); }
    __nv_bfloat16 *dA, *dB;
    float* dC;
    CK(cudaMalloc(&dA, A.size() * 2));
    CK(cudaMalloc(&dB, B.size() * 2));
    CK(cudaMalloc(&dC, (size_t)M * N * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemset(dC, 0, (size_t)M * N * 4));
    CUtensorMap am, bm;
    if (!make_map(&am, dA, M, K) || !make_map(&bm, dB, N, K)) { printf("map fail\n"); return 1; }
    const int smem = STAGES * kStage + 1024 + 256;
    CK(cudaFuncSetAttribute(gemm2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    gemm2<<<2 * P, 192, smem>>>(am, bm, dC, N);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> C((size_t)M * N);
    CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
    double err = 0, ref2 = 0;
    int bad = 0;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += (double)Af[i * K + k] * Bf[j * K + k];
            const double e = C[(size_t)i * N + j] - s;
            err += e * e;
            ref2 += s * s;
            if (std::fabs(e) > 1e-2 * (1 + std::fabs(s)) && bad++ < 5)
                printf("mismatch (%d,%d): got %f want %f\n", i, j, C[(size_t)i * N + j], s);
        }
    printf("rel-L2 %.3e, bad %d\n", std::sqrt(err / ref2), bad);
    return bad ? 1 : 0;
}
