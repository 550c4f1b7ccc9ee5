// Correctness probe for tcgen05.mma with A in tensor memory (kind::f16, M=128,
// N=64, K=16): A written lane-per-row with tcgen05.st (column j = bf16 pair
// k = 2j, 2j+1), B in SWIZZLE_128B K-major smem. Compares D with a CPU GEMM.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
    uint64_t d = (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32);
    d |= 1ull << 46; d |= 2ull << 61; return d;
}
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__global__ void ts_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int K) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    // B [64][K] -> SW128 K-major atoms of 64 K
    for (int i = threadIdx.x; i < 64 * K / 8; i += blockDim.x) {
        const int n = i / (K / 8), j = i % (K / 8);
        const uint4 v = *reinterpret_cast<const uint4*>(B + n * K + j * 8);
        const uint32_t addr = su32(smem) + (j / 8) * 64 * 128 + n * 128 + (((j & 7) ^ (n & 7)) << 4);
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
    }
    asm volatile("fence.proxy.async.shared::cta;");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = slot;
    // A rows -> TMEM columns 128.. (lane = row)
    {
        const int m = warp * 32 + lane;
        for (int c = 0; c < K / 2; c += 8) {
            uint32_t v[8];
            for (int e = 0; e < 8; ++e) {
                __nv_bfloat162 p = __halves2bfloat162(A[m * K + 2 * (c + e)], A[m * K + 2 * (c + e) + 1]);
                v[e] = *reinterpret_cast<uint32_t*>(&p);
            }
            const uint32_t ta = tm + 128 + c + ((uint32_t)(warp * 32) << 16);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                         :: "r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (threadIdx.x == 0) {
        for (int k = 0; k < K / 16; ++k) {
            const uint64_t bd = desc_sw128(su32(smem) + (k / 4) * 64 * 128 + (k % 4) * 32);
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}"
                         :: "r"(tm), "r"(tm + 128 + k * 8), "l"(bd), "r"(idesc(128, 64)), "r"(k));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&bar)));
    }
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}"
                     : "=r"(done) : "r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    {
        const int m = warp * 32 + lane;
        for (int c = 0; c < 64; c += 16) {
            uint32_t v[16];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                           "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                         : "r"(tm + c + ((uint32_t)(warp * 32) << 16)));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            for (int e = 0; e < 16; ++e) D[m * 64 + c + e] = __uint_as_float(v[e]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(tm));
}

int main() {
    const int K = 128;
    __nv_bfloat16 *hA = new __nv_bfloat16[128 * K], *hB = new __nv_bfloat16[64 * K];
    float* ref = new float[128 * 64];
    for (int i = 0; i < 128 * K; ++i) hA[i] = __float2bfloat16(((i * 37) % 17 - 8) / 8.0f);
    for (int i = 0; i < 64 * K; ++i) hB[i] = __float2bfloat16(((i * 53) % 13 - 6) / 4.0f);
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += (double)__bfloat162float(hA[m * K + k]) * __bfloat162float(hB[n * K + k]);
            ref[m * 64 + n] = (float)s;
        }
    __nv_bfloat16 *dA, *dB; float* dD;
    cudaMalloc(&dA, 128 * K * 2); cudaMalloc(&dB, 64 * K * 2); cudaMalloc(&dD, 128 * 64 * 4);
    cudaMemcpy(dA, hA, 128 * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, 64 * K * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    ts_kernel<<<1, 128, 64 * 1024>>>(dA, dB, dD, K);
    cudaError_t e = cudaDeviceSynchronize();
    float* hD = new float[128 * 64];
    cudaMemcpy(hD, dD, 128 * 64 * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0; int bad = 0;
    for (int i = 0; i < 128 * 64; ++i) {
        double d = fabs(hD[i] - ref[i]);
        if (d > maxerr) maxerr = d;
        if (d > 1e-2 && bad < 5) { printf("mismatch at m=%d n=%d: %f vs %f\n", i / 64, i % 64, hD[i], ref[i]); ++bad; }
    }
    printf("TS MMA probe: %s, max abs err %g\n", cudaGetErrorString(e), maxerr);
    return 0;
}
