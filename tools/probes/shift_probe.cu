// Probe: tcgen05.mma (kind::f16, M=128, N=64, K=16..64) with the A operand
// taken at an arbitrary ROW offset j of a SWIZZLE_128B K-major buffer written
// with the TMA/absolute-address swizzle (16-byte chunk c of row r stored at
// chunk c ^ (r & 7) of a 1024-byte-aligned buffer). Checks which descriptor
// "base offset" field value makes the MMA see rows j..j+127 correctly.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a, uint32_t base_off) {
    uint64_t d = (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32);
    d |= 1ull << 46; d |= (uint64_t)(base_off & 7) << 49; d |= 2ull << 61; return d;
}
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// A_all: [ROWS][64] bf16 (one 64-wide K atom), B: [64][64]
__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int j, int mode) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t abase = su32(smem), bbase = su32(smem + 32768);
    for (int i = threadIdx.x; i < 160 * 8; i += blockDim.x) {  // 160 rows of A
        const int r = i / 8, c = i % 8;
        const uint4 v = *reinterpret_cast<const uint4*>(A + r * 64 + c * 8);
        const uint32_t addr = abase + r * 128 + ((c ^ (r & 7)) << 4);
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
    }
    for (int i = threadIdx.x; i < 64 * 8; i += blockDim.x) {
        const int r = i / 8, c = i % 8;
        const uint4 v = *reinterpret_cast<const uint4*>(B + r * 64 + c * 8);
        const uint32_t addr = bbase + r * 128 + ((c ^ (r & 7)) << 4);
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" :: "r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
    }
    asm volatile("fence.proxy.async.shared::cta;");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" :: "r"(su32(&slot)));
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
    if (threadIdx.x == 0) {
        for (int k = 0; k < 4; ++k) {
            const uint32_t astart = abase + j * 128 + k * 32;
            const uint32_t bo = mode == 0 ? 0u : (mode == 1 ? (uint32_t)(j & 7) : (uint32_t)((astart >> 7) & 7));
            const uint64_t ad = desc_sw128(astart, bo);
            const uint64_t bd = desc_sw128(bbase + k * 32, 0);
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                         :: "r"(tm), "l"(ad), "l"(bd), "r"(idesc(128, 64)), "r"(k));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&bar)));
    }
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0,1,0,p;\n}"
                     : "=r"(done) : "r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
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
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" :: "r"(tm));
}

int main() {
    const int ROWS = 160;
    __nv_bfloat16 *hA = new __nv_bfloat16[ROWS * 64], *hB = new __nv_bfloat16[64 * 64];
    for (int i = 0; i < ROWS * 64; ++i) hA[i] = __float2bfloat16(((i * 37) % 17 - 8) / 8.0f);
    for (int i = 0; i < 64 * 64; ++i) hB[i] = __float2bfloat16(((i * 53) % 13 - 6) / 4.0f);
    __nv_bfloat16 *dA, *dB; float* dD;
    cudaMalloc(&dA, ROWS * 64 * 2); cudaMalloc(&dB, 64 * 64 * 2); cudaMalloc(&dD, 128 * 64 * 4);
    cudaMemcpy(dA, hA, ROWS * 64 * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, 64 * 64 * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    float* hD = new float[128 * 64];
    for (int mode = 0; mode < 3; ++mode) {
        printf("mode %d (%s):", mode, mode == 0 ? "base_offset 0" : mode == 1 ? "base_offset j&7" : "base_offset (addr>>7)&7");
        for (int j : {0, 1, 3, 7, 8, 9, 17, 31}) {
            probe<<<1, 128, 64 * 1024>>>(dA, dB, dD, j, mode);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(hD, dD, 128 * 64 * 4, cudaMemcpyDeviceToHost);
            double maxerr = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < 64; ++n) {
                    double s = 0;
                    for (int k = 0; k < 64; ++k)
                        s += (double)__bfloat162float(hA[(m + j) * 64 + k]) * __bfloat162float(hB[n * 64 + k]);
                    maxerr = fmax(maxerr, fabs(s - hD[m * 64 + n]));
                }
            printf(" j=%d:%s", j, e != cudaSuccess ? cudaGetErrorString(e) : (maxerr < 1e-3 ? "OK" : "BAD"));
        }
        printf("\n");
    }
    return 0;
}
