// FP32 FMA peak on this device: scalar FFMA and packed FFMA2 (fma.rn.f32x2),
// 8 independent chains per thread, 8 resident 256-thread CTAs per SM, CUDA
// events around 3 timed launches (median). Prints one JSON line per variant.
// Denominator of the SIMT (f32) rows: cfg1 Direct, f32 fused CBA, depthwise.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_peak fp32_peak.cu
#include <cstdio>
#include <algorithm>
#include <vector>

constexpr int kIters = 4096;

__global__ void ffma_kernel(float* out, float a, float b) {
    float x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678f) out[threadIdx.x] = s;
}

__global__ void ffma2_kernel(float* out, float a, float b) {
    unsigned long long x[8];
    unsigned long long av, bv;
    asm("mov.b64 %0, {%1, %1};" : "=l"(av) : "f"(a));
    asm("mov.b64 %0, {%1, %1};" : "=l"(bv) : "f"(b));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float lo = threadIdx.x * 1e-3f + i, hi = lo + 0.5f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(x[i]) : "f"(lo), "f"(hi));
    }
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(av), "l"(bv));
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[i]));
        s += lo + hi;
    }
    if (s == 12345.678f) out[threadIdx.x] = s;
}

template <typename K>
double run(K kern, int sms, double flop_per_thread_iter) {
    float* out;
    cudaMalloc(&out, 1024 * sizeof(float));
    const int blocks = sms * 8, threads = 256;
    kern<<<blocks, threads>>>(out, 0.999f, 0.001f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    std::vector<float> ms;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(out, 0.999f, 0.001f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float t = 0;
        cudaEventElapsedTime(&t, e0, e1);
        ms.push_back(t);
    }
    std::sort(ms.begin(), ms.end());
    cudaFree(out);
    const double flops = (double)blocks * threads * kIters * flop_per_thread_iter;
    return flops / (ms[1] * 1e-3) / 1e12;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const double t1 = run(ffma_kernel, sms, 8 * 2.0);
    const double t2 = run(ffma2_kernel, sms, 8 * 4.0);
    printf("{\"probe\": \"fp32_ffma\", \"tflops\": %.2f, \"sms\": %d, \"max_clock_mhz\": %d}\n", t1, sms, clk / 1000);
    printf("{\"probe\": \"fp32_ffma2_f32x2\", \"tflops\": %.2f, \"sms\": %d, \"max_clock_mhz\": %d}\n", t2, sms, clk / 1000);
    return 0;
}
