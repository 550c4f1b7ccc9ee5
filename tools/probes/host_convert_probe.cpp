// Host f32 -> bf16 (RNE) conversion throughput with T threads (the host-buffer ABI
// could halve its PCIe bytes for bf16 problems if the host converts fast enough).
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static inline uint16_t bf16_rne(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return (uint16_t)((u >> 16) | 0x40);
    return (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}

int main(int argc, char** argv) {
    const size_t n = (size_t)1 << 28;  // 1 GiB of f32
    std::vector<float> src(n);
    std::vector<uint16_t> dst(n);
    for (size_t i = 0; i < n; ++i) src[i] = (float)(i % 1000) * 0.001f - 0.5f;
    for (int t : {1, 4, 8, 16, 32}) {
        if (t > (int)std::thread::hardware_concurrency()) break;
        auto run = [&]() {
            std::vector<std::thread> th;
            for (int k = 0; k < t; ++k)
                th.emplace_back([&, k]() {
                    const size_t b = n * k / t, e = n * (k + 1) / t;
                    for (size_t i = b; i < e; ++i) dst[i] = bf16_rne(src[i]);
                });
            for (auto& x : th) x.join();
        };
        run();
        const auto t0 = std::chrono::steady_clock::now();
        for (int r = 0; r < 3; ++r) run();
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / 3;
        std::printf("threads %2d: %.1f G elem/s (%.1f GB/s f32 read)\n", t, n / s / 1e9, n * 4 / s / 1e9);
    }
    std::printf("hw threads %u\n", std::thread::hardware_concurrency());
}
