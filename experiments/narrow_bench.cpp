// Host narrowing throughput probe: int64 -> int32 for 256M weights with T threads.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>
int main() {
  const size_t m = 256u << 20;
  int64_t* w = (int64_t*)aligned_alloc(64, m * 8);
  int32_t* o = (int32_t*)aligned_alloc(64, m * 4);
  for (size_t i = 0; i < m; ++i) w[i] = (int64_t)(i % 201) - 100;
  for (size_t i = 0; i < m; ++i) o[i] = 0;
  for (int T : {1, 4, 8, 16, 32}) {
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([=] {
        const size_t lo = m * t / T, hi = m * (t + 1) / T;
        for (size_t i = lo; i < hi; ++i) o[i] = (int32_t)w[i];
      });
    for (auto& x : th) x.join();
    double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("T=%2d %.1f ms  %.1f GB/s (read+write)\n", T, s * 1e3, m * 12 / s / 1e9);
  }
  std::printf("hw threads %u\n", std::thread::hardware_concurrency());
}
