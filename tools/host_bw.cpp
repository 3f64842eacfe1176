// host_bw.cpp -- host memory read bandwidth with T threads over an 8 GiB
// buffer (the e2e upload's floor: narrowing reads the caller's uint64 matrix).
// Build: g++ -O3 -march=native -pthread -o tools/host_bw tools/host_bw.cpp
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

int main(int argc, char** argv) {
  const size_t bytes = (argc > 1 ? atoll(argv[1]) : 8ll) << 30;
  const size_t n = bytes / 8;
  uint64_t* a = static_cast<uint64_t*>(aligned_alloc(64, bytes));
  std::vector<std::thread> ts;
  const unsigned hw = std::thread::hardware_concurrency();
  for (unsigned t = 0; t < hw; ++t)  // first touch in parallel
    ts.emplace_back([=] { memset(a + n * t / hw, 1, (n * (t + 1) / hw - n * t / hw) * 8); });
  for (auto& t : ts) t.join();
  for (unsigned T : {1u, 2u, 4u, 8u, hw}) {
    std::vector<uint64_t> sums(T);
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> w;
    for (unsigned t = 0; t < T; ++t)
      w.emplace_back([&, t] {
        uint64_t s = 0;
        const size_t lo = n * t / T, hi = n * (t + 1) / T;
        for (size_t i = lo; i < hi; ++i) s += a[i];
        sums[t] = s;
      });
    for (auto& t : w) t.join();
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("{\"bench\": \"host_read\", \"threads\": %u, \"GBps\": %.1f, \"ms\": %.1f}\n", T, bytes / dt / 1e9,
           dt * 1e3);
  }
  return 0;
}
