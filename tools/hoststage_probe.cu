// Host staging probe: cost of moving a 1.84 MB pageable vector to the device (cfg2 e2e input).
//   nvcc -O3 -std=c++17 tools/hoststage_probe.cu -o tools/hoststage_probe -lpthread
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
using clk = std::chrono::steady_clock;
static double us(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::micro>(b - a).count(); }
int main() {
  const size_t bytes = 115200 * 16;
  std::vector<char> src(bytes, 1);
  char* pin; cudaHostAlloc(&pin, bytes, 0);
  char* dev; cudaMalloc(&dev, bytes);
  cudaStream_t s; cudaStreamCreate(&s);
  printf("hardware_concurrency %u\n", std::thread::hardware_concurrency());
  for (int rep = 0; rep < 3; ++rep) {
    auto t0 = clk::now(); std::memcpy(pin, src.data(), bytes); auto t1 = clk::now();
    printf("memcpy 1 thread: %.1f us\n", us(t0, t1));
    t0 = clk::now(); cudaMemcpyAsync(dev, src.data(), bytes, cudaMemcpyHostToDevice, s); cudaStreamSynchronize(s); t1 = clk::now();
    printf("cudaMemcpyAsync pageable + sync: %.1f us\n", us(t0, t1));
    t0 = clk::now(); cudaMemcpyAsync(dev, pin, bytes, cudaMemcpyHostToDevice, s); cudaStreamSynchronize(s); t1 = clk::now();
    printf("cudaMemcpyAsync pinned + sync: %.1f us\n", us(t0, t1));
  }
  for (int nt : {2, 4, 8}) {
    std::atomic<int> go{0}, fin{0};
    std::atomic<bool> stop{false};
    std::vector<std::thread> th;
    for (int i = 0; i < nt; ++i)
      th.emplace_back([&, i] {
        int seen = 0;
        while (!stop.load()) {
          const int g = go.load(std::memory_order_acquire);
          if (g == seen) continue;
          seen = g;
          const size_t per = (bytes + nt - 1) / nt, off = i * per, len = std::min(per, bytes - off);
          std::memcpy(pin + off, src.data() + off, len);
          fin.fetch_add(1, std::memory_order_acq_rel);
        }
      });
    for (int rep = 0; rep < 4; ++rep) {
      fin = 0;
      auto t0 = clk::now();
      go.fetch_add(1, std::memory_order_acq_rel);
      while (fin.load(std::memory_order_acquire) < nt) {}
      auto t1 = clk::now();
      printf("memcpy %d spinning threads: %.1f us\n", nt, us(t0, t1));
    }
    stop = true;
    for (auto& t : th) t.join();
  }
  return 0;
}
