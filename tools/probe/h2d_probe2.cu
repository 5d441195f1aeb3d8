// H2D variants after a 16-thread fill: pageable source, delay, chunked copies.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
static void fill(void* h, size_t n, int threads, int v) {
  std::vector<std::thread> ts;
  for (int t = 0; t < threads; ++t) ts.emplace_back([=] { memset((char*)h + n * t / threads, v, n / threads); });
  for (auto& t : ts) t.join();
}
int main() {
  const size_t n = 16u << 20;
  void* d = nullptr;
  cudaMalloc(&d, 64u << 20);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  void* pin = nullptr; cudaHostAlloc(&pin, 32u << 20, cudaHostAllocDefault);
  void* pg = malloc(32u << 20);
  auto run = [&](const char* name, void* h, int delay_us, int chunks) {
    for (int rep = 0; rep < 3; ++rep) {
      fill(h, n, 16, rep);
      if (delay_us) std::this_thread::sleep_for(std::chrono::microseconds(delay_us));
      cudaEventRecord(a, st);
      for (int c = 0; c < chunks; ++c)
        cudaMemcpyAsync((char*)d + n * c / chunks, (char*)h + n * c / chunks, n / chunks, cudaMemcpyHostToDevice, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("%-28s rep %d: %.3f ms  %.1f GB/s\n", name, rep, ms, n / ms / 1e6);
    }
  };
  run("pinned, no delay", pin, 0, 1);
  run("pinned, 2 ms delay", pin, 2000, 1);
  run("pinned, 20 ms delay", pin, 20000, 1);
  run("pinned, 16 chunks", pin, 0, 16);
  run("pageable", pg, 0, 1);
  return 0;
}
