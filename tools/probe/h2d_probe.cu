// H2D bandwidth probe: cudaHostAlloc'd source (default / write-combined),
// filled by 1 or 16 host threads right before the copy (the JPEG planner
// fills its staging with 16 threads).
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
static void fill(void* h, size_t n, int threads, int v) {
  std::vector<std::thread> ts;
  for (int t = 0; t < threads; ++t)
    ts.emplace_back([=] { memset((char*)h + n * t / threads, v, n / threads); });
  for (auto& t : ts) t.join();
}
int main() {
  const size_t n = 16u << 20;
  void* d = nullptr;
  cudaMalloc(&d, 64u << 20);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (unsigned flags : {cudaHostAllocDefault, cudaHostAllocWriteCombined}) {
    void* h = nullptr;
    cudaHostAlloc(&h, 32u << 20, flags);
    for (int threads : {1, 16}) {
      for (int rep = 0; rep < 3; ++rep) {
        fill(h, n, threads, rep);
        cudaEventRecord(a, st);
        cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("%s threads=%2d rep %d: %.3f ms  %.1f GB/s\n", flags ? "WC     " : "default", threads, rep, ms, n / ms / 1e6);
      }
    }
    cudaFreeHost(h);
  }
  return 0;
}
