// H2D after a 16-thread fill: plain stores vs stores + clflushopt vs non-temporal stores.
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <immintrin.h>
#include <cuda_runtime.h>
__attribute__((target("clflushopt"))) static void flush_range(char* p, size_t n) {
  for (size_t i = 0; i < n; i += 64) _mm_clflushopt(p + i);
  _mm_sfence();
}
static void nt_fill(char* p, size_t n, int v) {
  const __m128i x = _mm_set1_epi8((char)v);
  for (size_t i = 0; i < n; i += 16) _mm_stream_si128(reinterpret_cast<__m128i*>(p + i), x);
  _mm_sfence();
}
int main() {
  const size_t n = 16u << 20;
  void* d = nullptr;
  cudaMalloc(&d, 64u << 20);
  cudaStream_t st; cudaStreamCreate(&st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  char* h = nullptr; cudaHostAlloc((void**)&h, 32u << 20, cudaHostAllocDefault);
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      std::vector<std::thread> ts;
      for (int t = 0; t < 16; ++t)
        ts.emplace_back([=] {
          char* p = h + n * t / 16; size_t m = n / 16;
          if (mode == 2) nt_fill(p, m, rep); else memset(p, rep, m);
          if (mode == 1) flush_range(p, m);
        });
      for (auto& t : ts) t.join();
      cudaEventRecord(a, st);
      cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("%-22s rep %d: %.3f ms  %.1f GB/s\n", mode == 0 ? "plain stores" : mode == 1 ? "stores + clflushopt" : "non-temporal stores", rep, ms, n / ms / 1e6);
    }
  }
  return 0;
}
