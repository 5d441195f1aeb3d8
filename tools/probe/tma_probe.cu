// Minimal 3-D TMA tensor load (the warp_affine_tma_kernel pattern), checked against the source.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
__device__ inline uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <bool BIG>
__global__ void k(const __grid_constant__ CUtensorMap tm, float* out, int x0, int y0, int n, const double* dummy) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bar = (uint64_t*)smem;
  float* stage = (float*)(smem + 128);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(144 * 40 * 4) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(su32(stage)), "l"((uint64_t)&tm), "r"(x0), "r"(y0), "r"(n), "r"(su32(bar)) : "memory");
  }
  __syncthreads();
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(su32(bar)) : "memory");
  for (int i = threadIdx.x; i < 144 * 40; i += blockDim.x) out[i] = stage[i];
}
int main() {
  const int W = 1920 * 3, H = 1080, N = 2;
  std::vector<float> h((size_t)W * H * N);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(i % 100003);
  float *d, *o;
  cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 144 * 40 * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  CUtensorMap tm;
  cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
  cuuint32_t box[3] = {144, 40, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d entry=%d\n", (int)r, (int)q);
  for (int x0 : {304, -4, -8, -16, 5756}) {
    cudaFuncSetAttribute(k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 + 144 * 40 * 4);
    k<false><<<1, 128, 128 + 144 * 40 * 4>>>(tm, o, x0, 7, 1, nullptr);
    cudaError_t e = cudaDeviceSynchronize();
    printf("x0=%d launch: %s\n", x0, cudaGetErrorString(e));
    if (e) return 1;  // the context is dead after an illegal instruction
    std::vector<float> got(144 * 40);
    cudaMemcpy(got.data(), o, got.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int yy = 0; yy < 40; ++yy)
      for (int xx = 0; xx < 144; ++xx) {
        int gx = x0 + xx, gy = 7 + yy;
        float ref = (gx >= 0 && gx < W) ? h[(size_t)W * H * 1 + (size_t)gy * W + gx] : 0.f;
        bad += got[yy * 144 + xx] != ref;
      }
    printf("x0=%d mismatches %d\n", x0, bad);
  }
  return 0;
}
