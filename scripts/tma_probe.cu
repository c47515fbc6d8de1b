// Dev probe: TMA streaming rate of the GEMM's A operand pattern (128 x 32
// fp32 boxes, SWIZZLE_128B, 4-32 stage ring per CTA, consumer releases at
// once), independent of the GEMM kernel.  Reads X (n x 128 fp32) `passes` times.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(su(b)), "r"(ph) : "memory");
  } while (!done);
}

template <int S>
__global__ void __launch_bounds__(64, 1) k_stream(const __grid_constant__ CUtensorMap tm, int mtiles, int ksteps, int passes) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* ring = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[S], empty[S];
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int total = mtiles * passes;
  if (threadIdx.x == 0) {  // producer
    int it = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      const int m0 = (t % mtiles) * 128;
      for (int ks = 0; ks < ksteps; ++ks, ++it) {
        const int s = it % S;
        wait(&empty[s], ((it / S) & 1) ^ 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(16384) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     ::"r"(su(ring + s * 16384)), "l"((uint64_t)&tm), "r"(su(&full[s])), "r"(ks * 32), "r"(m0) : "memory");
      }
    }
  } else if (threadIdx.x == 32) {  // consumer
    int it = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x)
      for (int ks = 0; ks < ksteps; ++ks, ++it) {
        const int s = it % S;
        wait(&full[s], (it / S) & 1);
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
      }
  }
}

int main() {
  const int n = 169343, K = 128;
  float* X; cudaMalloc(&X, (size_t)n * K * 4); cudaMemset(X, 0, (size_t)n * K * 4);
  char* flush; cudaMalloc(&flush, 256 << 20);
  cudaDriverEntryPointQueryResult q; void* fp = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)n}; cuuint64_t str[1] = {(cuuint64_t)K * 4};
  cuuint32_t box[2] = {32, 128}; cuuint32_t es[2] = {1, 1};
  for (int prom = 0; prom < 2; ++prom) {
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, prom ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int mtiles = (n + 127) / 128;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](auto kern, int S, int passes) {
      const int smem = S * 16384 + 1024;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      float best = 1e9;
      for (int r = 0; r < 5; ++r) {
        cudaMemset(flush, r, 256 << 20);
        cudaEventRecord(a);
        kern<<<148, 64, smem>>>(tm, mtiles, K / 32, passes);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (r && ms < best) best = ms;
      }
      printf("prom%d S=%2d passes=%d: %.1f us  %.0f GB/s smem-fill\n", prom * 256, S, passes, best * 1e3,
             (double)n * K * 4 * passes / (best * 1e-3) / 1e9);
    };
    run(k_stream<4>, 4, 1); run(k_stream<4>, 4, 2); run(k_stream<8>, 8, 2); run(k_stream<12>, 12, 2);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
