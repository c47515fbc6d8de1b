// Dev probe: achievable throughput of random 512-byte row gathers (the SpMM
// access pattern) on this GPU, independent of the SpMM kernel.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

template <int U>
__global__ void gather(const float4* __restrict__ X, const int* __restrict__ idx, int nidx,
                       int per_warp, float4* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long i0 = warp * per_warp;
  if (i0 >= nidx) return;
  const long i1 = min((long)nidx, i0 + per_warp);
  float4 acc = make_float4(0, 0, 0, 0);
  for (long i = i0; i < i1; i += U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long j = i + u;
      const int r = j < i1 ? __ldg(idx + j) : 0;
      v[u] = __ldg(X + (long)r * 32 + lane);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
  }
  if (acc.x == 12345.f) out[warp] = acc;
}

int main() {
  const int n = 169343, nidx = 1335587;
  float4* X; int* idx; float4* out; char* flush;
  cudaMalloc(&X, (size_t)n * 512); cudaMemset(X, 0, (size_t)n * 512);
  cudaMalloc(&idx, nidx * 4); cudaMalloc(&out, 1 << 24); cudaMalloc(&flush, 256 << 20);
  std::vector<int> h(nidx);
  srand(1);
  for (int i = 0; i < nidx; ++i) h[i] = rand() % n;
  cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int U : {1, 2, 4, 8, 16}) {
    for (int pw : {8, 32, 128}) {
      const long warps = (nidx + pw - 1) / pw;
      const int grid = (int)((warps * 32 + 255) / 256);
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(flush, rep, 256 << 20);
        cudaEventRecord(a);
        switch (U) {
          case 1: gather<1><<<grid, 256>>>(X, idx, nidx, pw, out); break;
          case 2: gather<2><<<grid, 256>>>(X, idx, nidx, pw, out); break;
          case 4: gather<4><<<grid, 256>>>(X, idx, nidx, pw, out); break;
          case 8: gather<8><<<grid, 256>>>(X, idx, nidx, pw, out); break;
          case 16: gather<16><<<grid, 256>>>(X, idx, nidx, pw, out); break;
        }
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
      }
      printf("U=%2d per_warp=%3d: %.1f us  gather %.0f GB/s\n", U, pw, best * 1e3,
             (double)nidx * 512 / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}
