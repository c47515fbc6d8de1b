// powerlaw.cu -- a Chung-Lu power-law graph generator on the device.  The
// reference only generates uniform graphs (graph.hpp:160-190, an ER proxy);
// BASELINE config 5 asks for a large power-law graph, so this adds one with
// the same output contract as synthetic_graph: undirected, both directions
// emitted, no self loops, no duplicates, canonical (src, dst) order.
//
//   weight of node i:  w_i = (i + 1)^(-1/(gamma - 1))      (degree ~ w, P(deg) ~ deg^-gamma)
//   pairs = round(avg_degree * n / 2); pair p draws two endpoints independently
//   with probability w_i / sum w (inverse CDF over the float64 prefix sums,
//   the uniforms are the counter-based splitmix64 draws 2p and 2p+1 of
//   `seed`), drops self pairs, keeps one copy of every {a, b}.
// Deterministic for (n, avg_degree, gamma, seed) on any device.
#include <cub/cub.cuh>

#include <cmath>

#include "common.cuh"
#include "internal.cuh"

namespace sgnn {
namespace {

__device__ __forceinline__ uint64_t mix_at(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 2) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_weights(int32_t n, double a, double* w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    w[i] = pow((double)(i + 1), -a);
}

// first index with cdf[idx] > u
__device__ __forceinline__ int32_t draw(const double* __restrict__ cdf, int32_t n, double u) {
  int32_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (cdf[mid] > u) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

__global__ void k_pairs(int64_t pairs, int32_t n, uint64_t seed, const double* __restrict__ cdf,
                        uint64_t* __restrict__ keys) {
  const double total = cdf[n - 1];
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < pairs;
       p += (int64_t)gridDim.x * blockDim.x) {
    const double u1 = (double)(mix_at(seed, 2 * (uint64_t)p) >> 11) * 0x1.0p-53 * total;
    const double u2 = (double)(mix_at(seed, 2 * (uint64_t)p + 1) >> 11) * 0x1.0p-53 * total;
    const int32_t a = draw(cdf, n, u1), b = draw(cdf, n, u2);
    keys[p] = a == b ? ~0ull
                     : ((uint64_t)(uint32_t)min(a, b) << 32) | (uint64_t)(uint32_t)max(a, b);
  }
}

// both directions of every unique undirected pair (the sentinel sorts last)
__global__ void k_directed(int64_t m, const uint64_t* __restrict__ uniq, uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = uniq[i];
    out[2 * i] = k;
    out[2 * i + 1] = (k << 32) | (k >> 32);
  }
}

__global__ void k_split_keys(int64_t m, const uint64_t* __restrict__ k, int32_t* __restrict__ src,
                             int32_t* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    src[i] = (int32_t)(k[i] >> 32);
    dst[i] = (int32_t)(k[i] & 0xffffffffu);
  }
}

}  // namespace
}  // namespace sgnn

using namespace sgnn;

extern "C" {

int64_t sgnn_powerlaw_graph_capacity(int32_t n, double avg_degree) {
  if (n <= 1 || !(avg_degree > 0)) return 0;
  return 2 * (int64_t)std::llround(avg_degree * n / 2.0);
}

int sgnn_powerlaw_graph(sgnn_ctx ctx, int32_t n, double avg_degree, double exponent,
                        uint64_t seed, int32_t* src, int32_t* dst, int64_t* count) {
  SGNN_API_BEGIN
  require(ctx && count, "powerlaw_graph: null argument");
  require(n >= 0 && avg_degree >= 0, "powerlaw_graph: n and avg_degree must be non-negative");
  require(exponent > 1.0, "powerlaw_graph: exponent must be > 1");
  *count = 0;
  const int64_t pairs = sgnn_powerlaw_graph_capacity(n, avg_degree) / 2;
  if (pairs == 0) return SGNN_OK;
  // 2 * pairs directed edges go through CUB with an int item count
  require(pairs < ((int64_t)1 << 30), "powerlaw_graph: too many edges");
  cudaStream_t st = ctx->stream;
  DevBuf w((size_t)n * 8, st), cdf((size_t)n * 8, st);
  k_weights<<<grid_for(ctx, n, 256), 256, 0, st>>>(n, 1.0 / (exponent - 1.0), w.as<double>());
  launched(ctx);
  size_t tb = 0;
  SGNN_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, w.as<double>(), cdf.as<double>(), n, st));
  {
    DevBuf t(tb, st);
    SGNN_CUDA(cub::DeviceScan::InclusiveSum(t.get(), tb, w.as<double>(), cdf.as<double>(), n, st));
  }
  DevBuf keys((size_t)pairs * 8, st), sorted((size_t)pairs * 8, st);
  k_pairs<<<grid_for(ctx, pairs, 256), 256, 0, st>>>(pairs, n, seed, cdf.as<double>(),
                                                     keys.as<uint64_t>());
  launched(ctx);
  tb = 0;
  SGNN_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.as<uint64_t>(),
                                           sorted.as<uint64_t>(), (int)pairs, 0, 64, st));
  {
    DevBuf t(tb, st);
    SGNN_CUDA(cub::DeviceRadixSort::SortKeys(t.get(), tb, keys.as<uint64_t>(),
                                             sorted.as<uint64_t>(), (int)pairs, 0, 64, st));
  }
  DevBuf nu(8, st);
  tb = 0;
  SGNN_CUDA(cub::DeviceSelect::Unique(nullptr, tb, sorted.as<uint64_t>(), keys.as<uint64_t>(),
                                      nu.as<int64_t>(), (int)pairs, st));
  {
    DevBuf t(tb, st);
    SGNN_CUDA(cub::DeviceSelect::Unique(t.get(), tb, sorted.as<uint64_t>(), keys.as<uint64_t>(),
                                        nu.as<int64_t>(), (int)pairs, st));
  }
  int64_t m = 0;
  SGNN_CUDA(cudaMemcpyAsync(&m, nu.get(), 8, cudaMemcpyDeviceToHost, st));
  SGNN_CUDA(cudaStreamSynchronize(st));
  uint64_t last = 0;  // drop the self-pair sentinel (sorts last) if present
  if (m > 0) {
    SGNN_CUDA(cudaMemcpyAsync(&last, keys.as<uint64_t>() + m - 1, 8, cudaMemcpyDeviceToHost, st));
    SGNN_CUDA(cudaStreamSynchronize(st));
    if (last == ~0ull) --m;
  }
  const int64_t e = 2 * m;
  if (e == 0) return SGNN_OK;
  DevBuf dir((size_t)e * 8, st), dsort((size_t)e * 8, st);
  k_directed<<<grid_for(ctx, m, 256), 256, 0, st>>>(m, keys.as<uint64_t>(), dir.as<uint64_t>());
  launched(ctx);
  tb = 0;
  SGNN_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, dir.as<uint64_t>(), dsort.as<uint64_t>(),
                                           (int)e, 0, 64, st));
  {
    DevBuf t(tb, st);
    SGNN_CUDA(cub::DeviceRadixSort::SortKeys(t.get(), tb, dir.as<uint64_t>(),
                                             dsort.as<uint64_t>(), (int)e, 0, 64, st));
  }
  k_split_keys<<<grid_for(ctx, e, 256), 256, 0, st>>>(e, dsort.as<uint64_t>(), src, dst);
  launched(ctx);
  *count = e;
  SGNN_API_END
}

}  // extern "C"
