// dense.cu -- dense pieces of the path (dense.hpp): the general GEMM used for
// float64 (DFMA) and as the small-shape / non-tensor fallback, deterministic
// column sums, and counter-based generation of the reference's random inputs.
//
// float32 X.Theta-class GEMMs go to the tcgen05 kernel in gemm_tc.cu when the
// shape qualifies; float64 GEMMs run on the FP64 tensor cores (DMMA,
// k_gemm_dmma); the SIMT kernel handles small float32 shapes.
#include "common.cuh"
#include "internal.cuh"

namespace sgnn {

// ---------------------------------------------------------------------------
// SIMT GEMM: C[M x N] = op(A) op(B) (+bias), 64x64 tiles, 4x4 per thread,
// optional split-K into float64/partial workspace reduced in a fixed order.
// ---------------------------------------------------------------------------
constexpr int GBM = 64, GBN = 64, GBK = 16;

template <class T, class Acc>
__global__ void __launch_bounds__(256) k_gemm_simt(const T* __restrict__ A, const T* __restrict__ B,
                                                   int M, int N, int K, int lda, int ldb, bool ta,
                                                   bool tb, int kchunk, Acc* __restrict__ part,
                                                   T* __restrict__ C, const T* __restrict__ bias) {
  __shared__ T As[GBK][GBM + 4];
  __shared__ T Bs[GBK][GBN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
  const int k_begin = blockIdx.z * kchunk;
  const int k_end = min(K, k_begin + kchunk);
  Acc acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = Acc(0);

  for (int k0 = k_begin; k0 < k_end; k0 += GBK) {
    // A tile: GBM x GBK elements, 1024 / 256 = 4 per thread
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int idx = tid + t * 256;
      int mm, kk;
      if (ta) {  // A stored K x M: contiguous along m
        mm = idx % GBM;
        kk = idx / GBM;
      } else {
        kk = idx % GBK;
        mm = idx / GBK;
      }
      const int gm = m0 + mm, gk = k0 + kk;
      T v = T(0);
      if (gm < M && gk < k_end) v = ta ? A[(int64_t)gk * lda + gm] : A[(int64_t)gm * lda + gk];
      As[kk][mm] = v;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int idx = tid + t * 256;
      int nn, kk;
      if (tb) {  // B stored N x K: contiguous along k
        kk = idx % GBK;
        nn = idx / GBK;
      } else {
        nn = idx % GBN;
        kk = idx / GBN;
      }
      const int gn = n0 + nn, gk = k0 + kk;
      T v = T(0);
      if (gn < N && gk < k_end) v = tb ? B[(int64_t)gn * ldb + gk] : B[(int64_t)gk * ldb + gn];
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      Acc a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = (Acc)As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = (Acc)Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gm = m0 + ty + 16 * i, gn = n0 + tx + 16 * j;
      if (gm < M && gn < N) {
        if (part) {
          part[((int64_t)blockIdx.z * M + gm) * N + gn] = acc[i][j];
        } else {
          T v = (T)acc[i][j];
          if (bias) v = add_rn(v, bias[gn]);
          C[(int64_t)gm * N + gn] = v;
        }
      }
    }
}

// ---------------------------------------------------------------------------
// float64 GEMM on the FP64 tensor cores: the same 64 x 64 x 16 shared-memory
// tiles as k_gemm_simt, products by mma.sync.m8n8k4.f64 (DMMA).  8 warps as
// 2 (M) x 4 (N), each warp a 32 x 16 sub-tile = 4 x 2 DMMA 8x8 accumulators.
// Fragments (row.col): A 8x4 -- lane holds A[lane/4][lane%4]; B 4x8 -- lane
// holds B[lane%4][lane/4]; C 8x8 -- lane holds C[lane/4][2(lane%4) + {0,1}].
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) k_gemm_dmma(const double* __restrict__ A,
                                                   const double* __restrict__ B, int M, int N,
                                                   int K, int lda, int ldb, bool ta, bool tb,
                                                   int kchunk, double* __restrict__ part,
                                                   double* __restrict__ C,
                                                   const double* __restrict__ bias) {
  __shared__ double As[GBK][GBM + 1];
  __shared__ double Bs[GBK][GBN + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;  // warp sub-tile origin
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
  const int k_begin = blockIdx.z * kchunk;
  const int k_end = min(K, k_begin + kchunk);
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int k0 = k_begin; k0 < k_end; k0 += GBK) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int idx = tid + t * 256;
      int mm, kk;
      if (ta) {
        mm = idx % GBM;
        kk = idx / GBM;
      } else {
        kk = idx % GBK;
        mm = idx / GBK;
      }
      const int gm = m0 + mm, gk = k0 + kk;
      double v = 0.0;
      if (gm < M && gk < k_end) v = ta ? A[(int64_t)gk * lda + gm] : A[(int64_t)gm * lda + gk];
      As[kk][mm] = v;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int idx = tid + t * 256;
      int nn, kk;
      if (tb) {
        kk = idx % GBK;
        nn = idx / GBK;
      } else {
        nn = idx % GBN;
        kk = idx / GBN;
      }
      const int gn = n0 + nn, gk = k0 + kk;
      double v = 0.0;
      if (gn < N && gk < k_end) v = tb ? B[(int64_t)gn * ldb + gk] : B[(int64_t)gk * ldb + gn];
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < GBK; ks += 4) {
      const int kr = ks + (lane & 3);
      double a[4], b[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kr][wm + 8 * i + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = Bs[kr][wn + 8 * j + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gm = m0 + wm + 8 * i + (lane >> 2);
        const int gn = n0 + wn + 8 * j + 2 * (lane & 3) + h;
        if (gm < M && gn < N) {
          if (part) {
            part[((int64_t)blockIdx.z * M + gm) * N + gn] = acc[i][j][h];
          } else {
            double v = acc[i][j][h];
            if (bias) v = add_rn(v, bias[gn]);
            C[(int64_t)gm * N + gn] = v;
          }
        }
      }
}

template <class T, class Acc>
__global__ void k_splitk_reduce(int splits, int64_t MN, int N, const Acc* __restrict__ part,
                                T* __restrict__ C, const T* __restrict__ bias) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < MN;
       x += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += (double)part[(int64_t)z * MN + x];
    T v = (T)s;
    if (bias) v = add_rn(v, bias[x % N]);
    C[x] = v;
  }
}

template <class T>
void gemm_simt(sgnn_ctx ctx, const T* A, int32_t ra, int32_t ca, const T* B, int32_t rb,
               int32_t cb, bool ta, bool tb, T* C, const T* bias) {
  const int M = ta ? ca : ra, K = ta ? ra : ca, N = tb ? rb : cb;
  if (M == 0 || N == 0) return;
  const int tiles = (int)(ceil_div(M, GBM) * ceil_div(N, GBN));
  int splits = 1;
  const int target = 2 * ctx->num_sms;
  if (tiles < target && K > 2048) {
    splits = (int)std::min<int64_t>(ceil_div(target, tiles), ceil_div(K, 1024));
    if (splits > 256) splits = 256;
  }
  int kchunk = (int)ceil_div(ceil_div(K, splits), GBK) * GBK;
  if (K == 0) kchunk = GBK;
  splits = K == 0 ? 1 : (int)ceil_div(K, kchunk);
  dim3 grid((unsigned)ceil_div(N, GBN), (unsigned)ceil_div(M, GBM), (unsigned)splits);
  // float64 on the FP64 tensor cores (DMMA) unless disabled (dev switch)
  static const bool simt64 = getenv("SGNN_DMMA_OFF") != nullptr;
  const bool dmma = sizeof(T) == 8 && !simt64;
  if (splits == 1) {
    if constexpr (sizeof(T) == 8)
      if (dmma) {
        k_gemm_dmma<<<grid, 256, 0, ctx->stream>>>(A, B, M, N, K, ca, cb, ta, tb, kchunk,
                                                   nullptr, C, bias);
        launched(ctx);
        return;
      }
    k_gemm_simt<T, T><<<grid, 256, 0, ctx->stream>>>(A, B, M, N, K, ca, cb, ta, tb, kchunk,
                                                     (T*)nullptr, C, bias);
    launched(ctx);
  } else {
    // float32 partials of <= kchunk terms, combined in float64 in slice order
    using Acc = T;
    DevBuf part((size_t)splits * M * N * sizeof(Acc), ctx->stream);
    bool done = false;
    if constexpr (sizeof(T) == 8)
      if (dmma) {
        k_gemm_dmma<<<grid, 256, 0, ctx->stream>>>(A, B, M, N, K, ca, cb, ta, tb, kchunk,
                                                   part.as<double>(), C, bias);
        done = true;
      }
    if (!done)
      k_gemm_simt<T, Acc><<<grid, 256, 0, ctx->stream>>>(A, B, M, N, K, ca, cb, ta, tb, kchunk,
                                                         part.as<Acc>(), C, bias);
    launched(ctx);
    const int64_t MN = (int64_t)M * N;
    k_splitk_reduce<T, Acc><<<grid_for(ctx, MN, 256), 256, 0, ctx->stream>>>(
        splits, MN, N, part.as<Acc>(), C, bias);
    launched(ctx);
  }
}

template void gemm_simt<float>(sgnn_ctx, const float*, int32_t, int32_t, const float*, int32_t,
                               int32_t, bool, bool, float*, const float*);
template void gemm_simt<double>(sgnn_ctx, const double*, int32_t, int32_t, const double*,
                                int32_t, int32_t, bool, bool, double*, const double*);

// tcgen05 path (gemm_tc.cu); returns false when the shape is not supported
bool gemm_tc_f32(sgnn_ctx ctx, const float* A, int32_t ra, int32_t ca, const float* B,
                 int32_t rb, int32_t cb, bool ta, bool tb, float* C, const float* bias,
                 float* colsum_b, const float* att_src = nullptr, const float* att_dst = nullptr,
                 float* s_out = nullptr, float* d_out = nullptr, int heads = 0,
                 uint8_t* relu_out = nullptr, const uint8_t* mask_in = nullptr,
                 const float* elu_saved = nullptr);

// C = op(A) op(B) (+ bias) with ReLU fused into the epilogue: relu_out
// receives the mask (forward), or mask_in zeroes C where the mask is 0
// (backward).  false (nothing launched) when the shape does not allow it.
bool gemm_relu_f32(sgnn_ctx ctx, const float* A, int32_t ra, int32_t ca, const float* B,
                   int32_t rb, int32_t cb, bool ta, bool tb, float* C, const float* bias,
                   uint8_t* relu_out, const uint8_t* mask_in) {
  return gemm_tc_f32(ctx, A, ra, ca, B, rb, cb, ta, tb, C, bias, nullptr, nullptr, nullptr,
                     nullptr, nullptr, 0, relu_out, mask_in);
}

// C = op(A) op(B) with the ELU(1) backward fused into the epilogue (mask_in,
// saved = the activation's forward output); false when it does not apply
bool gemm_elu_bwd_f32(sgnn_ctx ctx, const float* A, int32_t ra, int32_t ca, const float* B,
                      int32_t rb, int32_t cb, bool ta, bool tb, float* C,
                      const uint8_t* mask_in, const float* saved) {
  return gemm_tc_f32(ctx, A, ra, ca, B, rb, cb, ta, tb, C, nullptr, nullptr, nullptr, nullptr,
                     nullptr, nullptr, 0, nullptr, mask_in, saved);
}

// M = X Theta with the GAT node scores s, d (n x h) computed in the GEMM
// epilogue; false when the fused form does not apply (nothing done)
bool gemm_scores_f32(sgnn_ctx ctx, const float* X, int32_t n, int32_t m, const float* theta,
                     int32_t hk, float* M, const float* a_src, const float* a_dst, int32_t h,
                     float* s, float* d) {
  return gemm_tc_f32(ctx, X, n, m, theta, m, hk, false, false, M, nullptr, nullptr, a_src, a_dst,
                     s, d, h);
}

template <>
void gemm<float>(sgnn_ctx ctx, const float* A, int32_t ra, int32_t ca, const float* B,
                 int32_t rb, int32_t cb, bool ta, bool tb, float* C, const float* bias) {
  const int32_t kk = ta ? ra : ca, kb = tb ? cb : rb;
  require(kk == kb, "gemm: inner dimensions do not match");
  if (gemm_tc_f32(ctx, A, ra, ca, B, rb, cb, ta, tb, C, bias, nullptr)) return;
  gemm_simt<float>(ctx, A, ra, ca, B, rb, cb, ta, tb, C, bias);
}
template <>
void gemm<double>(sgnn_ctx ctx, const double* A, int32_t ra, int32_t ca, const double* B,
                  int32_t rb, int32_t cb, bool ta, bool tb, double* C, const double* bias) {
  const int32_t kk = ta ? ra : ca, kb = tb ? cb : rb;
  require(kk == kb, "gemm: inner dimensions do not match");
  gemm_simt<double>(ctx, A, ra, ca, B, rb, cb, ta, tb, C, bias);
}

// ---------------------------------------------------------------------------
// column_sums (dense.hpp:272-282): blocks own contiguous row chunks and
// accumulate in float64 (coalesced row reads); the chunk partials are then
// combined by a fixed-shape tree -- deterministic, ~exact, HBM-bound.
// ---------------------------------------------------------------------------
template <class T>
__global__ void __launch_bounds__(256) k_colsum_partial(const T* __restrict__ X, int32_t rows,
                                                        int32_t cols, int32_t chunk,
                                                        double* __restrict__ part) {
  const int32_t r0 = blockIdx.x * chunk;
  const int32_t r1 = min(rows, r0 + chunk);
  for (int32_t j = threadIdx.x; j < cols; j += blockDim.x) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int32_t i = r0;
    for (; i + 3 < r1; i += 4) {
      s0 += (double)X[(int64_t)i * cols + j];
      s1 += (double)X[(int64_t)(i + 1) * cols + j];
      s2 += (double)X[(int64_t)(i + 2) * cols + j];
      s3 += (double)X[(int64_t)(i + 3) * cols + j];
    }
    for (; i < r1; ++i) s0 += (double)X[(int64_t)i * cols + j];
    part[(int64_t)blockIdx.x * cols + j] = (s0 + s1) + (s2 + s3);
  }
}

// out[j] = sum over nchunks partials; 8 warps split the chunk list, lanes own
// columns, smem combine in warp order.
template <class T>
__global__ void __launch_bounds__(256) k_colsum_final(int32_t nchunks, int32_t cols,
                                                      const double* __restrict__ part,
                                                      T* __restrict__ out) {
  __shared__ double sh[8][33];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t j = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (j < cols) {  // four independent chains: the partial list is read latency-free
    double s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int32_t c = w;
    for (; c + 24 < nchunks; c += 32) {
      s += part[(int64_t)c * cols + j];
      s1 += part[(int64_t)(c + 8) * cols + j];
      s2 += part[(int64_t)(c + 16) * cols + j];
      s3 += part[(int64_t)(c + 24) * cols + j];
    }
    for (; c < nchunks; c += 8) s += part[(int64_t)c * cols + j];
    s = (s + s1) + (s2 + s3);
  }
  sh[w][lane] = s;
  __syncthreads();
  if (w == 0 && j < cols) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += sh[k][lane];
    out[j] = (T)t;
  }
}

// out[j] = sum over nchunks partials, one block per column (narrow outputs:
// a 40-column d_bias took 29 us on two blocks of lane-per-column warps):
// threads stride the chunk list, then a fixed smem tree (deterministic)
template <class T>
__global__ void __launch_bounds__(256) k_colsum_final_col(int32_t nchunks, int32_t cols,
                                                          const double* __restrict__ part,
                                                          T* __restrict__ out) {
  __shared__ double sh[256];
  const int32_t j = blockIdx.x;
  double s = 0.0;
  for (int32_t c = threadIdx.x; c < nchunks; c += 256) s += part[(int64_t)c * cols + j];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[j] = (T)sh[0];
}

// float rows of cols % 4 == 0 (cols <= 1024): threads own float4 column
// vectors, 256 / (cols/4) row groups per block stride the chunk, float64
// accumulation, row groups combined in a fixed order in shared memory.
__global__ void __launch_bounds__(256) k_colsum_partial_v4(const float4* __restrict__ X,
                                                           int32_t rows, int32_t nv,
                                                           int32_t chunk,
                                                           double* __restrict__ part) {
  __shared__ double sh[256 * 4];
  const int groups = max(1, 256 / nv);
  const int tid = threadIdx.x, v = tid % nv, grp = tid / nv;
  const int32_t r0 = blockIdx.x * chunk, r1 = min(rows, r0 + chunk);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (grp < groups) {
    int32_t i = r0 + grp;
    for (; i + groups < r1; i += 2 * groups) {
      const float4 x = __ldg(X + (int64_t)i * nv + v);
      const float4 y = __ldg(X + (int64_t)(i + groups) * nv + v);
      a0 += (double)x.x + (double)y.x;
      a1 += (double)x.y + (double)y.y;
      a2 += (double)x.z + (double)y.z;
      a3 += (double)x.w + (double)y.w;
    }
    if (i < r1) {
      const float4 x = __ldg(X + (int64_t)i * nv + v);
      a0 += x.x;
      a1 += x.y;
      a2 += x.z;
      a3 += x.w;
    }
  }
  sh[tid * 4] = a0;
  sh[tid * 4 + 1] = a1;
  sh[tid * 4 + 2] = a2;
  sh[tid * 4 + 3] = a3;
  __syncthreads();
  if (grp == 0 && tid < nv) {
    for (int g = 1; g < groups; ++g) {
      a0 += sh[(g * nv + v) * 4];
      a1 += sh[(g * nv + v) * 4 + 1];
      a2 += sh[(g * nv + v) * 4 + 2];
      a3 += sh[(g * nv + v) * 4 + 3];
    }
    double* o = part + (int64_t)blockIdx.x * nv * 4 + v * 4;
    o[0] = a0;
    o[1] = a1;
    o[2] = a2;
    o[3] = a3;
  }
}

template <class T>
void column_sums(sgnn_ctx ctx, const T* X, int32_t rows, int32_t cols, T* out) {
  if (cols == 0) return;
  const int32_t target = ctx->num_sms * 4;
  int32_t chunk = rows > 0 ? (int32_t)ceil_div(rows, target) : 1;
  if (chunk < 16) chunk = 16;
  const int32_t nchunks = rows > 0 ? (int32_t)ceil_div(rows, chunk) : 1;
  DevBuf part((size_t)nchunks * cols * sizeof(double), ctx->stream);
  if (rows == 0) {
    SGNN_CUDA(cudaMemsetAsync(part.get(), 0, part.bytes(), ctx->stream));
  } else if (sizeof(T) == 4 && cols % 4 == 0 && cols <= 1024 &&
             reinterpret_cast<uintptr_t>(X) % 16 == 0) {
    k_colsum_partial_v4<<<nchunks, 256, 0, ctx->stream>>>(
        reinterpret_cast<const float4*>(X), rows, cols / 4, chunk, part.as<double>());
    launched(ctx);
  } else {
    k_colsum_partial<T><<<nchunks, 256, 0, ctx->stream>>>(X, rows, cols, chunk,
                                                          part.as<double>());
    launched(ctx);
  }
  if (cols <= 2 * ctx->num_sms)
    k_colsum_final_col<T><<<(unsigned)cols, 256, 0, ctx->stream>>>(nchunks, cols,
                                                                  part.as<double>(), out);
  else
    k_colsum_final<T><<<(unsigned)ceil_div(cols, 32), 256, 0, ctx->stream>>>(
        nchunks, cols, part.as<double>(), out);
  launched(ctx);
}
template void column_sums<float>(sgnn_ctx, const float*, int32_t, int32_t, float*);

// C = A^T B and colsum_b = 1^T B (dTheta and d_bias of one backward: B = dX'
// is read once when the tcgen05 kernel can fuse the column sums)
template <>
void gemm_tn_colsum<float>(sgnn_ctx ctx, const float* A, int32_t ra, int32_t ca, const float* B,
                           int32_t rb, int32_t cb, float* C, float* colsum_b) {
  require(ra == rb, "gemm: inner dimensions do not match");
  if (gemm_tc_f32(ctx, A, ra, ca, B, rb, cb, true, false, C, nullptr, colsum_b)) return;
  column_sums<float>(ctx, B, rb, cb, colsum_b);
  gemm<float>(ctx, A, ra, ca, B, rb, cb, true, false, C);
}
template <>
void gemm_tn_colsum<double>(sgnn_ctx ctx, const double* A, int32_t ra, int32_t ca,
                            const double* B, int32_t rb, int32_t cb, double* C,
                            double* colsum_b) {
  column_sums<double>(ctx, B, rb, cb, colsum_b);
  gemm<double>(ctx, A, ra, ca, B, rb, cb, true, false, C);
}
template void column_sums<double>(sgnn_ctx, const double*, int32_t, int32_t, double*);

// ---------------------------------------------------------------------------
// Counter-based form of the reference RNG (rng.hpp:13-42): after Rng(seed)
// the i-th next_u64() mixes seed + (i + 2) * golden, so every draw of
// DenseMatrix::random_uniform (dense.hpp:45-53) is computed independently on
// the device, bit-identical to the sequential host stream.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 2) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <class T>
__global__ void k_random_uniform(int64_t count, uint64_t seed, double lo, double hi, T* out) {
  const double span = __dsub_rn(hi, lo);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double u = __dmul_rn((double)(splitmix_at(seed, (uint64_t)i) >> 11), 0x1.0p-53);
    out[i] = (T)__dadd_rn(lo, __dmul_rn(span, u));
  }
}

template <class T>
void random_uniform(sgnn_ctx ctx, int64_t count, uint64_t seed, double lo, double hi, T* out) {
  if (count == 0) return;
  k_random_uniform<T><<<grid_for(ctx, count, 256), 256, 0, ctx->stream>>>(count, seed, lo, hi,
                                                                          out);
  launched(ctx);
}
template void random_uniform<float>(sgnn_ctx, int64_t, uint64_t, double, double, float*);
template void random_uniform<double>(sgnn_ctx, int64_t, uint64_t, double, double, double*);

}  // namespace sgnn

using namespace sgnn;

#define DISPATCH_T(dtype, ...)                 \
  do {                                         \
    if ((dtype) == SGNN_F32) {                 \
      using T = float;                         \
      __VA_ARGS__;                             \
    } else if ((dtype) == SGNN_F64) {          \
      using T = double;                        \
      __VA_ARGS__;                             \
    } else {                                   \
      throw invalid_argument("unknown dtype"); \
    }                                          \
  } while (0)

extern "C" {

int sgnn_gemm(sgnn_ctx ctx, int dtype, const void* A, int32_t ra, int32_t ca, const void* B,
              int32_t rb, int32_t cb, int ta, int tb, void* C) {
  SGNN_API_BEGIN
  DISPATCH_T(dtype, gemm<T>(ctx, static_cast<const T*>(A), ra, ca, static_cast<const T*>(B), rb,
                            cb, ta != 0, tb != 0, static_cast<T*>(C), nullptr));
  SGNN_API_END
}

int sgnn_gemm_ex(sgnn_ctx ctx, int dtype, const void* A, int32_t ra, int32_t ca, const void* B,
                 int32_t rb, int32_t cb, int ta, int tb, void* C, const void* bias,
                 void* colsum_b) {
  SGNN_API_BEGIN
  if (colsum_b) {
    require(ta != 0 && tb == 0 && bias == nullptr, "gemm: colsum_b needs C = A^T B, no bias");
    DISPATCH_T(dtype, gemm_tn_colsum<T>(ctx, static_cast<const T*>(A), ra, ca,
                                        static_cast<const T*>(B), rb, cb, static_cast<T*>(C),
                                        static_cast<T*>(colsum_b)));
  } else {
    DISPATCH_T(dtype, gemm<T>(ctx, static_cast<const T*>(A), ra, ca, static_cast<const T*>(B), rb,
                              cb, ta != 0, tb != 0, static_cast<T*>(C),
                              static_cast<const T*>(bias)));
  }
  SGNN_API_END
}

static void ok_rc(int rc) {
  if (rc == SGNN_OK) return;
  if (rc == SGNN_EINVAL) throw invalid_argument(sgnn_last_error());
  throw std::runtime_error(sgnn_last_error());
}

// gemm + activation (dense.hpp:197-268) with the activation fused into the
// tcgen05 epilogue where the shape allows it (float32), else two passes with
// identical results: act 0 = ReLU forward (C = relu(op(A) op(B) + bias),
// mask out), 1 = ReLU backward (C zeroed where mask == 0), 2 = ELU(1)
// backward (C scaled by saved + 1 where mask == 0; saved = the ELU output)
int sgnn_gemm_act(sgnn_ctx ctx, int dtype, const void* A, int32_t ra, int32_t ca, const void* B,
                  int32_t rb, int32_t cb, int ta, int tb, void* C, const void* bias, int act,
                  uint8_t* mask, const void* saved) {
  SGNN_API_BEGIN
  require(act >= 0 && act <= 2 && mask != nullptr, "gemm_act: unknown activation");
  require(act != 2 || saved != nullptr, "activation_backward: elu needs the saved output");
  const int64_t count = (int64_t)(ta ? ca : ra) * (tb ? rb : cb);
  bool fused = false;
  if (dtype == SGNN_F32 && !getenv("SGNN_NO_ACT_FUSION")) {
    const float* a = static_cast<const float*>(A);
    const float* b = static_cast<const float*>(B);
    float* c = static_cast<float*>(C);
    if (act == 0)
      fused = gemm_relu_f32(ctx, a, ra, ca, b, rb, cb, ta, tb, c,
                            static_cast<const float*>(bias), mask, nullptr);
    else if (act == 1 && !bias)
      fused = gemm_relu_f32(ctx, a, ra, ca, b, rb, cb, ta, tb, c, nullptr, nullptr, mask);
    else if (act == 2 && !bias)
      fused = gemm_elu_bwd_f32(ctx, a, ra, ca, b, rb, cb, ta, tb, c, mask,
                               static_cast<const float*>(saved));
  }
  if (!fused) {
    DISPATCH_T(dtype, gemm<T>(ctx, static_cast<const T*>(A), ra, ca, static_cast<const T*>(B), rb,
                              cb, ta != 0, tb != 0, static_cast<T*>(C),
                              static_cast<const T*>(bias)));
    if (act == 0) ok_rc(sgnn_activation(ctx, 0, dtype, C, count, C, mask));
    else ok_rc(sgnn_activation_backward(ctx, act == 1 ? 0 : 2, dtype, C, mask, saved, count, C));
  }
  SGNN_API_END
}

int sgnn_column_sums(sgnn_ctx ctx, int dtype, const void* X, int32_t rows, int32_t cols,
                     void* out) {
  SGNN_API_BEGIN
  DISPATCH_T(dtype, column_sums<T>(ctx, static_cast<const T*>(X), rows, cols,
                                   static_cast<T*>(out)));
  SGNN_API_END
}

int sgnn_random_uniform(sgnn_ctx ctx, int64_t rows, int64_t cols, uint64_t seed, double lo,
                        double hi, int dtype, void* out) {
  SGNN_API_BEGIN
  DISPATCH_T(dtype, random_uniform<T>(ctx, rows * cols, seed, lo, hi, static_cast<T*>(out)));
  SGNN_API_END
}

// gcn.hpp:54-62 -- bound = 1/sqrt(m) in double, theta from seed, bias Rng(seed+1)
int sgnn_gcn_params_init(sgnn_ctx ctx, int32_t m, int32_t k, uint64_t seed, int dtype,
                         void* theta, void* bias) {
  SGNN_API_BEGIN
  const double bound = 1.0 / std::sqrt((double)m);
  DISPATCH_T(dtype, {
    random_uniform<T>(ctx, (int64_t)m * k, seed, -bound, bound, static_cast<T*>(theta));
    random_uniform<T>(ctx, k, seed + 1, -bound, bound, static_cast<T*>(bias));
  });
  SGNN_API_END
}

// gat.hpp:36-52
int sgnn_gat_params_init(sgnn_ctx ctx, int32_t m, int32_t h, int32_t k, uint64_t seed,
                         int dtype, void* theta, void* a_src, void* a_dst, void* bias) {
  SGNN_API_BEGIN
  require(h >= 1, "GatParams: heads must be >= 1");
  const double bound = 1.0 / std::sqrt((double)m);
  const double abound = 1.0 / std::sqrt((double)k);
  DISPATCH_T(dtype, {
    random_uniform<T>(ctx, (int64_t)m * h * k, seed, -bound, bound, static_cast<T*>(theta));
    random_uniform<T>(ctx, (int64_t)h * k, seed + 1, -abound, abound, static_cast<T*>(a_src));
    random_uniform<T>(ctx, (int64_t)h * k, seed + 2, -abound, abound, static_cast<T*>(a_dst));
    random_uniform<T>(ctx, (int64_t)h * k, seed + 3, -bound, bound, static_cast<T*>(bias));
  });
  SGNN_API_END
}

}  // extern "C"
