// spmm.cu -- CSR SpMM for sm_100a (north-star subsystem 2, kernels.hpp:33-89).
//
// Mapping: a group of LPR lanes (1..32, power of two) owns one output row;
// each lane owns R 16-byte column vectors (float4 / double2) of that row, so a
// row's dense operand rows are fetched as fully coalesced 128-bit loads.  The
// group loads up to LPR (col, val) pairs of the row with one coalesced load,
// then broadcasts them with sub-warp shuffles.  Loads of U edges are issued
// before any of them is consumed (memory-level parallelism).
//
// Parity: each output element is accumulated by one thread in stored edge
// order with an unfused multiply then add (madd), which is exactly the
// reference's `crow[c] += v * brow[c]` (kernels.hpp:47-51): results are
// bit-identical to the reference CPU SpMM in float32 and float64.
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "internal.cuh"

namespace sgnn {

#ifndef SPMM_MINB
#define SPMM_MINB 4
#endif

template <class T, int W>
struct VecT;
template <class T>
struct VecT<T, 1> {
  using type = T;
};
template <>
struct VecT<float, 4> {
  using type = float4;
};
template <>
struct VecT<double, 2> {
  using type = double2;
};

template <class V>
__device__ __forceinline__ V ldg_v(const V* p) {
  return __ldg(p);
}

// Output rows are written once and never re-read by this kernel: stream them
// (evict-first) so the gathered dense operand keeps its L2 residency.
template <class V>
__device__ __forceinline__ void st_out(V* p, const V& v) {
  __stcs(p, v);
}

template <class T, int W>
struct Acc {
  T v[W];
};

template <class T, int W, class V>
__device__ __forceinline__ void acc_add(T* a, T s, const V& b);
template <>
__device__ __forceinline__ void acc_add<float, 4, float4>(float* a, float s, const float4& b) {
  a[0] = madd(a[0], s, b.x);
  a[1] = madd(a[1], s, b.y);
  a[2] = madd(a[2], s, b.z);
  a[3] = madd(a[3], s, b.w);
}
template <>
__device__ __forceinline__ void acc_add<double, 2, double2>(double* a, double s,
                                                            const double2& b) {
  a[0] = madd(a[0], s, b.x);
  a[1] = madd(a[1], s, b.y);
}
template <>
__device__ __forceinline__ void acc_add<float, 1, float>(float* a, float s, const float& b) {
  a[0] = madd(a[0], s, b);
}
template <>
__device__ __forceinline__ void acc_add<double, 1, double>(double* a, double s,
                                                           const double& b) {
  a[0] = madd(a[0], s, b);
}

template <class T, int W, class V>
__device__ __forceinline__ V pack(const T* a);
template <>
__device__ __forceinline__ float4 pack<float, 4, float4>(const float* a) {
  return make_float4(a[0], a[1], a[2], a[3]);
}
template <>
__device__ __forceinline__ double2 pack<double, 2, double2>(const double* a) {
  return make_double2(a[0], a[1]);
}
template <>
__device__ __forceinline__ float pack<float, 1, float>(const float* a) {
  return a[0];
}
template <>
__device__ __forceinline__ double pack<double, 1, double>(const double* a) {
  return a[0];
}

// LPR lanes per row, R vectors per lane, W scalars per vector, U edges in flight
template <class T, int LPR, int R, int W, int U>
__global__ void __launch_bounds__(256, (R == 1 && sizeof(T) == 4) ? SPMM_MINB : 1) k_spmm_csr(int32_t n_rows, const int32_t* __restrict__ rowptr,
                                                  const int32_t* __restrict__ cols,
                                                  const T* __restrict__ vals,
                                                  const T* __restrict__ B, int32_t f,
                                                  T* __restrict__ C, const T* __restrict__ bias,
                                                  int32_t ld, int32_t longest = 0x7fffffff,
                                                  const int32_t* __restrict__ seg_beg = nullptr) {
  // seg_beg != nullptr: rows are hub-row segments [seg_beg[r], rowptr[r]) (rowptr
  // then carries the segment ends) written to partial rows, see LongRows
  using V = typename VecT<T, W>::type;
  constexpr int RPW = 32 / LPR;  // rows per warp
  const int lane = threadIdx.x & 31;
  const int g = lane % LPR;      // lane within group
  const int grp = lane / LPR;
  const unsigned gmask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (grp * LPR));
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int fv = f / W;    // vectors in this column window
  const int ldv = ld / W;  // row stride in vectors
  const V* Bv = reinterpret_cast<const V*>(B);
  V* Cv = reinterpret_cast<V*>(C);
  const V* biasv = reinterpret_cast<const V*>(bias);

  for (int64_t row0 = warp * RPW; row0 < n_rows; row0 += nwarps * RPW) {
    const int64_t row = row0 + grp;
    bool active = row < n_rows;
    int32_t beg = 0, end = 0;
    if (active) {
      beg = seg_beg ? seg_beg[row] : rowptr[row];
      end = seg_beg ? rowptr[row] : rowptr[row + 1];
      if (end - beg > longest) active = false, end = beg;  // hub row: segments + combine
    }
    // column blocks of LPR*R vectors (one pass unless f > 32*R*W)
    for (int cb = 0; cb < fv; cb += LPR * R) {
      T acc[R][W];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int w = 0; w < W; ++w) acc[r][w] = T(0);
      for (int32_t base = beg; base < end; base += LPR) {
        const int32_t e = base + g;
        int32_t my_col = 0;
        T my_val = T(0);
        if (e < end) {
          my_col = __ldg(cols + e);
          my_val = __ldg(vals + e);
        }
        const int cnt = min(LPR, end - base);
        for (int j0 = 0; j0 < cnt; j0 += U) {
          V bv[U][R];
          T sv[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int j = j0 + u;
            int32_t c = 0;
            T s = T(0);
            if (LPR == 1) {
              c = my_col;
              s = my_val;
            } else {
              c = __shfl_sync(gmask, my_col, j & (LPR - 1), LPR);
              s = __shfl_sync(gmask, my_val, j & (LPR - 1), LPR);
            }
            sv[u] = s;
            const V* brow = Bv + (int64_t)c * ldv;
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const int cv = cb + r * LPR + g;
              if (j < cnt && cv < fv) bv[u][r] = ldg_v(brow + cv);
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (j0 + u < cnt) {
#pragma unroll
              for (int r = 0; r < R; ++r) acc_add<T, W, V>(acc[r], sv[u], bv[u][r]);
            }
          }
        }
      }
      if (active) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int cv = cb + r * LPR + g;
          if (cv < fv) {
            if (bias) {
              T b[W];
              const V bb = biasv[cv];
              const T* bp = reinterpret_cast<const T*>(&bb);
#pragma unroll
              for (int w = 0; w < W; ++w) b[w] = add_rn(acc[r][w], bp[w]);
              st_out(Cv + row * ldv + cv, pack<T, W, V>(b));
            } else {
              st_out(Cv + row * ldv + cv, pack<T, W, V>(acc[r]));
            }
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Lean fp32 row kernel (f <= 32*4*R): one warp per output row, no grid-stride
// loop, broadcast loads of (col, val) instead of shuffles, 32-bit vector
// offsets -- small enough for 64 resident warps/SM, which is what the random
// 512-byte row gathers need (the hardware gathers at ~12 TB/s when enough
// independent warps are in flight).  Same per-element edge order, unfused.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float4 ldB(const float4* p) { return __ldg(p); }

// Rows longer than `longest` edges are skipped (a LongRows plan covers them).
// SEG: the warp owns segment `row` of a long row instead: edges
// [seg_beg[row], rowptr[row]) -- in SEG mode `rowptr` carries the segment
// ends -- written without bias to its own partial row of C (combined in
// segment order by k_spmm_combine).
template <int R, int U, bool SEG = false>
__global__ void __launch_bounds__(256, (R == 1 ? (U <= 2 ? 8 : 6) : (U <= 2 ? 6 : 4)))
    k_spmm_lean(int32_t n_rows, const int32_t* __restrict__ rowptr,
                const int32_t* __restrict__ cols, const float* __restrict__ vals,
                const float4* __restrict__ B, int32_t fv, float4* __restrict__ C,
                const float4* __restrict__ bias, int32_t ldv, int32_t longest = 0x7fffffff,
                const int32_t* __restrict__ seg_beg = nullptr, int32_t ldc = 0) {
  // ldv: row stride of B (vectors); ldc: row stride of C (0: same as B)
  const int lane = threadIdx.x & 31;
  const int32_t row = (int32_t)((blockIdx.x * 256u + threadIdx.x) >> 5);
  if (row >= n_rows) return;
  int32_t beg, end;
  if (SEG) {
    beg = __ldg(seg_beg + row);
    end = __ldg(rowptr + row);
  } else {
    beg = __ldg(rowptr + row);
    end = __ldg(rowptr + row + 1);
    if (end - beg > longest) return;
  }
  float4 acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
  const bool ok1 = R < 2 || (32 + lane) < fv;
  const bool ok0 = lane < fv;
  int32_t e = beg;
  for (; e + U <= end; e += U) {
    int32_t c[U];
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = __ldg(cols + e + u);
      v[u] = __ldg(vals + e + u);
    }
    float4 b[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float4* src = B + (uint32_t)c[u] * (uint32_t)ldv + lane;
      if (ok0) b[u][0] = ldB(src);
      if (R > 1 && ok1) b[u][R - 1] = ldB(src + 32);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        acc[r].x = madd(acc[r].x, v[u], b[u][r].x);
        acc[r].y = madd(acc[r].y, v[u], b[u][r].y);
        acc[r].z = madd(acc[r].z, v[u], b[u][r].z);
        acc[r].w = madd(acc[r].w, v[u], b[u][r].w);
      }
  }
  for (; e < end; ++e) {
    const int32_t c = __ldg(cols + e);
    const float v = __ldg(vals + e);
    const float4* src = B + (uint32_t)c * (uint32_t)ldv + lane;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if ((r == 0 && ok0) || (r == 1 && ok1)) {
        const float4 b = __ldg(src + r * 32);
        acc[r].x = madd(acc[r].x, v, b.x);
        acc[r].y = madd(acc[r].y, v, b.y);
        acc[r].z = madd(acc[r].z, v, b.z);
        acc[r].w = madd(acc[r].w, v, b.w);
      }
    }
  }
  float4* dst = C + (uint32_t)row * (uint32_t)(ldc ? ldc : ldv) + lane;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if ((r == 0 && ok0) || (r == 1 && ok1)) {
      float4 o = acc[r];
      if (!SEG && bias) {
        const float4 bb = __ldg(bias + r * 32 + lane);
        o.x = __fadd_rn(o.x, bb.x);
        o.y = __fadd_rn(o.y, bb.y);
        o.z = __fadd_rn(o.z, bb.z);
        o.w = __fadd_rn(o.w, bb.w);
      }
      __stcs(dst + r * 32, o);
    }
  }
}

// Long rows: sum the segment partials of each long row in segment order
// (+ bias) -- warp per long row, lanes over 16-byte vectors.
__global__ void __launch_bounds__(256) k_spmm_combine(int32_t nlong,
                                                      const int32_t* __restrict__ long_row,
                                                      const int32_t* __restrict__ long_first,
                                                      const float4* __restrict__ part,
                                                      int32_t fv, float4* __restrict__ C,
                                                      const float4* __restrict__ bias,
                                                      int32_t ldv) {
  const int lane = threadIdx.x & 31;
  const int32_t j = (int32_t)((blockIdx.x * 256u + threadIdx.x) >> 5);
  if (j >= nlong) return;
  const int32_t row = __ldg(long_row + j), s0 = __ldg(long_first + j),
                s1 = __ldg(long_first + j + 1);
  for (int v = lane; v < fv; v += 32) {
    float4 a = __ldg(part + (int64_t)s0 * fv + v);
    for (int32_t s = s0 + 1; s < s1; ++s) {
      const float4 b = __ldg(part + (int64_t)s * fv + v);
      a.x = __fadd_rn(a.x, b.x);
      a.y = __fadd_rn(a.y, b.y);
      a.z = __fadd_rn(a.z, b.z);
      a.w = __fadd_rn(a.w, b.w);
    }
    if (bias) {
      const float4 bb = __ldg(bias + v);
      a.x = __fadd_rn(a.x, bb.x);
      a.y = __fadd_rn(a.y, bb.y);
      a.z = __fadd_rn(a.z, bb.z);
      a.w = __fadd_rn(a.w, bb.w);
    }
    C[(int64_t)row * ldv + v] = a;
  }
}

void spmm_combine(sgnn_ctx ctx, const LongRows& lr, const float* part, int32_t f, float* C,
                  const float* bias, int32_t ld) {
  if (lr.nlong == 0) return;
  k_spmm_combine<<<(unsigned)ceil_div(lr.nlong, 8), 256, 0, ctx->stream>>>(
      lr.nlong, lr.long_row.as<int32_t>(), lr.long_first.as<int32_t>(),
      reinterpret_cast<const float4*>(part), f / 4, reinterpret_cast<float4*>(C),
      reinterpret_cast<const float4*>(bias), ld / 4);
  launched(ctx);
}

__global__ void k_long_count(int32_t n, const int32_t* __restrict__ rowptr, int32_t seglen,
                             int32_t* __restrict__ segs, int32_t* __restrict__ islong) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t deg = i < n ? rowptr[i + 1] - rowptr[i] : 0;
    segs[i] = deg > seglen ? (deg + seglen - 1) / seglen : 0;
    islong[i] = deg > seglen ? 1 : 0;
  }
}

__global__ void k_long_fill(int32_t n, const int32_t* __restrict__ rowptr, int32_t seglen,
                            const int32_t* __restrict__ segoff, const int32_t* __restrict__ longoff,
                            int32_t* __restrict__ seg_beg, int32_t* __restrict__ seg_end,
                            int32_t* __restrict__ seg_row, int32_t* __restrict__ long_row,
                            int32_t* __restrict__ long_first) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t beg = rowptr[i], end = rowptr[i + 1];
    if (end - beg <= seglen) continue;
    const int32_t j = longoff[i], s0 = segoff[i];
    long_row[j] = (int32_t)i;
    long_first[j] = s0;
    int32_t s = s0;
    for (int32_t e = beg; e < end; e += seglen, ++s) {
      seg_beg[s] = e;
      seg_end[s] = min(e + seglen, end);
      seg_row[s] = (int32_t)i;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) long_first[longoff[n]] = segoff[n];  // sentinel
}

LongRows& long_rows(sgnn_ctx ctx, LongRows& plan, int32_t n, const int32_t* rowptr) {
  if (plan.built && plan.rowptr == rowptr) return plan;
  cudaStream_t st = ctx->stream;
  plan = LongRows();
  plan.rowptr = rowptr;
  plan.built = true;
  if (n <= 0) return plan;
  DevBuf segs((size_t)(n + 1) * 4, st), isl((size_t)(n + 1) * 4, st),
      segoff((size_t)(n + 1) * 4, st), longoff((size_t)(n + 1) * 4, st);
  k_long_count<<<grid_for(ctx, n + 1, 256), 256, 0, st>>>(n, rowptr, kLongRow, segs.as<int32_t>(),
                                                          isl.as<int32_t>());
  launched(ctx);
  size_t tb = 0;
  SGNN_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, segs.as<int32_t>(), segoff.as<int32_t>(),
                                          n + 1, st));
  {
    DevBuf t(tb, st);
    SGNN_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tb, segs.as<int32_t>(),
                                            segoff.as<int32_t>(), n + 1, st));
    SGNN_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tb, isl.as<int32_t>(),
                                            longoff.as<int32_t>(), n + 1, st));
  }
  int32_t cnt[2] = {0, 0};
  SGNN_CUDA(cudaMemcpyAsync(&cnt[0], segoff.as<int32_t>() + n, 4, cudaMemcpyDeviceToHost, st));
  SGNN_CUDA(cudaMemcpyAsync(&cnt[1], longoff.as<int32_t>() + n, 4, cudaMemcpyDeviceToHost, st));
  SGNN_CUDA(cudaStreamSynchronize(st));  // once per operator
  plan.nseg = cnt[0];
  plan.nlong = cnt[1];
  if (plan.nlong == 0) return plan;
  plan.seg_beg = DevBuf((size_t)plan.nseg * 4, st);
  plan.seg_end = DevBuf((size_t)plan.nseg * 4, st);
  plan.seg_row = DevBuf((size_t)plan.nseg * 4, st);
  plan.long_row = DevBuf((size_t)plan.nlong * 4, st);
  plan.long_first = DevBuf((size_t)(plan.nlong + 1) * 4, st);
  k_long_fill<<<grid_for(ctx, n, 256), 256, 0, st>>>(n, rowptr, kLongRow, segoff.as<int32_t>(),
                                                     longoff.as<int32_t>(), plan.seg_beg.as<int32_t>(),
                                                     plan.seg_end.as<int32_t>(),
                                                     plan.seg_row.as<int32_t>(),
                                                     plan.long_row.as<int32_t>(),
                                                     plan.long_first.as<int32_t>());
  launched(ctx);
  return plan;
}

template <int R>
static void launch_lean(sgnn_ctx ctx, int U, int32_t n_rows, const int32_t* rowptr,
                        const int32_t* cols, const float* vals, const float* B, int32_t f,
                        float* C, const float* bias, int32_t ld, const LongRows* lr = nullptr) {
  const int grid = (int)ceil_div(n_rows, 8);
  const float4* Bv = reinterpret_cast<const float4*>(B);
  float4* Cv = reinterpret_cast<float4*>(C);
  const float4* bv = reinterpret_cast<const float4*>(bias);
  const bool split = lr && lr->nlong > 0;
  const int32_t longest = split ? kLongRow : 0x7fffffff;
  if (U >= 4)
    k_spmm_lean<R, 4><<<grid, 256, 0, ctx->stream>>>(n_rows, rowptr, cols, vals, Bv, f / 4, Cv, bv, ld / 4, longest);
  else if (U >= 2)
    k_spmm_lean<R, 2><<<grid, 256, 0, ctx->stream>>>(n_rows, rowptr, cols, vals, Bv, f / 4, Cv, bv, ld / 4, longest);
  else
    k_spmm_lean<R, 1><<<grid, 256, 0, ctx->stream>>>(n_rows, rowptr, cols, vals, Bv, f / 4, Cv, bv, ld / 4, longest);
  launched(ctx);
  if (!split) return;
  // long rows: kLongRow-edge segments on their own warps, then an in-order combine
  DevBuf part((size_t)lr->nseg * f * 4, ctx->stream);
  float4* pv = part.as<float4>();
  k_spmm_lean<R, 2, true><<<(unsigned)ceil_div(lr->nseg, 8), 256, 0, ctx->stream>>>(
      lr->nseg, lr->seg_end.as<int32_t>(), cols, vals, Bv, f / 4, pv, nullptr, ld / 4, 0x7fffffff,
      lr->seg_beg.as<int32_t>(), f / 4);
  launched(ctx);
  k_spmm_combine<<<(unsigned)ceil_div(lr->nlong, 8), 256, 0, ctx->stream>>>(
      lr->nlong, lr->long_row.as<int32_t>(), lr->long_first.as<int32_t>(), pv, f / 4, Cv, bv,
      ld / 4);
  launched(ctx);
}

template <class T, int W, int LPR, int U>
static void launch_lpr(sgnn_ctx ctx, int R, int32_t n_rows, const int32_t* rowptr,
                       const int32_t* cols, const T* vals, const T* B, int32_t f, T* C,
                       const T* bias, int32_t ld, int32_t longest, const int32_t* seg_beg) {
  const int rpw = 32 / LPR;
  const int64_t warps = ceil_div(n_rows, rpw);
  const int block = 256;
  int64_t grid = ceil_div(warps * 32, block);
  const int64_t cap = (int64_t)ctx->num_sms * 64;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  switch (R) {
#define CASE(RR)                                                                         \
  case RR:                                                                               \
    k_spmm_csr<T, LPR, RR, W, U><<<(int)grid, block, 0, ctx->stream>>>(n_rows, rowptr, cols, \
                                                                      vals, B, f, C, bias, ld,  \
                                                                      longest, seg_beg);        \
    break;
    CASE(1) CASE(2) CASE(4) CASE(8)
#undef CASE
    default: throw invalid_argument("spmm: bad register blocking");
  }
  launched(ctx);
}

template <class T>
__global__ void __launch_bounds__(256) k_spmm_combine_t(int32_t nlong,
                                                        const int32_t* __restrict__ long_row,
                                                        const int32_t* __restrict__ long_first,
                                                        const T* __restrict__ part, int32_t f,
                                                        T* __restrict__ C,
                                                        const T* __restrict__ bias, int32_t ld) {
  const int lane = threadIdx.x & 31;
  const int32_t j = (int32_t)((blockIdx.x * 256u + threadIdx.x) >> 5);
  if (j >= nlong) return;
  const int32_t row = long_row[j], s0 = long_first[j], s1 = long_first[j + 1];
  for (int32_t c = lane; c < f; c += 32) {
    T a = part[(int64_t)s0 * f + c];
    for (int32_t sg = s0 + 1; sg < s1; ++sg) a = add_rn(a, part[(int64_t)sg * f + c]);
    if (bias) a = add_rn(a, bias[c]);
    C[(int64_t)row * ld + c] = a;
  }
}

template <class T, int W>
static void launch_w1(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr, const int32_t* cols,
                      const T* vals, const T* B, int32_t f, T* C, const T* bias, int32_t ld,
                      int32_t longest, const int32_t* seg_beg) {
  const int fv = f / W;
  int lpr = 1;
  while (lpr < 32 && lpr < fv) lpr <<= 1;
  int R = (int)ceil_div(fv, lpr);
  R = R <= 1 ? 1 : R <= 2 ? 2 : R <= 4 ? 4 : 8;  // R > 8: column-block loop in the kernel
  int U = lpr >= 4 ? 4 : (lpr == 2 ? 2 : 1);
  if (const char* e = getenv("SGNN_SPMM_CFG")) {  // dev tuning: "lpr,R,U"
    int a = 0, b = 0, c = 0;
    if (sscanf(e, "%d,%d,%d", &a, &b, &c) == 3 && a * b >= (lpr * R) / 1 && a <= 32) {
      lpr = a;
      R = b;
      U = c;
    }
  }
#define LPR_CASE(L)                                                                             \
  case L:                                                                                       \
    if (U >= 8) launch_lpr<T, W, L, 8>(ctx, R, n_rows, rowptr, cols, vals, B, f, C, bias, ld, longest, seg_beg);      \
    else if (U >= 4) launch_lpr<T, W, L, 4>(ctx, R, n_rows, rowptr, cols, vals, B, f, C, bias, ld, longest, seg_beg); \
    else if (U >= 2) launch_lpr<T, W, L, 2>(ctx, R, n_rows, rowptr, cols, vals, B, f, C, bias, ld, longest, seg_beg); \
    else launch_lpr<T, W, L, 1>(ctx, R, n_rows, rowptr, cols, vals, B, f, C, bias, ld, longest, seg_beg);             \
    break;
  switch (lpr) {
    LPR_CASE(1) LPR_CASE(2) LPR_CASE(4) LPR_CASE(8) LPR_CASE(16)
    default: LPR_CASE(32)
  }
#undef LPR_CASE
}

// generic path with hub-row splitting: normal rows, then the segments of the
// long rows into partial rows, then an in-order combine (+ bias)
template <class T, int W>
static void launch_w(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr, const int32_t* cols,
                     const T* vals, const T* B, int32_t f, T* C, const T* bias, int32_t ld,
                     const LongRows* lr = nullptr) {
  const bool split = lr && lr->nlong > 0;
  launch_w1<T, W>(ctx, n_rows, rowptr, cols, vals, B, f, C, bias, ld,
                  split ? kLongRow : 0x7fffffff, nullptr);
  if (!split) return;
  DevBuf part((size_t)lr->nseg * f * sizeof(T), ctx->stream);
  launch_w1<T, W>(ctx, lr->nseg, lr->seg_end.as<int32_t>(), cols, vals, B, f, part.as<T>(),
                  nullptr, f, 0x7fffffff, lr->seg_beg.as<int32_t>());
  k_spmm_combine_t<T><<<(unsigned)ceil_div(lr->nlong, 8), 256, 0, ctx->stream>>>(
      lr->nlong, lr->long_row.as<int32_t>(), lr->long_first.as<int32_t>(), part.as<T>(), f, C,
      bias, ld);
  launched(ctx);
}

// fp32 rows of 68..256 floats use the lean one-row-per-warp kernel (measured
// 84 us for the Arxiv f=128 product vs 125 us for the generic kernel); other
// widths and fp64 use the generic LPR-lane kernel.  SGNN_SPMM_MODE=1 forces
// the generic kernel (both are bit-identical to the reference).
template <class T>
void spmm_csr(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr, const int32_t* cols,
              const T* vals, const T* B, int32_t f, T* C, const T* bias, int64_t nnz,
              const LongRows* lr, int32_t b_rows) {
  if (n_rows == 0 || f == 0) return;
  constexpr int VW = sizeof(T) == 4 ? 4 : 2;
  if constexpr (sizeof(T) == 4) {
    // widths that are not a multiple of 4 (config 5's 47 classes): the scalar
    // kernel gathers 188-byte rows 4 bytes per lane; staging B into a
    // 16-byte-aligned padded copy lets the float4 kernels run (the padding
    // columns are zeros and never reach C; per-element order unchanged, so
    // the result is bit-identical).  Only for large products with known B.
    static const bool no_pad = getenv("SGNN_NO_PAD") != nullptr;
    if (!no_pad && b_rows > 0 && f % 4 != 0 && f > 4 && nnz >= (int64_t)1 << 20) {
      const int32_t f4 = (f + 3) & ~3;
      DevBuf bp((size_t)b_rows * f4 * 4, ctx->stream), cp((size_t)n_rows * f4 * 4, ctx->stream);
      pad_rows_f32(ctx, b_rows, f, B, f, f4, bp.as<float>());
      spmm_csr<float>(ctx, n_rows, rowptr, cols, vals, bp.as<float>(), f4, cp.as<float>(),
                      nullptr, nnz, lr, -1);
      unpad_rows_f32(ctx, n_rows, f, cp.as<float>(), f4, bias, C);
      return;
    }
  }
  const bool aligned = (reinterpret_cast<uintptr_t>(B) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(C) % 16 == 0) &&
                       (!bias || reinterpret_cast<uintptr_t>(bias) % 16 == 0);
  if constexpr (sizeof(T) == 4) {
    static const int mode = getenv("SGNN_SPMM_MODE") ? atoi(getenv("SGNN_SPMM_MODE")) : 0;
    static const int lu = getenv("SGNN_SPMM_U") ? atoi(getenv("SGNN_SPMM_U")) : 2;
    const bool vec_ok = aligned && f % 4 == 0 && nnz > 0;
    if (mode == 0 && vec_ok && f > 64 && f <= 256) {  // lean one-row-per-warp kernel
      if (f <= 128) launch_lean<1>(ctx, lu, n_rows, rowptr, cols, vals, B, f, C, bias, f, lr);
      else launch_lean<2>(ctx, lu, n_rows, rowptr, cols, vals, B, f, C, bias, f, lr);
      return;
    }
    if (mode == 0 && vec_ok && f > 256) {
      // wide rows: 256-column windows through the lean kernel (row stride f);
      // one thread still accumulates each output element in stored edge order
      for (int32_t c0 = 0; c0 < f; c0 += 256) {
        const int32_t w = f - c0 < 256 ? f - c0 : 256;
        const float* bw = bias ? bias + c0 : nullptr;
        if (w <= 128) launch_lean<1>(ctx, lu, n_rows, rowptr, cols, vals, B + c0, w, C + c0, bw, f, lr);
        else launch_lean<2>(ctx, lu, n_rows, rowptr, cols, vals, B + c0, w, C + c0, bw, f, lr);
      }
      return;
    }
  }
  if (f % VW == 0 && aligned)
    launch_w<T, VW>(ctx, n_rows, rowptr, cols, vals, B, f, C, bias, f, lr);
  else
    launch_w<T, 1>(ctx, n_rows, rowptr, cols, vals, B, f, C, bias, f, lr);
}

template void spmm_csr<float>(sgnn_ctx, int32_t, const int32_t*, const int32_t*, const float*,
                              const float*, int32_t, float*, const float*, int64_t,
                              const LongRows*, int32_t);
template void spmm_csr<double>(sgnn_ctx, int32_t, const int32_t*, const int32_t*, const double*,
                               const double*, int32_t, double*, const double*, int64_t,
                               const LongRows*, int32_t);

}  // namespace sgnn

using namespace sgnn;

extern "C" int sgnn_spmm(sgnn_ctx ctx, sgnn_adj adj, int transposed, const void* B, int32_t f,
                         void* C, const void* bias) {
  SGNN_API_BEGIN
  require(adj != nullptr, "spmm: null operator");
  require(f >= 0, "spmm: dimension mismatch");
  const int32_t n_out = transposed ? adj->n_cols : adj->n_rows;
  const int32_t* ptr = transposed ? adj->colptr.as<int32_t>() : adj->rowptr.as<int32_t>();
  const int32_t* idx = transposed ? adj->crows.as<int32_t>() : adj->cols.as<int32_t>();
  const LongRows* lr = &long_rows(ctx, transposed ? adj->long_bwd : adj->long_fwd, n_out, ptr);
  if (adj->dtype == SGNN_F32) {
    const float* v = transposed ? adj->cvals.as<float>() : adj->vals.as<float>();
    spmm_csr<float>(ctx, n_out, ptr, idx, v, static_cast<const float*>(B), f,
                    static_cast<float*>(C), static_cast<const float*>(bias), adj->nnz, lr,
                    transposed ? adj->n_rows : adj->n_cols);
  } else {
    const double* v = transposed ? adj->cvals.as<double>() : adj->vals.as<double>();
    spmm_csr<double>(ctx, n_out, ptr, idx, v, static_cast<const double*>(B), f,
                     static_cast<double*>(C), static_cast<const double*>(bias), adj->nnz, lr);
  }
  SGNN_API_END
}
