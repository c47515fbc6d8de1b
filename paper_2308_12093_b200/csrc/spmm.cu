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
#include "common.cuh"
#include "internal.cuh"

namespace sgnn {

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
__global__ void __launch_bounds__(256) k_spmm_csr(int32_t n_rows, const int32_t* __restrict__ rowptr,
                                                  const int32_t* __restrict__ cols,
                                                  const T* __restrict__ vals,
                                                  const T* __restrict__ B, int32_t f,
                                                  T* __restrict__ C, const T* __restrict__ bias) {
  using V = typename VecT<T, W>::type;
  constexpr int RPW = 32 / LPR;  // rows per warp
  const int lane = threadIdx.x & 31;
  const int g = lane % LPR;      // lane within group
  const int grp = lane / LPR;
  const unsigned gmask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (grp * LPR));
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int fv = f / W;  // vectors per row
  const V* Bv = reinterpret_cast<const V*>(B);
  V* Cv = reinterpret_cast<V*>(C);
  const V* biasv = reinterpret_cast<const V*>(bias);

  for (int64_t row0 = warp * RPW; row0 < n_rows; row0 += nwarps * RPW) {
    const int64_t row = row0 + grp;
    const bool active = row < n_rows;
    const int32_t beg = active ? rowptr[row] : 0;
    const int32_t end = active ? rowptr[row + 1] : 0;
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
            const V* brow = Bv + (int64_t)c * fv;
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
              Cv[row * fv + cv] = pack<T, W, V>(b);
            } else {
              Cv[row * fv + cv] = pack<T, W, V>(acc[r]);
            }
          }
        }
      }
    }
  }
}

template <class T, int W, int LPR>
static void launch_lpr(sgnn_ctx ctx, int R, int32_t n_rows, const int32_t* rowptr,
                       const int32_t* cols, const T* vals, const T* B, int32_t f, T* C,
                       const T* bias) {
  const int rpw = 32 / LPR;
  const int64_t warps = ceil_div(n_rows, rpw);
  const int block = 256;
  int64_t grid = ceil_div(warps * 32, block);
  const int64_t cap = (int64_t)ctx->num_sms * 64;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  constexpr int U = LPR >= 4 ? 4 : (LPR == 2 ? 2 : 1);
  switch (R) {
#define CASE(RR)                                                                         \
  case RR:                                                                               \
    k_spmm_csr<T, LPR, RR, W, U><<<(int)grid, block, 0, ctx->stream>>>(n_rows, rowptr, cols, \
                                                                      vals, B, f, C, bias); \
    break;
    CASE(1) CASE(2) CASE(4) CASE(8)
#undef CASE
    default: throw invalid_argument("spmm: bad register blocking");
  }
  launched(ctx);
}

template <class T, int W>
static void launch_w(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr, const int32_t* cols,
                     const T* vals, const T* B, int32_t f, T* C, const T* bias) {
  const int fv = f / W;
  int lpr = 1;
  while (lpr < 32 && lpr < fv) lpr <<= 1;
  int R = (int)ceil_div(fv, lpr);
  R = R <= 1 ? 1 : R <= 2 ? 2 : R <= 4 ? 4 : 8;  // R > 8: column-block loop in the kernel
  switch (lpr) {
    case 1: launch_lpr<T, W, 1>(ctx, R, n_rows, rowptr, cols, vals, B, f, C, bias); break;
    case 2: launch_lpr<T, W, 2>(ctx, R, n_rows, rowptr, cols, vals, B, f, C, bias); break;
    case 4: launch_lpr<T, W, 4>(ctx, R, n_rows, rowptr, cols, vals, B, f, C, bias); break;
    case 8: launch_lpr<T, W, 8>(ctx, R, n_rows, rowptr, cols, vals, B, f, C, bias); break;
    case 16: launch_lpr<T, W, 16>(ctx, R, n_rows, rowptr, cols, vals, B, f, C, bias); break;
    default: launch_lpr<T, W, 32>(ctx, R, n_rows, rowptr, cols, vals, B, f, C, bias); break;
  }
}

template <class T>
void spmm_csr(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr, const int32_t* cols,
              const T* vals, const T* B, int32_t f, T* C, const T* bias) {
  if (n_rows == 0 || f == 0) return;
  constexpr int VW = sizeof(T) == 4 ? 4 : 2;
  const bool aligned = (reinterpret_cast<uintptr_t>(B) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(C) % 16 == 0) &&
                       (!bias || reinterpret_cast<uintptr_t>(bias) % 16 == 0);
  if (f % VW == 0 && aligned)
    launch_w<T, VW>(ctx, n_rows, rowptr, cols, vals, B, f, C, bias);
  else
    launch_w<T, 1>(ctx, n_rows, rowptr, cols, vals, B, f, C, bias);
}

template void spmm_csr<float>(sgnn_ctx, int32_t, const int32_t*, const int32_t*, const float*,
                              const float*, int32_t, float*, const float*);
template void spmm_csr<double>(sgnn_ctx, int32_t, const int32_t*, const int32_t*, const double*,
                               const double*, int32_t, double*, const double*);

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
  if (adj->dtype == SGNN_F32) {
    const float* v = transposed ? adj->cvals.as<float>() : adj->vals.as<float>();
    spmm_csr<float>(ctx, n_out, ptr, idx, v, static_cast<const float*>(B), f,
                    static_cast<float*>(C), static_cast<const float*>(bias));
  } else {
    const double* v = transposed ? adj->cvals.as<double>() : adj->vals.as<double>();
    spmm_csr<double>(ctx, n_out, ptr, idx, v, static_cast<const double*>(B), f,
                     static_cast<double*>(C), static_cast<const double*>(bias));
  }
  SGNN_API_END
}
