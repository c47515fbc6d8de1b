// gat.cu -- GAT engine (north-star subsystem 3; gat.hpp:89-219, kernels.hpp:383-658).
//
// Forward: M = X Theta (GEMM) -> node scores s, d -> ONE fused row kernel per
// destination node (warp per row): per-head row max and 1/sum of exp
// (LeakyReLU(s_i + d_j) computed on the fly, never materialised), then
// batches of (edge, head) attention coefficients staged in shared memory and
// the multi-head aggregation out[i] = sum_e alpha_e M[j] + b with 128-bit
// loads of the M rows.  alpha + mask are written only at cache level `full`.
//
// Backward: row kernel (SDDMM dAlpha = <dX'_i, M_j> per (edge, head), softmax
// and LeakyReLU backward, row sums dS) -> column kernel over the CSC view
// (dD = column sums, dM = alpha^T dX' + dS a_src + dD a_dst) -> attention
// parameter reductions -> dTheta = X^T dM, dX = dM Theta^T (GEMMs).
//
// Order of accumulation follows the reference per output element (edge order,
// unfused multiply-add), so float64 results agree with the reference to a
// few ulps (exp() differs from glibc by <= 1 ulp).
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "internal.cuh"

namespace sgnn {

constexpr int HMAX = 64;  // heads supported by the fused kernels

template <class T>
__device__ __forceinline__ T dev_exp(T x);
template <>
__device__ __forceinline__ float dev_exp<float>(float x) {
  return expf(x);
}
template <>
__device__ __forceinline__ double dev_exp<double>(double x) {
  return exp(x);
}

template <class T>
__device__ __forceinline__ T leaky(T y, T beta, bool& pos) {
  pos = y > T(0);  // kernels.hpp:473-475
  return pos ? y : mul_rn(beta, y);
}

template <class T, int W>
struct V;
template <class T>
struct V<T, 1> {
  using t = T;
};
template <>
struct V<float, 4> {
  using t = float4;
};
template <>
struct V<double, 2> {
  using t = double2;
};

template <class T, int W>
__device__ __forceinline__ void vload(const T* p, T (&out)[W]) {
  using VT = typename V<T, W>::t;
  const VT v = __ldg(reinterpret_cast<const VT*>(p));
  const T* q = reinterpret_cast<const T*>(&v);
#pragma unroll
  for (int w = 0; w < W; ++w) out[w] = q[w];
}
template <class T, int W>
__device__ __forceinline__ void vstore(T* p, const T (&in)[W]) {
  using VT = typename V<T, W>::t;
  VT v;
  T* q = reinterpret_cast<T*>(&v);
#pragma unroll
  for (int w = 0; w < W; ++w) q[w] = in[w];
  *reinterpret_cast<VT*>(p) = v;
}

#include "gat_fast.cuh"
#include "gat_v2.cuh"
#include "gat_reorder.cuh"

// kernels.hpp:385-423 node_scores: one thread per (node, head), sequential dot
template <class T>
__global__ void k_node_scores(int32_t n, int32_t h, int32_t k, const T* __restrict__ M,
                              const T* __restrict__ a_src, const T* __restrict__ a_dst,
                              T* __restrict__ s, T* __restrict__ d) {
  const int64_t total = (int64_t)n * h;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int32_t t = (int32_t)(x % h);
    const T* mrow = M + x * k;
    const T* as = a_src + (int64_t)t * k;
    const T* ad = a_dst + (int64_t)t * k;
    T sv = T(0), dv = T(0);
    for (int32_t c = 0; c < k; ++c) {
      const T mv = mrow[c];
      sv = madd(sv, __ldg(as + c), mv);
      dv = madd(dv, __ldg(ad + c), mv);
    }
    s[x] = sv;
    d[x] = dv;
  }
}

// float32 node_scores for head widths the fused / fast paths do not cover
// (e.g. k = 256): one warp per (node, head), 16-byte loads across the head's
// k columns (coalesced rows of M, unlike thread-per-(node, head)), xor-tree
// reduction of the lane partials
__global__ void __launch_bounds__(256) k_node_scores_warp(int32_t n, int32_t h, int32_t k,
                                                          const float4* __restrict__ M,
                                                          const float4* __restrict__ a_src,
                                                          const float4* __restrict__ a_dst,
                                                          float* __restrict__ s,
                                                          float* __restrict__ d) {
  const int lane = threadIdx.x & 31;
  const int L = k >> 2;
  const int64_t total = (int64_t)n * h;
  const int64_t stride = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; x < total; x += stride) {
    const int32_t t = (int32_t)(x % h);
    const float4* mrow = M + x * L;
    const float4* as = a_src + (int64_t)t * L;
    const float4* ad = a_dst + (int64_t)t * L;
    float sv = 0.f, dv = 0.f;
#pragma unroll 4
    for (int c = lane; c < L; c += 32) {
      const float4 m = __ldg(mrow + c), a = __ldg(as + c), b = __ldg(ad + c);
      sv = fmaf(m.w, a.w, fmaf(m.z, a.z, fmaf(m.y, a.y, fmaf(m.x, a.x, sv))));
      dv = fmaf(m.w, b.w, fmaf(m.z, b.z, fmaf(m.y, b.y, fmaf(m.x, b.x, dv))));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sv += __shfl_xor_sync(0xffffffffu, sv, o);
      dv += __shfl_xor_sync(0xffffffffu, dv, o);
    }
    if (lane == 0) {
      s[x] = sv;
      d[x] = dv;
    }
  }
}

// heads of LPW whole 32-lane chunks (k = 128 LPW): a warp takes 4 (node,
// head) items at once and issues all 4 * LPW 16-byte loads before any
// reduction (memory-level parallelism; 8x256: 0.42 ms with one item at a time)
template <int LPW>
__global__ void __launch_bounds__(256) k_node_scores_warp4(int32_t n, int32_t h,
                                                           const float4* __restrict__ M,
                                                           const float4* __restrict__ a_src,
                                                           const float4* __restrict__ a_dst,
                                                           float* __restrict__ s,
                                                           float* __restrict__ d) {
  constexpr int L = 32 * LPW, IT = 4;
  const int lane = threadIdx.x & 31;
  const int64_t total = (int64_t)n * h;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t x0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * IT; x0 < total;
       x0 += nw * IT) {
    float4 m[IT][LPW];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int64_t x = min(x0 + it, total - 1);
#pragma unroll
      for (int c = 0; c < LPW; ++c) m[it][c] = __ldg(M + x * L + c * 32 + lane);
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int64_t x = x0 + it;
      const int32_t t = (int32_t)(min(x, total - 1) % h);
      float sv = 0.f, dv = 0.f;
#pragma unroll
      for (int c = 0; c < LPW; ++c) {
        const float4 a = __ldg(a_src + (int64_t)t * L + c * 32 + lane);
        const float4 b = __ldg(a_dst + (int64_t)t * L + c * 32 + lane);
        const float4 v = m[it][c];
        sv = fmaf(v.w, a.w, fmaf(v.z, a.z, fmaf(v.y, a.y, fmaf(v.x, a.x, sv))));
        dv = fmaf(v.w, b.w, fmaf(v.z, b.z, fmaf(v.y, b.y, fmaf(v.x, b.x, dv))));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sv += __shfl_xor_sync(0xffffffffu, sv, o);
        dv += __shfl_xor_sync(0xffffffffu, dv, o);
      }
      if (lane == 0 && x < total) {
        s[x] = sv;
        d[x] = dv;
      }
    }
  }
}

struct WarpSmem {
  static constexpr int kAlpha = 64;
};

// Per-row softmax statistics (kernels.hpp:517-531): lanes own heads and walk
// the row in stored order, exactly like the reference loop.
template <class T>
__device__ __forceinline__ void row_stats(int lane, int32_t i, int32_t beg, int32_t end,
                                          const int32_t* __restrict__ cols,
                                          const T* __restrict__ s, const T* __restrict__ d,
                                          int32_t h, T beta, T* smax, T* sinv) {
  for (int t = lane; t < h; t += 32) {
    const T si = s[(int64_t)i * h + t];
    bool pos;
    T gmax = leaky(add_rn(si, d[(int64_t)__ldg(cols + beg) * h + t]), beta, pos);
    for (int32_t e = beg + 1; e < end; ++e) {
      const T w = leaky(add_rn(si, d[(int64_t)__ldg(cols + e) * h + t]), beta, pos);
      gmax = gmax < w ? w : gmax;
    }
    T sum = T(0);
    for (int32_t e = beg; e < end; ++e) {
      const T w = leaky(add_rn(si, d[(int64_t)__ldg(cols + e) * h + t]), beta, pos);
      sum = add_rn(sum, dev_exp<T>(w - gmax));
    }
    smax[t] = gmax;
    sinv[t] = T(1) / sum;
  }
}

// Fused attention + aggregation. W scalars per vector, R vectors per lane per
// column block.  STORE: write alpha/mask (edge-major). AGG: aggregate.
template <class T, int W, int R, bool STORE, bool AGG>
__global__ void __launch_bounds__(256) k_gat_fwd(int32_t n, const int32_t* __restrict__ rowptr,
                                                 const int32_t* __restrict__ cols,
                                                 const T* __restrict__ M, const T* __restrict__ s,
                                                 const T* __restrict__ d, int32_t h, int32_t k,
                                                 T beta, const T* __restrict__ bias,
                                                 T* __restrict__ out, T* __restrict__ alpha,
                                                 uint8_t* __restrict__ mask) {
  __shared__ T sh_max[8][HMAX];
  __shared__ T sh_inv[8][HMAX];
  __shared__ T sh_al[8][HMAX];
  __shared__ int32_t sh_col[8][32];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* smax = sh_max[wib];
  T* sinv = sh_inv[wib];
  T* sal = sh_al[wib];
  int32_t* scol = sh_col[wib];
  const int32_t hk = h * k;
  const int fv = hk / W;
  int hp = 1;
  while (hp < h) hp <<= 1;
  const int EB = hp >= 32 ? 1 : 32 / hp;  // edges per batch
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;

  for (int64_t ii = warp; ii < n; ii += nwarps) {
    const int32_t i = (int32_t)ii;
    const int32_t beg = rowptr[i], end = rowptr[i + 1];
    row_stats<T>(lane, i, beg, end, cols, s, d, h, beta, smax, sinv);
    __syncwarp();
    const int ncb = AGG ? (int)ceil_div(fv, 32 * R) : 1;
    for (int cb = 0; cb < ncb; ++cb) {
      T acc[R][W];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int w = 0; w < W; ++w) acc[r][w] = T(0);
      for (int32_t base = beg; base < end; base += EB) {
        const int cnt = min(EB, end - base);
        for (int idx = lane; idx < EB * hp; idx += 32) {
          const int eb = idx / hp, t = idx % hp;
          if (t < h && eb < cnt) {
            const int32_t e = base + eb;
            const int32_t j = __ldg(cols + e);
            bool pos;
            const T w = leaky(add_rn(s[(int64_t)i * h + t], d[(int64_t)j * h + t]), beta, pos);
            const T a = mul_rn(dev_exp<T>(w - smax[t]), sinv[t]);
            sal[eb * hp + t] = a;
            if (STORE && cb == 0) {
              alpha[(int64_t)e * h + t] = a;
              mask[(int64_t)e * h + t] = pos ? 1 : 0;
            }
          }
        }
        if (lane < cnt) scol[lane] = __ldg(cols + base + lane);
        __syncwarp();
        if (AGG) {
          for (int eb = 0; eb < cnt; ++eb) {
            const T* mrow = M + (int64_t)scol[eb] * hk;
            T mv[R][W];
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const int v = cb * 32 * R + r * 32 + lane;
              if (v < fv) vload<T, W>(mrow + (int64_t)v * W, mv[r]);
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const int v = cb * 32 * R + r * 32 + lane;
              if (v < fv) {
#pragma unroll
                for (int w = 0; w < W; ++w) {
                  const int c = v * W + w;
                  acc[r][w] = madd(acc[r][w], sal[eb * hp + c / k], mv[r][w]);
                }
              }
            }
          }
        }
        __syncwarp();
      }
      if (AGG) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int v = cb * 32 * R + r * 32 + lane;
          if (v < fv) {
            T b[W], o[W];
            vload<T, W>(bias + (int64_t)v * W, b);
#pragma unroll
            for (int w = 0; w < W; ++w) o[w] = add_rn(acc[r][w], b[w]);
            vstore<T, W>(out + (int64_t)i * hk + (int64_t)v * W, o);
          }
        }
      }
    }
  }
}

// Backward, per destination row: alpha (cached or recomputed), dAlpha (SDDMM,
// kernels.hpp:342-377), softmax backward (:537-567), LeakyReLU backward
// (:481-495), row sums dS (:570-588).  dy and alpha written edge-major.
template <class T, int W, bool CACHED>
__global__ void __launch_bounds__(256) k_gat_bwd_row(
    int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
    const T* __restrict__ M, const T* __restrict__ s, const T* __restrict__ d,
    const T* __restrict__ G, int32_t h, int32_t k, T beta, const T* __restrict__ alpha_in,
    const uint8_t* __restrict__ mask_in, T* __restrict__ alpha_out,
    uint8_t* __restrict__ mask_out, T* __restrict__ da, T* __restrict__ dy,
    T* __restrict__ dS) {
  __shared__ T sh_max[8][HMAX];
  __shared__ T sh_inv[8][HMAX];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* smax = sh_max[wib];
  T* sinv = sh_inv[wib];
  const int32_t hk = h * k;
  int hp = 1;
  while (hp < h) hp <<= 1;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const T* al = CACHED ? alpha_in : alpha_out;
  const uint8_t* mk = CACHED ? mask_in : mask_out;

  for (int64_t ii = warp; ii < n; ii += nwarps) {
    const int32_t i = (int32_t)ii;
    const int32_t beg = rowptr[i], end = rowptr[i + 1];
    if (!CACHED) {
      row_stats<T>(lane, i, beg, end, cols, s, d, h, beta, smax, sinv);
      __syncwarp();
    }
    const T* grow = G + (int64_t)i * hk;
    const int64_t pairs = (int64_t)(end - beg) * hp;
    for (int64_t idx = lane; idx < pairs; idx += 32) {
      const int32_t e = beg + (int32_t)(idx / hp);
      const int t = (int)(idx % hp);
      if (t >= h) continue;
      const int32_t j = __ldg(cols + e);
      if (!CACHED) {
        bool pos;
        const T w = leaky(add_rn(s[(int64_t)i * h + t], d[(int64_t)j * h + t]), beta, pos);
        alpha_out[(int64_t)e * h + t] = mul_rn(dev_exp<T>(w - smax[t]), sinv[t]);
        mask_out[(int64_t)e * h + t] = pos ? 1 : 0;
      }
      const T* gr = grow + (int64_t)t * k;
      const T* mr = M + (int64_t)j * hk + (int64_t)t * k;
      T acc = T(0);
      for (int32_t c = 0; c < k; c += W) {
        T gv[W], mv[W];
        vload<T, W>(gr + c, gv);
        vload<T, W>(mr + c, mv);
#pragma unroll
        for (int w = 0; w < W; ++w) acc = madd(acc, gv[w], mv[w]);
      }
      da[(int64_t)e * h + t] = acc;
    }
    __syncwarp();
    for (int t = lane; t < h; t += 32) {
      T dot = T(0);
      for (int32_t e = beg; e < end; ++e)
        dot = madd(dot, al[(int64_t)e * h + t], da[(int64_t)e * h + t]);
      T rs = T(0);
      for (int32_t e = beg; e < end; ++e) {
        const T a = al[(int64_t)e * h + t];
        const T dw = mul_rn(a, da[(int64_t)e * h + t] - dot);
        const T g = mk[(int64_t)e * h + t] ? dw : mul_rn(beta, dw);
        dy[(int64_t)e * h + t] = g;
        rs = add_rn(rs, g);
      }
      dS[(int64_t)i * h + t] = rs;
    }
    __syncwarp();
  }
}

// Backward, per source column j over the CSC view: dD (kernels.hpp:639-658)
// and dM = alpha^T dX' (:258-295) + dS a_src + dD a_dst (:614-636).
template <class T, int W, int R>
__global__ void __launch_bounds__(256) k_gat_bwd_col(
    int32_t n, const int32_t* __restrict__ colptr, const int32_t* __restrict__ crows,
    const int32_t* __restrict__ perm, const T* __restrict__ G, const T* __restrict__ alpha,
    const T* __restrict__ dy, const T* __restrict__ dS, const T* __restrict__ a_src,
    const T* __restrict__ a_dst, int32_t h, int32_t k, T* __restrict__ dD, T* __restrict__ dM) {
  __shared__ T sh_dd[8][HMAX];
  __shared__ T sh_al[8][HMAX];
  __shared__ int32_t sh_row[8][32];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* sdd = sh_dd[wib];
  T* sal = sh_al[wib];
  int32_t* srow = sh_row[wib];
  const int32_t hk = h * k;
  const int fv = hk / W;
  int hp = 1;
  while (hp < h) hp <<= 1;
  const int EB = hp >= 32 ? 1 : 32 / hp;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;

  for (int64_t jj = warp; jj < n; jj += nwarps) {
    const int32_t j = (int32_t)jj;
    const int32_t beg = colptr[j], end = colptr[j + 1];
    for (int t = lane; t < h; t += 32) {
      T acc = T(0);
      for (int32_t p = beg; p < end; ++p) acc = add_rn(acc, dy[(int64_t)__ldg(perm + p) * h + t]);
      sdd[t] = acc;
      dD[(int64_t)j * h + t] = acc;
    }
    __syncwarp();
    const int ncb = (int)ceil_div(fv, 32 * R);
    for (int cb = 0; cb < ncb; ++cb) {
      T acc[R][W];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int w = 0; w < W; ++w) acc[r][w] = T(0);
      for (int32_t base = beg; base < end; base += EB) {
        const int cnt = min(EB, end - base);
        for (int idx = lane; idx < EB * hp; idx += 32) {
          const int eb = idx / hp, t = idx % hp;
          if (t < h && eb < cnt) sal[eb * hp + t] = alpha[(int64_t)__ldg(perm + base + eb) * h + t];
        }
        if (lane < cnt) srow[lane] = __ldg(crows + base + lane);
        __syncwarp();
        for (int eb = 0; eb < cnt; ++eb) {
          const T* grow = G + (int64_t)srow[eb] * hk;
          T gv[R][W];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int v = cb * 32 * R + r * 32 + lane;
            if (v < fv) vload<T, W>(grow + (int64_t)v * W, gv[r]);
          }
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int v = cb * 32 * R + r * 32 + lane;
            if (v < fv) {
#pragma unroll
              for (int w = 0; w < W; ++w)
                acc[r][w] = madd(acc[r][w], sal[eb * hp + (v * W + w) / k], gv[r][w]);
            }
          }
        }
        __syncwarp();
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int v = cb * 32 * R + r * 32 + lane;
        if (v < fv) {
          T o[W];
#pragma unroll
          for (int w = 0; w < W; ++w) {
            const int c = v * W + w;
            const int t = c / k, cc = c % k;
            T x = madd(acc[r][w], dS[(int64_t)j * h + t], __ldg(a_src + (int64_t)t * k + cc));
            o[w] = madd(x, sdd[t], __ldg(a_dst + (int64_t)t * k + cc));
          }
          vstore<T, W>(dM + (int64_t)j * hk + (int64_t)v * W, o);
        }
      }
    }
    __syncwarp();
  }
}

// attention_param_grad (kernels.hpp:592-611): out[t,c] = sum_i coeff[i,t] M[i,t,c]
template <class T>
__global__ void k_attgrad_partial(int32_t n, int32_t h, int32_t k, const T* __restrict__ M,
                                  const T* __restrict__ coeff, int32_t chunk,
                                  double* __restrict__ part) {
  const int32_t hk = h * k;
  const int32_t r0 = blockIdx.y * chunk, r1 = min(n, r0 + chunk);
  for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < hk; c += gridDim.x * blockDim.x) {
    const int32_t t = c / k;
    double acc = 0.0;
    for (int32_t i = r0; i < r1; ++i)
      acc += (double)coeff[(int64_t)i * h + t] * (double)M[(int64_t)i * hk + c];
    part[(int64_t)blockIdx.y * hk + c] = acc;
  }
}

template <class T>
__global__ void k_attgrad_final(int32_t nchunks, int32_t hk, const double* __restrict__ part,
                                T* __restrict__ out) {
  for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < hk; c += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int32_t z = 0; z < nchunks; ++z) s += part[(int64_t)z * hk + c];
    out[c] = (T)s;
  }
}

template <class T>
__global__ void k_edge_to_head_major(int64_t q, int32_t h, const T* __restrict__ eq,
                                     const uint8_t* __restrict__ mq, T* __restrict__ hq,
                                     uint8_t* __restrict__ mh) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < q * h;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = x / h, t = x % h;
    if (hq) hq[t * q + e] = eq[x];
    if (mh) mh[t * q + e] = mq[x];
  }
}

// kernels.hpp:500-534 edge_softmax over arbitrary scores (edge-major q x h)
template <class T>
__global__ void k_edge_softmax(int32_t n, const int32_t* __restrict__ rowptr, int32_t h,
                               const T* __restrict__ w, T* __restrict__ alpha) {
  const int64_t total = (int64_t)n * h;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = (int32_t)(x / h), t = (int32_t)(x % h);
    const int32_t beg = rowptr[i], end = rowptr[i + 1];
    T gmax = w[(int64_t)beg * h + t];
    for (int32_t e = beg + 1; e < end; ++e) {
      const T v = w[(int64_t)e * h + t];
      gmax = gmax < v ? v : gmax;
    }
    T sum = T(0);
    for (int32_t e = beg; e < end; ++e) sum = add_rn(sum, dev_exp<T>(w[(int64_t)e * h + t] - gmax));
    const T inv = T(1) / sum;
    for (int32_t e = beg; e < end; ++e)
      alpha[(int64_t)e * h + t] = mul_rn(dev_exp<T>(w[(int64_t)e * h + t] - gmax), inv);
  }
}

// kernels.hpp:301-337 sddmm (one head, no scale): thread per edge, sequential dot
template <class T>
__global__ void k_sddmm(int32_t n, const int32_t* __restrict__ rowptr,
                        const int32_t* __restrict__ cols, const T* __restrict__ B, int32_t f,
                        const T* __restrict__ C, int32_t ldc, T* __restrict__ out) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t i = warp; i < n; i += nwarps) {
    const T* brow = B + i * f;
    for (int32_t e = rowptr[i] + lane; e < rowptr[i + 1]; e += 32) {
      const int32_t j = cols[e];
      T acc = T(0);
      for (int32_t l = 0; l < f; ++l) acc = madd(acc, brow[l], C[(int64_t)l * ldc + j]);
      out[e] = acc;
    }
  }
}

// ---- host launchers ---------------------------------------------------------
static int pick_r(int fv) {
  const int need = (int)ceil_div(fv, 32);
  return need <= 1 ? 1 : need <= 2 ? 2 : need <= 4 ? 4 : need <= 8 ? 8 : 16;
}

template <class T, int W, bool STORE, bool AGG>
static void launch_fwd_w(sgnn_ctx ctx, int32_t n, const int32_t* rp, const int32_t* ci,
                         const T* M, const T* s, const T* d, int32_t h, int32_t k, T beta,
                         const T* bias, T* out, T* alpha, uint8_t* mask) {
  const int R = AGG ? pick_r(h * k / W) : 1;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 8),
                                                               (int64_t)ctx->num_sms * 32));
  switch (R) {
#define CASE(RR)                                                                             \
  case RR:                                                                                   \
    k_gat_fwd<T, W, RR, STORE, AGG><<<grid, 256, 0, ctx->stream>>>(n, rp, ci, M, s, d, h, k,    \
                                                                  beta, bias, out, alpha, mask); \
    break;
    CASE(1) CASE(2) CASE(4) CASE(8) CASE(16)
#undef CASE
  }
  launched(ctx);
}

template <class T, bool STORE, bool AGG>
static void launch_fwd(sgnn_ctx ctx, int32_t n, const int32_t* rp, const int32_t* ci,
                       const T* M, const T* s, const T* d, int32_t h, int32_t k, T beta,
                       const T* bias, T* out, T* alpha, uint8_t* mask) {
  constexpr int VW = sizeof(T) == 4 ? 4 : 2;
  const bool vec = k % VW == 0 && reinterpret_cast<uintptr_t>(M) % 16 == 0 &&
                   (!AGG || (reinterpret_cast<uintptr_t>(out) % 16 == 0 &&
                             reinterpret_cast<uintptr_t>(bias) % 16 == 0));
  if (vec)
    launch_fwd_w<T, VW, STORE, AGG>(ctx, n, rp, ci, M, s, d, h, k, beta, bias, out, alpha, mask);
  else
    launch_fwd_w<T, 1, STORE, AGG>(ctx, n, rp, ci, M, s, d, h, k, beta, bias, out, alpha, mask);
}

template <class T>
static void node_scores(sgnn_ctx ctx, int32_t n, int32_t h, int32_t k, const T* M,
                        const T* a_src, const T* a_dst, T* s, T* d) {
  if constexpr (sizeof(T) == 4) {
    const bool al = ((reinterpret_cast<uintptr_t>(M) | reinterpret_cast<uintptr_t>(a_src) |
                      reinterpret_cast<uintptr_t>(a_dst)) & 15) == 0;
    const int lpw = k % 128 == 0 ? k / 128 : 0;
    if (al && n > 0 && (lpw == 1 || lpw == 2 || lpw == 4 || lpw == 8)) {
      const unsigned g = (unsigned)std::min<int64_t>(ceil_div((int64_t)n * h, 32),
                                                     (int64_t)ctx->num_sms * 16);
      const float4* M4 = reinterpret_cast<const float4*>(M);
      const float4* as4 = reinterpret_cast<const float4*>(a_src);
      const float4* ad4 = reinterpret_cast<const float4*>(a_dst);
      float* sf = reinterpret_cast<float*>(s);
      float* df = reinterpret_cast<float*>(d);
      switch (lpw) {
        case 1: k_node_scores_warp4<1><<<g, 256, 0, ctx->stream>>>(n, h, M4, as4, ad4, sf, df); break;
        case 2: k_node_scores_warp4<2><<<g, 256, 0, ctx->stream>>>(n, h, M4, as4, ad4, sf, df); break;
        case 4: k_node_scores_warp4<4><<<g, 256, 0, ctx->stream>>>(n, h, M4, as4, ad4, sf, df); break;
        default: k_node_scores_warp4<8><<<g, 256, 0, ctx->stream>>>(n, h, M4, as4, ad4, sf, df); break;
      }
      launched(ctx);
      return;
    }
    if (k % 4 == 0 && al && n > 0) {
      const int64_t blocks = ceil_div((int64_t)n * h, 8);
      const unsigned g = (unsigned)std::min<int64_t>(blocks, (int64_t)ctx->num_sms * 16);
      k_node_scores_warp<<<g, 256, 0, ctx->stream>>>(
          n, h, k, reinterpret_cast<const float4*>(M), reinterpret_cast<const float4*>(a_src),
          reinterpret_cast<const float4*>(a_dst), reinterpret_cast<float*>(s),
          reinterpret_cast<float*>(d));
      launched(ctx);
      return;
    }
  }
  k_node_scores<T><<<grid_for(ctx, (int64_t)n * h, 256), 256, 0, ctx->stream>>>(n, h, k, M, a_src,
                                                                               a_dst, s, d);
  launched(ctx);
}

template <class T>
static void att_grad(sgnn_ctx ctx, int32_t n, int32_t h, int32_t k, const T* M, const T* coeff,
                     T* out) {
  const int32_t hk = h * k, chunk = 512;
  const int32_t nch = std::max<int32_t>(1, (int32_t)ceil_div(n, chunk));
  DevBuf part((size_t)nch * hk * 8, ctx->stream);
  if (n == 0) SGNN_CUDA(cudaMemsetAsync(part.get(), 0, part.bytes(), ctx->stream));
  else {
    dim3 g((unsigned)ceil_div(hk, 128), (unsigned)nch);
    k_attgrad_partial<T><<<g, 128, 0, ctx->stream>>>(n, h, k, M, coeff, chunk, part.as<double>());
    launched(ctx);
  }
  k_attgrad_final<T><<<(unsigned)ceil_div(hk, 128), 128, 0, ctx->stream>>>(nch, hk,
                                                                           part.as<double>(), out);
  launched(ctx);
}

template <class T>
static int rows_grid(sgnn_ctx ctx, int32_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 8), (int64_t)ctx->num_sms * 32));
}

// Fast-path eligibility (gat_fast.cuh): returns R (vectors per lane) or 0.
template <class T>
static int fast_R(int32_t h, int32_t k) {
  constexpr int VW = sizeof(T) == 4 ? 4 : 2;
  if (getenv("SGNN_GAT_GENERIC")) return 0;
  if (h > 8 || k % VW != 0) return 0;  // kernels instantiated for h <= 8
  const int lph = k / VW, fv = h * k / VW;
  const bool pow2 = (lph & (lph - 1)) == 0;
  if (!((pow2 && lph <= 32) || lph % 32 == 0)) return 0;
  const int R = pick_r(fv);
  if (R > 8) return 0;
  if (lph > 32 && R % (lph / 32) != 0) return 0;
  return R;
}

static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <class T>
static int wgrid(int32_t n) {
  constexpr int wpb = gf::WPB<T>::v;
  return (int)std::max<int64_t>(1, ceil_div(n, wpb));
}

#define R_SWITCH(R, ...)                  \
  switch (R) {                            \
    case 1: { constexpr int RR = 1; __VA_ARGS__; } break; \
    case 2: { constexpr int RR = 2; __VA_ARGS__; } break; \
    case 4: { constexpr int RR = 4; __VA_ARGS__; } break; \
    default: { constexpr int RR = 8; __VA_ARGS__; } break; \
  }

// float32 compile-time-heads path (gat_v2.cuh): h in {1,2,4,8}, k % 4 == 0,
// h*k <= 1024.  Returns R (16-byte vectors per lane) or 0.
template <class T>
static int v2_R(int32_t h, int32_t k) {
  if (sizeof(T) != 4 || getenv("SGNN_GAT_V1")) return 0;
  if (!(h == 1 || h == 2 || h == 4 || h == 8) || k % 4 != 0) return 0;
  const int fv = h * k / 4, L = k / 4;
  int R = pick_r(fv);
  if (h == 8 && R == 4 && fv <= 96) return 3;  // 257..384 wide: 3 vectors per lane
  // slabs wider than 32 * wr vectors run in column windows (gridDim.y) of
  // 32 * w vectors, heads whole per window: more warps per row and fewer
  // registers per lane keep more rows in flight (Arxiv 8 x 256: the three
  // gather kernels 8.7 ms at w = 8 -> 6.1 ms at w = 2)
  static const int wr = [] {
    const char* e = getenv("SGNN_GAT_WIDE_R");  // dev knob: 1, 2 (default), 4, 8
    return e ? (e[0] == '1' ? 1 : e[0] == '4' ? 4 : e[0] == '8' ? 8 : 2) : 2;
  }();
  if (R > wr)
    for (int w = wr; w <= 8; w *= 2)
      if ((32 * w) % L == 0) return w;
  return R <= 8 ? R : 0;
}

// column windows of the dense-row gather kernels: slabs wider than 32R vectors
template <class T>
static unsigned v2_windows(int32_t h, int32_t k) {
  const int fv = h * k / 4, R = v2_R<T>(h, k);
  return (unsigned)((fv + 32 * R - 1) / (32 * R));
}

// (H, R) -> constexpr instantiation: every pair v2_R can return
#define HR_SWITCH(H_, R_, ...)                                                        \
  switch (H_ * 16 + R_) {                                                             \
    case 1 * 16 + 1: { constexpr int HH = 1, RR = 1; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    case 2 * 16 + 1: { constexpr int HH = 2, RR = 1; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    case 1 * 16 + 2: { constexpr int HH = 1, RR = 2; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    case 1 * 16 + 4: { constexpr int HH = 1, RR = 4; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    case 2 * 16 + 4: { constexpr int HH = 2, RR = 4; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    case 2 * 16 + 2: { constexpr int HH = 2, RR = 2; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    case 4 * 16 + 1: { constexpr int HH = 4, RR = 1; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    case 4 * 16 + 2: { constexpr int HH = 4, RR = 2; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    case 4 * 16 + 4: { constexpr int HH = 4, RR = 4; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    case 4 * 16 + 8: { constexpr int HH = 4, RR = 8; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    case 2 * 16 + 8: { constexpr int HH = 2, RR = 8; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    case 1 * 16 + 8: { constexpr int HH = 1, RR = 8; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    case 8 * 16 + 1: { constexpr int HH = 8, RR = 1; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    case 8 * 16 + 2: { constexpr int HH = 8, RR = 2; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    case 8 * 16 + 3: { constexpr int HH = 8, RR = 3; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    case 8 * 16 + 4: { constexpr int HH = 8, RR = 4; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    case 8 * 16 + 8: { constexpr int HH = 8, RR = 8; (void)HH; (void)RR; __VA_ARGS__; } break;          \
    default: throw invalid_argument("gat: no v2 kernel for this head/width");        \
  }

static unsigned v2_grid(int32_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, g2::WPB)); }

// k_gat_sddmm2 reduction mode for head width L = k/4 vectors at R vectors per
// lane: 1 = power-of-two heads of <= 32 lanes, C in {2,4,8} = heads of C whole
// 32-lane chunks (R % C == 0), 0 = shared-memory fold (any other width)
static int sddmm_mode(int L, int R) {
  if ((L & (L - 1)) == 0 && L <= 32) return 1;
  const int C = L / 32;
  if (L % 32 == 0 && (C == 2 || C == 4 || C == 8) && R % C == 0) return C;
  return 0;
}

template <int HH, int RR, bool SEGB>
static void sddmm2_launch(int mode, dim3 grid, cudaStream_t st, int32_t n, const int32_t* rp,
                          const int32_t* ci, const float4* M4, const float4* G4, int32_t k,
                          float* da, const g2::SegArgs& sa) {
#define SDDMM2_GO(PM) g2::k_gat_sddmm2<HH, RR, PM, SEGB><<<grid, 256, 0, st>>>(n, rp, ci, M4, G4, k, da, sa)
  // heads of L < 16 vectors, L not a power of two, one window: padded lanes
  if (mode == 0 && grid.y == 1 && (k / 4) < 16 && HH >= 2) {
    if ((k / 4) < 8) {
      g2::k_gat_sddmm_pad<HH, 8, SEGB><<<grid, 256, 0, st>>>(n, rp, ci, M4, G4, k, da, sa);
    } else {
      g2::k_gat_sddmm_pad<HH, 16, SEGB><<<grid, 256, 0, st>>>(n, rp, ci, M4, G4, k, da, sa);
    }
    return;
  }
  switch (mode) {
    case 1: SDDMM2_GO(1); return;
    case 2: if constexpr (RR % 2 == 0) { SDDMM2_GO(2); return; } break;
    case 4: if constexpr (RR % 4 == 0) { SDDMM2_GO(4); return; } break;
    case 8: if constexpr (RR % 8 == 0) { SDDMM2_GO(8); return; } break;
    default: break;
  }
  SDDMM2_GO(0);
#undef SDDMM2_GO
}

template <int HH, int RR>
static void sddmm_sbwd_launch(int mode, cudaStream_t st, int32_t n, const int32_t* rp,
                              const int32_t* ci, const float4* M4, const float4* G4, int32_t k,
                              const float* al, const uint8_t* mk, double beta, float* da,
                              float* dy, float* dS, const g2::SegArgs& sa, float* rec,
                              const int32_t* pinv) {
  const unsigned grid = (unsigned)std::max<int64_t>(1, ceil_div(n, 16));  // two rows per warp
#define SDSB_GO(PM) \
  g2::k_gat_sddmm_sbwd<HH, RR, PM><<<grid, 256, 0, st>>>(n, rp, ci, M4, G4, k, al, mk, \
                                                         (float)beta, da, dy, dS, sa, rec, pinv)
  switch (mode) {
    case 1: SDSB_GO(1); return;
    case 2: if constexpr (RR % 2 == 0) { SDSB_GO(2); return; } break;
    case 4: if constexpr (RR % 4 == 0) { SDSB_GO(4); return; } break;
    case 8: if constexpr (RR % 8 == 0) { SDSB_GO(8); return; } break;
    default: break;
  }
#undef SDSB_GO
  throw invalid_argument("gat: no fused SDDMM kernel for this head width");
}

// inverse of the pattern's CSC permutation: pinv[perm[p]] = p (CSR edge ->
// CSC position), built once per pattern on first use (outside graph capture:
// the first call of a layer runs eagerly, like the LongRows plans)
__global__ void k_perm_inverse(int64_t q, const int32_t* __restrict__ perm,
                               int32_t* __restrict__ pinv) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < q;
       p += (int64_t)gridDim.x * blockDim.x)
    pinv[__ldg(perm + p)] = (int32_t)p;
}
static const int32_t* pattern_pinv(sgnn_ctx ctx, sgnn_pattern P) {
  if (!P->pinv.get() && P->nnz > 0) {
    // not built inside a stream capture (a graph-owned buffer): the caller
    // then keeps the perm-indirect column pass
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    SGNN_CUDA(cudaStreamIsCapturing(ctx->stream, &cs));
    if (cs != cudaStreamCaptureStatusNone) return nullptr;
    P->pinv = DevBuf((size_t)P->nnz * 4, ctx->stream);
    k_perm_inverse<<<grid_for(ctx, P->nnz, 256), 256, 0, ctx->stream>>>(
        P->nnz, P->perm.as<int32_t>(), P->pinv.as<int32_t>());
    launched(ctx);
  }
  return P->pinv.as<int32_t>();
}

// hub rows / columns of a pattern (LongRows plan): segment arguments
static g2::SegArgs seg_args(const LongRows& pl, float* part = nullptr, float* ddpart = nullptr) {
  g2::SegArgs a;
  a.longest = 0x7fffffff;
  a.row = pl.seg_row.as<int32_t>();
  a.beg = pl.seg_beg.as<int32_t>();
  a.end = pl.seg_end.as<int32_t>();
  a.part = reinterpret_cast<float4*>(part);
  a.ddpart = ddpart;
  return a;
}
static g2::SegArgs skip_long(const LongRows& pl) {
  g2::SegArgs a;
  a.longest = pl.nlong ? kLongRow : 0x7fffffff;
  return a;
}

template <class T>
static void node_scores_fast(sgnn_ctx ctx, int R, int32_t n, int32_t h, int32_t k, const T* M,
                             const T* a_src, const T* a_dst, T* s, T* d) {
  constexpr int VW = sizeof(T) == 4 ? 4 : 2;
  constexpr int wpb = gf::WPB<T>::v;
  R_SWITCH(R, (gf::k_node_scores_fast<T, VW, RR><<<wgrid<T>(n), 32 * wpb, 0, ctx->stream>>>(
                  n, h, k, M, a_src, a_dst, s, d)));
  launched(ctx);
}

// ---------------------------------------------------------------------------
// Operator-reordered layer for wide heads (gat_reorder.cuh): every edge
// gather moves from the k-wide rows of M = X Theta onto the m-wide rows of X
// (and, in the backward, the h x m rows of Gtheta = G_t Theta_t^T); the
// per-head transforms run on the tcgen05 GEMM with pitched operands.  Taken
// when the caller allows it (sgnn_gat_forward_ex SGNN_GAT_REORDER, the Gat2
// model) and the shape gains: float32, k > m, h in {1,2,4,8}, m and k
// multiples of 4, the h x m Gtheta row fits a warp's registers, no hub rows.
// SGNN_GAT_REORDER=0 turns it off (A/B switch).
// ---------------------------------------------------------------------------
#define REO_H(H_, ...)                                               \
  switch (H_) {                                                      \
    case 1: { constexpr int HH = 1; __VA_ARGS__; } break;            \
    case 2: { constexpr int HH = 2; __VA_ARGS__; } break;            \
    case 4: { constexpr int HH = 4; __VA_ARGS__; } break;            \
    case 8: { constexpr int HH = 8; __VA_ARGS__; } break;            \
    default: throw std::logic_error("gat reorder: unsupported head count"); \
  }
#define REO_HRM(H_, RM_, ...)                                                      \
  switch ((H_) * 8 + (RM_)) {                                                      \
    case 1 * 8 + 1: { constexpr int HH = 1, RM = 1; __VA_ARGS__; } break;          \
    case 1 * 8 + 2: { constexpr int HH = 1, RM = 2; __VA_ARGS__; } break;          \
    case 1 * 8 + 3: { constexpr int HH = 1, RM = 3; __VA_ARGS__; } break;          \
    case 1 * 8 + 4: { constexpr int HH = 1, RM = 4; __VA_ARGS__; } break;          \
    case 2 * 8 + 1: { constexpr int HH = 2, RM = 1; __VA_ARGS__; } break;          \
    case 2 * 8 + 2: { constexpr int HH = 2, RM = 2; __VA_ARGS__; } break;          \
    case 2 * 8 + 3: { constexpr int HH = 2, RM = 3; __VA_ARGS__; } break;          \
    case 2 * 8 + 4: { constexpr int HH = 2, RM = 4; __VA_ARGS__; } break;          \
    case 4 * 8 + 1: { constexpr int HH = 4, RM = 1; __VA_ARGS__; } break;          \
    case 4 * 8 + 2: { constexpr int HH = 4, RM = 2; __VA_ARGS__; } break;          \
    case 4 * 8 + 3: { constexpr int HH = 4, RM = 3; __VA_ARGS__; } break;          \
    case 4 * 8 + 4: { constexpr int HH = 4, RM = 4; __VA_ARGS__; } break;          \
    case 8 * 8 + 1: { constexpr int HH = 8, RM = 1; __VA_ARGS__; } break;          \
    case 8 * 8 + 2: { constexpr int HH = 8, RM = 2; __VA_ARGS__; } break;          \
    default: throw std::logic_error("gat reorder: unsupported shape");            \
  }

static bool reorder_env_off() {
  static const bool off = [] {
    const char* e = getenv("SGNN_GAT_REORDER");
    return e && e[0] == '0';
  }();
  return off;
}

static int reo_rm(int32_t m) { return (int)ceil_div(m / 4, 32); }

static bool reorder_shape_ok(int32_t n, int32_t m, int32_t h, int32_t k) {
  if (reorder_env_off() || !gemm_tc_available() || n <= 0) return false;
  if (!(h == 1 || h == 2 || h == 4 || h == 8)) return false;
  if (k <= m || (m & 3) || (k & 3)) return false;
  const int RM = reo_rm(m);
  return RM <= 4 && h * RM <= 16;
}

// W = [Theta_t a_src_t ; Theta_t a_dst_t] (2 x h x m)
static void reo_wvec(sgnn_ctx ctx, int32_t m, int32_t h, int32_t k, const float* theta,
                     const float* a_src, const float* a_dst, float* W) {
  g2::k_gat_wvec<<<(unsigned)ceil_div(2LL * h * m, 8), 256, 0, ctx->stream>>>(m, h, k, theta,
                                                                              a_src, a_dst, W);
  launched(ctx);
}

static void reo_scores(sgnn_ctx ctx, int32_t n, int32_t m, int32_t h, const float* X,
                       const float* W, float* s, float* d) {
  const int32_t mv = m / 4;
  const size_t smem = (size_t)2 * h * mv * sizeof(float4);
  const float4* X4 = reinterpret_cast<const float4*>(X);
  const float4* W4 = reinterpret_cast<const float4*>(W);
  REO_HRM(h, reo_rm(m), (g2::k_gat_xscores<HH, RM><<<v2_grid(n), 256, smem, ctx->stream>>>(
                            n, mv, X4, W4, s, d)));
  launched(ctx);
}

// alpha (and mask) of the reordered layer from the scores (k_gat_attn4)
static void reo_attention(sgnn_ctx ctx, sgnn_pattern p, int32_t h, float beta, const float* s,
                          const float* d, float* alpha, uint8_t* mask) {
  const int32_t n = p->n;
  REO_H(h, (g2::k_gat_attn4<HH><<<g2::sub_grid(n), 256, 0, ctx->stream>>>(
               n, p->rowptr.as<int32_t>(), p->cols.as<int32_t>(), s, d, beta, alpha, mask,
               0x7fffffff)));
  launched(ctx);
}

static void reo_aggregate(sgnn_ctx ctx, sgnn_pattern p, int32_t m, int32_t h, const float* alpha,
                          const float* X, float* Z) {
  const int32_t n = p->n, mv = m / 4;
  const float4* X4 = reinterpret_cast<const float4*>(X);
  float4* Z4 = reinterpret_cast<float4*>(Z);
  REO_HRM(h, reo_rm(m), (g2::k_gat_aggx<HH, RM><<<v2_grid(n), 256, 0, ctx->stream>>>(
                            n, p->rowptr.as<int32_t>(), p->cols.as<int32_t>(), alpha, X4, mv, Z4)));
  launched(ctx);
}

static void reo_gemm(sgnn_ctx ctx, const float* A, int32_t ra, int32_t ca, int32_t lda,
                     const float* B, int32_t rb, int32_t cb, int32_t ldb, bool ta, bool tb,
                     float* C, int32_t ldc, const float* bias, float* colsum_b = nullptr) {
  if (!gemm_tc_f32_pitched(ctx, A, ra, ca, lda, B, rb, cb, ldb, ta, tb, C, ldc, bias, colsum_b))
    throw std::runtime_error("gat reorder: pitched tcgen05 GEMM rejected its operands");
}

static void gat_forward_reordered(sgnn_ctx ctx, sgnn_pattern p, const float* X, int32_t m,
                                  const float* theta, const float* a_src, const float* a_dst,
                                  const float* bias, int32_t h, int32_t k, float beta, int level,
                                  float* out, sgnn_gat_cache c, uint8_t* elu_mask,
                                  bool* elu_fused) {
  const int32_t n = p->n, hk = h * k, hm = h * m;
  const int64_t q = p->nnz;
  cudaStream_t st = ctx->stream;
  DevBuf W((size_t)2 * hm * 4, st), s((size_t)n * h * 4 + 16, st), d((size_t)n * h * 4 + 16, st),
      Z((size_t)n * hm * 4, st), alpha((size_t)q * h * 4 + 16, st), mask;
  if (level == SGNN_GAT_FULL) mask = DevBuf((size_t)q * h + 16, st);
  reo_wvec(ctx, m, h, k, theta, a_src, a_dst, W.as<float>());
  reo_scores(ctx, n, m, h, X, W.as<float>(), s.as<float>(), d.as<float>());
  reo_attention(ctx, p, h, beta, s.as<float>(), d.as<float>(), alpha.as<float>(),
                mask.as<uint8_t>());
  reo_aggregate(ctx, p, m, h, alpha.as<float>(), X, Z.as<float>());
  // out_t = Z_t Theta_t + b_t, with the caller's ELU(1) in the epilogue when
  // the heads are whole 32-column chunks (the first head decides; all share
  // shape, pitch and alignment)
  bool fuse = elu_mask != nullptr;
  for (int32_t t = 0; t < h; ++t) {
    const float* A = Z.as<float>() + (size_t)t * m;
    const float* B = theta + (size_t)t * k;
    float* C = out + (size_t)t * k;
    if (fuse) {
      if (gemm_tc_f32_pitched(ctx, A, n, m, hm, B, m, k, hk, false, false, C, hk,
                              bias + (size_t)t * k, nullptr, elu_mask + (size_t)t * k)) {
        if (elu_fused) *elu_fused = true;
        continue;
      }
      if (t > 0) throw std::logic_error("gat reorder: ELU epilogue rejected after head 0");
      fuse = false;
    }
    reo_gemm(ctx, A, n, m, hm, B, m, k, hk, false, false, C, hk, bias + (size_t)t * k);
  }
  c->reordered = true;
  c->saved_input = X;
  c->q = q;
  if (level >= SGNN_GAT_FEATURES) {
    c->Z = std::move(Z);
    c->Z.track(kCache, (size_t)n * hm * 4);
  }
  if (level == SGNN_GAT_NODE_ATTENTION) {
    c->s = std::move(s);
    c->d = std::move(d);
    c->s.track(kCache, (size_t)n * h * 4);
    c->d.track(kCache, (size_t)n * h * 4);
  }
  if (level == SGNN_GAT_FULL) {
    c->alpha = std::move(alpha);
    c->mask = std::move(mask);
    c->alpha.track(kCache, (size_t)q * h * 4);
    c->mask.track(kCache, (size_t)q * h);
  }
}

// alpha / mask of a reordered cache (kept at level full, else recomputed from
// the kept or recomputed scores)
struct ReoEdges {
  DevBuf alpha, mask, s, d;
  const float* a = nullptr;
  const uint8_t* mk = nullptr;
};
static void reo_edges(sgnn_ctx ctx, sgnn_pattern p, sgnn_gat_cache c, const float* W,
                      ReoEdges& r) {
  const int32_t n = p->n, h = c->h;
  const int64_t q = p->nnz;
  cudaStream_t st = ctx->stream;
  if (c->level == SGNN_GAT_FULL) {
    r.a = c->alpha.as<float>();
    r.mk = c->mask.as<uint8_t>();
    return;
  }
  const float *sp, *dp;
  if (c->level == SGNN_GAT_NODE_ATTENTION) {
    sp = c->s.as<float>();
    dp = c->d.as<float>();
  } else {
    r.s = DevBuf((size_t)n * h * 4 + 16, st);
    r.d = DevBuf((size_t)n * h * 4 + 16, st);
    reo_scores(ctx, n, c->m, h, static_cast<const float*>(c->saved_input), W, r.s.as<float>(),
               r.d.as<float>());
    sp = r.s.as<float>();
    dp = r.d.as<float>();
  }
  r.alpha = DevBuf((size_t)q * h * 4 + 16, st);
  r.mask = DevBuf((size_t)q * h + 16, st);
  reo_attention(ctx, p, h, (float)c->beta, sp, dp, r.alpha.as<float>(), r.mask.as<uint8_t>());
  r.a = r.alpha.as<float>();
  r.mk = r.mask.as<uint8_t>();
}

static void gat_backward_reordered(sgnn_ctx ctx, sgnn_pattern p, const float* G,
                                   const float* theta, const float* a_src, const float* a_dst,
                                   sgnn_gat_cache c, bool fg, float* d_theta, float* d_a_src,
                                   float* d_a_dst, float* d_bias, float* d_input) {
  const int32_t n = p->n, h = c->h, k = c->k, m = c->m, hk = h * k, hm = h * m, mv = m / 4;
  const int RM = reo_rm(m);
  const int64_t q = p->nnz;
  const float* X = static_cast<const float*>(c->saved_input);
  cudaStream_t st = ctx->stream;
  const int32_t* rp = p->rowptr.as<int32_t>();
  const int32_t* ci = p->cols.as<int32_t>();
  DevBuf W((size_t)2 * hm * 4, st);
  reo_wvec(ctx, m, h, k, theta, a_src, a_dst, W.as<float>());
  ReoEdges e;
  reo_edges(ctx, p, c, W.as<float>(), e);
  DevBuf Zt;
  const float* Z;
  if (c->level >= SGNN_GAT_FEATURES) {
    Z = c->Z.as<float>();
  } else {
    Zt = DevBuf((size_t)n * hm * 4, st);
    reo_aggregate(ctx, p, m, h, e.a, X, Zt.as<float>());
    Z = Zt.as<float>();
  }
  // Gtheta_t = G_t Theta_t^T  (n x h x m)
  DevBuf Gt((size_t)n * hm * 4, st);
  for (int32_t t = 0; t < h; ++t)
    reo_gemm(ctx, G + (size_t)t * k, n, k, hk, theta + (size_t)t * k, m, k, hk, false, true,
             Gt.as<float>() + (size_t)t * m, hm, nullptr);
  // dAlpha, then the softmax / LeakyReLU backward (k_gat_sbwd4: dy, dS)
  DevBuf da((size_t)q * h * 4 + 16, st), dy((size_t)q * h * 4 + 16, st),
      dS((size_t)n * h * 4 + 16, st), dD((size_t)n * h * 4 + 16, st);
  const float4* X4 = reinterpret_cast<const float4*>(X);
  const float4* Gt4 = reinterpret_cast<const float4*>(Gt.get());
  REO_HRM(h, RM, (g2::k_gat_sddmmx<HH, RM><<<v2_grid(n), 256, 0, st>>>(n, rp, ci, Gt4, X4, mv,
                                                                       da.as<float>())));
  launched(ctx);
  REO_H(h, (g2::k_gat_sbwd4<HH><<<g2::sub_grid(n), 256, 0, st>>>(
               n, rp, e.a, e.mk, da.as<float>(), (float)c->beta, dy.as<float>(), dS.as<float>())));
  launched(ctx);
  const int32_t* cp = p->colptr.as<int32_t>();
  const int32_t* pm = p->perm.as<int32_t>();
  if (fg) {  // d_input and dD in one column pass
    REO_HRM(h, RM, (g2::k_gat_colx<HH, RM><<<v2_grid(n), 256, 0, st>>>(
                       n, cp, p->rows.as<int32_t>(), pm, Gt4, e.a, dy.as<float>(), dS.as<float>(),
                       reinterpret_cast<const float4*>(W.get()), mv, dD.as<float>(),
                       reinterpret_cast<float4*>(d_input))));
  } else {
    REO_H(h, (g2::k_gat_colsum_dy<HH><<<v2_grid(n), 256, 0, st>>>(n, cp, pm, dy.as<float>(),
                                                                  dD.as<float>())));
  }
  launched(ctx);
  // U_S = X^T dS, U_D = X^T dD (m x h); dTheta_t = Z_t^T G_t + rank-1 terms
  DevBuf us((size_t)m * h * 4 + 16, st), ud((size_t)m * h * 4 + 16, st);
  gemm<float>(ctx, X, n, m, dS.as<float>(), n, h, true, false, us.as<float>());
  gemm<float>(ctx, X, n, m, dD.as<float>(), n, h, true, false, ud.as<float>());
  // d_bias = 1^T G fused into the dTheta GEMMs (column sums of their B = G_t)
  for (int32_t t = 0; t < h; ++t)
    reo_gemm(ctx, Z + (size_t)t * m, n, m, hm, G + (size_t)t * k, n, k, hk, true, false,
             d_theta + (size_t)t * k, hk, nullptr, d_bias + (size_t)t * k);
  g2::k_gat_reorder_grads<<<dim3((unsigned)ceil_div(hk, 32)), 256, 0, st>>>(
      m, h, k, theta, a_src, a_dst, us.as<float>(), ud.as<float>(), d_theta, d_a_src, d_a_dst);
  launched(ctx);
}

// SGNN_GAT_FUSE=0: the forward runs attention and aggregation as two
// kernels (A/B switch; the results are bit-identical either way)
static bool gat_fuse_on() {
  static const bool on = [] {
    const char* e = getenv("SGNN_GAT_FUSE");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class T>
void gat_forward_t(sgnn_ctx ctx, sgnn_pattern p, const T* X, int32_t m, const T* theta,
                   const T* a_src, const T* a_dst, const T* bias, int32_t h, int32_t k,
                   T beta, int level, T* out, sgnn_gat_cache c, uint8_t* elu_mask = nullptr,
                   bool* elu_fused = nullptr, bool reorder = false) {
  const int32_t n = p->n;
  const int64_t q = p->nnz;
  const int32_t hk = h * k;
  cudaStream_t st = ctx->stream;
  if constexpr (sizeof(T) == 4) {
    if (reorder && reorder_shape_ok(n, m, h, k) && al16(X) && al16(theta) && al16(a_src) &&
        al16(a_dst) && al16(bias) && al16(out) &&
        long_rows(ctx, p->long_rows, n, p->rowptr.as<int32_t>()).nlong == 0) {
      gat_forward_reordered(ctx, p, X, m, theta, a_src, a_dst, bias, h, k, beta, level, out, c,
                            elu_mask, elu_fused);
      return;
    }
  }
  DevBuf M((size_t)n * hk * sizeof(T), st), s((size_t)n * h * sizeof(T) + 8, st),
      d((size_t)n * h * sizeof(T) + 8, st), alpha, mask;
  const int32_t* rp = p->rowptr.as<int32_t>();
  const int32_t* ci = p->cols.as<int32_t>();
  const int R = fast_R<T>(h, k);
  const int R2 = v2_R<T>(h, k);
  const bool v2 = R2 && al16(out) && al16(bias) && al16(a_src) && al16(a_dst);
  bool scored = false;  // node scores fused into the X.Theta epilogue (whole heads per tile)
  if constexpr (sizeof(T) == 4)
    if (v2)
      scored = gemm_scores_f32(ctx, X, n, m, theta, hk, M.as<float>(), a_src, a_dst, h,
                               s.as<float>(), d.as<float>());
  if (!scored) gemm<T>(ctx, X, n, m, theta, m, hk, false, false, M.as<T>());
  if (v2) {
    if (scored) {
    } else if (R) {
      node_scores_fast<T>(ctx, R, n, h, k, M.as<T>(), a_src, a_dst, s.as<T>(), d.as<T>());
    } else {
      node_scores<T>(ctx, n, h, k, M.as<T>(), a_src, a_dst, s.as<T>(), d.as<T>());
    }
    const float4* M4 = reinterpret_cast<const float4*>(M.get());
    const float4* b4 = reinterpret_cast<const float4*>(bias);
    float4* o4 = reinterpret_cast<float4*>(out);
    const float* sp = reinterpret_cast<const float*>(s.get());
    const float* dp = reinterpret_cast<const float*>(d.get());
    DevBuf alpha_tmp;
    float* ap;
    uint8_t* mp = nullptr;
    if (level == SGNN_GAT_FULL) {
      alpha = DevBuf((size_t)q * h * sizeof(T) + 16, st);
      mask = DevBuf((size_t)q * h + 16, st);
      ap = alpha.as<float>();
      mp = mask.as<uint8_t>();
    } else {
      alpha_tmp = DevBuf((size_t)q * h * sizeof(T) + 16, st);
      ap = alpha_tmp.as<float>();
    }
    const LongRows& pr = long_rows(ctx, p->long_rows, n, rp);
    g2::SegArgs sk = skip_long(pr);
    if (elu_mask && pr.nlong == 0) {  // ELU in the aggregation epilogue (no hub combine)
      sk.elu_mask = elu_mask;
      if (elu_fused) *elu_fused = true;
    }
    if (v2_windows<T>(h, k) == 1 && gat_fuse_on()) {
      // attention + aggregation of the hub-free rows in one kernel
      // (bit-identical to k_gat_attn4 + k_gat_agg2; SGNN_GAT_FUSE=0 splits them)
      HR_SWITCH(h, R2, (g2::k_gat_attnagg<HH, RR><<<(unsigned)ceil_div(n, 16), 256, 0, st>>>(
                           n, rp, ci, sp, dp, (float)beta, ap, mp, M4, k, b4, o4, sk)));
      launched(ctx);
      if (pr.nlong) {  // hub rows: a block per row
        HR_SWITCH(h, 1, (g2::k_gat_attn_long<HH><<<pr.nlong, 256, 0, st>>>(
                            pr.long_row.as<int32_t>(), rp, ci, sp, dp, (float)beta, ap, mp)));
        launched(ctx);
      }
    } else {
      HR_SWITCH(h, R2, (g2::k_gat_attn4<HH><<<g2::sub_grid(n), 256, 0, st>>>(
                           n, rp, ci, sp, dp, (float)beta, ap, mp, sk.longest)));
      launched(ctx);
      if (pr.nlong) {  // hub rows: a block per row
        HR_SWITCH(h, 1, (g2::k_gat_attn_long<HH><<<pr.nlong, 256, 0, st>>>(
                            pr.long_row.as<int32_t>(), rp, ci, sp, dp, (float)beta, ap, mp)));
        launched(ctx);
      }
      HR_SWITCH(h, R2, (g2::k_gat_agg2<HH, RR><<<dim3(v2_grid(n), v2_windows<T>(h, k)), 256, 0, st>>>(n, rp, ci, ap, M4, k,
                                                                          b4, o4, sk)));
      launched(ctx);
    }
    if (pr.nlong) {  // hub rows: segment partials, combined in order (+ bias)
      DevBuf part((size_t)pr.nseg * hk * sizeof(float), st);
      HR_SWITCH(h, R2, (g2::k_gat_agg2<HH, RR, true><<<dim3(v2_grid(pr.nseg), v2_windows<T>(h, k)), 256, 0, st>>>(
                           pr.nseg, rp, ci, ap, M4, k, b4, o4, seg_args(pr, part.as<float>()))));
      launched(ctx);
      spmm_combine(ctx, pr, part.as<float>(), hk, reinterpret_cast<float*>(out),
                   reinterpret_cast<const float*>(bias), hk);
    }
  } else if (R && al16(M.get()) && al16(out) && al16(bias) && al16(a_src) && al16(a_dst)) {
    constexpr int VW = sizeof(T) == 4 ? 4 : 2;
    constexpr int wpb = gf::WPB<T>::v;
    node_scores_fast<T>(ctx, R, n, h, k, M.as<T>(), a_src, a_dst, s.as<T>(), d.as<T>());
    if (level == SGNN_GAT_FULL) {
      alpha = DevBuf((size_t)q * h * sizeof(T) + 8, st);
      mask = DevBuf((size_t)q * h + 8, st);
      R_SWITCH(R, (gf::k_gat_fwd_fast<T, VW, RR, 8, true><<<wgrid<T>(n), 32 * wpb, 0, st>>>(
                      n, rp, ci, M.as<T>(), s.as<T>(), d.as<T>(), h, k, beta, bias, out,
                      alpha.as<T>(), mask.as<uint8_t>())));
    } else {
      R_SWITCH(R, (gf::k_gat_fwd_fast<T, VW, RR, 8, false><<<wgrid<T>(n), 32 * wpb, 0, st>>>(
                      n, rp, ci, M.as<T>(), s.as<T>(), d.as<T>(), h, k, beta, bias, out,
                      (T*)nullptr, (uint8_t*)nullptr)));
    }
    launched(ctx);
  } else if (level == SGNN_GAT_FULL) {
    node_scores<T>(ctx, n, h, k, M.as<T>(), a_src, a_dst, s.as<T>(), d.as<T>());
    alpha = DevBuf((size_t)q * h * sizeof(T) + 8, st);
    mask = DevBuf((size_t)q * h + 8, st);
    launch_fwd<T, true, true>(ctx, n, rp, ci, M.as<T>(), s.as<T>(), d.as<T>(), h, k, beta, bias,
                              out, alpha.as<T>(), mask.as<uint8_t>());
  } else {
    node_scores<T>(ctx, n, h, k, M.as<T>(), a_src, a_dst, s.as<T>(), d.as<T>());
    launch_fwd<T, false, true>(ctx, n, rp, ci, M.as<T>(), s.as<T>(), d.as<T>(), h, k, beta,
                               bias, out, nullptr, nullptr);
  }
  // reclassify retained buffers into the cache (gat.hpp:123-137); charged
  // with the reference's sizes (cost.hpp:236-248 footprint)
  c->saved_input = X;
  c->q = q;
  if (level >= SGNN_GAT_FEATURES) {
    c->M = std::move(M);
    c->M.track(kCache, (size_t)n * hk * sizeof(T));
  }
  if (level == SGNN_GAT_NODE_ATTENTION) {
    c->s = std::move(s);
    c->d = std::move(d);
    c->s.track(kCache, (size_t)n * h * sizeof(T));
    c->d.track(kCache, (size_t)n * h * sizeof(T));
  }
  if (level == SGNN_GAT_FULL) {
    c->alpha = std::move(alpha);
    c->mask = std::move(mask);
    c->alpha.track(kCache, (size_t)q * h * sizeof(T));
    c->mask.track(kCache, (size_t)q * h);
  }
}

// gat.hpp:150-170 gat_recompute of the pieces the level did not keep
template <class T>
struct Recomputed {
  DevBuf M, s, d;
  const T* Mp = nullptr;
  const T* sp = nullptr;
  const T* dp = nullptr;
};

template <class T>
static void recompute(sgnn_ctx ctx, sgnn_pattern p, sgnn_gat_cache c, const T* theta,
                      const T* a_src, const T* a_dst, Recomputed<T>& r) {
  const int32_t n = p->n, h = c->h, k = c->k, hk = h * k;
  cudaStream_t st = ctx->stream;
  if (c->level >= SGNN_GAT_FEATURES) {
    r.Mp = c->M.as<T>();
  } else {
    r.M = DevBuf((size_t)n * hk * sizeof(T), st);
    bool scored = false;
    if constexpr (sizeof(T) == 4) {  // level none: M and s, d from one GEMM
      if (v2_R<T>(h, k) && al16(a_src) && al16(a_dst)) {
        r.s = DevBuf((size_t)n * h * sizeof(T) + 8, st);
        r.d = DevBuf((size_t)n * h * sizeof(T) + 8, st);
        scored = gemm_scores_f32(ctx, static_cast<const float*>(c->saved_input), n, c->m, theta,
                                 hk, r.M.template as<float>(), a_src, a_dst, h,
                                 r.s.template as<float>(), r.d.template as<float>());
      }
    }
    if (!scored)
      gemm<T>(ctx, static_cast<const T*>(c->saved_input), n, c->m, theta, c->m, hk, false, false,
              r.M.template as<T>());
    r.Mp = r.M.template as<T>();
    if (scored) {
      r.sp = r.s.template as<T>();
      r.dp = r.d.template as<T>();
      return;
    }
  }
  if (c->level == SGNN_GAT_FULL) return;
  if (c->level == SGNN_GAT_NODE_ATTENTION) {
    r.sp = c->s.as<T>();
    r.dp = c->d.as<T>();
  } else {
    r.s = DevBuf((size_t)n * h * sizeof(T) + 8, st);
    r.d = DevBuf((size_t)n * h * sizeof(T) + 8, st);
    const int R = fast_R<T>(h, k);
    if (R && al16(r.Mp) && al16(a_src) && al16(a_dst))
      node_scores_fast<T>(ctx, R, n, h, k, r.Mp, a_src, a_dst, r.s.template as<T>(),
                          r.d.template as<T>());
    else
      node_scores<T>(ctx, n, h, k, r.Mp, a_src, a_dst, r.s.template as<T>(), r.d.template as<T>());
    r.sp = r.s.template as<T>();
    r.dp = r.d.template as<T>();
  }
}

template <class T>
void gat_backward_t(sgnn_ctx ctx, sgnn_pattern p, const T* G, const T* theta, const T* a_src,
                    const T* a_dst, sgnn_gat_cache c, bool fg, T* d_theta, T* d_a_src,
                    T* d_a_dst, T* d_bias, T* d_input, const uint8_t* elu_mask = nullptr,
                    const T* elu_saved = nullptr, bool* elu_fused = nullptr) {
  // d_input = dM Theta^T, with the ELU(1) backward of the layer below fused
  // into the GEMM epilogue when asked for and the tcgen05 path applies
  auto dx_gemm = [&](const T* dM) {
    if constexpr (sizeof(T) == 4) {
      if (elu_mask && elu_saved &&
          gemm_elu_bwd_f32(ctx, dM, c->n, c->h * c->k, theta, c->m, c->h * c->k, false, true,
                           d_input, elu_mask, elu_saved)) {
        if (elu_fused) *elu_fused = true;
        return;
      }
    }
    gemm<T>(ctx, dM, c->n, c->h * c->k, theta, c->m, c->h * c->k, false, true, d_input);
  };
  if constexpr (sizeof(T) == 4) {
    if (c->reordered) {
      gat_backward_reordered(ctx, p, G, theta, a_src, a_dst, c, fg, d_theta, d_a_src, d_a_dst,
                             d_bias, d_input);
      return;
    }
  }
  const int32_t n = p->n, h = c->h, k = c->k, hk = h * k, m = c->m;
  const int64_t q = p->nnz;
  const T beta = (T)c->beta;
  cudaStream_t st = ctx->stream;
  const int R2 = v2_R<T>(h, k);
  const bool v2 = R2 && al16(G) && al16(a_src) && al16(a_dst);
  if (!v2) column_sums<T>(ctx, G, n, hk, d_bias);  // v2: fused with the attention grads
  Recomputed<T> r;
  recompute<T>(ctx, p, c, theta, a_src, a_dst, r);
  const bool cached = c->level == SGNN_GAT_FULL;
  DevBuf alpha_t, mask_t, da((size_t)q * h * sizeof(T) + 8, st), dy((size_t)q * h * sizeof(T) + 8, st),
      dS((size_t)n * h * sizeof(T) + 8, st), dD((size_t)n * h * sizeof(T) + 8, st),
      dM((size_t)n * hk * sizeof(T), st);
  if (!cached) {
    alpha_t = DevBuf((size_t)q * h * sizeof(T) + 8, st);
    mask_t = DevBuf((size_t)q * h + 8, st);
  }
  const T* alpha = cached ? c->alpha.as<T>() : alpha_t.as<T>();
  if (v2) {  // M, dM come from the 256-byte-aligned pool / cache
    const int32_t* rp = p->rowptr.as<int32_t>();
    const int32_t* ci = p->cols.as<int32_t>();
    const float4* M4 = reinterpret_cast<const float4*>(r.Mp);
    const float4* G4 = reinterpret_cast<const float4*>(G);
    const float* sp = reinterpret_cast<const float*>(r.sp);
    const float* dp = reinterpret_cast<const float*>(r.dp);
    const LongRows& pr = long_rows(ctx, p->long_rows, n, rp);
    const LongRows& pc = long_rows(ctx, p->long_cols, n, p->colptr.as<int32_t>());
    const g2::SegArgs sk = skip_long(pr), skc = skip_long(pc);
    if (!cached) {  // attention + mask recomputed like gat_recompute (gat.hpp:150-170)
      HR_SWITCH(h, R2, (g2::k_gat_attn4<HH><<<g2::sub_grid(n), 256, 0, st>>>(
                           n, rp, ci, sp, dp, (float)beta, alpha_t.as<float>(),
                           mask_t.as<uint8_t>(), sk.longest)));
      launched(ctx);
      if (pr.nlong) {
        HR_SWITCH(h, 1, (g2::k_gat_attn_long<HH><<<pr.nlong, 256, 0, st>>>(
                            pr.long_row.as<int32_t>(), rp, ci, sp, dp, (float)beta,
                            alpha_t.as<float>(), mask_t.as<uint8_t>())));
        launched(ctx);
      }
    }
    const float* al = reinterpret_cast<const float*>(alpha);
    const uint8_t* mk = cached ? c->mask.as<uint8_t>() : mask_t.as<uint8_t>();
    const int L = k / 4;
    const unsigned wn = v2_windows<T>(h, k);
    const int smode = sddmm_mode(L, R2);
    // SDDMM + softmax backward of the hub-free rows in one kernel when the
    // head dots reduce in registers (bit-identical to k_gat_sddmm2 +
    // k_gat_sbwd4; SGNN_GAT_FUSE=0 splits them)
    const bool fuse = wn == 1 && smode >= 1 && gat_fuse_on();
    // fused path: the softmax backward writes (alpha, dy) records at each
    // edge's CSC position, so the column pass reads them sequentially
    // instead of through perm (bit-identical values and order)
    const int32_t* pinv = fuse ? pattern_pinv(ctx, p) : nullptr;
    const bool use_rec = pinv != nullptr;
    DevBuf rec(use_rec ? (size_t)q * 2 * h * sizeof(float) + 16 : 0, st);
    if (fuse) {
      HR_SWITCH(h, R2, (sddmm_sbwd_launch<HH, RR>(smode, st, n, rp, ci, M4, G4, k, al, mk, beta,
                                                  da.as<float>(), dy.as<float>(), dS.as<float>(),
                                                  sk, rec.as<float>(), pinv)));
    } else {
      HR_SWITCH(h, R2, (sddmm2_launch<HH, RR, false>(smode, dim3(v2_grid(n), wn), st, n, rp, ci,
                                                     M4, G4, k, da.as<float>(), sk)));
    }
    if (pr.nlong)  // hub rows: per-edge outputs, segments write them directly
      HR_SWITCH(h, R2, (sddmm2_launch<HH, RR, true>(smode, dim3(v2_grid(pr.nseg), wn), st, pr.nseg,
                                                    rp, ci, M4, G4, k, da.as<float>(), seg_args(pr))));
    launched(ctx);
    if (!fuse) {
      HR_SWITCH(h, R2, (g2::k_gat_sbwd4<HH><<<g2::sub_grid(n), 256, 0, st>>>(
                           n, rp, al, mk, da.as<float>(), (float)beta, dy.as<float>(),
                           dS.as<float>(), sk.longest)));
      launched(ctx);
    }
    if (pr.nlong) {
      HR_SWITCH(h, 1, (g2::k_gat_sbwd_long<HH><<<pr.nlong, 256, 0, st>>>(
                          pr.long_row.as<int32_t>(), rp, al, mk, da.as<float>(), (float)beta,
                          dy.as<float>(), dS.as<float>(), nullptr,
                          rec.as<float>(), pinv)));
      launched(ctx);
    }
    const int32_t* cpp = p->colptr.as<int32_t>();
    const int32_t* crw = p->rows.as<int32_t>();
    const int32_t* prm = p->perm.as<int32_t>();
    const float4* as4 = reinterpret_cast<const float4*>(a_src);
    const float4* ad4 = reinterpret_cast<const float4*>(a_dst);
    float4* dM4 = reinterpret_cast<float4*>(dM.get());
    // alpha / dy of the column pass: the interleaved CSC records (fused path)
    // or the edge-major arrays read through perm
    const float* cal = use_rec ? rec.as<float>() : al;
    const float* cdy = use_rec ? nullptr : dy.as<float>();
    if (use_rec) {
      HR_SWITCH(h, R2, (g2::k_gat_col2<HH, RR, false, true><<<dim3(v2_grid(n), wn), 256, 0, st>>>(
                           n, cpp, crw, prm, G4, cal, cdy, dS.as<float>(), as4, ad4, k,
                           dD.as<float>(), dM4, skc)));
    } else {
      HR_SWITCH(h, R2, (g2::k_gat_col2<HH, RR><<<dim3(v2_grid(n), wn), 256, 0, st>>>(
                           n, cpp, crw, prm, G4, cal, cdy, dS.as<float>(), as4, ad4, k,
                           dD.as<float>(), dM4, skc)));
    }
    launched(ctx);
    if (pc.nlong) {  // hub columns: segment partials + in-order combine
      DevBuf part((size_t)pc.nseg * hk * sizeof(float), st), ddp((size_t)pc.nseg * h * 4, st);
      if (use_rec) {
        HR_SWITCH(h, R2, (g2::k_gat_col2<HH, RR, true, true><<<dim3(v2_grid(pc.nseg), wn), 256, 0, st>>>(
                             pc.nseg, cpp, crw, prm, G4, cal, cdy, dS.as<float>(), as4, ad4, k,
                             dD.as<float>(), dM4, seg_args(pc, part.as<float>(), ddp.as<float>()))));
      } else {
        HR_SWITCH(h, R2, (g2::k_gat_col2<HH, RR, true><<<dim3(v2_grid(pc.nseg), wn), 256, 0, st>>>(
                             pc.nseg, cpp, crw, prm, G4, cal, cdy, dS.as<float>(), as4, ad4, k,
                             dD.as<float>(), dM4, seg_args(pc, part.as<float>(), ddp.as<float>()))));
      }
      launched(ctx);
      HR_SWITCH(h, 1, (g2::k_gat_col_combine<HH><<<v2_grid(pc.nlong), 256, 0, st>>>(
                          pc.nlong, pc.long_row.as<int32_t>(), pc.long_first.as<int32_t>(),
                          part.as<float4>(), ddp.as<float>(), dS.as<float>(), as4, ad4, k,
                          dD.as<float>(), dM4)));
      launched(ctx);
    }
    // dTheta = X^T dM on the side stream, overlapped with the attention
    // gradients and dX = dM Theta^T here (independent consumers of dM)
    SideStream side(ctx);
    side.side();
    gemm<T>(ctx, static_cast<const T*>(c->saved_input), n, m, dM.as<T>(), n, hk, true, false,
            d_theta);
    side.main();
    {  // d_bias, d_a_src, d_a_dst: one pass over dX' and M
      const int32_t nb = std::max<int32_t>(1, std::min<int32_t>(4 * ctx->num_sms, n));
      const int32_t chunk = (int32_t)ceil_div(n, nb);
      DevBuf part((size_t)nb * 3 * hk * sizeof(double), st);
      switch (h) {
        case 1: g2::k_grads3_partial<1><<<dim3(nb, (unsigned)ceil_div(hk / 4, 256)), 256, 0, st>>>(n, k, G4, M4, dS.as<float>(), dD.as<float>(), chunk, part.as<double>()); break;
        case 2: g2::k_grads3_partial<2><<<dim3(nb, (unsigned)ceil_div(hk / 4, 256)), 256, 0, st>>>(n, k, G4, M4, dS.as<float>(), dD.as<float>(), chunk, part.as<double>()); break;
        case 4: g2::k_grads3_partial<4><<<dim3(nb, (unsigned)ceil_div(hk / 4, 256)), 256, 0, st>>>(n, k, G4, M4, dS.as<float>(), dD.as<float>(), chunk, part.as<double>()); break;
        default: g2::k_grads3_partial<8><<<dim3(nb, (unsigned)ceil_div(hk / 4, 256)), 256, 0, st>>>(n, k, G4, M4, dS.as<float>(), dD.as<float>(), chunk, part.as<double>()); break;
      }
      launched(ctx);
      g2::k_grads3_final_col<<<dim3((unsigned)hk, 3), 256, 0, st>>>(
          nb, hk, part.as<double>(), reinterpret_cast<float*>(d_bias),
          reinterpret_cast<float*>(d_a_src), reinterpret_cast<float*>(d_a_dst));
      launched(ctx);
    }
    if (fg) dx_gemm(dM.as<T>());
    side.join();
    return;
  }
  {
    const int R = fast_R<T>(h, k);
    if (R && al16(G) && al16(r.Mp) && al16(dM.get()) && al16(a_src) && al16(a_dst)) {
      constexpr int VW = sizeof(T) == 4 ? 4 : 2;
      constexpr int wpb = gf::WPB<T>::v;
      const int32_t* rp = p->rowptr.as<int32_t>();
      const int32_t* ci = p->cols.as<int32_t>();
      if (cached) {
        R_SWITCH(R, (gf::k_gat_bwd_row_fast<T, VW, RR, 8, true><<<wgrid<T>(n), 32 * wpb, 0, st>>>(
                        n, rp, ci, r.Mp, r.sp, r.dp, G, h, k, beta, c->alpha.as<T>(),
                        c->mask.as<uint8_t>(), (T*)nullptr, da.as<T>(), dy.as<T>(), dS.as<T>())));
      } else {
        R_SWITCH(R, (gf::k_gat_bwd_row_fast<T, VW, RR, 8, false><<<wgrid<T>(n), 32 * wpb, 0, st>>>(
                        n, rp, ci, r.Mp, r.sp, r.dp, G, h, k, beta, (const T*)nullptr,
                        (const uint8_t*)nullptr, alpha_t.as<T>(), da.as<T>(), dy.as<T>(),
                        dS.as<T>())));
      }
      launched(ctx);
      R_SWITCH(R, (gf::k_gat_bwd_col_fast<T, VW, RR><<<wgrid<T>(n), 32 * wpb, 0, st>>>(
                      n, p->colptr.as<int32_t>(), p->rows.as<int32_t>(), p->perm.as<int32_t>(),
                      G, alpha, dy.as<T>(), dS.as<T>(), a_src, a_dst, h, k, dD.as<T>(),
                      dM.as<T>())));
      launched(ctx);
      // attention-parameter gradients: one pass over M for a_src and a_dst
      const int32_t chunk = (int32_t)std::max<int64_t>(64, ceil_div(n, ctx->num_sms * 4));
      const int32_t nch = (int32_t)std::max<int64_t>(1, ceil_div(n, chunk));
      DevBuf psrc((size_t)nch * hk * 8, st), pdst((size_t)nch * hk * 8, st);
      gf::k_attgrad2_partial<T, VW><<<nch, 256, 0, st>>>(n, h, k, r.Mp, dS.as<T>(), dD.as<T>(), chunk,
                                                    psrc.as<double>(), pdst.as<double>());
      launched(ctx);
      gf::k_reduce_partials<T><<<(unsigned)ceil_div(hk, 32), 256, 0, st>>>(nch, hk,
                                                                        psrc.as<double>(), d_a_src);
      launched(ctx);
      gf::k_reduce_partials<T><<<(unsigned)ceil_div(hk, 32), 256, 0, st>>>(nch, hk,
                                                                        pdst.as<double>(), d_a_dst);
      launched(ctx);
      gemm<T>(ctx, static_cast<const T*>(c->saved_input), n, m, dM.as<T>(), n, hk, true, false,
              d_theta);
      if (fg) dx_gemm(dM.as<T>());
      return;
    }
  }
  const int32_t* rp = p->rowptr.as<int32_t>();
  const int32_t* ci = p->cols.as<int32_t>();
  constexpr int VW = sizeof(T) == 4 ? 4 : 2;
  const bool vec = k % VW == 0 && reinterpret_cast<uintptr_t>(G) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(r.Mp) % 16 == 0;
  const int g = rows_grid<T>(ctx, n);
#define ROW(W, CACHED)                                                                        \
  k_gat_bwd_row<T, W, CACHED><<<g, 256, 0, st>>>(n, rp, ci, r.Mp, r.sp, r.dp, G, h, k, beta,  \
                                                c->alpha.as<T>(), c->mask.as<uint8_t>(),       \
                                                alpha_t.as<T>(), mask_t.as<uint8_t>(),        \
                                                da.as<T>(), dy.as<T>(), dS.as<T>())
  if (vec) {
    if (cached) ROW(VW, true); else ROW(VW, false);
  } else {
    if (cached) ROW(1, true); else ROW(1, false);
  }
#undef ROW
  launched(ctx);
  // column pass over the CSC view
  const int32_t* cp = p->colptr.as<int32_t>();
  const int32_t* cr = p->rows.as<int32_t>();
  const int32_t* pm = p->perm.as<int32_t>();
  const bool cvec = vec && reinterpret_cast<uintptr_t>(dM.get()) % 16 == 0;
  const int W = cvec ? VW : 1;
  const int R = pick_r(hk / W);
#define COL(WW, RR)                                                                            \
  k_gat_bwd_col<T, WW, RR><<<g, 256, 0, st>>>(n, cp, cr, pm, G, alpha, dy.as<T>(), dS.as<T>(), \
                                             a_src, a_dst, h, k, dD.as<T>(), dM.as<T>())
#define COLR(WW)                    \
  switch (R) {                      \
    case 1: COL(WW, 1); break;      \
    case 2: COL(WW, 2); break;      \
    case 4: COL(WW, 4); break;      \
    case 8: COL(WW, 8); break;      \
    default: COL(WW, 16); break;    \
  }
  if (W == VW) {
    COLR(VW)
  } else {
    COLR(1)
  }
#undef COLR
#undef COL
  launched(ctx);
  att_grad<T>(ctx, n, h, k, r.Mp, dS.as<T>(), d_a_src);
  att_grad<T>(ctx, n, h, k, r.Mp, dD.as<T>(), d_a_dst);
  gemm<T>(ctx, static_cast<const T*>(c->saved_input), n, m, dM.as<T>(), n, hk, true, false,
          d_theta);
  if (fg) dx_gemm(dM.as<T>());
}

template <class T>
void gat_edge_values_t(sgnn_ctx ctx, sgnn_pattern p, sgnn_gat_cache c, const T* theta,
                       const T* a_src, const T* a_dst, T* alpha_hq, uint8_t* mask_hq) {
  const int32_t n = p->n, h = c->h, k = c->k;
  const int64_t q = p->nnz;
  cudaStream_t st = ctx->stream;
  DevBuf al, mk;
  const T* ae;
  const uint8_t* me;
  if constexpr (sizeof(T) == 4) {
    if (c->reordered) {
      DevBuf W((size_t)2 * h * c->m * 4, st);
      reo_wvec(ctx, c->m, h, k, theta, a_src, a_dst, W.as<float>());
      ReoEdges e;
      reo_edges(ctx, p, c, W.as<float>(), e);
      k_edge_to_head_major<T><<<grid_for(ctx, q * h, 256), 256, 0, st>>>(q, h, e.a, e.mk,
                                                                         alpha_hq, mask_hq);
      launched(ctx);
      return;
    }
  }
  if (c->level == SGNN_GAT_FULL) {
    ae = c->alpha.as<T>();
    me = c->mask.as<uint8_t>();
  } else {
    Recomputed<T> r;
    recompute<T>(ctx, p, c, theta, a_src, a_dst, r);
    al = DevBuf((size_t)q * h * sizeof(T) + 8, st);
    mk = DevBuf((size_t)q * h + 8, st);
    launch_fwd<T, true, false>(ctx, n, p->rowptr.as<int32_t>(), p->cols.as<int32_t>(), r.Mp,
                               r.sp, r.dp, h, k, (T)c->beta, nullptr, nullptr, al.as<T>(),
                               mk.as<uint8_t>());
    ae = al.as<T>();
    me = mk.as<uint8_t>();
  }
  k_edge_to_head_major<T><<<grid_for(ctx, q * h, 256), 256, 0, st>>>(q, h, ae, me, alpha_hq,
                                                                     mask_hq);
  launched(ctx);
}

}  // namespace sgnn

using namespace sgnn;

extern "C" {

int sgnn_gat_forward(sgnn_ctx ctx, sgnn_pattern p, const void* X, int32_t m, const void* theta,
                     const void* a_src, const void* a_dst, const void* bias, int32_t heads,
                     int32_t k, double beta, int level, int dtype, void* out,
                     sgnn_gat_cache* cache) {
  return sgnn::gat_forward_elu(ctx, p, X, m, theta, a_src, a_dst, bias, heads, k, beta, level,
                               dtype, out, cache, nullptr, nullptr, false);
}

int sgnn_gat_forward_ex(sgnn_ctx ctx, sgnn_pattern p, const void* X, int32_t m, const void* theta,
                        const void* a_src, const void* a_dst, const void* bias, int32_t heads,
                        int32_t k, double beta, int level, int dtype, void* out,
                        sgnn_gat_cache* cache, int flags) {
  if (flags & ~SGNN_GAT_REORDER) {
    set_last_error("gat_forward_ex: unknown flags");
    return SGNN_EINVAL;
  }
  return sgnn::gat_forward_elu(ctx, p, X, m, theta, a_src, a_dst, bias, heads, k, beta, level,
                               dtype, out, cache, nullptr, nullptr, (flags & SGNN_GAT_REORDER) != 0);
}

int sgnn_gat_cache_reordered(sgnn_gat_cache c, int* out) {
  SGNN_API_BEGIN
  require(c != nullptr && out != nullptr, "gat cache: null argument");
  *out = c->reordered ? 1 : 0;
  SGNN_API_END
}

int sgnn_gat_backward(sgnn_ctx ctx, sgnn_pattern p, const void* d_out, const void* theta,
                      const void* a_src, const void* a_dst, int32_t m, int32_t heads, int32_t k,
                      double beta, sgnn_gat_cache c, int fg, void* d_theta, void* d_a_src,
                      void* d_a_dst, void* d_bias, void* d_input) {
  (void)beta;  // the forward's beta is kept in the cache
  return sgnn::gat_backward_elu(ctx, p, d_out, theta, a_src, a_dst, m, heads, k, c, fg, d_theta,
                                d_a_src, d_a_dst, d_bias, d_input, nullptr, nullptr, nullptr);
}

}  // extern "C"

int sgnn::gat_forward_elu(sgnn_ctx ctx, sgnn_pattern p, const void* X, int32_t m,
                          const void* theta, const void* a_src, const void* a_dst,
                          const void* bias, int32_t heads, int32_t k, double beta, int level,
                          int dtype, void* out, sgnn_gat_cache* cache, uint8_t* elu_mask,
                          bool* fused, bool reorder) {
  if (fused) *fused = false;
  SGNN_API_BEGIN
  require(p && p->all_self_loops, "gat_forward: pattern must contain all self loops");
  require(m >= 1 && heads >= 1 && k >= 1, "gat_forward: input width does not match theta");
  require(beta > 0, "gat_forward: beta must be positive");
  require(heads <= HMAX, "gat_forward: more than 64 heads is not supported on the device");
  require(level >= SGNN_GAT_NONE && level <= SGNN_GAT_FULL, "unknown caching level");
  auto* c = new sgnn_gat_cache_s;
  c->level = level;
  c->dtype = dtype;
  c->n = p->n;
  c->m = m;
  c->h = heads;
  c->k = k;
  c->beta = beta;
  try {
    if (dtype == SGNN_F32)
      gat_forward_t<float>(ctx, p, (const float*)X, m, (const float*)theta, (const float*)a_src,
                           (const float*)a_dst, (const float*)bias, heads, k, (float)beta, level,
                           (float*)out, c, elu_mask, fused, reorder);
    else if (dtype == SGNN_F64)
      gat_forward_t<double>(ctx, p, (const double*)X, m, (const double*)theta,
                            (const double*)a_src, (const double*)a_dst, (const double*)bias,
                            heads, k, beta, level, (double*)out, c);
    else
      throw invalid_argument("unknown dtype");
  } catch (...) {
    delete c;
    throw;
  }
  *cache = c;
  SGNN_API_END
}

int sgnn::gat_backward_elu(sgnn_ctx ctx, sgnn_pattern p, const void* d_out, const void* theta,
                           const void* a_src, const void* a_dst, int32_t m, int32_t heads,
                           int32_t k, sgnn_gat_cache c, int fg, void* d_theta, void* d_a_src,
                           void* d_a_dst, void* d_bias, void* d_input, const uint8_t* elu_mask,
                           const void* elu_saved, bool* fused) {
  if (fused) *fused = false;
  SGNN_API_BEGIN
  require(c != nullptr, "gat_backward: missing saved input");
  require(!c->consumed, "gat_backward: cache already consumed");
  c->consumed = true;  // gat.hpp:177-178
  require(p && p->n == c->n && heads == c->h && k == c->k,
          "gat_backward: gradient shape mismatch");
  require(c->saved_input != nullptr && m == c->m, "gat_backward: missing saved input");
  if (c->level >= SGNN_GAT_FEATURES)
    require((c->reordered ? c->Z.get() : c->M.get()) != nullptr,
            "gat_backward: cache level promises M but it is absent");
  if (c->level == SGNN_GAT_FULL)
    require(c->alpha.get() != nullptr && c->mask.get() != nullptr,
            "gat_backward: cache level promises alpha/mask but they are absent");
  require(!fg || d_input != nullptr, "gat_backward: d_input required for feature gradients");
  if (c->dtype == SGNN_F32)
    gat_backward_t<float>(ctx, p, (const float*)d_out, (const float*)theta,
                          (const float*)a_src, (const float*)a_dst, c, fg != 0,
                          (float*)d_theta, (float*)d_a_src, (float*)d_a_dst, (float*)d_bias,
                          (float*)d_input, elu_mask, (const float*)elu_saved, fused);
  else
    gat_backward_t<double>(ctx, p, (const double*)d_out, (const double*)theta,
                           (const double*)a_src, (const double*)a_dst, c, fg != 0,
                           (double*)d_theta, (double*)d_a_src, (double*)d_a_dst,
                           (double*)d_bias, (double*)d_input);
  SGNN_API_END
}

extern "C" {

int sgnn_gat_cache_destroy(sgnn_gat_cache c) {
  SGNN_API_BEGIN
  delete c;
  SGNN_API_END
}

// device arrays the cache retains (NULL where the level does not keep them):
// M (n x hk), s / d (n x h), alpha / mask edge-major (q x h)
int sgnn_gat_cache_arrays(sgnn_gat_cache c, const void** M, const void** s, const void** d,
                          const void** alpha, const uint8_t** mask) {
  SGNN_API_BEGIN
  require(c != nullptr, "gat cache: null handle");
  if (M) *M = c->M.get();
  if (s) *s = c->s.get();
  if (d) *d = c->d.get();
  if (alpha) *alpha = c->alpha.get();
  if (mask) *mask = c->mask.as<uint8_t>();
  SGNN_API_END
}

int sgnn_gat_cache_extra_bytes(sgnn_gat_cache c, int64_t* out) {
  SGNN_API_BEGIN
  // gat.hpp:66-71: bytes owned beyond the retained input; buffers carry +8
  // bytes of slack for empty shapes, so report the logical sizes.
  const int64_t sb = c->dtype == SGNN_F32 ? 4 : 8;
  int64_t b = 0;
  if (c->M.get()) b += sb * c->n * c->h * c->k;
  if (c->Z.get()) b += sb * c->n * c->h * c->m;  // reordered layer: Z in place of M
  if (c->s.get()) b += 2 * sb * c->n * c->h;
  if (c->alpha.get()) b += (sb + 1) * c->q * c->h;
  *out = b;
  SGNN_API_END
}

int sgnn_gat_cache_edge_values(sgnn_ctx ctx, sgnn_pattern p, sgnn_gat_cache c,
                               const void* theta, const void* a_src, const void* a_dst,
                               void* alpha_hq, uint8_t* mask_hq) {
  SGNN_API_BEGIN
  require(c && p, "gat_cache_edge_values: null argument");
  if (c->dtype == SGNN_F32)
    gat_edge_values_t<float>(ctx, p, c, (const float*)theta, (const float*)a_src,
                             (const float*)a_dst, (float*)alpha_hq, mask_hq);
  else
    gat_edge_values_t<double>(ctx, p, c, (const double*)theta, (const double*)a_src,
                              (const double*)a_dst, (double*)alpha_hq, mask_hq);
  SGNN_API_END
}

int sgnn_edge_softmax(sgnn_ctx ctx, sgnn_pattern p, int32_t heads, const void* w, int dtype,
                      void* alpha) {
  SGNN_API_BEGIN
  require(p && p->all_self_loops, "edge_softmax: pattern must contain all self loops");
  const int64_t total = (int64_t)p->n * heads;
  if (total == 0) return SGNN_OK;
  if (dtype == SGNN_F32)
    k_edge_softmax<float><<<grid_for(ctx, total, 256), 256, 0, ctx->stream>>>(
        p->n, p->rowptr.as<int32_t>(), heads, (const float*)w, (float*)alpha);
  else
    k_edge_softmax<double><<<grid_for(ctx, total, 256), 256, 0, ctx->stream>>>(
        p->n, p->rowptr.as<int32_t>(), heads, (const double*)w, (double*)alpha);
  launched(ctx);
  SGNN_API_END
}

int sgnn_sddmm(sgnn_ctx ctx, sgnn_pattern p, const void* B, int32_t f, const void* C,
               int32_t ldc, int dtype, void* out) {
  SGNN_API_BEGIN
  require(p != nullptr, "sddmm: outer dimension mismatch");
  require(ldc == p->n, "sddmm: outer dimension mismatch");
  if (p->n == 0) return SGNN_OK;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(p->n, 8), 148 * 32));
  if (dtype == SGNN_F32)
    k_sddmm<float><<<grid, 256, 0, ctx->stream>>>(p->n, p->rowptr.as<int32_t>(),
                                                  p->cols.as<int32_t>(), (const float*)B, f,
                                                  (const float*)C, ldc, (float*)out);
  else
    k_sddmm<double><<<grid, 256, 0, ctx->stream>>>(p->n, p->rowptr.as<int32_t>(),
                                                   p->cols.as<int32_t>(), (const double*)B, f,
                                                   (const double*)C, ldc, (double*)out);
  launched(ctx);
  SGNN_API_END
}


// ---------------------------------------------------------------------------
// Kernel-level GAT pieces over row / column blocks (float32, the v2 shapes:
// h in {1,2,4,8}, k % 4 == 0, h*k <= 1024).  They are the reference's kernel
// functions (kernels.hpp) as separate calls so a row-partitioned layer can
// interleave them with NCCL exchanges: column ids index a (gathered) operand
// of any row count, row ids are block-local.  All pointers 16-byte aligned.
// ---------------------------------------------------------------------------
}  // extern "C"

struct sgnn_rowplan_s {
  LongRows plan;
};

static const LongRows* plan_of(sgnn_rowplan rp) {
  return rp && rp->plan.nlong > 0 ? &rp->plan : nullptr;
}

extern "C" {

// hub-row plan of a block CSR (rows longer than 128 edges split into
// segments), for the block entry points below; NULL plans are allowed there
int sgnn_rowplan_create(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr, sgnn_rowplan* out) {
  SGNN_API_BEGIN
  require(ctx && out && (n_rows == 0 || rowptr), "rowplan: null argument");
  auto* p = new sgnn_rowplan_s;
  long_rows(ctx, p->plan, n_rows, rowptr);
  *out = p;
  SGNN_API_END
}

int sgnn_rowplan_destroy(sgnn_rowplan p) {
  SGNN_API_BEGIN
  delete p;
  SGNN_API_END
}

static void block_check(int32_t h, int32_t k) {
  require(v2_R<float>(h, k) != 0, "gat block: needs h in {1,2,4,8}, k % 4 == 0, h*k <= 1024");
}

// node_scores (kernels.hpp:385-423) fused into M = X Theta when whole heads fit
// a GEMM tile (k % 4 == 0, tile width % k == 0)
int sgnn_gat_transform(sgnn_ctx ctx, const float* X, int32_t n_rows, int32_t m,
                       const float* theta, int32_t h, int32_t k, const float* a_src,
                       const float* a_dst, float* M, float* s, float* d) {
  SGNN_API_BEGIN
  block_check(h, k);
  if (n_rows == 0) return SGNN_OK;
  if (!gemm_scores_f32(ctx, X, n_rows, m, theta, h * k, M, a_src, a_dst, h, s, d)) {
    gemm<float>(ctx, X, n_rows, m, theta, m, h * k, false, false, M);
    const int R = fast_R<float>(h, k);
    if (R) node_scores_fast<float>(ctx, R, n_rows, h, k, M, a_src, a_dst, s, d);
    else node_scores<float>(ctx, n_rows, h, k, M, a_src, a_dst, s, d);
  }
  SGNN_API_END
}

// edge_scores + leaky_relu_edges + edge_softmax (kernels.hpp:427-534):
// alpha, mask edge-major (q_local x h) for the block's rows; s block-local,
// d indexed by column id.  row_stats (optional, n_rows x h x 4): s, max and
// 1 / sum per row and head -- what sgnn_gat_column_pass_stats rebuilds alpha
// from on the ranks that own the columns
int sgnn_gat_attention_ex(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr,
                          const int32_t* cols, int32_t h, const float* s, const float* d,
                          double beta, float* alpha, uint8_t* mask, float* row_stats,
                          sgnn_rowplan plan) {
  SGNN_API_BEGIN
  require(beta > 0, "gat_forward: beta must be positive");
  require(h == 1 || h == 2 || h == 4 || h == 8, "gat block: needs h in {1,2,4,8}");
  if (n_rows == 0) return SGNN_OK;
  const LongRows* pl = plan_of(plan);
  HR_SWITCH(h, 1, (g2::k_gat_attn4<HH><<<g2::sub_grid(n_rows), 256, 0, ctx->stream>>>(
                      n_rows, rowptr, cols, s, d, (float)beta, alpha, mask,
                      pl ? kLongRow : 0x7fffffff, row_stats)));
  launched(ctx);
  if (pl) {
    HR_SWITCH(h, 1, (g2::k_gat_attn_long<HH><<<pl->nlong, 256, 0, ctx->stream>>>(
                        pl->long_row.as<int32_t>(), rowptr, cols, s, d, (float)beta, alpha,
                        mask, row_stats)));
    launched(ctx);
  }
  SGNN_API_END
}

int sgnn_gat_attention(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr,
                       const int32_t* cols, int32_t h, const float* s, const float* d,
                       double beta, float* alpha, uint8_t* mask, sgnn_rowplan plan) {
  return sgnn_gat_attention_ex(ctx, n_rows, rowptr, cols, h, s, d, beta, alpha, mask, nullptr,
                               plan);
}

// spmm_semibatched + bias (kernels.hpp:219-254): out rows of the block
int sgnn_gat_aggregate(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr, const int32_t* cols,
                       int32_t h, int32_t k, const float* alpha, const float* M,
                       const float* bias, float* out, sgnn_rowplan plan) {
  SGNN_API_BEGIN
  block_check(h, k);
  if (n_rows == 0) return SGNN_OK;
  const int R2 = v2_R<float>(h, k);
  const LongRows* pl = plan_of(plan);
  const unsigned wn = v2_windows<float>(h, k);
  const float4* M4 = reinterpret_cast<const float4*>(M);
  const float4* b4 = reinterpret_cast<const float4*>(bias);
  float4* o4 = reinterpret_cast<float4*>(out);
  g2::SegArgs sk;
  sk.longest = pl ? kLongRow : 0x7fffffff;
  HR_SWITCH(h, R2, (g2::k_gat_agg2<HH, RR><<<dim3(v2_grid(n_rows), wn), 256, 0, ctx->stream>>>(
                       n_rows, rowptr, cols, alpha, M4, k, b4, o4, sk)));
  launched(ctx);
  if (pl) {
    DevBuf part((size_t)pl->nseg * h * k * 4, ctx->stream);
    HR_SWITCH(h, R2, (g2::k_gat_agg2<HH, RR, true><<<dim3(v2_grid(pl->nseg), wn), 256, 0, ctx->stream>>>(
                         pl->nseg, rowptr, cols, alpha, M4, k, b4, o4,
                         seg_args(*pl, part.as<float>()))));
    launched(ctx);
    spmm_combine(ctx, *pl, part.as<float>(), h * k, out, bias, h * k);
  }
  SGNN_API_END
}

// sddmm_semibatched (kernels.hpp:342-377): dAlpha edge-major for the block's rows
int sgnn_gat_sddmm(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr, const int32_t* cols,
                   int32_t h, int32_t k, const float* M, const float* G, float* da,
                   sgnn_rowplan plan) {
  SGNN_API_BEGIN
  block_check(h, k);
  if (n_rows == 0) return SGNN_OK;
  const int R2 = v2_R<float>(h, k);
  const int L = k / 4;
  const float4* M4 = reinterpret_cast<const float4*>(M);
  const float4* G4 = reinterpret_cast<const float4*>(G);
  const LongRows* pl = plan_of(plan);
  const unsigned wn = v2_windows<float>(h, k);
  g2::SegArgs sk;
  sk.longest = pl ? kLongRow : 0x7fffffff;
  const int smode = sddmm_mode(L, R2);
  HR_SWITCH(h, R2, (sddmm2_launch<HH, RR, false>(smode, dim3(v2_grid(n_rows), wn), ctx->stream,
                                                 n_rows, rowptr, cols, M4, G4, k, da, sk)));
  if (pl)
    HR_SWITCH(h, R2, (sddmm2_launch<HH, RR, true>(smode, dim3(v2_grid(pl->nseg), wn), ctx->stream,
                                                  pl->nseg, rowptr, cols, M4, G4, k, da,
                                                  seg_args(*pl))));
  launched(ctx);
  SGNN_API_END
}

// edge_softmax_backward + leaky_relu_edges_backward + edge_row_sums
// (kernels.hpp:481-495, 537-588).  row_stats (optional): the 4th slot of each
// row gets dot = sum_e alpha dAlpha per head
int sgnn_gat_softmax_backward_ex(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr, int32_t h,
                                 const float* alpha, const uint8_t* mask, const float* da,
                                 double beta, float* dy, float* dS, float* row_stats,
                                 sgnn_rowplan plan) {
  SGNN_API_BEGIN
  require(h == 1 || h == 2 || h == 4 || h == 8, "gat block: needs h in {1,2,4,8}");
  if (n_rows == 0) return SGNN_OK;
  const LongRows* pl = plan_of(plan);
  HR_SWITCH(h, 1, (g2::k_gat_sbwd4<HH><<<g2::sub_grid(n_rows), 256, 0, ctx->stream>>>(
                      n_rows, rowptr, alpha, mask, da, (float)beta, dy, dS,
                      pl ? kLongRow : 0x7fffffff, row_stats)));
  launched(ctx);
  if (pl) {
    HR_SWITCH(h, 1, (g2::k_gat_sbwd_long<HH><<<pl->nlong, 256, 0, ctx->stream>>>(
                        pl->long_row.as<int32_t>(), rowptr, alpha, mask, da, (float)beta, dy,
                        dS, row_stats)));
    launched(ctx);
  }
  SGNN_API_END
}

int sgnn_gat_softmax_backward(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr, int32_t h,
                              const float* alpha, const uint8_t* mask, const float* da,
                              double beta, float* dy, float* dS, sgnn_rowplan plan) {
  return sgnn_gat_softmax_backward_ex(ctx, n_rows, rowptr, h, alpha, mask, da, beta, dy, dS,
                                      nullptr, plan);
}

// spmm_semibatched_transposed + edge_col_sums + add_scaled_rows_inplace
// (kernels.hpp:258-295, 614-658) over a block of columns: colptr / rows /
// perm of the block (rows and perm index the gathered G and alpha / dy)
int sgnn_gat_column_pass(sgnn_ctx ctx, int32_t n_cols, const int32_t* colptr,
                         const int32_t* rows, const int32_t* perm, int32_t h, int32_t k,
                         const float* G, const float* alpha, const float* dy, const float* dS,
                         const float* a_src, const float* a_dst, float* dD, float* dM,
                         sgnn_rowplan plan) {
  SGNN_API_BEGIN
  block_check(h, k);
  if (n_cols == 0) return SGNN_OK;
  const int R2 = v2_R<float>(h, k);
  const LongRows* pl = plan_of(plan);
  const unsigned wn = v2_windows<float>(h, k);
  const float4* G4 = reinterpret_cast<const float4*>(G);
  const float4* as4 = reinterpret_cast<const float4*>(a_src);
  const float4* ad4 = reinterpret_cast<const float4*>(a_dst);
  float4* dM4 = reinterpret_cast<float4*>(dM);
  g2::SegArgs sk;
  sk.longest = pl ? kLongRow : 0x7fffffff;
  HR_SWITCH(h, R2, (g2::k_gat_col2<HH, RR><<<dim3(v2_grid(n_cols), wn), 256, 0, ctx->stream>>>(
                       n_cols, colptr, rows, perm, G4, alpha, dy, dS, as4, ad4, k, dD, dM4, sk)));
  launched(ctx);
  if (pl) {
    DevBuf part((size_t)pl->nseg * h * k * 4, ctx->stream), ddp((size_t)pl->nseg * h * 4, ctx->stream);
    HR_SWITCH(h, R2, (g2::k_gat_col2<HH, RR, true><<<dim3(v2_grid(pl->nseg), wn), 256, 0, ctx->stream>>>(
                         pl->nseg, colptr, rows, perm, G4, alpha, dy, dS, as4, ad4, k, dD, dM4,
                         seg_args(*pl, part.as<float>(), ddp.as<float>()))));
    launched(ctx);
    HR_SWITCH(h, 1, (g2::k_gat_col_combine<HH><<<v2_grid(pl->nlong), 256, 0, ctx->stream>>>(
                        pl->nlong, pl->long_row.as<int32_t>(), pl->long_first.as<int32_t>(),
                        part.as<float4>(), ddp.as<float>(), dS, as4, ad4, k, dD, dM4)));
    launched(ctx);
  }
  SGNN_API_END
}

// 1 when sgnn_gat_column_pass_stats supports (h, k): the v2 shapes whose
// head dot reduces by xor (k/4 a power of two <= 32, or 32C with whole heads
// per lane group)
int sgnn_gat_column_stats_supported(int32_t h, int32_t k) {
  const int R2 = v2_R<float>(h, k);
  return R2 != 0 && R2 != 3 && sddmm_mode(k / 4, R2) != 0 ? 1 : 0;
}

// The column pass of a row-partitioned layer from per-row statistics (see
// g2::k_gat_col3): rows index the gathered dX' (G) and the gathered row_stats
// ([row][head][4]: s, max, 1/sum, dot); d_own / M_own / dS are the block's own
// rows (= its columns).  Replaces shipping alpha and dy (2 q' h values) with
// 4 n h statistics.
int sgnn_gat_column_pass_stats(sgnn_ctx ctx, int32_t n_cols, const int32_t* colptr,
                               const int32_t* rows, int32_t h, int32_t k, const float* G,
                               const float* row_stats, const float* d_own, const float* M_own,
                               double beta, const float* dS, const float* a_src,
                               const float* a_dst, float* dD, float* dM, sgnn_rowplan plan) {
  SGNN_API_BEGIN
  block_check(h, k);
  require(sgnn_gat_column_stats_supported(h, k), "gat block: column statistics need k/4 a power of two <= 32 or a multiple of 32");
  if (n_cols == 0) return SGNN_OK;
  const int R2 = v2_R<float>(h, k);
  const LongRows* pl = plan_of(plan);
  const unsigned wn = v2_windows<float>(h, k);
  const float4* G4 = reinterpret_cast<const float4*>(G);
  const float4* M4 = reinterpret_cast<const float4*>(M_own);
  const float4* as4 = reinterpret_cast<const float4*>(a_src);
  const float4* ad4 = reinterpret_cast<const float4*>(a_dst);
  float4* dM4 = reinterpret_cast<float4*>(dM);
  const float b = (float)beta;
  g2::SegArgs sk;
  sk.longest = pl ? kLongRow : 0x7fffffff;
  HR_SWITCH(h, R2, (g2::k_gat_col3<HH, RR><<<dim3(v2_grid(n_cols), wn), 256, 0, ctx->stream>>>(
                       n_cols, colptr, rows, G4, row_stats, d_own, M4, b, dS, as4, ad4, k, dD,
                       dM4, sk)));
  launched(ctx);
  if (pl) {
    DevBuf part((size_t)pl->nseg * h * k * 4, ctx->stream), ddp((size_t)pl->nseg * h * 4, ctx->stream);
    HR_SWITCH(h, R2, (g2::k_gat_col3<HH, RR, true><<<dim3(v2_grid(pl->nseg), wn), 256, 0, ctx->stream>>>(
                         pl->nseg, colptr, rows, G4, row_stats, d_own, M4, b, dS, as4, ad4, k,
                         dD, dM4, seg_args(*pl, part.as<float>(), ddp.as<float>()))));
    launched(ctx);
    HR_SWITCH(h, 1, (g2::k_gat_col_combine<HH><<<v2_grid(pl->nlong), 256, 0, ctx->stream>>>(
                        pl->nlong, pl->long_row.as<int32_t>(), pl->long_first.as<int32_t>(),
                        part.as<float4>(), ddp.as<float>(), dS, as4, ad4, k, dD, dM4)));
    launched(ctx);
  }
  SGNN_API_END
}

// column_sums (d_bias) + attention_param_grad for a_src / a_dst
// (dense.hpp:272-282, kernels.hpp:592-611) over the block's rows
int sgnn_gat_param_grads(sgnn_ctx ctx, int32_t n_rows, int32_t h, int32_t k, const float* G,
                         const float* M, const float* dS, const float* dD, float* d_bias,
                         float* d_a_src, float* d_a_dst) {
  SGNN_API_BEGIN
  block_check(h, k);
  const int32_t hk = h * k;
  if (n_rows == 0) {
    SGNN_CUDA(cudaMemsetAsync(d_bias, 0, hk * 4, ctx->stream));
    SGNN_CUDA(cudaMemsetAsync(d_a_src, 0, hk * 4, ctx->stream));
    SGNN_CUDA(cudaMemsetAsync(d_a_dst, 0, hk * 4, ctx->stream));
    return SGNN_OK;
  }
  cudaStream_t st = ctx->stream;
  const int32_t nb = std::max<int32_t>(1, std::min<int32_t>(4 * ctx->num_sms, n_rows));
  const int32_t chunk = (int32_t)ceil_div(n_rows, nb);
  DevBuf part((size_t)nb * 3 * hk * sizeof(double), st);
  const float4* G4 = reinterpret_cast<const float4*>(G);
  const float4* M4 = reinterpret_cast<const float4*>(M);
  switch (h) {
    case 1: g2::k_grads3_partial<1><<<dim3(nb, (unsigned)ceil_div(hk / 4, 256)), 256, 0, st>>>(n_rows, k, G4, M4, dS, dD, chunk, part.as<double>()); break;
    case 2: g2::k_grads3_partial<2><<<dim3(nb, (unsigned)ceil_div(hk / 4, 256)), 256, 0, st>>>(n_rows, k, G4, M4, dS, dD, chunk, part.as<double>()); break;
    case 4: g2::k_grads3_partial<4><<<dim3(nb, (unsigned)ceil_div(hk / 4, 256)), 256, 0, st>>>(n_rows, k, G4, M4, dS, dD, chunk, part.as<double>()); break;
    default: g2::k_grads3_partial<8><<<dim3(nb, (unsigned)ceil_div(hk / 4, 256)), 256, 0, st>>>(n_rows, k, G4, M4, dS, dD, chunk, part.as<double>()); break;
  }
  launched(ctx);
  g2::k_grads3_final_col<<<dim3((unsigned)hk, 3), 256, 0, st>>>(
      nb, hk, part.as<double>(), d_bias, d_a_src, d_a_dst);
  launched(ctx);
  SGNN_API_END
}

}  // extern "C"
