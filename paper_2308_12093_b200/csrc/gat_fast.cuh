// gat_fast.cuh -- fast-path GAT kernels (included by gat.cu inside namespace sgnn).
//
// All kernels run one warp per row/column with lanes owning 16-byte column
// vectors of the n x hk slab (vector v = r*32 + lane, columns W*v..W*v+W-1,
// head (W*v)/k), so every gathered M / dX' row is a fully coalesced 128-bit
// load -- the same structure as the lean SpMM.  Per-edge scalars never take
// a dependent global round trip per head:
//   * softmax statistics: lanes over edges (32 per batch), the whole d-row of
//     a neighbour (h scores) in registers, per-head warp max/sum shuffles;
//   * attention during aggregation: each lane recomputes alpha for its own
//     head from s_i, d_j, (max, 1/sum) -- one broadcast 4-byte load + exp;
//   * SDDMM dAlpha: head-segmented xor-shuffle reductions of the per-lane
//     partial dot products.
// Eligible when h <= 16, k % W == 0, k/W a power of two <= 32 or a multiple of
// 32, and hk <= 32*R*W with R <= 8.  Other shapes use the generic kernels.
#pragma once

namespace gf {

constexpr int HF = 16;  // max heads on the fast path

template <class T>
__device__ __forceinline__ T wmax(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const T u = __shfl_xor_sync(0xffffffffu, v, o);
    v = v < u ? u : v;
  }
  return v;
}
template <class T>
__device__ __forceinline__ T wsum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = add_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <class T>
__device__ __forceinline__ T neg_inf();
template <>
__device__ __forceinline__ float neg_inf<float>() {
  return -INFINITY;
}
template <>
__device__ __forceinline__ double neg_inf<double>() {
  return -(double)INFINITY;
}

__device__ __forceinline__ float rcp_rn(float x) { return __frcp_rn(x); }
__device__ __forceinline__ double rcp_rn(double x) { return __drcp_rn(x); }

// Stage w[e][t] = LeakyReLU(s_i,t + d_j,t) for a batch of <= 32 edges (lanes
// over edges, one read of the neighbour's score row per edge).
template <class T, int HT>
__device__ __forceinline__ int32_t stage_scores(int lane, int32_t base, int cnt,
                                                const int32_t* __restrict__ cols,
                                                const T* __restrict__ d,
                                                const T* __restrict__ srow, int h, T beta,
                                                T (*sw)[HT + 1]) {
  int32_t j = 0;
  if (lane < cnt) {
    j = __ldg(cols + base + lane);
    const T* dr = d + (int64_t)j * h;
#pragma unroll
    for (int t = 0; t < HT; ++t)
      if (t < h) {
        bool pos;
        sw[lane][t] = leaky(add_rn(srow[t], dr[t]), beta, pos);
      }
  }
  __syncwarp();
  return j;
}

// Row softmax statistics (kernels.hpp:517-531) in the reference order: lane t
// folds the max, then the sum of exp(w - max), over the row's edges in stored
// order from the staged scores.  Writes smax[t], sinv[t] (= 1/sum).
template <class T, int HT>
__device__ __forceinline__ void row_stats_seq(int lane, int32_t beg, int32_t end,
                                              const int32_t* __restrict__ cols,
                                              const T* __restrict__ d,
                                              const T* __restrict__ srow, int h, T beta,
                                              T (*sw)[HT + 1], T* smax, T* sinv) {
  T m = T(0), sum = T(0);
  for (int32_t base = beg; base < end; base += 32) {
    const int cnt = min(32, end - base);
    if (end - beg > 32 || base == beg) stage_scores<T, HT>(lane, base, cnt, cols, d, srow, h, beta, sw);
    if (lane < h) {
      int e0 = 0;
      if (base == beg) {
        m = sw[0][lane];
        e0 = 1;
      }
      for (int e = e0; e < cnt; ++e) {
        const T w = sw[e][lane];
        m = m < w ? w : m;
      }
    }
    __syncwarp();
  }
  for (int32_t base = beg; base < end; base += 32) {
    const int cnt = min(32, end - base);
    if (end - beg > 32) stage_scores<T, HT>(lane, base, cnt, cols, d, srow, h, beta, sw);
    if (lane < h)
      for (int e = 0; e < cnt; ++e) sum = add_rn(sum, dev_exp<T>(sw[e][lane] - m));
    __syncwarp();
  }
  if (lane < h) {
    smax[lane] = m;
    sinv[lane] = rcp_rn(sum);
  }
  __syncwarp();
}

template <class T>
struct WPB {
  static constexpr int v = 8;
};

// Row softmax statistics (kernels.hpp:517-531) for all heads: smax[t], sinv[t]
// in shared memory.  Lanes over edges; rows of <= 32 edges keep their scores
// in registers (one load of the neighbour's score row per edge); longer rows
// re-read them in a second pass.  With STORE the edge-major alpha and mask of
// cache level `full` are written from the same registers.
template <class T, int HT, bool STORE>
__device__ __forceinline__ void row_stats(int lane, int32_t beg, int32_t end,
                                          const int32_t* __restrict__ cols,
                                          const T* __restrict__ d, const T* __restrict__ srow,
                                          int h, T beta, T* smax, T* sinv,
                                          T* __restrict__ alpha = nullptr,
                                          uint8_t* __restrict__ mask = nullptr) {
  T si[HT], m[HT], sm[HT], w0[HT];
#pragma unroll
  for (int t = 0; t < HT; ++t) {
    si[t] = t < h ? srow[t] : T(0);
    m[t] = neg_inf<T>();
    sm[t] = T(0);
    w0[t] = neg_inf<T>();
  }
  const bool single = end - beg <= 32;
  for (int32_t e = beg + lane; e < end; e += 32) {
    const T* dr = d + (int64_t)__ldg(cols + e) * h;
#pragma unroll
    for (int t = 0; t < HT; ++t)
      if (t < h) {
        bool pos;
        const T w = leaky(add_rn(si[t], dr[t]), beta, pos);
        m[t] = m[t] < w ? w : m[t];
        w0[t] = w;
      }
  }
#pragma unroll
  for (int t = 0; t < HT; ++t)
    if (t < h) m[t] = wmax(m[t]);
  if (single) {
    if (beg + lane < end)
#pragma unroll
      for (int t = 0; t < HT; ++t)
        if (t < h) sm[t] = dev_exp<T>(w0[t] - m[t]);
  } else {
    for (int32_t e = beg + lane; e < end; e += 32) {
      const T* dr = d + (int64_t)__ldg(cols + e) * h;
#pragma unroll
      for (int t = 0; t < HT; ++t)
        if (t < h) {
          bool pos;
          const T w = leaky(add_rn(si[t], dr[t]), beta, pos);
          sm[t] = add_rn(sm[t], dev_exp<T>(w - m[t]));
        }
    }
  }
  T inv[HT];
#pragma unroll
  for (int t = 0; t < HT; ++t)
    if (t < h) {
      inv[t] = T(1) / wsum(sm[t]);
      if (lane == 0) {
        smax[t] = m[t];
        sinv[t] = inv[t];
      }
    }
  if (STORE) {
    for (int32_t e = beg + lane; e < end; e += 32) {
      const T* dr = single ? nullptr : d + (int64_t)__ldg(cols + e) * h;
#pragma unroll
      for (int t = 0; t < HT; ++t)
        if (t < h) {
          T w = w0[t];
          if (!single) {
            bool p2;
            w = leaky(add_rn(si[t], dr[t]), beta, p2);
          }
          // mask records y > 0; for beta > 0 that is w > 0
          alpha[(int64_t)e * h + t] = mul_rn(dev_exp<T>(w - m[t]), inv[t]);
          mask[(int64_t)e * h + t] = w > T(0) ? 1 : 0;
        }
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// node scores s, d (kernels.hpp:385-423): warp per row, coalesced row read,
// head-segmented reduction.
// ---------------------------------------------------------------------------
template <class T, int W, int R>
__global__ void __launch_bounds__(256) k_node_scores_fast(int32_t n, int32_t h, int32_t k,
                                                          const T* __restrict__ M,
                                                          const T* __restrict__ a_src,
                                                          const T* __restrict__ a_dst,
                                                          T* __restrict__ s, T* __restrict__ d) {
  const int lane = threadIdx.x & 31;
  const int32_t i = (int32_t)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (i >= n) return;
  const int32_t hk = h * k;
  const int fv = hk / W, lph = k / W;
  const T* mrow = M + (int64_t)i * hk;
  T ps[R], pd[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int v = r * 32 + lane;
    ps[r] = pd[r] = T(0);
    if (v < fv) {
      T mv[W], as[W], ad[W];
      vload<T, W>(mrow + (int64_t)v * W, mv);
      vload<T, W>(a_src + (int64_t)v * W, as);
      vload<T, W>(a_dst + (int64_t)v * W, ad);
#pragma unroll
      for (int w = 0; w < W; ++w) {
        ps[r] = madd(ps[r], as[w], mv[w]);
        pd[r] = madd(pd[r], ad[w], mv[w]);
      }
    }
  }
  if (lph <= 32) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      for (int o = lph >> 1; o > 0; o >>= 1) {
        ps[r] = add_rn(ps[r], __shfl_xor_sync(0xffffffffu, ps[r], o));
        pd[r] = add_rn(pd[r], __shfl_xor_sync(0xffffffffu, pd[r], o));
      }
      const int v = r * 32 + lane;
      if (v < fv && (lane & (lph - 1)) == 0) {
        s[(int64_t)i * h + v / lph] = ps[r];
        d[(int64_t)i * h + v / lph] = pd[r];
      }
    }
  } else {
    const int cph = lph / 32;  // a head spans cph whole r-chunks
    for (int r0 = 0; r0 < R; r0 += cph) {
      T a = T(0), b = T(0);
      for (int r = r0; r < r0 + cph && r < R; ++r) {
        a = add_rn(a, ps[r]);
        b = add_rn(b, pd[r]);
      }
      a = wsum(a);
      b = wsum(b);
      if (lane == 0 && r0 * 32 < fv) {
        s[(int64_t)i * h + r0 * 32 / lph] = a;
        d[(int64_t)i * h + r0 * 32 / lph] = b;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// forward: scores staged per batch of 32 edges (lanes over edges), softmax
// statistics folded by lanes over heads in stored order, attention computed
// once per (edge, head), then the warp aggregates with two 128-bit M-row
// gathers in flight (32-bit vector offsets), + bias.  STORE writes alpha /
// mask edge-major (cache level full).
// ---------------------------------------------------------------------------
template <class T, int W, int R, int HT, bool STORE>
__global__ void __launch_bounds__(256) k_gat_fwd_fast(int32_t n, const int32_t* __restrict__ rowptr,
                                                      const int32_t* __restrict__ cols,
                                                      const T* __restrict__ M,
                                                      const T* __restrict__ s,
                                                      const T* __restrict__ d, int32_t h,
                                                      int32_t k, T beta,
                                                      const T* __restrict__ bias,
                                                      T* __restrict__ out, T* __restrict__ alpha,
                                                      uint8_t* __restrict__ mask) {
  using VT = typename V<T, W>::t;
  __shared__ T sh_max[8][HT], sh_inv[8][HT];
  __shared__ T sh_w[8][32][HT + 1];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t i = (int32_t)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (i >= n) return;
  const int32_t hk = h * k, fv = hk / W;
  const int32_t beg = rowptr[i], end = rowptr[i + 1];
  const T* srow = s + (int64_t)i * h;
  T (*sw)[HT + 1] = sh_w[wib];
  row_stats_seq<T, HT>(lane, beg, end, cols, d, srow, h, beta, sw, sh_max[wib], sh_inv[wib]);
  const VT* Mv = reinterpret_cast<const VT*>(M);
  int tr[R];
  T acc[R][W];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int v = r * 32 + lane;
    tr[r] = v < fv ? (v * W) / k : 0;
#pragma unroll
    for (int w = 0; w < W; ++w) acc[r][w] = T(0);
  }
  const bool multi = end - beg > 32;
  for (int32_t base = beg; base < end; base += 32) {
    const int cnt = min(32, end - base);
    int32_t mycol;
    if (multi) mycol = stage_scores<T, HT>(lane, base, cnt, cols, d, srow, h, beta, sw);
    else mycol = lane < cnt ? __ldg(cols + base + lane) : 0;
    // attention of every head for the lane's edge, in place over the scores
    if (lane < cnt) {
      const int32_t e = base + lane;
      uint32_t mb = 0;
#pragma unroll
      for (int t = 0; t < HT; ++t)
        if (t < h) {
          const T w = sw[lane][t];
          const T a = mul_rn(dev_exp<T>(w - sh_max[wib][t]), sh_inv[wib][t]);
          sw[lane][t] = a;
          if (w > T(0)) mb |= 1u << t;  // y > 0 <=> w > 0 (beta > 0)
        }
      if (STORE)
#pragma unroll
        for (int t = 0; t < HT; ++t)
          if (t < h) mask[(int64_t)e * h + t] = (mb >> t) & 1u;
    }
    __syncwarp();
    if (STORE)  // edge-major alpha of the batch: one contiguous, coalesced span
      for (int x = lane; x < cnt * h; x += 32) alpha[(int64_t)base * h + x] = sw[x / h][x % h];
    for (int eb = 0; eb < cnt; eb += 2) {
      const bool two = eb + 1 < cnt;
      const uint32_t o0 = (uint32_t)__shfl_sync(0xffffffffu, mycol, eb) * (uint32_t)fv;
      const uint32_t o1 =
          (uint32_t)__shfl_sync(0xffffffffu, mycol, two ? eb + 1 : eb) * (uint32_t)fv;
      VT m0[R], m1[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t v = r * 32 + lane;
        if (v < (uint32_t)fv) {
          m0[r] = __ldg(Mv + o0 + v);
          if (two) m1[r] = __ldg(Mv + o1 + v);
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int v = r * 32 + lane;
        if (v < fv) {
          const T a0 = sw[eb][tr[r]];
          const T* q0 = reinterpret_cast<const T*>(&m0[r]);
#pragma unroll
          for (int q = 0; q < W; ++q) acc[r][q] = madd(acc[r][q], a0, q0[q]);
          if (two) {
            const T a1 = sw[eb + 1][tr[r]];
            const T* q1 = reinterpret_cast<const T*>(&m1[r]);
#pragma unroll
            for (int q = 0; q < W; ++q) acc[r][q] = madd(acc[r][q], a1, q1[q]);
          }
        }
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int v = r * 32 + lane;
    if (v < fv) {
      T b[W], o[W];
      vload<T, W>(bias + (int64_t)v * W, b);
#pragma unroll
      for (int q = 0; q < W; ++q) o[q] = add_rn(acc[r][q], b[q]);
      vstore<T, W>(out + (int64_t)i * hk + (int64_t)v * W, o);
    }
  }
}

// ---------------------------------------------------------------------------
// backward, per destination row (kernels.hpp:342-377, 481-495, 537-588).
// Per batch of 32 edges: attention per (edge, head) staged in smem (cached, or
// recomputed like gat_recompute), dAlpha from two 128-bit M-row gathers in
// flight and head-segmented xor reductions; lanes over heads fold the softmax
// dot and the row sums dS in stored edge order.  Rows longer than 32 edges
// spill alpha / dAlpha to global scratch between the two passes.
// ---------------------------------------------------------------------------
template <class T, int W, int R, int HT, bool CACHED>
__global__ void __launch_bounds__(256) k_gat_bwd_row_fast(
    int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
    const T* __restrict__ M, const T* __restrict__ s, const T* __restrict__ d,
    const T* __restrict__ G, int32_t h, int32_t k, T beta, const T* __restrict__ alpha_in,
    const uint8_t* __restrict__ mask_in, T* __restrict__ alpha_out, T* __restrict__ da,
    T* __restrict__ dy, T* __restrict__ dS) {
  using VT = typename V<T, W>::t;
  __shared__ T sh_max[8][HT], sh_inv[8][HT], sh_dot[8][HT];
  __shared__ T sh_w[8][32][HT + 1];
  __shared__ T sh_da[8][32][HT + 1];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t i = (int32_t)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (i >= n) return;
  const int32_t hk = h * k, fv = hk / W, lph = k / W;
  const int32_t beg = rowptr[i], end = rowptr[i + 1];
  const T* srow = s + (int64_t)i * h;
  T (*sw)[HT + 1] = sh_w[wib];
  T (*sd)[HT + 1] = sh_da[wib];
  const bool multi = end - beg > 32;
  if (!CACHED)
    row_stats_seq<T, HT>(lane, beg, end, cols, d, srow, h, beta, sw, sh_max[wib], sh_inv[wib]);
  const VT* Mv = reinterpret_cast<const VT*>(M);
  const VT* Gv = reinterpret_cast<const VT*>(G);
  T g[R][W];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t v = r * 32 + lane;
    if (v < (uint32_t)fv) {
      const VT x = __ldg(Gv + (uint32_t)i * (uint32_t)fv + v);
      const T* px = reinterpret_cast<const T*>(&x);
#pragma unroll
      for (int q = 0; q < W; ++q) g[r][q] = px[q];
    } else {
#pragma unroll
      for (int q = 0; q < W; ++q) g[r][q] = T(0);
    }
  }
  auto head_reduce = [&](T (&p)[R], int eb) {
    if (lph <= 32) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        for (int o = lph >> 1; o > 0; o >>= 1)
          p[r] = add_rn(p[r], __shfl_xor_sync(0xffffffffu, p[r], o));
        const int v = r * 32 + lane;
        if (v < fv && (lane & (lph - 1)) == 0) sd[eb][v / lph] = p[r];
      }
    } else {
      const int cph = lph / 32;
      for (int r0 = 0; r0 < R; r0 += cph) {
        T a = T(0);
        for (int r = r0; r < r0 + cph && r < R; ++r) a = add_rn(a, p[r]);
        a = wsum(a);
        if (lane == 0 && r0 * 32 < fv) sd[eb][r0 * 32 / lph] = a;
      }
    }
  };
  T dot = T(0);  // lane t: sum_e alpha dAlpha for head t
  uint32_t mbits = 0;
  for (int32_t base = beg; base < end; base += 32) {
    const int cnt = min(32, end - base);
    int32_t mycol = 0;
    if (!CACHED && multi) {
      mycol = stage_scores<T, HT>(lane, base, cnt, cols, d, srow, h, beta, sw);
    } else if (lane < cnt) {
      mycol = __ldg(cols + base + lane);
    }
    if (lane < cnt) {  // attention and mask of the lane's edge for every head
      const int32_t e = base + lane;
#pragma unroll
      for (int t = 0; t < HT; ++t)
        if (t < h) {
          T a;
          bool pos;
          if (CACHED) {
            a = alpha_in[(int64_t)e * h + t];
            pos = mask_in[(int64_t)e * h + t] != 0;
          } else {
            const T w = sw[lane][t];
            a = mul_rn(dev_exp<T>(w - sh_max[wib][t]), sh_inv[wib][t]);
            pos = w > T(0);
          }
          sw[lane][t] = a;
          if (pos) mbits |= 1u << t;
        }
    }
    __syncwarp();
    if (!CACHED)  // alpha for the column pass: contiguous edge-major span
      for (int x = lane; x < cnt * h; x += 32) alpha_out[(int64_t)base * h + x] = sw[x / h][x % h];
    for (int eb = 0; eb < cnt; eb += 2) {  // dAlpha[eb][t], two gathers in flight
      const bool two = eb + 1 < cnt;
      const uint32_t o0 = (uint32_t)__shfl_sync(0xffffffffu, mycol, eb) * (uint32_t)fv;
      const uint32_t o1 =
          (uint32_t)__shfl_sync(0xffffffffu, mycol, two ? eb + 1 : eb) * (uint32_t)fv;
      VT x0[R], x1[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t v = r * 32 + lane;
        if (v < (uint32_t)fv) {
          x0[r] = __ldg(Mv + o0 + v);
          if (two) x1[r] = __ldg(Mv + o1 + v);
        }
      }
      T p0[R], p1[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int v = r * 32 + lane;
        p0[r] = p1[r] = T(0);
        if (v < fv) {
          const T* q0 = reinterpret_cast<const T*>(&x0[r]);
#pragma unroll
          for (int q = 0; q < W; ++q) p0[r] = madd(p0[r], g[r][q], q0[q]);
          if (two) {
            const T* q1 = reinterpret_cast<const T*>(&x1[r]);
#pragma unroll
            for (int q = 0; q < W; ++q) p1[r] = madd(p1[r], g[r][q], q1[q]);
          }
        }
      }
      head_reduce(p0, eb);
      if (two) head_reduce(p1, eb + 1);
    }
    __syncwarp();
    if (lane < h)  // softmax-backward dot, stored edge order
      for (int eb = 0; eb < cnt; ++eb) dot = madd(dot, sw[eb][lane], sd[eb][lane]);
    if (multi)  // spill dAlpha for the second pass
      for (int x = lane; x < cnt * h; x += 32) da[(int64_t)base * h + x] = sd[x / h][x % h];
    __syncwarp();
  }
  if (lane < h) sh_dot[wib][lane] = dot;
  __syncwarp();
  // dy = mask ? dw : beta dw with dw = alpha (dAlpha - dot); dS in edge order
  T rs = T(0);
  for (int32_t base = beg; base < end; base += 32) {
    const int cnt = min(32, end - base);
    if (lane < cnt) {
      const int32_t e = base + lane;
      const uint32_t mb = mbits;
#pragma unroll
      for (int t = 0; t < HT; ++t)
        if (t < h) {
          T a, dd;
          bool pos;
          if (multi) {
            a = CACHED ? alpha_in[(int64_t)e * h + t] : alpha_out[(int64_t)e * h + t];
            dd = da[(int64_t)e * h + t];
            if (CACHED) {
              pos = mask_in[(int64_t)e * h + t] != 0;
            } else {
              pos = add_rn(srow[t], d[(int64_t)__ldg(cols + e) * h + t]) > T(0);
            }
          } else {
            a = sw[lane][t];
            dd = sd[lane][t];
            pos = (mb >> t) & 1u;
          }
          const T dw = mul_rn(a, dd - sh_dot[wib][t]);
          const T gg = pos ? dw : mul_rn(beta, dw);
          sd[lane][t] = gg;
        }
    }
    __syncwarp();
    for (int x = lane; x < cnt * h; x += 32) dy[(int64_t)base * h + x] = sd[x / h][x % h];
    if (lane < h)
      for (int eb = 0; eb < cnt; ++eb) rs = add_rn(rs, sd[eb][lane]);
    __syncwarp();
  }
  if (lane < h) dS[(int64_t)i * h + lane] = rs;
}

// ---------------------------------------------------------------------------
// backward, per source column j over the CSC view (kernels.hpp:258-295,
// 614-658): dD[j] and dM[j] = alpha^T dX' + dS a_src + dD a_dst.  Lanes of
// head t accumulate dD_t redundantly in CSC (edge) order; dX' rows are
// 128-bit gathers as in the SpMM.
// ---------------------------------------------------------------------------
template <class T, int W, int R>
__global__ void __launch_bounds__(256) k_gat_bwd_col_fast(
    int32_t n, const int32_t* __restrict__ colptr, const int32_t* __restrict__ crows,
    const int32_t* __restrict__ perm, const T* __restrict__ G, const T* __restrict__ alpha,
    const T* __restrict__ dy, const T* __restrict__ dS, const T* __restrict__ a_src,
    const T* __restrict__ a_dst, int32_t h, int32_t k, T* __restrict__ dD,
    T* __restrict__ dM) {
  const int lane = threadIdx.x & 31;
  const int32_t j = (int32_t)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (j >= n) return;
  const int32_t hk = h * k, fv = hk / W;
  const int32_t beg = colptr[j], end = colptr[j + 1];
  int tr[R];
  T acc[R][W], dd[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int v = r * 32 + lane;
    tr[r] = v < fv ? (v * W) / k : 0;
    dd[r] = T(0);
#pragma unroll
    for (int q = 0; q < W; ++q) acc[r][q] = T(0);
  }
  for (int32_t base = beg; base < end; base += 32) {
    const int cnt = min(32, end - base);
    const int32_t my_e = lane < cnt ? __ldg(perm + base + lane) : 0;
    const int32_t my_r = lane < cnt ? __ldg(crows + base + lane) : 0;
    for (int pb = 0; pb < cnt; pb += 2) {
      const bool two = pb + 1 < cnt;
      const int32_t e0 = __shfl_sync(0xffffffffu, my_e, pb);
      const int32_t r0 = __shfl_sync(0xffffffffu, my_r, pb);
      const int32_t e1 = __shfl_sync(0xffffffffu, my_e, two ? pb + 1 : pb);
      const int32_t r1 = __shfl_sync(0xffffffffu, my_r, two ? pb + 1 : pb);
      const T* g0 = G + (int64_t)r0 * hk;
      const T* g1 = G + (int64_t)r1 * hk;
      T gv0[R][W], gv1[R][W], a0[R], a1[R], y0[R], y1[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int v = r * 32 + lane;
        if (v < fv) {
          vload<T, W>(g0 + (int64_t)v * W, gv0[r]);
          a0[r] = alpha[(int64_t)e0 * h + tr[r]];
          y0[r] = dy[(int64_t)e0 * h + tr[r]];
          if (two) {
            vload<T, W>(g1 + (int64_t)v * W, gv1[r]);
            a1[r] = alpha[(int64_t)e1 * h + tr[r]];
            y1[r] = dy[(int64_t)e1 * h + tr[r]];
          }
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int v = r * 32 + lane;
        if (v < fv) {
          dd[r] = add_rn(dd[r], y0[r]);
#pragma unroll
          for (int q = 0; q < W; ++q) acc[r][q] = madd(acc[r][q], a0[r], gv0[r][q]);
          if (two) {
            dd[r] = add_rn(dd[r], y1[r]);
#pragma unroll
            for (int q = 0; q < W; ++q) acc[r][q] = madd(acc[r][q], a1[r], gv1[r][q]);
          }
        }
      }
    }
  }
  const T* sj = dS + (int64_t)j * h;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int v = r * 32 + lane;
    if (v < fv) {
      const int t = tr[r];
      if (((v * W) % k) == 0) dD[(int64_t)j * h + t] = dd[r];
      T as[W], ad[W], o[W];
      vload<T, W>(a_src + (int64_t)v * W, as);
      vload<T, W>(a_dst + (int64_t)v * W, ad);
      const T sv = sj[t];
#pragma unroll
      for (int q = 0; q < W; ++q) o[q] = madd(madd(acc[r][q], sv, as[q]), dd[r], ad[q]);
      vstore<T, W>(dM + (int64_t)j * hk + (int64_t)v * W, o);
    }
  }
}

// attention_param_grad (kernels.hpp:592-611) for a_src and a_dst in one pass
// over M (fv <= 256 on the fast path): a block owns a row chunk; threads own
// W-column vectors, 256/fv row
// groups per block stride the chunk; float64 accumulation; block partials
// combined in a fixed order by k_reduce_partials.
template <class T, int W>
__global__ void __launch_bounds__(256) k_attgrad2_partial(int32_t n, int32_t h, int32_t k,
                                                          const T* __restrict__ M,
                                                          const T* __restrict__ dS,
                                                          const T* __restrict__ dD, int32_t chunk,
                                                          double* __restrict__ ps,
                                                          double* __restrict__ pd) {
  __shared__ double sh_s[256 * W], sh_d[256 * W];
  const int32_t hk = h * k, fv = hk / W;
  const int groups = max(1, 256 / fv);
  const int tid = threadIdx.x;
  const int v = tid % fv, grp = tid / fv;
  const int32_t r0 = blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  double a[W], b[W];
#pragma unroll
  for (int q = 0; q < W; ++q) a[q] = b[q] = 0.0;
  if (grp < groups) {
    const int t = (v * W) / k;
    for (int32_t i = r0 + grp; i < r1; i += groups) {
      T mv[W];
      vload<T, W>(M + (int64_t)i * hk + (int64_t)v * W, mv);
      const double cs = (double)dS[(int64_t)i * h + t], cd = (double)dD[(int64_t)i * h + t];
#pragma unroll
      for (int q = 0; q < W; ++q) {
        a[q] += cs * (double)mv[q];
        b[q] += cd * (double)mv[q];
      }
    }
  }
#pragma unroll
  for (int q = 0; q < W; ++q) {
    sh_s[tid * W + q] = a[q];
    sh_d[tid * W + q] = b[q];
  }
  __syncthreads();
  if (grp == 0) {
    for (int gg = 1; gg < groups; ++gg)
#pragma unroll
      for (int q = 0; q < W; ++q) {
        a[q] += sh_s[(gg * fv + v) * W + q];
        b[q] += sh_d[(gg * fv + v) * W + q];
      }
#pragma unroll
    for (int q = 0; q < W; ++q) {
      ps[(int64_t)blockIdx.x * hk + (int64_t)v * W + q] = a[q];
      pd[(int64_t)blockIdx.x * hk + (int64_t)v * W + q] = b[q];
    }
  }
}

// partials [nw][hk] -> out[hk] (8 warps split the partial list, fixed order)
template <class T>
__global__ void __launch_bounds__(256) k_reduce_partials(int32_t nw, int32_t hk,
                                                         const double* __restrict__ part,
                                                         T* __restrict__ out) {
  __shared__ double sh[8][33];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t c = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (c < hk) {  // four independent chains
    double s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int32_t z = w;
    for (; z + 24 < nw; z += 32) {
      s += part[(int64_t)z * hk + c];
      s1 += part[(int64_t)(z + 8) * hk + c];
      s2 += part[(int64_t)(z + 16) * hk + c];
      s3 += part[(int64_t)(z + 24) * hk + c];
    }
    for (; z < nw; z += 8) s += part[(int64_t)z * hk + c];
    s = (s + s1) + (s2 + s3);
  }
  sh[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < hk) {
    double t = 0.0;
    for (int q = 0; q < 8; ++q) t += sh[q][lane];
    out[c] = (T)t;
  }
}

}  // namespace gf
