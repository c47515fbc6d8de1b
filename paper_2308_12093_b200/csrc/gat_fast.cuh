// gat_fast.cuh -- fast-path GAT kernels (included by gat.cu).
//
// Layout: one warp per destination row (forward, backward-row) or source
// column (backward-column); lanes own 16-byte column vectors of the n x hk
// slab (vector v = cb*32R + r*32 + lane, columns W*v .. W*v+W-1, head W*v/k),
// so every gathered M / dX' row is read with fully coalesced 128-bit loads.
// Per-edge scalars (attention, scores) are computed with lanes over edges in
// batches of 32 and staged in shared memory; softmax statistics use warp
// shuffle reductions; the SDDMM dot products use head-segmented xor-shuffle
// reductions.  Eligible when k % W == 0, k/W is a power of two <= 32 or a
// multiple of 32, h <= 16.  Other shapes use the generic kernels in gat.cu.
#pragma once

// (included inside namespace sgnn)
namespace gf {

constexpr int HF = 16;  // max heads on the fast path
// warps per block: keeps the per-warp staging arrays under the 48 KB static limit
template <class T>
struct WPB {
  static constexpr int v = sizeof(T) == 4 ? 8 : 4;
};

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

// Row softmax statistics for heads 0..h-1: smax[t], sinv[t] (kernels.hpp:517-531).
// Lanes over edges, two passes (max, then sum of exp(w - max)).
template <class T>
__device__ __forceinline__ void row_stats_fast(int lane, int32_t beg, int32_t end,
                                               const int32_t* __restrict__ cols,
                                               const T* __restrict__ d, const T* ss, int h,
                                               T beta, T* smax, T* sinv) {
  for (int t = 0; t < h; ++t) {
    T m = neg_inf<T>();
    for (int32_t e = beg + lane; e < end; e += 32) {
      bool pos;
      const T w = leaky(add_rn(ss[t], d[(int64_t)__ldg(cols + e) * h + t]), beta, pos);
      m = m < w ? w : m;
    }
    m = wmax(m);
    T s = T(0);
    for (int32_t e = beg + lane; e < end; e += 32) {
      bool pos;
      const T w = leaky(add_rn(ss[t], d[(int64_t)__ldg(cols + e) * h + t]), beta, pos);
      s = add_rn(s, dev_exp<T>(w - m));
    }
    s = wsum(s);
    if (lane == 0) {
      smax[t] = m;
      sinv[t] = T(1) / s;
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
  for (int cb = 0; cb < fv; cb += 32 * R) {
    T ps[R], pd[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int v = cb + r * 32 + lane;
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
        const int v = cb + r * 32 + lane;
        if (v < fv && (lane & (lph - 1)) == 0) {
          const int t = v / lph;
          s[(int64_t)i * h + t] = ps[r];
          d[(int64_t)i * h + t] = pd[r];
        }
      }
    } else {
      // a head spans lph/32 whole r-chunks: sum chunks, then the full warp
      const int cph = lph / 32;
      for (int r0 = 0; r0 < R; r0 += cph) {
        T a = T(0), b = T(0);
        for (int r = r0; r < r0 + cph && r < R; ++r) {
          a = add_rn(a, ps[r]);
          b = add_rn(b, pd[r]);
        }
        a = wsum(a);
        b = wsum(b);
        const int v = cb + r0 * 32;
        if (lane == 0 && v < fv) {
          const int t = v / lph;
          s[(int64_t)i * h + t] = a;
          d[(int64_t)i * h + t] = b;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// forward: stats + attention + multi-head aggregation + bias, one warp per row
// ---------------------------------------------------------------------------
template <class T, int W, int R, bool STORE>
__global__ void __launch_bounds__(256) k_gat_fwd_fast(int32_t n, const int32_t* __restrict__ rowptr,
                                                      const int32_t* __restrict__ cols,
                                                      const T* __restrict__ M,
                                                      const T* __restrict__ s,
                                                      const T* __restrict__ d, int32_t h,
                                                      int32_t k, T beta,
                                                      const T* __restrict__ bias,
                                                      T* __restrict__ out, T* __restrict__ alpha,
                                                      uint8_t* __restrict__ mask) {
  __shared__ T sh_ss[WPB<T>::v][HF], sh_max[WPB<T>::v][HF], sh_inv[WPB<T>::v][HF];
  __shared__ T sh_al[WPB<T>::v][32][HF + 1];
  __shared__ int32_t sh_col[WPB<T>::v][32];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t i = (int32_t)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (i >= n) return;
  T* ss = sh_ss[wib];
  T* smax = sh_max[wib];
  T* sinv = sh_inv[wib];
  const int32_t hk = h * k, fv = hk / W;
  const int32_t beg = rowptr[i], end = rowptr[i + 1];
  if (lane < h) ss[lane] = s[(int64_t)i * h + lane];
  __syncwarp();
  row_stats_fast<T>(lane, beg, end, cols, d, ss, h, beta, smax, sinv);
  for (int cb = 0; cb < fv; cb += 32 * R) {
    T acc[R][W];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int w = 0; w < W; ++w) acc[r][w] = T(0);
    for (int32_t base = beg; base < end; base += 32) {
      const int cnt = min(32, end - base);
      if (lane < cnt) {
        const int32_t e = base + lane;
        const int32_t j = __ldg(cols + e);
        sh_col[wib][lane] = j;
        for (int t = 0; t < h; ++t) {
          bool pos;
          const T w = leaky(add_rn(ss[t], d[(int64_t)j * h + t]), beta, pos);
          const T a = mul_rn(dev_exp<T>(w - smax[t]), sinv[t]);
          sh_al[wib][lane][t] = a;
          if (STORE && cb == 0) {
            alpha[(int64_t)e * h + t] = a;
            mask[(int64_t)e * h + t] = pos ? 1 : 0;
          }
        }
      }
      __syncwarp();
      for (int eb = 0; eb < cnt; ++eb) {
        const T* mrow = M + (int64_t)sh_col[wib][eb] * hk;
        T mv[R][W];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int v = cb + r * 32 + lane;
          if (v < fv) vload<T, W>(mrow + (int64_t)v * W, mv[r]);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int v = cb + r * 32 + lane;
          if (v < fv) {
            const T a = sh_al[wib][eb][(v * W) / k];
#pragma unroll
            for (int w = 0; w < W; ++w) acc[r][w] = madd(acc[r][w], a, mv[r][w]);
          }
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int v = cb + r * 32 + lane;
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

// ---------------------------------------------------------------------------
// backward, per destination row: alpha (cached or recomputed), SDDMM dAlpha,
// softmax + LeakyReLU backward, dS.  Persistent warps also accumulate the
// column sums of dX' (d_bias) for the rows they own.
// ---------------------------------------------------------------------------
template <class T, int W, int R, bool CACHED>
__global__ void __launch_bounds__(256) k_gat_bwd_row_fast(
    int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
    const T* __restrict__ M, const T* __restrict__ s, const T* __restrict__ d,
    const T* __restrict__ G, int32_t h, int32_t k, T beta, const T* __restrict__ alpha_in,
    const uint8_t* __restrict__ mask_in, T* __restrict__ alpha_out, T* __restrict__ da,
    T* __restrict__ dy, T* __restrict__ dS) {
  __shared__ T sh_ss[WPB<T>::v][HF], sh_max[WPB<T>::v][HF], sh_inv[WPB<T>::v][HF], sh_dot[WPB<T>::v][HF];
  __shared__ T sh_al[WPB<T>::v][32][HF + 1];
  __shared__ T sh_da[WPB<T>::v][32][HF + 1];
  __shared__ int32_t sh_col[WPB<T>::v][32];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t i = (int32_t)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (i >= n) return;
  T* ss = sh_ss[wib];
  T* smax = sh_max[wib];
  T* sinv = sh_inv[wib];
  T* sdot = sh_dot[wib];
  const int32_t hk = h * k, fv = hk / W, lph = k / W;
  const int32_t beg = rowptr[i], end = rowptr[i + 1];
  if (!CACHED) {
    if (lane < h) ss[lane] = s[(int64_t)i * h + lane];
    __syncwarp();
    row_stats_fast<T>(lane, beg, end, cols, d, ss, h, beta, smax, sinv);
  }
  if (lane < h) sdot[lane] = T(0);
  __syncwarp();
  const T* grow = G + (int64_t)i * hk;
  // pass 1: alpha (write for the column pass) and dAlpha per (edge, head)
  for (int32_t base = beg; base < end; base += 32) {
    const int cnt = min(32, end - base);
    if (lane < cnt) {
      const int32_t e = base + lane;
      const int32_t j = __ldg(cols + e);
      sh_col[wib][lane] = j;
      for (int t = 0; t < h; ++t) {
        T a;
        if (CACHED) {
          a = alpha_in[(int64_t)e * h + t];
        } else {
          bool pos;
          const T w = leaky(add_rn(ss[t], d[(int64_t)j * h + t]), beta, pos);
          a = mul_rn(dev_exp<T>(w - smax[t]), sinv[t]);
          alpha_out[(int64_t)e * h + t] = a;
        }
        sh_al[wib][lane][t] = a;
      }
    }
    __syncwarp();
    for (int cb = 0; cb < fv; cb += 32 * R) {
      T g[R][W];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int v = cb + r * 32 + lane;
        if (v < fv) vload<T, W>(grow + (int64_t)v * W, g[r]);
        else
#pragma unroll
          for (int w = 0; w < W; ++w) g[r][w] = T(0);
      }
      for (int eb = 0; eb < cnt; ++eb) {
        const T* mrow = M + (int64_t)sh_col[wib][eb] * hk;
        T p[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int v = cb + r * 32 + lane;
          p[r] = T(0);
          if (v < fv) {
            T mv[W];
            vload<T, W>(mrow + (int64_t)v * W, mv);
#pragma unroll
            for (int w = 0; w < W; ++w) p[r] = madd(p[r], g[r][w], mv[w]);
          }
        }
        if (lph <= 32) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            for (int o = lph >> 1; o > 0; o >>= 1)
              p[r] = add_rn(p[r], __shfl_xor_sync(0xffffffffu, p[r], o));
            const int v = cb + r * 32 + lane;
            if (v < fv && (lane & (lph - 1)) == 0) sh_da[wib][eb][v / lph] = p[r];
          }
        } else {
          const int cph = lph / 32;
          for (int r0 = 0; r0 < R; r0 += cph) {
            T a = T(0);
            for (int r = r0; r < r0 + cph && r < R; ++r) a = add_rn(a, p[r]);
            a = wsum(a);
            const int v = cb + r0 * 32;
            if (lane == 0 && v < fv) sh_da[wib][eb][v / lph] = a;
          }
        }
      }
    }
    __syncwarp();
    // dot_t = sum_e alpha * dAlpha in edge order; spill dAlpha for pass 2
    for (int t = lane; t < h; t += 32) {
      T dt = sdot[t];
      for (int eb = 0; eb < cnt; ++eb) dt = madd(dt, sh_al[wib][eb][t], sh_da[wib][eb][t]);
      sdot[t] = dt;
    }
    for (int x = lane; x < cnt * h; x += 32) {
      const int eb = x / h, t = x % h;
      da[(int64_t)(base + eb) * h + t] = sh_da[wib][eb][t];
    }
    __syncwarp();
  }
  // pass 2: dw = alpha (dAlpha - dot), dy = mask ? dw : beta dw, dS = row sums
  for (int t = lane; t < h; t += 32) {
    const T dt = sdot[t];
    T rs = T(0);
    for (int32_t e = beg; e < end; ++e) {
      const T a = CACHED ? alpha_in[(int64_t)e * h + t] : alpha_out[(int64_t)e * h + t];
      const T dw = mul_rn(a, da[(int64_t)e * h + t] - dt);
      bool pos;
      if (CACHED) {
        pos = mask_in[(int64_t)e * h + t] != 0;
      } else {
        const int32_t j = __ldg(cols + e);
        pos = add_rn(ss[t], d[(int64_t)j * h + t]) > T(0);
      }
      const T gg = pos ? dw : mul_rn(beta, dw);
      dy[(int64_t)e * h + t] = gg;
      rs = add_rn(rs, gg);
    }
    dS[(int64_t)i * h + t] = rs;
  }
}

// ---------------------------------------------------------------------------
// backward, per source column j (CSC view): dD, dM = alpha^T dX' + dS a_src +
// dD a_dst, and per-warp partials of the attention-parameter gradients
// sum_j dS[j,t] M[j,t,:] and sum_j dD[j,t] M[j,t,:] (kernels.hpp:592-611).
// Grid-stride warps; partial[warp] written once at the end (deterministic).
// ---------------------------------------------------------------------------
template <class T, int W, int R>
__global__ void __launch_bounds__(256) k_gat_bwd_col_fast(
    int32_t n, const int32_t* __restrict__ colptr, const int32_t* __restrict__ crows,
    const int32_t* __restrict__ perm, const T* __restrict__ G, const T* __restrict__ M,
    const T* __restrict__ alpha, const T* __restrict__ dy, const T* __restrict__ dS,
    const T* __restrict__ a_src, const T* __restrict__ a_dst, int32_t h, int32_t k,
    T* __restrict__ dD, T* __restrict__ dM, double* __restrict__ part_src,
    double* __restrict__ part_dst) {
  __shared__ T sh_dd[WPB<T>::v][HF], sh_sj[WPB<T>::v][HF];
  __shared__ T sh_al[WPB<T>::v][32][HF + 1];
  __shared__ T sh_dy[WPB<T>::v][32][HF + 1];
  __shared__ int32_t sh_row[WPB<T>::v][32];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  T* sdd = sh_dd[wib];
  T* ssj = sh_sj[wib];
  const int32_t hk = h * k, fv = hk / W;
  // attention-parameter gradient partials for this warp (lane's vectors of the
  // first column block; fv <= 32R is required on this path)
  double ps[R][W], pdd[R][W];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int w = 0; w < W; ++w) ps[r][w] = pdd[r][w] = 0.0;
  for (int64_t jj = warp; jj < n; jj += nwarps) {
    const int32_t j = (int32_t)jj;
    const int32_t beg = colptr[j], end = colptr[j + 1];
    if (lane < h) {
      sdd[lane] = T(0);
      ssj[lane] = dS[(int64_t)j * h + lane];
    }
    T acc[R][W];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int w = 0; w < W; ++w) acc[r][w] = T(0);
    __syncwarp();
    for (int32_t base = beg; base < end; base += 32) {
      const int cnt = min(32, end - base);
      if (lane < cnt) {
        const int32_t p = base + lane;
        const int32_t e = __ldg(perm + p);
        sh_row[wib][lane] = __ldg(crows + p);
        for (int t = 0; t < h; ++t) {
          sh_al[wib][lane][t] = alpha[(int64_t)e * h + t];
          sh_dy[wib][lane][t] = dy[(int64_t)e * h + t];
        }
      }
      __syncwarp();
      for (int t = lane; t < h; t += 32) {  // dD in CSC (edge) order
        T a = sdd[t];
        for (int eb = 0; eb < cnt; ++eb) a = add_rn(a, sh_dy[wib][eb][t]);
        sdd[t] = a;
      }
      for (int eb = 0; eb < cnt; ++eb) {
        const T* grow = G + (int64_t)sh_row[wib][eb] * hk;
        T gv[R][W];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int v = r * 32 + lane;
          if (v < fv) vload<T, W>(grow + (int64_t)v * W, gv[r]);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int v = r * 32 + lane;
          if (v < fv) {
            const T a = sh_al[wib][eb][(v * W) / k];
#pragma unroll
            for (int w = 0; w < W; ++w) acc[r][w] = madd(acc[r][w], a, gv[r][w]);
          }
        }
      }
      __syncwarp();
    }
    if (lane < h) dD[(int64_t)j * h + lane] = sdd[lane];
    __syncwarp();
    const T* mrow = M + (int64_t)j * hk;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int v = r * 32 + lane;
      if (v < fv) {
        const int t = (v * W) / k;
        const T sj = ssj[t], dj = sdd[t];
        T as[W], ad[W], mv[W], o[W];
        vload<T, W>(a_src + (int64_t)v * W, as);
        vload<T, W>(a_dst + (int64_t)v * W, ad);
        vload<T, W>(mrow + (int64_t)v * W, mv);
#pragma unroll
        for (int w = 0; w < W; ++w) {
          // dM = (alpha^T dX') + dS a_src + dD a_dst (add_scaled_rows order)
          o[w] = madd(madd(acc[r][w], sj, as[w]), dj, ad[w]);
          ps[r][w] += (double)sj * (double)mv[w];
          pdd[r][w] += (double)dj * (double)mv[w];
        }
        vstore<T, W>(dM + (int64_t)j * hk + (int64_t)v * W, o);
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int v = r * 32 + lane;
    if (v < fv)
#pragma unroll
      for (int w = 0; w < W; ++w) {
        part_src[warp * hk + (int64_t)v * W + w] = ps[r][w];
        part_dst[warp * hk + (int64_t)v * W + w] = pdd[r][w];
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
  if (c < hk)
    for (int32_t z = w; z < nw; z += 8) s += part[(int64_t)z * hk + c];
  sh[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < hk) {
    double t = 0.0;
    for (int q = 0; q < 8; ++q) t += sh[q][lane];
    out[c] = (T)t;
  }
}

}  // namespace gf
