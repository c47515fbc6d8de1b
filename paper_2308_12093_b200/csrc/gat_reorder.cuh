// Operator-reordered GAT layer for wide heads (k > m, e.g. the first layer of
// Gat2 128 -> 8 x 256).  The reference evaluates, per head t,
//   M_t = X Theta_t,  s = M a_src, d = M a_dst,  out_i,t = sum_j alpha_ij,t M_j,t + b_t
// (gat.hpp:99-121) and gathers k-wide M rows per edge in the aggregation, the
// SDDMM and the transposed SpMM.  Reassociating the products moves every edge
// gather onto the m-wide input rows:
//   s_i,t = X_i . (Theta_t a_src_t),          d_j,t = X_j . (Theta_t a_dst_t)
//   Z_i,t = sum_j alpha_ij,t X_j,             out_t = Z_t Theta_t + b_t
//   dAlpha_ij,t = (G_i,t Theta_t^T) . X_j     (Gtheta = G_t Theta_t^T, n x h x m)
//   dTheta_t = Z_t^T G_t + (X^T dS_t) a_src_t^T + (X^T dD_t) a_dst_t^T
//   d a_src_t = (X^T dS_t)^T Theta_t,          d a_dst_t = (X^T dD_t)^T Theta_t
//   dX_j = sum_i sum_t alpha_ij,t Gtheta_i,t + sum_t dS_j,t W_src,t + dD_j,t W_dst,t
// with dS / dD the row / column sums of the softmax-backward edge values (as in
// k_gat_sbwd4 / k_gat_col2).  M is never formed; the per-head transforms run on
// the tcgen05 GEMM with pitched operands (gemm_tc_f32_pitched).  Float32.
#pragma once

namespace g2 {

// Sum NV per-lane values over the warp: lane l ends with the total of value
// index l >> (5 - log2 NV) (a transposing butterfly: log2 NV exchange steps
// that halve the values each lane carries, then a plain xor reduction) --
// NV - 1 + 5 - log2 NV shuffles instead of 5 NV.
template <int NV>
__device__ __forceinline__ float warp_multi_sum(float (&v)[NV]) {
  const int lane = threadIdx.x & 31;
  int off = 16;
#pragma unroll
  for (int w = NV; w > 1; w >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int j = 0; j < w / 2; ++j) {
      const float send = up ? v[j] : v[j + w / 2];
      const float keep = up ? v[j + w / 2] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
    off >>= 1;
  }
  float r = v[0];
  for (; off > 0; off >>= 1) r += __shfl_xor_sync(0xffffffffu, r, off);
  return r;
}
template <int NV>
__device__ __forceinline__ constexpr int multi_sum_shift() {
  return NV >= 32 ? 0 : (NV >= 16 ? 1 : (NV >= 8 ? 2 : (NV >= 4 ? 3 : (NV >= 2 ? 4 : 5))));
}

// W[w][t][v] = sum_c Theta[v][t k + c] a_w[t k + c]  (w = 0: a_src, 1: a_dst);
// warp per output, lanes over c.
__global__ void __launch_bounds__(256) k_gat_wvec(int32_t m, int32_t h, int32_t k,
                                                  const float* __restrict__ theta,
                                                  const float* __restrict__ a_src,
                                                  const float* __restrict__ a_dst,
                                                  float* __restrict__ W) {
  const int lane = threadIdx.x & 31;
  const int64_t o = (int64_t)(blockIdx.x * 256u + threadIdx.x) >> 5;
  if (o >= 2LL * h * m) return;
  const int32_t v = (int32_t)(o % m), t = (int32_t)((o / m) % h), w = (int32_t)(o / ((int64_t)m * h));
  const float* a = (w == 0 ? a_src : a_dst) + (int64_t)t * k;
  const float* th = theta + (int64_t)v * h * k + (int64_t)t * k;
  float acc = 0.f;
  for (int32_t c = lane; c < k; c += 32) acc = fmaf(__ldg(th + c), __ldg(a + c), acc);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) W[o] = acc;
}

// s_i,t = X_i . W_src,t and d_i,t = X_i . W_dst,t: warp per row, lanes own RM
// 16-byte vectors of X_i, W (2 h m floats) staged in shared memory.
template <int H, int RM>
__global__ void __launch_bounds__(256) k_gat_xscores(int32_t n, int32_t mv,
                                                     const float4* __restrict__ X,
                                                     const float4* __restrict__ W,
                                                     float* __restrict__ s, float* __restrict__ d) {
  extern __shared__ float4 w_s[];  // [2H][mv]
  for (int q = threadIdx.x; q < 2 * H * mv; q += 256) w_s[q] = __ldg(W + q);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int32_t i = (int32_t)((blockIdx.x * 256u + threadIdx.x) >> 5);
  if (i >= n) return;
  float4 x[RM];
#pragma unroll
  for (int r = 0; r < RM; ++r) {
    const int v = r * 32 + lane;
    x[r] = v < mv ? __ldg(X + (int64_t)i * mv + v) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float p[2 * H];
#pragma unroll
  for (int w = 0; w < 2 * H; ++w) {
    p[w] = 0.f;
#pragma unroll
    for (int r = 0; r < RM; ++r) {
      const int v = r * 32 + lane;
      if (v < mv) p[w] += dot4(x[r], w_s[w * mv + v]);
    }
  }
  const float tot = warp_multi_sum<2 * H>(p);
  constexpr int SH = multi_sum_shift<2 * H>();
  if ((lane & ((1 << SH) - 1)) == 0) {
    const int w = lane >> SH;
    if (w < H) s[(int64_t)i * H + w] = tot;
    else d[(int64_t)i * H + (w - H)] = tot;
  }
}

// Z_i,t = sum_{e in row i} alpha_e,t X_{col_e}: warp per row, lanes own RM
// 16-byte vectors of an m-wide row, per-head accumulators in registers;
// stored edge order, FMA.  Z is n x h x m.
template <int H, int RM>
__global__ void __launch_bounds__(256) k_gat_aggx(int32_t n, const int32_t* __restrict__ rowptr,
                                                  const int32_t* __restrict__ cols,
                                                  const float* __restrict__ alpha,
                                                  const float4* __restrict__ X, int32_t mv,
                                                  float4* __restrict__ Z) {
  const int lane = threadIdx.x & 31;
  const int32_t i = (int32_t)((blockIdx.x * 256u + threadIdx.x) >> 5);
  if (i >= n) return;
  const int32_t beg = __ldg(rowptr + i), end = __ldg(rowptr + i + 1);
  float4 acc[H][RM];
#pragma unroll
  for (int t = 0; t < H; ++t)
#pragma unroll
    for (int r = 0; r < RM; ++r) acc[t][r] = make_float4(0.f, 0.f, 0.f, 0.f);
  int32_t e = beg;
  for (; e + 2 <= end; e += 2) {
    const uint32_t c0 = (uint32_t)__ldg(cols + e), c1 = (uint32_t)__ldg(cols + e + 1);
    float a0[H], a1[H];
    ld_heads<H>(alpha + (int64_t)e * H, a0);
    ld_heads<H>(alpha + (int64_t)(e + 1) * H, a1);
    float4 x0[RM], x1[RM];
#pragma unroll
    for (int r = 0; r < RM; ++r) {
      const int v = r * 32 + lane;
      x0[r] = v < mv ? __ldg(X + c0 * (uint32_t)mv + v) : make_float4(0.f, 0.f, 0.f, 0.f);
      x1[r] = v < mv ? __ldg(X + c1 * (uint32_t)mv + v) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int t = 0; t < H; ++t)
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        fma4(acc[t][r], a0[t], x0[r]);
        fma4(acc[t][r], a1[t], x1[r]);
      }
  }
  if (e < end) {
    const uint32_t c0 = (uint32_t)__ldg(cols + e);
    float a0[H];
    ld_heads<H>(alpha + (int64_t)e * H, a0);
#pragma unroll
    for (int r = 0; r < RM; ++r) {
      const int v = r * 32 + lane;
      if (v < mv) {
        const float4 x0 = __ldg(X + c0 * (uint32_t)mv + v);
#pragma unroll
        for (int t = 0; t < H; ++t) fma4(acc[t][r], a0[t], x0);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < H; ++t)
#pragma unroll
    for (int r = 0; r < RM; ++r) {
      const int v = r * 32 + lane;
      if (v < mv) __stcs(Z + ((int64_t)i * H + t) * mv + v, acc[t][r]);
    }
}

// dAlpha_e,t = Gtheta_i,t . X_{col_e} for the edges of row i: warp per row,
// the row's Gtheta (h x m) held in registers, one m-wide X row gathered per
// edge (two edges in flight), the h dots reduced by the transposing butterfly.
template <int H, int RM>
__global__ void __launch_bounds__(256) k_gat_sddmmx(int32_t n, const int32_t* __restrict__ rowptr,
                                                    const int32_t* __restrict__ cols,
                                                    const float4* __restrict__ Gt,
                                                    const float4* __restrict__ X, int32_t mv,
                                                    float* __restrict__ da) {
  const int lane = threadIdx.x & 31;
  const int32_t i = (int32_t)((blockIdx.x * 256u + threadIdx.x) >> 5);
  if (i >= n) return;
  const int32_t beg = __ldg(rowptr + i), end = __ldg(rowptr + i + 1);
  float4 g[H][RM];
#pragma unroll
  for (int t = 0; t < H; ++t)
#pragma unroll
    for (int r = 0; r < RM; ++r) {
      const int v = r * 32 + lane;
      g[t][r] = v < mv ? __ldcs(Gt + ((int64_t)i * H + t) * mv + v) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  constexpr int SH = multi_sum_shift<H>();
  const bool writer = (lane & ((1 << SH) - 1)) == 0;
  const int wt = lane >> SH;
  for (int32_t e = beg; e < end; e += 2) {
    const bool two = e + 1 < end;
    const uint32_t c0 = (uint32_t)__ldg(cols + e);
    const uint32_t c1 = two ? (uint32_t)__ldg(cols + e + 1) : c0;
    float4 x0[RM], x1[RM];
#pragma unroll
    for (int r = 0; r < RM; ++r) {
      const int v = r * 32 + lane;
      x0[r] = v < mv ? __ldg(X + c0 * (uint32_t)mv + v) : make_float4(0.f, 0.f, 0.f, 0.f);
      x1[r] = v < mv ? __ldg(X + c1 * (uint32_t)mv + v) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float p0[H], p1[H];
#pragma unroll
    for (int t = 0; t < H; ++t) {
      p0[t] = 0.f;
      p1[t] = 0.f;
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        p0[t] += dot4(g[t][r], x0[r]);
        p1[t] += dot4(g[t][r], x1[r]);
      }
    }
    const float r0 = warp_multi_sum<H>(p0);
    const float r1 = warp_multi_sum<H>(p1);
    if (writer) {
      da[(int64_t)e * H + wt] = r0;
      if (two) da[(int64_t)(e + 1) * H + wt] = r1;
    }
  }
}

// dD_j,t = sum over the edges into column j of dy_e,t (k_gat_col2's column
// sums without the dM rows): warp per column, lanes = (32 / H) edge slots x H
// heads, xor reduction over the slots.
template <int H>
__global__ void __launch_bounds__(256) k_gat_colsum_dy(int32_t n, const int32_t* __restrict__ colptr,
                                                       const int32_t* __restrict__ perm,
                                                       const float* __restrict__ dy,
                                                       float* __restrict__ dD) {
  const int lane = threadIdx.x & 31;
  const int32_t j = (int32_t)((blockIdx.x * 256u + threadIdx.x) >> 5);
  if (j >= n) return;
  constexpr int SL = 32 / H;
  const int t = lane % H, slot = lane / H;
  const int32_t beg = __ldg(colptr + j), end = __ldg(colptr + j + 1);
  float acc = 0.f;
  for (int32_t p = beg + slot; p < end; p += SL) acc += __ldg(dy + (int64_t)__ldg(perm + p) * H + t);
#pragma unroll
  for (int off = 16; off >= H; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane < H) dD[(int64_t)j * H + t] = acc;
}

// Input gradient and dD in one pass over the CSC view: warp per column j,
//   dX_j = sum_{e into j} sum_t alpha_e,t Gtheta_{row_e},t
//          + sum_t dS_j,t W_src,t + dD_j,t W_dst,t,   dD_j,t = sum_e dy_e,t
// gathering one h x m Gtheta row per edge.
template <int H, int RM>
__global__ void __launch_bounds__(256) k_gat_colx(int32_t n, const int32_t* __restrict__ colptr,
                                                  const int32_t* __restrict__ crows,
                                                  const int32_t* __restrict__ perm,
                                                  const float4* __restrict__ Gt,
                                                  const float* __restrict__ alpha,
                                                  const float* __restrict__ dy,
                                                  const float* __restrict__ dS,
                                                  const float4* __restrict__ W, int32_t mv,
                                                  float* __restrict__ dD,
                                                  float4* __restrict__ dX) {
  const int lane = threadIdx.x & 31;
  const int32_t j = (int32_t)((blockIdx.x * 256u + threadIdx.x) >> 5);
  if (j >= n) return;
  const int32_t beg = __ldg(colptr + j), end = __ldg(colptr + j + 1);
  float4 acc[RM];
  float dd[H];
#pragma unroll
  for (int r = 0; r < RM; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int t = 0; t < H; ++t) dd[t] = 0.f;
  for (int32_t p = beg; p < end; ++p) {
    const int32_t e = __ldg(perm + p);
    const uint32_t row = (uint32_t)__ldg(crows + p);
    float a[H], y[H];
    ld_heads<H>(alpha + (int64_t)e * H, a);
    ld_heads<H>(dy + (int64_t)e * H, y);
#pragma unroll
    for (int t = 0; t < H; ++t) dd[t] += y[t];
#pragma unroll
    for (int t = 0; t < H; ++t)
#pragma unroll
      for (int r = 0; r < RM; ++r) {
        const int v = r * 32 + lane;
        if (v < mv) fma4(acc[r], a[t], __ldg(Gt + ((int64_t)row * H + t) * mv + v));
      }
  }
  float cs[H];
  ld_heads<H>(dS + (int64_t)j * H, cs);
#pragma unroll
  for (int r = 0; r < RM; ++r) {
    const int v = r * 32 + lane;
    if (v < mv) {
      float4 o = acc[r];
#pragma unroll
      for (int t = 0; t < H; ++t) {
        fma4(o, cs[t], __ldg(W + (int64_t)t * mv + v));
        fma4(o, dd[t], __ldg(W + (int64_t)(H + t) * mv + v));
      }
      __stcs(dX + (int64_t)j * mv + v, o);
    }
  }
  if (lane == 0) st_heads<H>(dD + (int64_t)j * H, dd);
}

// Attention-parameter gradients and the rank-1 terms of dTheta from
// U = [X^T dS | X^T dD] (m x h each), t = c / k for column c of h k:
//   d a_src[c] = sum_v U_S[v][t] Theta[v][c],  d a_dst[c] likewise,
//   dTheta[v][c] += U_S[v][t] a_src[c] + U_D[v][t] a_dst[c]
// Block per 32 columns: 8 warps split the m rows (lane = column, coalesced),
// the per-warp float64 partials of the two dots summed in fixed order.
__global__ void __launch_bounds__(256) k_gat_reorder_grads(int32_t m, int32_t h, int32_t k,
                                                           const float* __restrict__ theta,
                                                           const float* __restrict__ a_src,
                                                           const float* __restrict__ a_dst,
                                                           const float* __restrict__ us,
                                                           const float* __restrict__ ud,
                                                           float* __restrict__ d_theta,
                                                           float* __restrict__ d_a_src,
                                                           float* __restrict__ d_a_dst) {
  __shared__ double part[2][8][32];
  const int32_t hk = h * k;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t c = (int32_t)blockIdx.x * 32 + lane;
  double gs = 0.0, gd = 0.0;
  if (c < hk) {
    const int32_t t = c / k;
    const float as = __ldg(a_src + c), ad = __ldg(a_dst + c);
    for (int32_t v = w; v < m; v += 8) {
      const float uS = __ldg(us + (int64_t)v * h + t), uD = __ldg(ud + (int64_t)v * h + t);
      const float th = __ldg(theta + (int64_t)v * hk + c);
      gs += (double)uS * th;
      gd += (double)uD * th;
      float* o = d_theta + (int64_t)v * hk + c;
      *o = fmaf(uD, ad, fmaf(uS, as, *o));
    }
  }
  part[0][w][lane] = gs;
  part[1][w][lane] = gd;
  __syncthreads();
  if (w < 2 && c < hk) {
    double tot = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) tot += part[w][q][lane];
    (w == 0 ? d_a_src : d_a_dst)[c] = (float)tot;
  }
}

}  // namespace g2
