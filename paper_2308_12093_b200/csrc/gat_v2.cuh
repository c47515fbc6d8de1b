// gat_v2.cuh -- float32 GAT row/column kernels with compile-time head count
// (included by gat.cu inside namespace sgnn).  Used when T = float, h is 1, 2,
// 4 or 8, k % 4 == 0 and k/4 is a power of two <= 32 (a head spans k/4 lanes
// of one 32-lane chunk); other shapes use gat_fast.cuh / the generic kernels.
//
// Against gat_fast.cuh (which folds the softmax statistics by lanes over heads
// in stored edge order, one dependent shared-memory round trip per edge) these
// kernels keep every per-edge scalar in registers of the lane that owns the
// edge and reduce over the warp with a transposed butterfly: h values per lane
// are reduced across 32 lanes in (h-1) + (5-log2 h) shuffles, then broadcast
// back in h shuffles -- 17 shuffles for 8 heads instead of 40.  The float32
// path is checked against the float64 oracle at the north-star tolerance
// (1e-4 under max_rel_diff, dense.hpp:303-316); softmax sums therefore use a
// tree order and products use FMA, where gat_fast.cuh reproduces the
// reference's sequential order.  Dense-row gathers are issued U = 4 edges
// ahead (R 16-byte vectors per lane per edge) to keep more bytes in flight.
//
// Reference semantics followed: kernels.hpp:427-534 (scores, LeakyReLU, edge
// softmax, alpha = exp(w - max) * (1 / sum)), 219-254 (semibatched SpMM),
// 342-377 (SDDMM dAlpha), 481-495 + 537-588 (softmax / LeakyReLU backward,
// row sums), 258-295 + 614-658 (transposed semibatched SpMM, column sums,
// add_scaled_rows).
#pragma once

namespace g2 {

constexpr int WPB = 8;  // warps (rows) per block
#ifndef GAT_U2
#define GAT_U2 2    // dense-row gathers in flight per warp when R <= 2
#endif
#ifndef GAT_MINB8
#define GAT_MINB8 3  // ... at 8 vectors per lane (2 = no spills, but measured slower)
#endif
#ifndef GAT_MINB
#define GAT_MINB 5  // resident blocks per SM the gather kernels are built for
#endif

// Hub rows / columns (a LongRows plan, internal.cuh): the row kernels skip rows
// longer than `longest`; their SEG instantiation runs one warp per segment
// (row[s], edges [beg[s], end[s])) and writes partials (combined in segment
// order afterwards) or, for per-edge outputs, the final values directly.
struct SegArgs {
  int32_t longest = 0x7fffffff;
  const int32_t* row = nullptr;
  const int32_t* beg = nullptr;
  const int32_t* end = nullptr;
  float4* part = nullptr;  // nseg x fv partial rows
  float* ddpart = nullptr; // nseg x h partial column sums (column pass)
  // aggregation epilogue: ELU(1) on the output and its byte mask (x > 0),
  // row-major like the output (dense.hpp:197-228 activation fused)
  uint8_t* elu_mask = nullptr;
};

// dense-row gathers in flight per warp: 4 16-byte vectors per lane in total
template <int R>
struct Unroll {
  static constexpr int v = R >= 4 ? 1 : 4 / R;
};

template <int H>
struct Log2 {
  static constexpr int v = H == 1 ? 0 : H == 2 ? 1 : H == 4 ? 2 : H == 8 ? 3 : 4;
};

struct OpMax {
  __device__ __forceinline__ float operator()(float a, float b) const { return fmaxf(a, b); }
};
struct OpSum {
  __device__ __forceinline__ float operator()(float a, float b) const { return a + b; }
};

// Reduce v[0..H) over all 32 lanes; on return every lane holds all H results.
template <int H, class Op>
__device__ __forceinline__ void allreduce(float (&v)[H], int lane, Op op) {
  constexpr int LG = Log2<H>::v;
#pragma unroll
  for (int s = 0; s < LG; ++s) {  // reduce-scatter: halve the live values each step
    const int o = 16 >> s;
    const int half = H >> (s + 1);
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int q = 0; q < half; ++q) {
      const float send = up ? v[q] : v[q + half];
      const float keep = up ? v[q + half] : v[q];
      v[q] = op(keep, __shfl_xor_sync(0xffffffffu, send, o));
    }
  }
#pragma unroll
  for (int o = 16 >> LG; o > 0; o >>= 1) v[0] = op(v[0], __shfl_xor_sync(0xffffffffu, v[0], o));
  // lane l now holds head ((l >> (5 - LG)) bit-reversed order below) -- gather back
  const float mine = v[0];
#pragma unroll
  for (int t = 0; t < H; ++t) {
    // head t was kept by lanes whose bits (4, 3, ...) spell t from the top half down
    int src = 0;
#pragma unroll
    for (int s = 0; s < LG; ++s)
      if (t & (H >> (s + 1))) src |= 16 >> s;
    v[t] = __shfl_sync(0xffffffffu, mine, src);
  }
}

// CG: load through L2 (__ldcg) -- values this kernel wrote earlier (the
// read-only __ldg path is not coherent with them)
template <int H, bool CG = false>
__device__ __forceinline__ void ld_heads(const float* __restrict__ p, float (&v)[H]) {
  if constexpr (H % 4 == 0) {
#pragma unroll
    for (int q = 0; q < H / 4; ++q) {
      const float4 x = CG ? __ldcg(reinterpret_cast<const float4*>(p) + q)
                          : __ldg(reinterpret_cast<const float4*>(p) + q);
      v[4 * q] = x.x;
      v[4 * q + 1] = x.y;
      v[4 * q + 2] = x.z;
      v[4 * q + 3] = x.w;
    }
  } else if constexpr (H == 2) {
    const float2 x = CG ? __ldcg(reinterpret_cast<const float2*>(p))
                        : __ldg(reinterpret_cast<const float2*>(p));
    v[0] = x.x;
    v[1] = x.y;
  } else {
    v[0] = CG ? __ldcg(p) : __ldg(p);
  }
}

template <int H>
__device__ __forceinline__ void st_heads(float* __restrict__ p, const float (&v)[H]) {
  if constexpr (H % 4 == 0) {
#pragma unroll
    for (int q = 0; q < H / 4; ++q)
      reinterpret_cast<float4*>(p)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  } else if constexpr (H == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else {
    p[0] = v[0];
  }
}

// (alpha, dy) edge record, head-interleaved: r[2t] = alpha_t, r[2t+1] = dy_t
template <int H>
__device__ __forceinline__ void st_rec(float* __restrict__ r, const float (&a)[H],
                                       const float (&y)[H]) {
  if constexpr (H % 2 == 0) {
#pragma unroll
    for (int t = 0; t < H; t += 2)
      reinterpret_cast<float4*>(r)[t / 2] = make_float4(a[t], y[t], a[t + 1], y[t + 1]);
  } else {
    *reinterpret_cast<float2*>(r) = make_float2(a[0], y[0]);
  }
}

// per-row statistics of the partitioned column pass, [row][head][4] =
// (s, max, 1 / sum, dot): one 16-byte load per (edge, head) in k_gat_col3
template <int H>
__device__ __forceinline__ void st_stats3(float* __restrict__ p, const float (&s)[H],
                                          const float (&mx)[H], const float (&inv)[H]) {
#pragma unroll
  for (int t = 0; t < H; ++t) {
    p[4 * t] = s[t];
    p[4 * t + 1] = mx[t];
    p[4 * t + 2] = inv[t];
  }
}
template <int H>
__device__ __forceinline__ void st_stat(float* __restrict__ p, const float (&v)[H]) {
#pragma unroll
  for (int t = 0; t < H; ++t) p[4 * t] = v[t];
}

template <int H>
__device__ __forceinline__ void st_mask(uint8_t* __restrict__ p, uint32_t bits) {
  if constexpr (H == 8) {
    uint2 w;
    w.x = (bits & 1u) | ((bits >> 1) & 1u) << 8 | ((bits >> 2) & 1u) << 16 | ((bits >> 3) & 1u) << 24;
    w.y = ((bits >> 4) & 1u) | ((bits >> 5) & 1u) << 8 | ((bits >> 6) & 1u) << 16 |
          ((bits >> 7) & 1u) << 24;
    *reinterpret_cast<uint2*>(p) = w;
  } else if constexpr (H == 4) {
    *reinterpret_cast<uint32_t*>(p) =
        (bits & 1u) | ((bits >> 1) & 1u) << 8 | ((bits >> 2) & 1u) << 16 | ((bits >> 3) & 1u) << 24;
  } else if constexpr (H == 2) {
    *reinterpret_cast<uint16_t*>(p) = (uint16_t)((bits & 1u) | ((bits >> 1) & 1u) << 8);
  } else {
    p[0] = (uint8_t)(bits & 1u);
  }
}

template <int H>
__device__ __forceinline__ uint32_t ld_mask(const uint8_t* __restrict__ p) {
  uint32_t w0 = 0, w1 = 0;
  if constexpr (H == 8) {
    const uint2 w = __ldg(reinterpret_cast<const uint2*>(p));
    w0 = w.x;
    w1 = w.y;
  } else if constexpr (H == 4) {
    w0 = __ldg(reinterpret_cast<const uint32_t*>(p));
  } else if constexpr (H == 2) {
    w0 = __ldg(reinterpret_cast<const uint16_t*>(p));
  } else {
    w0 = __ldg(p);
  }
  uint32_t bits = 0;
#pragma unroll
  for (int t = 0; t < H; ++t) {
    const uint32_t b = t < 4 ? (w0 >> (8 * t)) & 0xffu : (w1 >> (8 * (t - 4))) & 0xffu;
    bits |= (b != 0u ? 1u : 0u) << t;
  }
  return bits;
}

__device__ __forceinline__ float lrelu(float y, float beta) { return y > 0.f ? y : beta * y; }

__device__ __forceinline__ void fma4(float4& a, float s, const float4& b) {
  a.x = fmaf(s, b.x, a.x);
  a.y = fmaf(s, b.y, a.y);
  a.z = fmaf(s, b.z, a.z);
  a.w = fmaf(s, b.w, a.w);
}
__device__ __forceinline__ float dot4(const float4& a, const float4& b) {
  return fmaf(a.w, b.w, fmaf(a.z, b.z, fmaf(a.y, b.y, a.x * b.x)));
}

// Per-row softmax statistics over [beg, end): mx[t] = max_e w, inv[t] =
// 1 / sum_e exp(w - mx).  Rows of <= 32 edges keep the lane's scores in
// e[] (= exp(w - mx)) for the caller; longer rows recompute.
template <int H>
__device__ __forceinline__ void row_stats(int lane, int32_t beg, int32_t end,
                                          const int32_t* __restrict__ cols,
                                          const float* __restrict__ d, const float (&si)[H],
                                          float beta, float (&mx)[H], float (&inv)[H],
                                          float (&e)[H], uint32_t& pos) {
  float w[H];
  pos = 0;
#pragma unroll
  for (int t = 0; t < H; ++t) mx[t] = -INFINITY;
  for (int32_t base = beg; base < end; base += 32) {
    const int32_t ee = base + lane;
    if (ee < end) {
      float dj[H];
      ld_heads<H>(d + (int64_t)__ldg(cols + ee) * H, dj);
#pragma unroll
      for (int t = 0; t < H; ++t) {
        const float y = si[t] + dj[t];
        w[t] = lrelu(y, beta);
        if (base == beg && y > 0.f) pos |= 1u << t;
        mx[t] = fmaxf(mx[t], w[t]);
      }
    }
  }
  allreduce<H>(mx, lane, OpMax());
  float sm[H];
  const bool single = end - beg <= 32;
#pragma unroll
  for (int t = 0; t < H; ++t) {
    e[t] = (single && beg + lane < end) ? expf(w[t] - mx[t]) : 0.f;
    sm[t] = e[t];
  }
  if (!single) {
    for (int32_t base = beg; base < end; base += 32) {
      const int32_t ee = base + lane;
      if (ee < end) {
        float dj[H];
        ld_heads<H>(d + (int64_t)__ldg(cols + ee) * H, dj);
#pragma unroll
        for (int t = 0; t < H; ++t) sm[t] += expf(lrelu(si[t] + dj[t], beta) - mx[t]);
      }
    }
  }
  allreduce<H>(sm, lane, OpSum());
#pragma unroll
  for (int t = 0; t < H; ++t) inv[t] = 1.f / sm[t];
}

// alpha of the lane's edge ee for every head (multi-batch rows: recomputed)
template <int H>
__device__ __forceinline__ void edge_alpha(int32_t ee, const int32_t* __restrict__ cols,
                                           const float* __restrict__ d, const float (&si)[H],
                                           float beta, const float (&mx)[H], const float (&inv)[H],
                                           float (&a)[H], uint32_t& pos) {
  float dj[H];
  ld_heads<H>(d + (int64_t)__ldg(cols + ee) * H, dj);
  pos = 0;
#pragma unroll
  for (int t = 0; t < H; ++t) {
    const float y = si[t] + dj[t];
    if (y > 0.f) pos |= 1u << t;
    a[t] = expf(lrelu(y, beta) - mx[t]) * inv[t];
  }
}

// Aggregate one staged batch: acc[r] += sum_j alpha[j][head(r)] * X[col_j] (R
// 16-byte vectors per lane), U gathers in flight.
template <int H, int R>
__device__ __forceinline__ void aggregate(int lane, int cnt, int32_t mycol, int fv,
                                          const float4* __restrict__ X,
                                          float (*sa)[H + 1], const int (&tr)[R],
                                          float4 (&acc)[R]) {
  constexpr int U = Unroll<R>::v;
  for (int jb = 0; jb < cnt; jb += U) {
    float4 x[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = jb + u;
      const uint32_t c = (uint32_t)__shfl_sync(0xffffffffu, mycol, j < cnt ? j : jb);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t v = r * 32 + lane;
        if (j < cnt && v < (uint32_t)fv) x[u][r] = __ldg(X + c * (uint32_t)fv + v);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (jb + u < cnt) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (r * 32 + lane < fv) fma4(acc[r], sa[jb + u][tr[r]], x[u][r]);
      }
    }
  }
}

// Softmax statistics of a row, staged for the warp: single-batch rows (<= 32
// edges) leave alpha of every (edge, head) in sa[lane][t]; longer rows leave
// (s_i, max, 1/sum) in st[0..2][t] for per-batch recomputation.  pos = the
// lane's LeakyReLU mask bits (single-batch rows).
template <int H>
__device__ __forceinline__ uint32_t stage_stats(int lane, int32_t i, int32_t beg, int32_t end,
                                                const int32_t* __restrict__ cols,
                                                const float* __restrict__ s,
                                                const float* __restrict__ d, float beta,
                                                float (*sa)[H + 1], float (*st)[H]) {
  float si[H], mx[H], inv[H], e[H];
  uint32_t pos = 0;
  ld_heads<H>(s + (int64_t)i * H, si);
  row_stats<H>(lane, beg, end, cols, d, si, beta, mx, inv, e, pos);
  if (end - beg <= 32) {
    if (beg + lane < end)
#pragma unroll
      for (int t = 0; t < H; ++t) sa[lane][t] = e[t] * inv[t];
  } else if (lane == 0) {
#pragma unroll
    for (int t = 0; t < H; ++t) {
      st[0][t] = si[t];
      st[1][t] = mx[t];
      st[2][t] = inv[t];
    }
  }
  __syncwarp();
  return pos;
}

// alpha of edge ee of a multi-batch row from the staged statistics
template <int H>
__device__ __forceinline__ uint32_t restage_alpha(int32_t ee, const int32_t* __restrict__ cols,
                                                  const float* __restrict__ d, float beta,
                                                  const float (*st)[H], float* a) {
  float dj[H];
  ld_heads<H>(d + (int64_t)__ldg(cols + ee) * H, dj);
  uint32_t pos = 0;
#pragma unroll
  for (int t = 0; t < H; ++t) {
    const float y = st[0][t] + dj[t];
    if (y > 0.f) pos |= 1u << t;
    a[t] = expf(lrelu(y, beta) - st[1][t]) * st[2][t];
  }
  return pos;
}

// ---------------------------------------------------------------------------
// forward, part 2 (kernels.hpp:219-254 semibatched SpMM + bias):
// out[i, t, :] = sum_e alpha[e, t] M[col_e, t, :] + b.  Lean like the GCN
// SpMM: one warp per row, per edge a broadcast column index, one 4-byte
// attention load per lane (its head; 32-byte sector per edge) and R 16-byte
// row vectors, U edges in flight; <= 40 registers for 48 resident warps/SM.
// ---------------------------------------------------------------------------
// LDA: the attention load (__ldg; __ldcg when the same kernel just wrote it)
struct LdgA {
  static __device__ __forceinline__ float ld(const float* p) { return __ldg(p); }
};
struct LdcgA {
  static __device__ __forceinline__ float ld(const float* p) { return __ldcg(p); }
};

template <int H, int R, bool SEG, class LDA>
__device__ __forceinline__ void agg2_row(int32_t i, int vo, int32_t n,
                                         const int32_t* __restrict__ rowptr,
                                         const int32_t* __restrict__ cols,
                                         const float* __restrict__ alpha,
                                         const float4* __restrict__ M, int32_t k,
                                         const float4* __restrict__ bias,
                                         float4* __restrict__ out, const SegArgs& sg) {
  constexpr int U = R >= 4 ? 1 : (R <= 2 ? GAT_U2 : 2);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int fv = H * k / 4, L = k / 4;
  int32_t beg, end;
  if (SEG) {
    beg = __ldg(sg.beg + i);
    end = __ldg(sg.end + i);
  } else {
    beg = __ldg(rowptr + i);
    end = __ldg(rowptr + i + 1);
    if (end - beg > sg.longest) return;
  }
  int tr[R];
  float4 acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    tr[r] = min(H - 1, (vo + r * 32 + lane) / L);
    acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // 32-lane chunks per head (k/4 = 32C; only the 8-vector wide-slab kernels
  // test it, the narrow ones keep C = 1 at compile time)
  const int C = (R == 8 && (L & 31) == 0) ? L >> 5 : 1;
  int32_t e = beg;
  for (; e + U <= end; e += U) {
    uint32_t c[U];
    float a[U][R];
    float4 x[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = (uint32_t)__ldg(cols + e + u);
#pragma unroll
      for (int r = 0; r < R; ++r)  // once per head when heads span whole chunks
        a[u][r] = r % C == 0 ? LDA::ld(alpha + (int64_t)(e + u) * H + tr[r]) : a[u][r - 1];
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t v = vo + r * 32 + lane;
        if (v < (uint32_t)fv) x[u][r] = __ldg(M + c[u] * (uint32_t)fv + v);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (vo + r * 32 + lane < fv) fma4(acc[r], a[u][r], x[u][r]);
  }
  for (; e < end; ++e) {
    const uint32_t c = (uint32_t)__ldg(cols + e);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t v = vo + r * 32 + lane;
      if (v < (uint32_t)fv)
        fma4(acc[r], LDA::ld(alpha + (int64_t)e * H + tr[r]), __ldg(M + c * (uint32_t)fv + v));
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int v = vo + r * 32 + lane;
    if (v < fv) {
      if (SEG) {
        sg.part[(int64_t)i * fv + v] = acc[r];
        continue;
      }
      const float4 b = __ldg(bias + v);
      float4 o = acc[r];
      o.x += b.x;
      o.y += b.y;
      o.z += b.z;
      o.w += b.w;
      if (sg.elu_mask) {  // same expressions as the separate activation pass
        const uint32_t mb = (o.x > 0.f ? 1u : 0u) | (o.y > 0.f ? 1u : 0u) << 8 |
                            (o.z > 0.f ? 1u : 0u) << 16 | (o.w > 0.f ? 1u : 0u) << 24;
        o.x = o.x > 0.f ? o.x : __fmul_rn(1.f, expf(o.x) - 1.f);
        o.y = o.y > 0.f ? o.y : __fmul_rn(1.f, expf(o.y) - 1.f);
        o.z = o.z > 0.f ? o.z : __fmul_rn(1.f, expf(o.z) - 1.f);
        o.w = o.w > 0.f ? o.w : __fmul_rn(1.f, expf(o.w) - 1.f);
        reinterpret_cast<uint32_t*>(sg.elu_mask)[(int64_t)i * fv + v] = mb;
      }
      __stcs(out + (int64_t)i * fv + v, o);
    }
  }
}

template <int H, int R, bool SEG = false>
__global__ void __launch_bounds__(256, R <= 2 ? GAT_MINB : (R >= 8 ? GAT_MINB8 : 3))
    k_gat_agg2(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
               const float* __restrict__ alpha, const float4* __restrict__ M, int32_t k,
               const float4* __restrict__ bias, float4* __restrict__ out, SegArgs sg = {}) {
  // column window blockIdx.y (slabs wider than 32R vectors), one warp per row
  agg2_row<H, R, SEG, LdgA>((int32_t)((blockIdx.x * 256u + threadIdx.x) >> 5),
                            blockIdx.y * 32 * R, n, rowptr, cols, alpha, M, k, bias, out, sg);
}

// ---------------------------------------------------------------------------
// backward, part 1 (kernels.hpp:342-377 semibatched SDDMM): dAlpha[e, t] =
// <dX'[i, t, :], M[col_e, t, :]>, edge-major.  Lean warp per row: the row of
// dX' stays in registers, R 16-byte vectors of M gathered per edge, U edges
// in flight.  P2 = 1 (k/4 a power of two <= 32, heads aligned to lane groups):
// head-segmented xor reductions over the k/4 lanes of a head; P2 = C >= 2
// (k/4 = 32C, a head spans C whole 32-lane chunks): the chunks are folded in
// registers and the heads' dots reduce-scattered over the warp; P2 = 0: the
// per-vector partial dots go through shared memory and H*U lanes fold the
// k/4 partials of their (edge, head).
// ---------------------------------------------------------------------------
template <int R>
struct SddmmU {
  static constexpr int v = R >= 4 ? 1 : (R <= 2 ? GAT_U2 : 2);
};

// one row (or hub segment) i of the SDDMM over column window vo; sh_p: the
// warp's shared-memory fold buffer (P2 == 0 only)
template <int H, int R, int P2, bool SEG>
__device__ __forceinline__ void sddmm2_row(int32_t i, int vo, int32_t n,
                                           const int32_t* __restrict__ rowptr,
                                           const int32_t* __restrict__ cols,
                                           const float4* __restrict__ M,
                                           const float4* __restrict__ G, int32_t k,
                                           float* __restrict__ da, const SegArgs& sg,
                                           float (*sh_p)[P2 ? 1 : 32 * R]) {
  constexpr int U = SddmmU<R>::v;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int fv = H * k / 4, L = k / 4;
  int32_t beg, end, grow = i;  // grow: the row of dX' this warp dots against
  if (SEG) {
    beg = __ldg(sg.beg + i);
    end = __ldg(sg.end + i);
    grow = __ldg(sg.row + i);
  } else {
    beg = __ldg(rowptr + i);
    end = __ldg(rowptr + i + 1);
    if (end - beg > sg.longest) return;
  }
  int tr[R];
  float4 g[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int v = vo + r * 32 + lane;
    tr[r] = min(H - 1, v / L);
    g[r] = v < fv ? __ldg(G + (int64_t)grow * fv + v) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const bool lead = P2 == 1 && (lane & (L - 1)) == 0;
  for (int32_t e = beg; e < end; e += U) {
    uint32_t c[U];
    float4 x[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = (uint32_t)__ldg(cols + min(e + u, end - 1));
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t v = vo + r * 32 + lane;
        if (v < (uint32_t)fv) x[u][r] = __ldg(M + c[u] * (uint32_t)fv + v);
      }
    if constexpr (P2 >= 2) {
      // heads of C = P2 whole chunks: fold chunk partials per head (in chunk
      // order), then reduce the NV = U * R / C head dots over all 32 lanes by a
      // reduce-scatter (log2(NV) halving steps, then plain xor steps)
      constexpr int C = P2, NH = R / C, NV = U * NH;
      static_assert(R % C == 0 && (NV & (NV - 1)) == 0 && NV <= 32, "wide-head SDDMM shape");
      float p[NV];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int qh = 0; qh < NH; ++qh) {
          float a = 0.f;
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const int r = qh * C + c;
            a += vo + r * 32 + lane < fv ? dot4(g[r], x[u][r]) : 0.f;
          }
          p[u * NH + qh] = a;
        }
      int off = 16;
#pragma unroll
      for (int half = NV / 2; half >= 1; half >>= 1, off >>= 1) {
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int q = 0; q < half; ++q) {
          const float send = up ? p[q] : p[q + half];
          const float keep = up ? p[q + half] : p[q];
          p[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      for (; off > 0; off >>= 1) p[0] += __shfl_xor_sync(0xffffffffu, p[0], off);
      int idx = 0;
      {
        int o2 = 16;
#pragma unroll
        for (int half = NV / 2; half >= 1; half >>= 1, o2 >>= 1)
          if (lane & o2) idx += half;
      }
      const int u = idx / NH, t = vo / L + idx % NH;
      if ((lane & ((32 / NV) - 1)) == 0 && e + u < end && t < H) da[(int64_t)(e + u) * H + t] = p[0];
      continue;
    }
    if (P2 == 1 && U * R <= L) {
      // transposed reduction: the U*R partial dots of a lane are reduced over
      // the L lanes of its head by a reduce-scatter (each step halves the live
      // values) -- log2(U*R) + ... shuffles instead of U*R*log2(L); lane bits
      // above the remaining xor range then name the (edge, chunk) it holds
      constexpr int NV = U * R;
      float p[NV];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < R; ++r)
          p[u * R + r] = vo + r * 32 + lane < fv ? dot4(g[r], x[u][r]) : 0.f;
      int off = L >> 1;
#pragma unroll
      for (int half = NV / 2; half >= 1; half >>= 1, off >>= 1) {
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int q = 0; q < half; ++q) {
          const float send = up ? p[q] : p[q + half];
          const float keep = up ? p[q + half] : p[q];
          p[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      for (; off > 0; off >>= 1) p[0] += __shfl_xor_sync(0xffffffffu, p[0], off);
      // value index held: bits of (lane & (L/2 .. L/NV)) from the top down
      int idx = 0;
      {
        int o2 = L >> 1;
#pragma unroll
        for (int half = NV / 2; half >= 1; half >>= 1, o2 >>= 1)
          if (lane & o2) idx += half;
      }
      const int u = idx / R, r = idx % R;
      if ((lane & ((L / NV) - 1)) == 0 && e + u < end && vo + r * 32 + lane < fv)
        da[(int64_t)(e + u) * H + min(H - 1, (vo + r * 32 + lane) / L)] = p[0];
      continue;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float p[R];
#pragma unroll
      for (int r = 0; r < R; ++r) p[r] = vo + r * 32 + lane < fv ? dot4(g[r], x[u][r]) : 0.f;
      if constexpr (P2 == 1) {
        for (int o = L >> 1; o > 0; o >>= 1)
#pragma unroll
          for (int r = 0; r < R; ++r) p[r] += __shfl_xor_sync(0xffffffffu, p[r], o);
        if (lead && e + u < end)
#pragma unroll
          for (int r = 0; r < R; ++r)
            if (vo + r * 32 + lane < fv) da[(int64_t)(e + u) * H + tr[r]] = p[r];
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (vo + r * 32 + lane < fv) sh_p[u][r * 32 + lane] = p[r];
      }
    }
    if constexpr (P2 == 0) {
      __syncwarp();
      const int hw = min(H, (32 * R) / L);  // heads of this window (whole: L | 32R)
      if (lane < U * hw) {
        const int u = lane / hw, tl = lane % hw, t = vo / L + tl;
        float acc = 0.f;
        for (int q = 0; q < L; ++q) acc += sh_p[u][tl * L + q];
        if (e + u < end && t < H) da[(int64_t)(e + u) * H + t] = acc;
      }
      __syncwarp();
    }
  }
}

template <int H, int R, int P2, bool SEG = false>
__global__ void __launch_bounds__(256, R <= 2 ? GAT_MINB : (R >= 8 ? GAT_MINB8 : 3))
    k_gat_sddmm2(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
                 const float4* __restrict__ M, const float4* __restrict__ G, int32_t k,
                 float* __restrict__ da, SegArgs sg = {}) {
  __shared__ float sh_p[P2 ? 1 : WPB][P2 ? 1 : SddmmU<R>::v][P2 ? 1 : 32 * R];  // P2 == 0 only
  const int wib = threadIdx.x >> 5;
  // column window blockIdx.y (slabs wider than 32R vectors), one warp per row
  sddmm2_row<H, R, P2, SEG>((int32_t)((blockIdx.x * 256u + threadIdx.x) >> 5),
                            blockIdx.y * 32 * R, n, rowptr, cols, M, G, k, da, sg,
                            sh_p[P2 ? 0 : wib]);
}

// ---------------------------------------------------------------------------
// SDDMM for head widths L = k/4 that are not a power of two (e.g. k = 40):
// each head gets LP = 8 or 16 lanes (the next power of two, lanes q >= L
// idle), so the per-head dots reduce with the transposed xor reduce-scatter
// of the power-of-two path instead of the shared-memory fold.  One column
// window (H * LP <= 32 R lanes' worth); U = 2 edges in flight.
// ---------------------------------------------------------------------------
template <int H, int LP, bool SEG = false>
__global__ void __launch_bounds__(256, 3)
    k_gat_sddmm_pad(int32_t n, const int32_t* __restrict__ rowptr,
                    const int32_t* __restrict__ cols, const float4* __restrict__ M,
                    const float4* __restrict__ G, int32_t k, float* __restrict__ da,
                    SegArgs sg = {}) {
  constexpr int R = (H * LP + 31) / 32, U = 2, NV = U * R;
  static_assert(NV <= LP && (NV & (NV - 1)) == 0, "padded SDDMM shape");
  const int lane = threadIdx.x & 31;
  const int32_t i = (int32_t)((blockIdx.x * 256u + threadIdx.x) >> 5);
  if (i >= n) return;
  const int L = k / 4, fv = H * L;
  int32_t beg, end, grow = i;
  if (SEG) {
    beg = __ldg(sg.beg + i);
    end = __ldg(sg.end + i);
    grow = __ldg(sg.row + i);
  } else {
    beg = __ldg(rowptr + i);
    end = __ldg(rowptr + i + 1);
    if (end - beg > sg.longest) return;
  }
  int vv[R];  // vector of slot (r, lane), -1 for a padding lane
  float4 g[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int slot = r * 32 + lane, t = slot / LP, q = slot % LP;
    vv[r] = (q < L && t < H) ? t * L + q : -1;
    g[r] = vv[r] >= 0 ? __ldg(G + (int64_t)grow * fv + vv[r]) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // value index a lane holds after the reduce-scatter: bits LP/2 .. LP/NV
  int idx = 0;
  {
    int o2 = LP >> 1;
#pragma unroll
    for (int half = NV / 2; half >= 1; half >>= 1, o2 >>= 1)
      if (lane & o2) idx += half;
  }
  const int ou = idx / R, orr = idx % R;
  const int ot = (orr * 32 + lane) / LP;
  const bool writer = (lane & ((LP / NV) - 1)) == 0 && ot < H;
  for (int32_t e = beg; e < end; e += U) {
    uint32_t c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = (uint32_t)__ldg(cols + min(e + u, end - 1));
    float p[NV];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float4 x[R];
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (vv[r] >= 0) x[r] = __ldg(M + c[u] * (uint32_t)fv + vv[r]);
#pragma unroll
      for (int r = 0; r < R; ++r) p[u * R + r] = vv[r] >= 0 ? dot4(g[r], x[r]) : 0.f;
    }
    int off = LP >> 1;
#pragma unroll
    for (int half = NV / 2; half >= 1; half >>= 1, off >>= 1) {
      const bool up = (lane & off) != 0;
#pragma unroll
      for (int q = 0; q < half; ++q) {
        const float send = up ? p[q] : p[q + half];
        const float keep = up ? p[q + half] : p[q];
        p[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
    for (; off > 0; off >>= 1) p[0] += __shfl_xor_sync(0xffffffffu, p[0], off);
    if (writer && e + ou < end) da[(int64_t)(e + ou) * H + ot] = p[0];
  }
}

// ---------------------------------------------------------------------------
// backward, part 3, per source column j over the CSC view (kernels.hpp:
// 258-295 transposed semibatched SpMM, 640-658 column sums, 614-636
// add_scaled_rows): dM[j] = sum_e alpha[e] dX'[row_e] + dS[j] a_src + dD[j]
// a_dst with dD[j, t] = sum_e dy[e, t].  Lean warp per column: per edge the
// canonical index and row are broadcast loads, alpha / dy one 4-byte load per
// lane (its head), the dX' row R 16-byte vectors; the lanes of a head carry
// identical dD sums, so no reduction is needed.
// ---------------------------------------------------------------------------
// REC: alpha points at (alpha, dy) records in CSC order (st_rec layout, 2H
// floats per position, written by the softmax backward at the edge's CSC
// position): one 8-byte load per (edge, head) at p instead of two 4-byte loads
// through perm (dy unused)
template <int H, int R, bool SEG = false, bool REC = false>
__global__ void __launch_bounds__(256, R <= 2 ? GAT_MINB : (R >= 8 ? GAT_MINB8 : 3)) k_gat_col2(
    int32_t n, const int32_t* __restrict__ colptr, const int32_t* __restrict__ crows,
    const int32_t* __restrict__ perm, const float4* __restrict__ G,
    const float* __restrict__ alpha, const float* __restrict__ dy, const float* __restrict__ dS,
    const float4* __restrict__ a_src, const float4* __restrict__ a_dst, int32_t k,
    float* __restrict__ dD, float4* __restrict__ dM, SegArgs sg = {}) {
  constexpr int U = R >= 4 ? 1 : (R <= 2 ? GAT_U2 : 2);
  const int lane = threadIdx.x & 31;
  const int vo = blockIdx.y * 32 * R;  // column window (slabs wider than 32R vectors)
  const int32_t j = (int32_t)((blockIdx.x * 256u + threadIdx.x) >> 5);
  if (j >= n) return;
  const int fv = H * k / 4, L = k / 4;
  int32_t beg, end;
  if (SEG) {
    beg = __ldg(sg.beg + j);
    end = __ldg(sg.end + j);
  } else {
    beg = __ldg(colptr + j);
    end = __ldg(colptr + j + 1);
    if (end - beg > sg.longest) return;
  }
  int tr[R];
  float4 acc[R];
  float dd[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    tr[r] = min(H - 1, (vo + r * 32 + lane) / L);
    acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    dd[r] = 0.f;
  }
  // heads of C whole 32-lane chunks (k/4 = 32C): alpha / dy are loaded once per
  // head, the other chunks reuse alpha and take the head's dy sum at the end
  const int C = (R == 8 && (L & 31) == 0) ? L >> 5 : 1;
  int32_t p = beg;
  for (; p + U <= end; p += U) {
    uint32_t row[U];
    int32_t e[U];
    float a[U][R];
    float4 x[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if constexpr (!REC) e[u] = __ldg(perm + p + u);
      row[u] = (uint32_t)__ldg(crows + p + u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t v = vo + r * 32 + lane;
        if (r % C == 0) {  // first chunk of its head (every chunk when C == 1)
          if constexpr (REC) {
            const float2 ay = __ldg(reinterpret_cast<const float2*>(alpha) + (int64_t)(p + u) * H + tr[r]);
            a[u][r] = ay.x;
            dd[r] += ay.y;
          } else {
            a[u][r] = __ldg(alpha + (int64_t)e[u] * H + tr[r]);
            dd[r] += __ldg(dy + (int64_t)e[u] * H + tr[r]);
          }
        } else {
          a[u][r] = a[u][r - 1];
        }
        if (v < (uint32_t)fv) x[u][r] = __ldg(G + row[u] * (uint32_t)fv + v);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (vo + r * 32 + lane < fv) fma4(acc[r], a[u][r], x[u][r]);
  }
  for (; p < end; ++p) {
    const int32_t e = REC ? 0 : __ldg(perm + p);
    const uint32_t row = (uint32_t)__ldg(crows + p);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t v = vo + r * 32 + lane;
      float a;
      if constexpr (REC) {
        const float2 ay = __ldg(reinterpret_cast<const float2*>(alpha) + (int64_t)p * H + tr[r]);
        a = ay.x;
        dd[r] += ay.y;
      } else {
        a = __ldg(alpha + (int64_t)e * H + tr[r]);
        dd[r] += __ldg(dy + (int64_t)e * H + tr[r]);
      }
      if (v < (uint32_t)fv) fma4(acc[r], a, __ldg(G + row * (uint32_t)fv + v));
    }
  }
#pragma unroll
  for (int r = 1; r < R; ++r)  // chunks after a head's first take its dy sum
    if (r % C != 0) dd[r] = dd[r - 1];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int v = vo + r * 32 + lane;
    if (v < fv) {
      if (SEG) {
        sg.part[(int64_t)j * fv + v] = acc[r];
        if (v % L == 0) sg.ddpart[(int64_t)j * H + tr[r]] = dd[r];
        continue;
      }
      if (v % L == 0) dD[(int64_t)j * H + tr[r]] = dd[r];
      const float cs = __ldg(dS + (int64_t)j * H + tr[r]);
      const float4 as = __ldg(a_src + v), ad = __ldg(a_dst + v);
      float4 o = acc[r];
      fma4(o, cs, as);
      fma4(o, dd[r], ad);
      __stcs(dM + (int64_t)j * fv + v, o);
    }
  }
}

// ---------------------------------------------------------------------------
// Column pass of the row-partitioned layer (dist.DistGatLayer) that rebuilds
// the per-edge values from per-row statistics instead of reading alpha / dy
// (all-gather 4 n h row statistics, not 2 q' h edge values).
// Row statistics, [row][H][4]: s (node score), max and 1 / sum of the softmax
// (k_gat_attn4 / k_gat_attn_long), and dot = sum_e alpha dAlpha
// (k_gat_sbwd4 / k_gat_sbwd_long) -- one 16-byte load per (edge, head).  Per edge (row i, column j):
//   y = s_i + d_j, alpha = exp(lrelu(y) - max_i) * inv_i      (= k_gat_attn4)
//   dAlpha = <dX'_i, M_j> per head                            (kernels.hpp:342-377)
//   dy = alpha (dAlpha - dot_i), times beta where y <= 0      (= k_gat_sbwd4)
// and then exactly what k_gat_col2 accumulates.  dX'_i is the row the column
// pass gathers anyway and M_j is the column's own row, so rebuilding dAlpha
// costs shuffles, not bytes.  Head reductions: L = k/4 <= 32 a power of two
// (xor over the head's lanes) or L = 32C with R % C == 0 (chunks folded in
// registers, then xor over the warp).  Every lane of a head ends with the
// head's dAlpha, so dD needs no reduction (as in k_gat_col2).
// ---------------------------------------------------------------------------
template <int H, int R, bool SEG = false>
__global__ void __launch_bounds__(256, R >= 8 ? 1 : (R >= 3 ? 2 : 4)) k_gat_col3(
    int32_t n, const int32_t* __restrict__ colptr, const int32_t* __restrict__ crows,
    const float4* __restrict__ G, const float* __restrict__ stats, const float* __restrict__ dloc,
    const float4* __restrict__ Mloc, float beta, const float* __restrict__ dS,
    const float4* __restrict__ a_src, const float4* __restrict__ a_dst, int32_t k,
    float* __restrict__ dD, float4* __restrict__ dM, SegArgs sg = {}) {
  constexpr int U = R >= 4 ? 1 : 2;
  const int lane = threadIdx.x & 31;
  const int vo = blockIdx.y * 32 * R;
  const int32_t q = (int32_t)((blockIdx.x * 256u + threadIdx.x) >> 5);
  if (q >= n) return;
  const int fv = H * k / 4, L = k / 4;
  int32_t beg, end, j = q;
  if (SEG) {
    beg = __ldg(sg.beg + q);
    end = __ldg(sg.end + q);
    j = __ldg(sg.row + q);
  } else {
    beg = __ldg(colptr + q);
    end = __ldg(colptr + q + 1);
    if (end - beg > sg.longest) return;
  }
  // heads of C whole chunks (L = 32C): fold the C chunk partials of a head
  const int C = L > 32 ? L >> 5 : 1;
  const int red = L > 32 ? 32 : L;  // lanes the head dot is xor-reduced over
  int tr[R];
  float4 acc[R], mj[R];
  float dd[R], dj[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int v = vo + r * 32 + lane;
    tr[r] = min(H - 1, v / L);
    acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    dd[r] = 0.f;
    mj[r] = v < fv ? __ldg(Mloc + (int64_t)j * fv + v) : make_float4(0.f, 0.f, 0.f, 0.f);
    dj[r] = __ldg(dloc + (int64_t)j * H + tr[r]);
  }
  for (int32_t p = beg; p < end; p += U) {
    uint32_t row[U];
    float4 x[U][R];
    float pd[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u) row[u] = (uint32_t)__ldg(crows + min(p + u, end - 1));
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t v = vo + r * 32 + lane;
        x[u][r] = v < (uint32_t)fv ? __ldg(G + row[u] * (uint32_t)fv + v)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
        pd[u][r] = dot4(x[u][r], mj[r]);
      }
    // per-head dAlpha on every lane of the head
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (C > 1) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (r % C == 0) {
            float a = 0.f;
#pragma unroll
            for (int c = 0; c < R; ++c)
              if (c < C && r + c < R) a += pd[u][r + c];
            pd[u][r] = a;
          }
      }
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (r % C == 0)
          for (int o = red >> 1; o > 0; o >>= 1)
            pd[u][r] += __shfl_xor_sync(0xffffffffu, pd[u][r], o);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (p + u >= end) break;
      const float4* st = reinterpret_cast<const float4*>(stats) + (int64_t)row[u] * H;
      float a[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r % C == 0) {  // first chunk of its head: alpha and dy of (edge, head)
          const float4 q = __ldg(st + tr[r]);  // (s, max, 1 / sum, dot) of (row, head)
          const float y = q.x + dj[r];
          a[r] = expf(lrelu(y, beta) - q.y) * q.z;
          const float dw = a[r] * (pd[u][r] - q.w);
          dd[r] += y > 0.f ? dw : beta * dw;
        } else {
          a[r] = a[r - 1];
        }
        if (vo + r * 32 + lane < fv) fma4(acc[r], a[r], x[u][r]);
      }
    }
  }
#pragma unroll
  for (int r = 1; r < R; ++r)
    if (r % C != 0) dd[r] = dd[r - 1];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int v = vo + r * 32 + lane;
    if (v < fv) {
      if (SEG) {
        sg.part[(int64_t)q * fv + v] = acc[r];
        if (v % L == 0) sg.ddpart[(int64_t)q * H + tr[r]] = dd[r];
        continue;
      }
      if (v % L == 0) dD[(int64_t)j * H + tr[r]] = dd[r];
      const float cs = __ldg(dS + (int64_t)j * H + tr[r]);
      const float4 as = __ldg(a_src + v), ad = __ldg(a_dst + v);
      float4 o = acc[r];
      fma4(o, cs, as);
      fma4(o, dd[r], ad);
      __stcs(dM + (int64_t)j * fv + v, o);
    }
  }
}

// ---------------------------------------------------------------------------
// backward, part 4: the three column-sum gradients in one pass over the rows
// (dense.hpp:272-282 column_sums for d_bias = 1^T dX'; kernels.hpp:592-611
// attention_param_grad for d_a_src = sum_i dS[i,t] M[i,t,:] and d_a_dst with
// dD).  Block partials in float64, threads own 16-byte column vectors, row
// groups combined in a fixed order; k_grads3_final_col folds the partials.
// part layout: [block][3][hk] (db | d_a_src | d_a_dst, the latter h x k).
// ---------------------------------------------------------------------------
template <int H>
__global__ void __launch_bounds__(256) k_grads3_partial(int32_t n, int32_t k,
                                                        const float4* __restrict__ G,
                                                        const float4* __restrict__ M,
                                                        const float* __restrict__ dS,
                                                        const float* __restrict__ dD,
                                                        int32_t chunk, double* __restrict__ part) {
  __shared__ double sh[3][256][4];
  const int fv = H * k / 4, L = k / 4;
  const int fvw = min(fv, 256);  // vectors of this column window (gridDim.y windows)
  const int groups = max(1, 256 / fvw);
  const int tid = threadIdx.x, v = blockIdx.y * 256 + tid % fvw, grp = tid / fvw;
  const int t = min(H - 1, v / L);
  const int32_t r0 = blockIdx.x * chunk, r1 = min(n, r0 + chunk);
  double a[3][4] = {};
  if (grp < groups && v < fv) {
#pragma unroll 2
    for (int32_t i = r0 + grp; i < r1; i += groups) {
      const float4 g = __ldg(G + (int64_t)i * fv + v);
      const float4 mm = __ldg(M + (int64_t)i * fv + v);
      const double cs = (double)__ldg(dS + (int64_t)i * H + t);
      const double cd = (double)__ldg(dD + (int64_t)i * H + t);
      a[0][0] += g.x;
      a[0][1] += g.y;
      a[0][2] += g.z;
      a[0][3] += g.w;
      a[1][0] += cs * mm.x;
      a[1][1] += cs * mm.y;
      a[1][2] += cs * mm.z;
      a[1][3] += cs * mm.w;
      a[2][0] += cd * mm.x;
      a[2][1] += cd * mm.y;
      a[2][2] += cd * mm.z;
      a[2][3] += cd * mm.w;
    }
  }
#pragma unroll
  for (int q = 0; q < 3; ++q)
#pragma unroll
    for (int c = 0; c < 4; ++c) sh[q][tid][c] = a[q][c];
  __syncthreads();
  if (grp == 0 && v < fv) {
    for (int gg = 1; gg < groups; ++gg)
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int c = 0; c < 4; ++c) a[q][c] += sh[q][gg * fvw + tid % fvw][c];
    double* o = part + (int64_t)blockIdx.x * 3 * fv * 4;
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int c = 0; c < 4; ++c) o[(int64_t)q * fv * 4 + v * 4 + c] = a[q][c];
  }
}

// out[q][c] = sum over blocks of part[b][q][c], one block per output column
// (grid hk x 3): threads stride the nb partials, then a fixed smem tree -- a
// few L2 round trips instead of nb / 32 dependent ones per lane (hk = 256:
// 18 -> 6 us)
__global__ void __launch_bounds__(256) k_grads3_final_col(int32_t nb, int32_t hk,
                                                          const double* __restrict__ part,
                                                          float* __restrict__ db,
                                                          float* __restrict__ das,
                                                          float* __restrict__ dad) {
  __shared__ double sh[256];
  const int32_t c = blockIdx.x;
  const int q = blockIdx.y;
  const int64_t st = 3LL * hk;
  const double* p = part + (int64_t)q * hk + c;
  double s = 0.0;
  for (int32_t b = threadIdx.x; b < nb; b += 256) s += p[b * st];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) (q == 0 ? db : q == 1 ? das : dad)[c] = (float)sh[0];
}

// ---------------------------------------------------------------------------
// Sub-warp variants of the attention and softmax-backward kernels: a group of
// GS = 16 lanes owns a row (2 rows per warp), lanes over the row's edges, so
// the per-edge vectors (d rows, alpha, dAlpha, dy, mask: h values each) are
// read and written as contiguous, coalesced spans.  Group reductions are the
// transposed butterfly of allreduce() restricted to the 16 lanes; loops run a
// warp-uniform trip count (the longer of the two rows) so every shuffle has
// all lanes.
// ---------------------------------------------------------------------------
constexpr int GS = 16;

template <int H, class Op>
__device__ __forceinline__ void group_allreduce(float (&v)[H], int gl, Op op) {
  constexpr int LG = Log2<H>::v;
#pragma unroll
  for (int st = 0; st < LG; ++st) {
    const int o = (GS / 2) >> st;
    const int half = H >> (st + 1);
    const bool up = (gl & o) != 0;
#pragma unroll
    for (int q = 0; q < half; ++q) {
      const float send = up ? v[q] : v[q + half];
      const float keep = up ? v[q + half] : v[q];
      v[q] = op(keep, __shfl_xor_sync(0xffffffffu, send, o));
    }
  }
#pragma unroll
  for (int o = (GS / 2) >> LG; o > 0; o >>= 1)
    v[0] = op(v[0], __shfl_xor_sync(0xffffffffu, v[0], o));
  const float mine = v[0];
#pragma unroll
  for (int t = 0; t < H; ++t) {
    int src = 0;
#pragma unroll
    for (int st = 0; st < LG; ++st)
      if (t & (H >> (st + 1))) src |= (GS / 2) >> st;
    v[t] = __shfl_sync(0xffffffffu, mine, src, GS);
  }
}

template <int H>
__device__ __forceinline__ void attn4_rows(int32_t i, int32_t n, const int32_t* __restrict__ rowptr,
                                           const int32_t* __restrict__ cols,
                                           const float* __restrict__ s,
                                           const float* __restrict__ d, float beta,
                                           float* __restrict__ alpha,
                                           uint8_t* __restrict__ mask, int32_t longest,
                                           float* __restrict__ stats) {
  // i: this 16-lane group's row (two rows per warp)
  const int lane = threadIdx.x & 31, gl = lane & (GS - 1);
  int32_t beg = 0, end = 0;
  if (i < n) {
    beg = __ldg(rowptr + i);
    end = __ldg(rowptr + i + 1);
  }
  const int32_t deg = end - beg > longest ? 0 : end - beg;  // hub rows: k_gat_attn_long
  const int32_t wdeg = max(deg, __shfl_xor_sync(0xffffffffu, deg, GS));  // warp-uniform
  if (wdeg == 0) return;
  float si[H];
  if (i < n) ld_heads<H>(s + (int64_t)i * H, si);
  float w[H], mx[H], sm[H];
#pragma unroll
  for (int t = 0; t < H; ++t) {
    mx[t] = -INFINITY;
    sm[t] = 0.f;
  }
  uint32_t pos1 = 0;  // mask bits of the lane's edge (single-pass rows)
  for (int32_t off = 0; off < wdeg; off += GS) {  // max
    const int32_t e = beg + off + gl;
    if (off + gl < deg) {
      float dj[H];
      ld_heads<H>(d + (int64_t)__ldg(cols + e) * H, dj);
      pos1 = 0;
#pragma unroll
      for (int t = 0; t < H; ++t) {
        const float y = si[t] + dj[t];
        if (y > 0.f) pos1 |= 1u << t;
        w[t] = lrelu(y, beta);
        mx[t] = fmaxf(mx[t], w[t]);
      }
    }
  }
  group_allreduce<H>(mx, gl, OpMax());
  const bool one = wdeg <= GS;  // the lane's scores are still in w[]
  for (int32_t off = 0; off < wdeg; off += GS) {  // sum
    const int32_t e = beg + off + gl;
    if (off + gl < deg) {
      if (!one) {
        float dj[H];
        ld_heads<H>(d + (int64_t)__ldg(cols + e) * H, dj);
#pragma unroll
        for (int t = 0; t < H; ++t) w[t] = lrelu(si[t] + dj[t], beta);
      }
#pragma unroll
      for (int t = 0; t < H; ++t) {
        const float ex = expf(w[t] - mx[t]);
        sm[t] += ex;
        if (one) w[t] = ex;  // single-pass rows keep exp(w - max) for alpha
      }
    }
  }
  group_allreduce<H>(sm, gl, OpSum());
#pragma unroll
  for (int t = 0; t < H; ++t) sm[t] = 1.f / sm[t];
  if (stats && gl == 0 && deg > 0) {  // row statistics for k_gat_col3: s, max, 1 / sum
    st_stats3<H>(stats + (int64_t)i * 4 * H, si, mx, sm);
  }
  for (int32_t off = 0; off < wdeg; off += GS) {  // alpha, mask
    const int32_t e = beg + off + gl;
    if (off + gl < deg) {
      float a[H];
      uint32_t pos = pos1;
      if (one) {  // exp(w - max) still in registers: no second gather or exp
#pragma unroll
        for (int t = 0; t < H; ++t) a[t] = w[t] * sm[t];
      } else {
        float dj[H];
        pos = 0;
        ld_heads<H>(d + (int64_t)__ldg(cols + e) * H, dj);
#pragma unroll
        for (int t = 0; t < H; ++t) {
          const float y = si[t] + dj[t];
          if (y > 0.f) pos |= 1u << t;
          a[t] = expf(lrelu(y, beta) - mx[t]) * sm[t];
        }
      }
      st_heads<H>(alpha + (int64_t)e * H, a);
      if (mask) st_mask<H>(mask + (int64_t)e * H, pos);
    }
  }
}

template <int H>
__global__ void __launch_bounds__(256) k_gat_attn4(int32_t n, const int32_t* __restrict__ rowptr,
                                                   const int32_t* __restrict__ cols,
                                                   const float* __restrict__ s,
                                                   const float* __restrict__ d, float beta,
                                                   float* __restrict__ alpha,
                                                   uint8_t* __restrict__ mask,
                                                   int32_t longest = 0x7fffffff,
                                                   float* __restrict__ stats = nullptr) {
  attn4_rows<H>((int32_t)((blockIdx.x * 256u + threadIdx.x) / GS), n, rowptr, cols, s, d, beta,
                alpha, mask, longest, stats);
}

// ---------------------------------------------------------------------------
// Attention + aggregation in one kernel (one column window, hub-free rows):
// a warp computes the attention of its two rows exactly as k_gat_attn4 (16
// lanes per row; alpha / mask written edge-major, the cache at level full)
// and then aggregates each of the two rows as k_gat_agg2 (the whole warp per
// row), reading the attention back through L2 (__ldcg: written by this warp,
// ordered by __syncwarp) -- bit-identical to the two-kernel path, one launch
// and one alpha round trip to HBM fewer, and the latency-bound softmax phase
// overlaps other warps' gathers.
// ---------------------------------------------------------------------------
#ifndef GAT_AA_MINB
#define GAT_AA_MINB 5  // resident blocks per SM at R <= 2 (4: no spills, 10 us slower at Arxiv 8x32; 6 slower again)
#endif
template <int H, int R>
__global__ void __launch_bounds__(256, R <= 2 ? GAT_AA_MINB : (R <= 4 ? 3 : 2))
    k_gat_attnagg(int32_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
                  const float* __restrict__ s, const float* __restrict__ d, float beta,
                  float* __restrict__ alpha, uint8_t* __restrict__ mask,
                  const float4* __restrict__ M, int32_t k, const float4* __restrict__ bias,
                  float4* __restrict__ out, SegArgs sg) {
  const int32_t w = (int32_t)((blockIdx.x * 256u + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  attn4_rows<H>(2 * w + (lane >= GS ? 1 : 0), n, rowptr, cols, s, d, beta, alpha, mask,
                sg.longest, nullptr);
  __syncwarp();
  agg2_row<H, R, false, LdcgA>(2 * w, 0, n, rowptr, cols, alpha, M, k, bias, out, sg);
  agg2_row<H, R, false, LdcgA>(2 * w + 1, 0, n, rowptr, cols, alpha, M, k, bias, out, sg);
}

// softmax / LeakyReLU backward of row i (16 lanes per row); CG: dAlpha was
// written by the same kernel (read through L2)
template <int H, bool CG>
__device__ __forceinline__ void sbwd4_rows(int32_t i, int32_t n,
                                           const int32_t* __restrict__ rowptr,
                                           const float* __restrict__ alpha,
                                           const uint8_t* __restrict__ mask,
                                           const float* __restrict__ da, float beta,
                                           float* __restrict__ dy, float* __restrict__ dS,
                                           int32_t longest, float* __restrict__ stats,
                                           float* __restrict__ rec = nullptr,
                                           const int32_t* __restrict__ pinv = nullptr) {
  const int lane = threadIdx.x & 31, gl = lane & (GS - 1);
  int32_t beg = 0, end = 0;
  if (i < n) {
    beg = __ldg(rowptr + i);
    end = __ldg(rowptr + i + 1);
  }
  const bool hub = end - beg > longest;  // done by k_gat_sbwd_long
  const int32_t deg = hub ? 0 : end - beg;
  const int32_t wdeg = max(deg, __shfl_xor_sync(0xffffffffu, deg, GS));
  if (wdeg == 0) {
    if (i < n && gl == 0 && !hub) {
      float z[H];
#pragma unroll
      for (int t = 0; t < H; ++t) z[t] = 0.f;
      st_heads<H>(dS + (int64_t)i * H, z);
    }
    return;
  }
  float a[H], g[H], dot[H], rs[H];
#pragma unroll
  for (int t = 0; t < H; ++t) dot[t] = rs[t] = 0.f;
  for (int32_t off = 0; off < wdeg; off += GS) {
    const int32_t e = beg + off + gl;
    if (off + gl < deg) {
      ld_heads<H>(alpha + (int64_t)e * H, a);
      ld_heads<H, CG>(da + (int64_t)e * H, g);
#pragma unroll
      for (int t = 0; t < H; ++t) dot[t] = fmaf(a[t], g[t], dot[t]);
    }
  }
  group_allreduce<H>(dot, gl, OpSum());
  if (stats && gl == 0 && deg > 0) st_stat<H>(stats + (int64_t)i * 4 * H + 3, dot);
  const bool one = wdeg <= GS;  // a[], g[] still hold the lane's edge
  for (int32_t off = 0; off < wdeg; off += GS) {
    const int32_t e = beg + off + gl;
    if (off + gl < deg) {
      if (!one) {
        ld_heads<H>(alpha + (int64_t)e * H, a);
        ld_heads<H, CG>(da + (int64_t)e * H, g);
      }
      const uint32_t pos = ld_mask<H>(mask + (int64_t)e * H);
      float y[H];
#pragma unroll
      for (int t = 0; t < H; ++t) {
        const float dw = a[t] * (g[t] - dot[t]);
        y[t] = (pos >> t) & 1u ? dw : beta * dw;
        rs[t] += y[t];
      }
      if (rec) {  // (alpha, dy) record at the edge's CSC position
        st_rec<H>(rec + (int64_t)__ldg(pinv + e) * (2 * H), a, y);
      } else {
        st_heads<H>(dy + (int64_t)e * H, y);
      }
    }
  }
  group_allreduce<H>(rs, gl, OpSum());
  if (i < n && gl == 0 && !hub) st_heads<H>(dS + (int64_t)i * H, rs);
}


template <int H>
__global__ void __launch_bounds__(256) k_gat_sbwd4(int32_t n, const int32_t* __restrict__ rowptr,
                                                   const float* __restrict__ alpha,
                                                   const uint8_t* __restrict__ mask,
                                                   const float* __restrict__ da, float beta,
                                                   float* __restrict__ dy,
                                                   float* __restrict__ dS,
                                                   int32_t longest = 0x7fffffff,
                                                   float* __restrict__ stats = nullptr) {
  sbwd4_rows<H, false>((int32_t)((blockIdx.x * 256u + threadIdx.x) / GS), n, rowptr, alpha, mask,
                       da, beta, dy, dS, longest, stats);
}

// ---------------------------------------------------------------------------
// SDDMM + softmax / LeakyReLU backward in one kernel (one column window,
// hub-free rows, P2 >= 1): a warp computes dAlpha of its two rows exactly as
// k_gat_sddmm2 (the whole warp per row), then the softmax backward of each row
// exactly as k_gat_sbwd4 (16 lanes per row), reading dAlpha back through L2
// (__ldcg: written by this warp, ordered by __syncwarp) -- bit-identical to the
// two-kernel path, one launch and one dAlpha round trip to HBM fewer, and the
// latency-bound row reductions overlap other warps' gathers.
// ---------------------------------------------------------------------------
#ifndef GAT_SDSB_MINB
#define GAT_SDSB_MINB 5  // resident blocks per SM at R <= 2 (4: no spills, measured slower)
#endif
template <int H, int R, int P2>
__global__ void __launch_bounds__(256, R <= 2 ? GAT_SDSB_MINB : (R <= 4 ? 3 : 2))
    k_gat_sddmm_sbwd(int32_t n, const int32_t* __restrict__ rowptr,
                     const int32_t* __restrict__ cols, const float4* __restrict__ M,
                     const float4* __restrict__ G, int32_t k, const float* __restrict__ alpha,
                     const uint8_t* __restrict__ mask, float beta, float* __restrict__ da,
                     float* __restrict__ dy, float* __restrict__ dS, SegArgs sg,
                     float* __restrict__ rec, const int32_t* __restrict__ pinv) {
  static_assert(P2 >= 1, "fused SDDMM: register reductions only");
  const int32_t w = (int32_t)((blockIdx.x * 256u + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  sddmm2_row<H, R, P2, false>(2 * w, 0, n, rowptr, cols, M, G, k, da, sg, nullptr);
  sddmm2_row<H, R, P2, false>(2 * w + 1, 0, n, rowptr, cols, M, G, k, da, sg, nullptr);
  __syncwarp();
  sbwd4_rows<H, true>(2 * w + (lane >= GS ? 1 : 0), n, rowptr, alpha, mask, da, beta, dy, dS,
                      sg.longest, nullptr, rec, pinv);
}

static inline unsigned sub_grid(int32_t n) { return (unsigned)((n + 256 / GS - 1) / (256 / GS)); }

// Hub columns of the column pass: sum the segment partials (dM rows and the
// per-head dD sums) in segment order, then the add_scaled_rows epilogue.
template <int H>
__global__ void __launch_bounds__(256) k_gat_col_combine(
    int32_t nlong, const int32_t* __restrict__ long_col, const int32_t* __restrict__ long_first,
    const float4* __restrict__ part, const float* __restrict__ ddpart, const float* __restrict__ dS,
    const float4* __restrict__ a_src, const float4* __restrict__ a_dst, int32_t k,
    float* __restrict__ dD, float4* __restrict__ dM) {
  const int lane = threadIdx.x & 31;
  const int32_t q = (int32_t)((blockIdx.x * 256u + threadIdx.x) >> 5);
  if (q >= nlong) return;
  const int fv = H * k / 4, L = k / 4;
  const int32_t j = __ldg(long_col + q), s0 = __ldg(long_first + q), s1 = __ldg(long_first + q + 1);
  for (int v = lane; v < fv; v += 32) {
    const int t = min(H - 1, v / L);
    float4 acc = __ldg(part + (int64_t)s0 * fv + v);
    float dd = __ldg(ddpart + (int64_t)s0 * H + t);
    for (int32_t sgi = s0 + 1; sgi < s1; ++sgi) {
      const float4 b = __ldg(part + (int64_t)sgi * fv + v);
      acc.x += b.x;
      acc.y += b.y;
      acc.z += b.z;
      acc.w += b.w;
      dd += __ldg(ddpart + (int64_t)sgi * H + t);
    }
    if (v % L == 0) dD[(int64_t)j * H + t] = dd;
    const float cs = __ldg(dS + (int64_t)j * H + t);
    fma4(acc, cs, __ldg(a_src + v));
    fma4(acc, dd, __ldg(a_dst + v));
    dM[(int64_t)j * fv + v] = acc;
  }
}

// block-wide reduction of H values (8 warps): every thread gets the totals
template <int H, class Op>
__device__ __forceinline__ void block_allreduce(float (&v)[H], float (*sh)[H], Op op) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  allreduce<H>(v, lane, op);
  if (lane == 0)
#pragma unroll
    for (int t = 0; t < H; ++t) sh[w][t] = v[t];
  __syncthreads();
#pragma unroll
  for (int t = 0; t < H; ++t) {
    float a = sh[0][t];
    for (int q = 1; q < WPB; ++q) a = op(a, sh[q][t]);
    v[t] = a;
  }
  __syncthreads();
}

// Hub rows of the attention (kernels.hpp:427-534): one block per row, three
// strided passes (max, sum of exp, alpha + mask) with block reductions.
template <int H>
__global__ void __launch_bounds__(256) k_gat_attn_long(const int32_t* __restrict__ long_row,
                                                       const int32_t* __restrict__ rowptr,
                                                       const int32_t* __restrict__ cols,
                                                       const float* __restrict__ s,
                                                       const float* __restrict__ d, float beta,
                                                       float* __restrict__ alpha,
                                                       uint8_t* __restrict__ mask,
                                                       float* __restrict__ stats = nullptr) {
  __shared__ float sh[WPB][H];
  const int32_t i = __ldg(long_row + blockIdx.x);
  const int32_t beg = __ldg(rowptr + i), end = __ldg(rowptr + i + 1);
  float si[H], mx[H], sm[H];
  ld_heads<H>(s + (int64_t)i * H, si);
#pragma unroll
  for (int t = 0; t < H; ++t) {
    mx[t] = -INFINITY;
    sm[t] = 0.f;
  }
  for (int32_t e = beg + threadIdx.x; e < end; e += blockDim.x) {
    float dj[H];
    ld_heads<H>(d + (int64_t)__ldg(cols + e) * H, dj);
#pragma unroll
    for (int t = 0; t < H; ++t) mx[t] = fmaxf(mx[t], lrelu(si[t] + dj[t], beta));
  }
  block_allreduce<H>(mx, sh, OpMax());
  for (int32_t e = beg + threadIdx.x; e < end; e += blockDim.x) {
    float dj[H];
    ld_heads<H>(d + (int64_t)__ldg(cols + e) * H, dj);
#pragma unroll
    for (int t = 0; t < H; ++t) sm[t] += expf(lrelu(si[t] + dj[t], beta) - mx[t]);
  }
  block_allreduce<H>(sm, sh, OpSum());
#pragma unroll
  for (int t = 0; t < H; ++t) sm[t] = 1.f / sm[t];
  if (stats && threadIdx.x == 0) {
    st_stats3<H>(stats + (int64_t)i * 4 * H, si, mx, sm);
  }
  for (int32_t e = beg + threadIdx.x; e < end; e += blockDim.x) {
    float dj[H], a[H];
    ld_heads<H>(d + (int64_t)__ldg(cols + e) * H, dj);
    uint32_t pos = 0;
#pragma unroll
    for (int t = 0; t < H; ++t) {
      const float y = si[t] + dj[t];
      if (y > 0.f) pos |= 1u << t;
      a[t] = expf(lrelu(y, beta) - mx[t]) * sm[t];
    }
    st_heads<H>(alpha + (int64_t)e * H, a);
    if (mask) st_mask<H>(mask + (int64_t)e * H, pos);
  }
}

// Hub rows of the softmax / LeakyReLU backward and row sums (kernels.hpp:
// 481-495, 537-588): one block per row, two strided passes.
template <int H>
__global__ void __launch_bounds__(256) k_gat_sbwd_long(const int32_t* __restrict__ long_row,
                                                       const int32_t* __restrict__ rowptr,
                                                       const float* __restrict__ alpha,
                                                       const uint8_t* __restrict__ mask,
                                                       const float* __restrict__ da, float beta,
                                                       float* __restrict__ dy,
                                                       float* __restrict__ dS,
                                                       float* __restrict__ stats = nullptr,
                                                       float* __restrict__ rec = nullptr,
                                                       const int32_t* __restrict__ pinv = nullptr) {
  __shared__ float sh[WPB][H];
  const int32_t i = __ldg(long_row + blockIdx.x);
  const int32_t beg = __ldg(rowptr + i), end = __ldg(rowptr + i + 1);
  float dot[H], rs[H];
#pragma unroll
  for (int t = 0; t < H; ++t) dot[t] = rs[t] = 0.f;
  for (int32_t e = beg + threadIdx.x; e < end; e += blockDim.x) {
    float a[H], g[H];
    ld_heads<H>(alpha + (int64_t)e * H, a);
    ld_heads<H>(da + (int64_t)e * H, g);
#pragma unroll
    for (int t = 0; t < H; ++t) dot[t] = fmaf(a[t], g[t], dot[t]);
  }
  block_allreduce<H>(dot, sh, OpSum());
  if (stats && threadIdx.x == 0) st_stat<H>(stats + (int64_t)i * 4 * H + 3, dot);
  for (int32_t e = beg + threadIdx.x; e < end; e += blockDim.x) {
    float a[H], g[H], y[H];
    ld_heads<H>(alpha + (int64_t)e * H, a);
    ld_heads<H>(da + (int64_t)e * H, g);
    const uint32_t pos = ld_mask<H>(mask + (int64_t)e * H);
#pragma unroll
    for (int t = 0; t < H; ++t) {
      const float dw = a[t] * (g[t] - dot[t]);
      y[t] = (pos >> t) & 1u ? dw : beta * dw;
      rs[t] += y[t];
    }
    if (rec) {
      st_rec<H>(rec + (int64_t)__ldg(pinv + e) * (2 * H), a, y);
    } else {
      st_heads<H>(dy + (int64_t)e * H, y);
    }
  }
  block_allreduce<H>(rs, sh, OpSum());
  if (threadIdx.x == 0) st_heads<H>(dS + (int64_t)i * H, rs);
}

}  // namespace g2
