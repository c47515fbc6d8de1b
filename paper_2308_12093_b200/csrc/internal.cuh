// internal.cuh -- device-side object layouts and the kernel launchers shared
// between translation units of libsgnn_cuda.so.
#pragma once

#include "common.cuh"

namespace sgnn {
// Rows longer than kLongRow edges (power-law hubs) are split into kLongRow-edge
// segments, each on its own warp, combined in segment order: without it one
// warp would walk a hub row alone while the rest of the GPU idles.  Built
// once per operator (and direction) on first use.
constexpr int32_t kLongRow = 128;
struct LongRows {
  bool built = false;
  const int32_t* rowptr = nullptr;  // the CSR the plan belongs to
  int32_t nseg = 0, nlong = 0;
  DevBuf seg_beg, seg_end, seg_row;  // nseg: edge range and row of every segment
  DevBuf long_row;    // nlong: row id
  DevBuf long_first;  // nlong + 1: first segment of every long row (+ sentinel)
};
LongRows& long_rows(sgnn_ctx ctx, LongRows& plan, int32_t n_rows, const int32_t* rowptr);
// C[long_row[j]] = sum of the segment partials of row j in order (+ bias)
void spmm_combine(sgnn_ctx ctx, const LongRows& lr, const float* part, int32_t f, float* C,
                  const float* bias, int32_t ld);
}  // namespace sgnn

// AdjacencyOp (kernels.hpp:191-211): forward CSR and the CSC arrays that are
// the CSR of A^T (zero-copy transpose of sparse.hpp:400-420), owned here.
struct sgnn_adj_s {
  int32_t n_rows = 0, n_cols = 0;
  int64_t nnz = 0;
  int dtype = SGNN_F32;
  int format = SGNN_CSC;
  sgnn::DevBuf rowptr, cols, vals;    // CSR of A
  sgnn::DevBuf colptr, crows, cvals;  // CSC of A == CSR of A^T
  sgnn::LongRows long_fwd, long_bwd;  // hub-row plans of the CSR / CSC
  ~sgnn_adj_s();
};

// SparsePattern (pattern.hpp:17-95)
struct sgnn_pattern_s {
  int32_t n = 0;
  int64_t nnz = 0;
  bool all_self_loops = false;
  sgnn::DevBuf rowptr, cols, colptr, rows, perm, diag;
  sgnn::LongRows long_rows, long_cols;  // hub-row / hub-column plans
  sgnn::DevBuf pinv;  // CSR edge -> CSC position (lazy; the column pass's edge records)
  ~sgnn_pattern_s();
};

// GcnCache (gcn.hpp:66-76): exactly one of the borrowed X / owned P
struct sgnn_gcn_cache_s {
  sgnn_scheme scheme{};
  int dtype = SGNN_F32;
  int32_t n = 0, m = 0;
  const void* saved_input = nullptr;  // borrowed (aliases the caller's X)
  sgnn::DevBuf saved_propagated;      // owned P = A'X
  bool consumed = false;
};

// GatCache (gat.hpp:56-72); edge values edge-major q x h
struct sgnn_gat_cache_s {
  int level = SGNN_GAT_NONE;
  int dtype = SGNN_F32;
  int32_t n = 0, m = 0, h = 0, k = 0;
  int64_t q = 0;  // pattern nnz
  double beta = 0.2;
  const void* saved_input = nullptr;  // borrowed, always retained
  sgnn::DevBuf M;                     // level >= features
  sgnn::DevBuf s, d;                  // level == node_attention
  sgnn::DevBuf alpha, mask;           // level == full
  // operator-reordered layer (gat_reorder.cuh): Z = alpha-aggregated input
  // (n x h x m) in place of M at level >= features
  bool reordered = false;
  sgnn::DevBuf Z;
  bool consumed = false;
};

namespace sgnn {

// Copy streams, events and reusable device staging buffers of the host-buffer
// layer steps (pipeline.cu); owned by the context.
struct Pipe {
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev[8] = {};
  void* ws[8] = {};
  size_t cap[8] = {};
  ~Pipe();
  void* buf(int slot, size_t bytes);
};
Pipe& pipe(sgnn_ctx ctx);
void destroy_pipe(sgnn_ctx ctx);

void build_ptr(sgnn_ctx ctx, const int32_t* sorted_ids, int64_t nnz, int32_t n, int32_t* ptr);

// M = X Theta (tcgen05) with the GAT node scores fused into the epilogue;
// returns false (nothing launched) when the shape does not allow it
bool gemm_scores_f32(sgnn_ctx ctx, const float* X, int32_t n, int32_t m, const float* theta,
                     int32_t hk, float* M, const float* a_src, const float* a_dst, int32_t h,
                     float* s, float* d);

// split a contiguous fp32 matrix into tf32 hi / lo (the tcgen05 GEMM's
// pre-split B) on ctx->stream; true if the GEMM of an ra x ca A would use a
// pre-split B of `elems` elements
void gemm_presplit_f32(sgnn_ctx ctx, const float* B, int64_t elems, float* hi, float* lo);
bool gemm_uses_presplit(int64_t elems, int32_t ra, int32_t ca);
bool gemm_relu_f32(sgnn_ctx ctx, const float* A, int32_t ra, int32_t ca, const float* B,
                   int32_t rb, int32_t cb, bool ta, bool tb, float* C, const float* bias,
                   uint8_t* relu_out, const uint8_t* mask_in);

bool gemm_elu_bwd_f32(sgnn_ctx ctx, const float* A, int32_t ra, int32_t ca, const float* B,
                      int32_t rb, int32_t cb, bool ta, bool tb, float* C,
                      const uint8_t* mask_in, const float* saved);

// GAT layer calls of Gat2 with the ELU(1) fused where the producing kernel
// allows it: the forward's aggregation epilogue applies ELU to out and writes
// the mask (*fused = false: out is the plain layer output); the backward's
// d_input GEMM applies the ELU backward (mask, saved output).  gat.cu.
int gat_forward_elu(sgnn_ctx ctx, sgnn_pattern p, const void* X, int32_t m, const void* theta,
                    const void* a_src, const void* a_dst, const void* bias, int32_t heads,
                    int32_t k, double beta, int level, int dtype, void* out,
                    sgnn_gat_cache* cache, uint8_t* elu_mask, bool* fused,
                    bool reorder = false);
int gat_backward_elu(sgnn_ctx ctx, sgnn_pattern p, const void* d_out, const void* theta,
                     const void* a_src, const void* a_dst, int32_t m, int32_t heads, int32_t k,
                     sgnn_gat_cache c, int fg, void* d_theta, void* d_a_src, void* d_a_dst,
                     void* d_bias, void* d_input, const uint8_t* elu_mask,
                     const void* elu_saved, bool* fused);

// GCN layer calls of the models with ReLU fused where the producing kernel is
// a tcgen05 GEMM (else a separate activation pass): forward writes the mask
// and applies ReLU to out; backward applies the ReLU backward (mask_in) to
// d_input.  gcn.cu.
int gcn_forward_relu(sgnn_ctx ctx, sgnn_adj A, const void* X, int32_t m, const void* theta,
                     const void* bias, int32_t k, const sgnn_scheme* s, void* out,
                     sgnn_gcn_cache* cache, uint8_t* relu_mask);
int gcn_backward_relu(sgnn_ctx ctx, sgnn_adj A, const void* d_out, const void* theta, int32_t m,
                      int32_t k, sgnn_gcn_cache c, int fg, void* d_theta, void* d_bias,
                      void* d_input, const uint8_t* relu_mask_in);

// C (n_rows x f) = A B (+bias) for a CSR (rowptr, cols, vals); b_rows = the
// row count of B when known (float32 widths that are not a multiple of 4 are
// then staged into 16-byte-aligned padded copies for the vector kernels)
template <class T>
void spmm_csr(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr, const int32_t* cols,
              const T* vals, const T* B, int32_t f, T* C, const T* bias, int64_t nnz,
              const LongRows* lr = nullptr, int32_t b_rows = -1);

// tcgen05 GEMM on blocks of wider matrices (row pitches lda / ldb / ldc,
// multiples of 4 floats); false when the shape is not supported
// false when SGNN_DISABLE_TCGEN05=1 (A/B switch of the tcgen05 GEMMs)
bool gemm_tc_available();
// colsum_b: fused column sums of B (MN-major B only, as gemm_tn_colsum);
// elu_mask: ELU(1) applied to C (+ bias) with its byte mask written at the
// same pitch as C (k_act_fwd's expressions; whole 32-column chunks).  false:
// nothing was written, the caller runs the unfused pieces.
bool gemm_tc_f32_pitched(sgnn_ctx ctx, const float* A, int32_t ra, int32_t ca, int32_t lda,
                         const float* B, int32_t rb, int32_t cb, int32_t ldb, bool ta, bool tb,
                         float* C, int32_t ldc, const float* bias, float* colsum_b = nullptr,
                         uint8_t* elu_mask = nullptr);

// row-padded staging copies of float32 matrices (gemm_tc.cu): zero-padded to
// ocols columns / back to ocols columns with an optional bias add
void pad_rows_f32(sgnn_ctx ctx, int32_t rows, int32_t cols, const float* src, int32_t ld,
                  int32_t ocols, float* dst);
void unpad_rows_f32(sgnn_ctx ctx, int32_t rows, int32_t ocols, const float* src, int32_t ld,
                    const float* bias, float* dst);

// C = op(A) op(B) (row-major); A ra x ca, B rb x cb; bias added per column of C
template <class T>
void gemm(sgnn_ctx ctx, const T* A, int32_t ra, int32_t ca, const T* B, int32_t rb, int32_t cb,
          bool ta, bool tb, T* C, const T* bias = nullptr);

template <class T>
void column_sums(sgnn_ctx ctx, const T* X, int32_t rows, int32_t cols, T* out);
template <class T>
void gemm_tn_colsum(sgnn_ctx ctx, const T* A, int32_t ra, int32_t ca, const T* B, int32_t rb,
                    int32_t cb, T* C, T* colsum_b);

template <class T>
void random_uniform(sgnn_ctx ctx, int64_t count, uint64_t seed, double lo, double hi, T* out);

}  // namespace sgnn
