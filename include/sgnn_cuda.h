/*
 * sgnn_cuda.h -- C-ABI of the B200-native (sm_100a) GCN/GAT layer library
 * (libsgnn_cuda.so).  Plain pointers and sizes only; no torch or C++ types.
 *
 * This is the drop-in boundary for the reference `sgnn` layer API
 * (/root/reference/proj/include/sgnn/): every entry point names the reference
 * interface it replaces.  The reference binds its C++ API to Python through
 * pybind11 (python/bindings.cpp); the binding a maintainer would add over this
 * ABI (ctypes) is shown in INTEGRATION.md and implemented in
 * paper_2308_12093_b200/_capi.py.
 *
 * Conventions
 *  - Device pointers unless a parameter says "host".  All work is enqueued on
 *    the stream of the sgnn_ctx; calls that return a size through a host
 *    pointer synchronize that stream.
 *  - Indices int32 (ref common.hpp:16), counts int64 (common.hpp:17).
 *  - Dense matrices row-major.  Multi-head operands are n x (h*k) slabs with
 *    the head in the middle (ref gat.hpp:19-20).  Per-edge per-head values on
 *    the device are EDGE-major (q x h); the reference stores them head-major
 *    (h x q, pattern.hpp:99-123) -- sgnn_gat_cache_edge_values converts.
 *  - Errors: int status; SGNN_EINVAL where the reference throws
 *    std::invalid_argument (common.hpp:37-43) with the same message text,
 *    retrievable through sgnn_last_error() (thread-local).
 */
#ifndef SGNN_CUDA_H
#define SGNN_CUDA_H

#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif
#ifdef __cplusplus
extern "C" {
#endif

#define SGNN_OK 0
#define SGNN_EINVAL 1   /* std::invalid_argument in the reference */
#define SGNN_ERUNTIME 2 /* std::runtime_error in the reference      */
#define SGNN_ECUDA 3
#define SGNN_ENCCL 4

typedef enum { SGNN_F32 = 0, SGNN_F64 = 1 } sgnn_dtype;

/* sparse.hpp:22 SparseFormat */
typedef enum {
  SGNN_COO = 0,
  SGNN_CSR = 1,
  SGNN_CSC = 2,
  SGNN_ELLPACK = 3,
  SGNN_HYBRID = 4
} sgnn_format;

/* cost.hpp:114-122 GcnForward / GcnBackward / SchemeChoice */
typedef enum {
  SGNN_TRANSFORM_FIRST = 0,
  SGNN_PROPAGATE_FIRST = 1,
  SGNN_PROPAGATE_FIRST_CACHED = 2
} sgnn_gcn_forward_scheme;
typedef enum {
  SGNN_FUSED_PROPAGATE = 0,
  SGNN_SPLIT_PROPAGATE = 1,
  SGNN_SPLIT_PROPAGATE_CACHED = 2
} sgnn_gcn_backward_scheme;
typedef struct {
  int32_t forward;  /* sgnn_gcn_forward_scheme  */
  int32_t backward; /* sgnn_gcn_backward_scheme */
  int32_t caching;  /* bool */
} sgnn_scheme;

/* gcn.hpp:23 SchemePolicy */
typedef enum {
  SGNN_POLICY_ADAPTIVE = 0,
  SGNN_POLICY_TRANSFORM_FIRST = 1,
  SGNN_POLICY_PROPAGATE_FIRST = 2
} sgnn_policy;

/* cost.hpp:229 GatCacheLevel */
typedef enum {
  SGNN_GAT_NONE = 0,
  SGNN_GAT_FEATURES = 1,
  SGNN_GAT_NODE_ATTENTION = 2,
  SGNN_GAT_FULL = 3
} sgnn_gat_level;

typedef struct sgnn_ctx_s* sgnn_ctx;
typedef struct sgnn_adj_s* sgnn_adj;
typedef struct sgnn_pattern_s* sgnn_pattern;
typedef struct sgnn_gcn_cache_s* sgnn_gcn_cache;
typedef struct sgnn_gat_cache_s* sgnn_gat_cache;

/* ---- errors / context ------------------------------------------------ */
/* common.hpp:37-43 require() message of the last failing call on this thread */
const char* sgnn_last_error(void);
const char* sgnn_version(void);
/* stream: a cudaStream_t; NULL = the default stream (CUDA convention) */
int sgnn_ctx_create(int device, void* stream, sgnn_ctx* out);
/* memtrack.hpp:19-94 MemTracker for the device engine: live / peak / total
 * bytes per class (0 untracked, 1 transient, 2 cache, 3 output, 4 = all) of
 * the layer intermediates, charged with their logical sizes (the reference's
 * Array sizes); kernel scratch stays untracked.  Process-wide. */
typedef enum {
  SGNN_MEM_UNTRACKED = 0,
  SGNN_MEM_TRANSIENT = 1,
  SGNN_MEM_CACHE = 2,
  SGNN_MEM_OUTPUT = 3,
  SGNN_MEM_ALL = 4
} sgnn_mem_class;
int sgnn_mem_stats(int mem_class, int64_t* live, int64_t* peak, int64_t* total);
/* peaks restart from the live level, totals from zero (memtrack.hpp:79-87) */
int sgnn_mem_reset_peaks(void);
int sgnn_ctx_destroy(sgnn_ctx ctx);
int sgnn_ctx_set_stream(sgnn_ctx ctx, void* stream);
int sgnn_ctx_synchronize(sgnn_ctx ctx);
/* number of kernels this context has launched (bench gpu_launches) */
int sgnn_ctx_launch_count(sgnn_ctx ctx, int64_t* out);

/* ---- host-pure: selector and analytic model (cost.hpp, gcn.hpp) --------- */
/* cost.hpp:201-223 gcn_select_scheme */
int sgnn_gcn_select_scheme(int64_t m, int64_t k, int needs_feature_grad, int caching,
                           sgnn_scheme* out);
/* gcn.hpp:34-47 resolve_scheme */
int sgnn_resolve_scheme(int policy, int64_t m, int64_t k, int needs_feature_grad, int caching,
                        sgnn_scheme* out);
/* cost.hpp:143-197 */
int64_t sgnn_gcn_forward_flops(int fwd, int64_t n, int64_t m, int64_t k, int64_t q);
int64_t sgnn_gcn_backward_flops(int bwd, int64_t n, int64_t m, int64_t k, int64_t q, int fg);
int64_t sgnn_gcn_forward_transients(int fwd, int64_t n, int64_t m, int64_t k);
int64_t sgnn_gcn_backward_transients(int bwd, int64_t n, int64_t m, int64_t k, int fg);
/* cost.hpp:63-101 spmm_cost / sddmm_cost */
int sgnn_spmm_cost(int format, int64_t n, int64_t q, int64_t p, int64_t f, int64_t scalar_bytes,
                   int64_t index_bytes, int64_t* flops, int64_t* bytes, double* oi);
int sgnn_sddmm_cost(int format, int64_t n, int64_t q, int64_t p, int64_t f,
                    int64_t scalar_bytes, int64_t index_bytes, int64_t* flops, int64_t* bytes,
                    double* oi);
/* cost.hpp:243-252 gat_cache_footprint */
int64_t sgnn_gat_cache_footprint(int level, int64_t n, int64_t h, int64_t k, int64_t q,
                                 int64_t scalar_bytes);

/* ---- deterministic inputs (graph.hpp, dense.hpp, gcn.hpp, gat.hpp) ------- */
/* graph.hpp:160-190 synthetic_graph; host buffers of sgnn_synthetic_graph_edges() */
int64_t sgnn_synthetic_graph_edges(int32_t n, double avg_degree);
int sgnn_synthetic_graph(int32_t n, double avg_degree, uint64_t seed, int32_t* host_src,
                         int32_t* host_dst);
/* dense.hpp:45-53 DenseMatrix::random_uniform, generated ON DEVICE: the
 * splitmix64 stream is counter-based, draw i = mix(seed + (i+2)*golden) */
int sgnn_random_uniform(sgnn_ctx ctx, int64_t rows, int64_t cols, uint64_t seed, double lo,
                        double hi, int dtype, void* out);
/* gcn.hpp:54-62 GcnParams::init (device outputs theta m x k, bias k) */
int sgnn_gcn_params_init(sgnn_ctx ctx, int32_t m, int32_t k, uint64_t seed, int dtype,
                         void* theta, void* bias);
/* gat.hpp:36-52 GatParams::init */
int sgnn_gat_params_init(sgnn_ctx ctx, int32_t m, int32_t h, int32_t k, uint64_t seed,
                         int dtype, void* theta, void* a_src, void* a_dst, void* bias);

/* Chung-Lu power-law graph on the device (no reference counterpart: the
 * reference generator graph.hpp:160-190 is uniform; BASELINE config 5 asks for
 * a power-law graph).  w_i = (i+1)^(-1/(exponent-1)); round(avg_degree*n/2)
 * pair draws from the counter-based splitmix64 stream of seed; undirected,
 * both directions, no self loops or duplicates, canonical order.  src / dst:
 * device buffers of sgnn_powerlaw_graph_capacity(n, avg_degree) entries;
 * *count receives the number written (synchronises the context stream). */
int64_t sgnn_powerlaw_graph_capacity(int32_t n, double avg_degree);
int sgnn_powerlaw_graph(sgnn_ctx ctx, int32_t n, double avg_degree, double exponent,
                        uint64_t seed, int32_t* src, int32_t* dst, int64_t* count);

/* ---- sparse-format layer, on device (sparse.hpp, pattern.hpp) ------------ */
/* sparse.hpp:110-142 coo_from_triplets: range check, stable sort by (row,col),
 * duplicates keep the LAST value.  Outputs have capacity nnz. */
int sgnn_coo_canonicalize(sgnn_ctx ctx, int32_t n_rows, int32_t n_cols, int64_t nnz,
                          const int32_t* rows, const int32_t* cols, const void* vals, int dtype,
                          int32_t* out_rows, int32_t* out_cols, void* out_vals,
                          int64_t* host_out_nnz);
/* sparse.hpp:151-171 coo_to_csr (input canonical) */
int sgnn_csr_from_coo(sgnn_ctx ctx, int32_t n_rows, int64_t nnz, const int32_t* rows,
                      int32_t* rowptr);
/* sparse.hpp:195-218 coo_to_csc; perm[p] = canonical index of CSC entry p
 * (pattern.hpp:35-44).  out_vals/perm may be NULL. */
int sgnn_csc_from_coo(sgnn_ctx ctx, int32_t n_cols, int64_t nnz, const int32_t* rows,
                      const int32_t* cols, const void* vals, int dtype, int32_t* colptr,
                      int32_t* out_rows, void* out_vals, int32_t* perm);
/* sparse.hpp:457-472 add_self_loops (input canonical; capacity nnz + n) */
int sgnn_add_self_loops(sgnn_ctx ctx, int32_t n, int64_t nnz, const int32_t* rows,
                        const int32_t* cols, const void* vals, int dtype, int32_t* out_rows,
                        int32_t* out_cols, void* out_vals, int64_t* host_out_nnz);
/* sparse.hpp:474-495 gcn_normalize (input canonical; capacity nnz + n);
 * degrees in float64 in canonical order, bit-identical to the reference */
int sgnn_gcn_normalize(sgnn_ctx ctx, int32_t n, int64_t nnz, const int32_t* rows,
                       const int32_t* cols, const void* vals, int dtype, int32_t* out_rows,
                       int32_t* out_cols, void* out_vals, int64_t* host_out_nnz);

/* kernels.hpp:191-211 AdjacencyOp: canonical COO -> device CSR (forward) and
 * CSC (= CSR of A^T, the zero-copy transpose of sparse.hpp:400-420).  Any
 * `format` is accepted: every reference format accumulates each output row
 * in ascending column order, so results are identical. */
int sgnn_adj_create(sgnn_ctx ctx, int32_t n_rows, int32_t n_cols, int64_t nnz,
                    const int32_t* rows, const int32_t* cols, const void* vals, int dtype,
                    int format, sgnn_adj* out);
int sgnn_adj_destroy(sgnn_adj adj);
int sgnn_adj_info(sgnn_adj adj, int32_t* n_rows, int32_t* n_cols, int64_t* nnz, int* dtype);
/* device arrays of the operator (borrowed; valid while adj lives) */
int sgnn_adj_arrays(sgnn_adj adj, const int32_t** rowptr, const int32_t** cols,
                    const void** vals, const int32_t** colptr, const int32_t** crows,
                    const void** cvals);

/* pattern.hpp:19-59 SparsePattern::build from a device CSR */
int sgnn_pattern_create(sgnn_ctx ctx, int32_t n, int64_t nnz, const int32_t* rowptr,
                        const int32_t* cols, sgnn_pattern* out);
int sgnn_pattern_destroy(sgnn_pattern p);
int sgnn_pattern_info(sgnn_pattern p, int32_t* n, int64_t* nnz, int* all_self_loops);
int sgnn_pattern_arrays(sgnn_pattern p, const int32_t** rowptr, const int32_t** cols,
                        const int32_t** colptr, const int32_t** rows, const int32_t** perm,
                        const int32_t** diag);

/* ---- kernels (kernels.hpp, dense.hpp) ----------------------------------- */
/* kernels.hpp:167-186 spmm / AdjacencyOp::multiply[_transposed]:
 * C (n_rows x f) = A B (+ 1 bias^T if bias != NULL) */
int sgnn_spmm(sgnn_ctx ctx, sgnn_adj adj, int transposed, const void* B, int32_t f, void* C,
              const void* bias);
/* kernels.hpp:301-337 sddmm (one head, no scale): out_e = B[i,:] . C[:,j];
 * B n x f, C f x ldc */
int sgnn_sddmm(sgnn_ctx ctx, sgnn_pattern p, const void* B, int32_t f, const void* C,
               int32_t ldc, int dtype, void* out);
/* kernels.hpp:500-534 edge_softmax, edge-major w/alpha (q x heads) */
int sgnn_edge_softmax(sgnn_ctx ctx, sgnn_pattern p, int32_t heads, const void* w, int dtype,
                      void* alpha);
/* dense.hpp:97-157 gemm: C = op(A) op(B); A is ra x ca, B is rb x cb */
int sgnn_gemm(sgnn_ctx ctx, int dtype, const void* A, int32_t ra, int32_t ca, const void* B,
              int32_t rb, int32_t cb, int trans_a, int trans_b, void* C);
/* gemm with the bias add fused into the epilogue (dense.hpp:159-170), or --
 * for C = A^T B -- with colsum_b = 1^T B computed from the same read of B
 * (d_bias fused into dTheta, gcn.hpp:139-141); either extra may be NULL */
int sgnn_gemm_ex(sgnn_ctx ctx, int dtype, const void* A, int32_t ra, int32_t ca, const void* B,
                 int32_t rb, int32_t cb, int trans_a, int trans_b, void* C, const void* bias,
                 void* colsum_b);
/* gemm + activation (dense.hpp:197-268), the activation fused into the
 * tcgen05 epilogue where the shape allows it, else two passes (identical
 * results): act 0 = ReLU forward (C = relu(op(A) op(B) + bias), mask out),
 * 1 = ReLU backward (C zeroed where mask == 0), 2 = ELU(1) backward (C times
 * saved + 1 where mask == 0; saved = the ELU output); bias only with act 0 */
int sgnn_gemm_act(sgnn_ctx ctx, int dtype, const void* A, int32_t ra, int32_t ca, const void* B,
                  int32_t rb, int32_t cb, int ta, int tb, void* C, const void* bias, int act,
                  uint8_t* mask, const void* saved);
/* dense.hpp:272-282 column_sums: out (cols) = sum over rows */
int sgnn_column_sums(sgnn_ctx ctx, int dtype, const void* X, int32_t rows, int32_t cols,
                     void* out);

/* ---- GCN layer (gcn.hpp:91-193) ------------------------------------------ */
/* gcn_forward: out (n x k) = A' X Theta + 1 b^T with the given scheme.  The
 * returned cache borrows X (uncached schemes, gcn.hpp:111) -- X must stay
 * valid until backward -- or owns P = A'X (propagate_first_cached). */
int sgnn_gcn_forward(sgnn_ctx ctx, sgnn_adj adj, const void* X, int32_t m, const void* theta,
                     const void* bias, int32_t k, const sgnn_scheme* scheme, void* out,
                     sgnn_gcn_cache* cache);
/* gcn_backward: consume-once cache (gcn.hpp:137-138: marked consumed before
 * any other check); d_input may be NULL when needs_feature_grad == 0 */
int sgnn_gcn_backward(sgnn_ctx ctx, sgnn_adj adj, const void* d_out, const void* theta,
                      int32_t m, int32_t k, sgnn_gcn_cache cache, int needs_feature_grad,
                      void* d_theta, void* d_bias, void* d_input);
int sgnn_gcn_cache_destroy(sgnn_gcn_cache cache);
/* gcn.hpp:72-75 retained_bytes */
int sgnn_gcn_cache_retained_bytes(sgnn_gcn_cache cache, int64_t* out);
/* gcn.hpp:66-76 GcnCache fields: device X (borrowed; uncached schemes) or the
 * owned P = A'X (cached scheme); the absent one is NULL */
int sgnn_gcn_cache_arrays(sgnn_gcn_cache cache, const void** saved_input,
                          const void** saved_propagated);

/* ---- GAT layer (gat.hpp:89-219) ------------------------------------------ */
int sgnn_gat_forward(sgnn_ctx ctx, sgnn_pattern p, const void* X, int32_t m, const void* theta,
                     const void* a_src, const void* a_dst, const void* bias, int32_t heads,
                     int32_t k, double beta, int level, int dtype, void* out,
                     sgnn_gat_cache* cache);
/* gat_forward with options.  SGNN_GAT_REORDER lets the layer run operator-
 * reordered when the heads are wider than the input (k > m; float32, h in
 * {1,2,4,8}, m and k multiples of 4, no rows over 128 edges): the attention
 * scores as X (Theta_t a_t), the aggregation over the m-wide input rows
 * (Z_t = sum_j alpha_t X_j) and out_t = Z_t Theta_t + b_t, so M = X Theta is
 * never formed -- same outputs and gradients within float32 rounding.  Such a
 * cache keeps Z (n x h x m) where the reference keeps M (gat_cache_arrays
 * returns M = NULL; extra_bytes counts Z); backward and edge_values accept it
 * as any other.  Without the flag this is sgnn_gat_forward. */
#define SGNN_GAT_REORDER 1
int sgnn_gat_forward_ex(sgnn_ctx ctx, sgnn_pattern p, const void* X, int32_t m, const void* theta,
                        const void* a_src, const void* a_dst, const void* bias, int32_t heads,
                        int32_t k, double beta, int level, int dtype, void* out,
                        sgnn_gat_cache* cache, int flags);
int sgnn_gat_backward(sgnn_ctx ctx, sgnn_pattern p, const void* d_out, const void* theta,
                      const void* a_src, const void* a_dst, int32_t m, int32_t heads, int32_t k,
                      double beta, sgnn_gat_cache cache, int needs_feature_grad, void* d_theta,
                      void* d_a_src, void* d_a_dst, void* d_bias, void* d_input);
int sgnn_gat_cache_destroy(sgnn_gat_cache cache);
/* 1 when the forward ran operator-reordered (sgnn_gat_forward_ex) */
int sgnn_gat_cache_reordered(sgnn_gat_cache cache, int* out);
/* gat.hpp:66-71 extra_bytes (== gat_cache_footprint at every level) */
int sgnn_gat_cache_extra_bytes(sgnn_gat_cache cache, int64_t* out);
/* gat.hpp:56-72 GatCache fields retained at the cache level (NULL otherwise):
 * M (n x hk), s / d node scores (n x h), alpha / mask edge-major (q x h) */
int sgnn_gat_cache_arrays(sgnn_gat_cache cache, const void** M, const void** s, const void** d,
                          const void** alpha, const uint8_t** mask);
/* cached (level full) or recomputed (gat.hpp:150-170) attention, converted to
 * the reference head-major layout: alpha (h x q, dtype), mask (h x q bytes) */
int sgnn_gat_cache_edge_values(sgnn_ctx ctx, sgnn_pattern p, sgnn_gat_cache cache,
                               const void* theta, const void* a_src, const void* a_dst,
                               void* alpha_hq, uint8_t* mask_hq);

/* ---- kernel-level GAT pieces over row / column blocks -----------------------
 * float32, h in {1,2,4,8}, k % 4 == 0, h*k <= 1024.  The reference's kernel
 * functions as separate calls, so a row-partitioned layer can interleave them
 * with NCCL exchanges (dist.DistGatLayer): column ids index a (gathered)
 * operand of any row count, row ids are block-local, edge values are
 * edge-major (edges x h) in the block's CSR order. */
/* hub-row plan of a block CSR / CSC (rows longer than 128 edges run as
 * segments); every block entry point below accepts one (or NULL) */
typedef struct sgnn_rowplan_s* sgnn_rowplan;
int sgnn_rowplan_create(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr, sgnn_rowplan* out);
int sgnn_rowplan_destroy(sgnn_rowplan plan);
/* gemm + node_scores (kernels.hpp:385-423): M = X Theta, s/d per head */
int sgnn_gat_transform(sgnn_ctx ctx, const float* X, int32_t n_rows, int32_t m,
                       const float* theta, int32_t h, int32_t k, const float* a_src,
                       const float* a_dst, float* M, float* s, float* d);
/* edge_scores + leaky_relu_edges + edge_softmax (kernels.hpp:427-534) */
int sgnn_gat_attention(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr,
                       const int32_t* cols, int32_t h, const float* s, const float* d,
                       double beta, float* alpha, uint8_t* mask, sgnn_rowplan plan);
/* ... plus the per-row statistics (n_rows x h x 4: s, max, 1/sum, [dot]; NULL = none)
 * that sgnn_gat_column_pass_stats rebuilds alpha from */
int sgnn_gat_attention_ex(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr,
                          const int32_t* cols, int32_t h, const float* s, const float* d,
                          double beta, float* alpha, uint8_t* mask, float* row_stats,
                          sgnn_rowplan plan);
/* spmm_semibatched + bias (kernels.hpp:219-254) */
int sgnn_gat_aggregate(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr, const int32_t* cols,
                       int32_t h, int32_t k, const float* alpha, const float* M,
                       const float* bias, float* out, sgnn_rowplan plan);
/* sddmm_semibatched (kernels.hpp:342-377) */
int sgnn_gat_sddmm(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr, const int32_t* cols,
                   int32_t h, int32_t k, const float* M, const float* G, float* da,
                   sgnn_rowplan plan);
/* edge_softmax_backward + leaky_relu_edges_backward + edge_row_sums (481-588) */
int sgnn_gat_softmax_backward(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr, int32_t h,
                              const float* alpha, const uint8_t* mask, const float* da,
                              double beta, float* dy, float* dS, sgnn_rowplan plan);
/* ... plus dot = sum_e alpha dAlpha per row and head into row_stats[row][head][3] */
int sgnn_gat_softmax_backward_ex(sgnn_ctx ctx, int32_t n_rows, const int32_t* rowptr, int32_t h,
                                 const float* alpha, const uint8_t* mask, const float* da,
                                 double beta, float* dy, float* dS, float* row_stats,
                                 sgnn_rowplan plan);
/* spmm_semibatched_transposed + edge_col_sums + add_scaled_rows (258-295,
 * 614-658) over a block of columns (rows / perm index gathered G / edges) */
int sgnn_gat_column_pass(sgnn_ctx ctx, int32_t n_cols, const int32_t* colptr,
                         const int32_t* rows, const int32_t* perm, int32_t h, int32_t k,
                         const float* G, const float* alpha, const float* dy, const float* dS,
                         const float* a_src, const float* a_dst, float* dD, float* dM,
                         sgnn_rowplan plan);
/* The same column pass rebuilding alpha / dy per edge from the gathered row
 * statistics and dAlpha = <dX'_i, M_j> (kernels.hpp:342-377, 427-588 restated
 * per column): the row-partitioned layer all-gathers 4 n h statistics
 * instead of 2 q' h edge values.  d_own, M_own, dS: the block's own rows. */
int sgnn_gat_column_stats_supported(int32_t h, int32_t k);
int sgnn_gat_column_pass_stats(sgnn_ctx ctx, int32_t n_cols, const int32_t* colptr,
                               const int32_t* rows, int32_t h, int32_t k, const float* G,
                               const float* row_stats, const float* d_own, const float* M_own,
                               double beta, const float* dS, const float* a_src,
                               const float* a_dst, float* dD, float* dM, sgnn_rowplan plan);
/* column_sums + attention_param_grad (dense.hpp:272-282, kernels.hpp:592-611) */
int sgnn_gat_param_grads(sgnn_ctx ctx, int32_t n_rows, int32_t h, int32_t k, const float* G,
                         const float* M, const float* dS, const float* dD, float* d_bias,
                         float* d_a_src, float* d_a_dst);

/* ---- two-layer models (model.hpp:16-245) ---------------------------------
 * Gcn2 = GCN -> ReLU -> GCN, Gat2 = GAT -> ELU(1) -> GAT; replaces Gcn2Model /
 * Gat2Model + loss_mse (model.hpp) and activation / activation_backward
 * (dense.hpp:190-270).  Parameters are device buffers owned by the model,
 * initialised like the constructors (layer 2 from seed+101 / seed+201). */
typedef struct {
  int32_t kind;          /* ModelKind: 0 gcn2, 1 gat2 (model.hpp:16) */
  int32_t in_features;   /* ModelConfig (model.hpp:18-29) */
  int32_t hidden;
  int32_t out_features;
  int32_t heads;         /* gat2 */
  int32_t scheme_policy; /* SchemePolicy: 0 adaptive, 1 transform-first, 2 propagate-first */
  int32_t caching;       /* gcn2: retain A'X */
  int32_t gat_level;     /* gat2: sgnn_gat_level */
  double leaky_slope;    /* gat attention slope */
  int32_t input_grad;    /* compute d(input features) */
} sgnn_model_config;
typedef struct sgnn_model_s* sgnn_model;
/* activation (dense.hpp:197-228): kind 0 relu, 2 elu(alpha = 1); out may
 * alias x; mask[i] = x[i] > 0 (count bytes) */
int sgnn_activation(sgnn_ctx ctx, int kind, int dtype, const void* x, int64_t count, void* out,
                    uint8_t* mask);
/* activation_backward (dense.hpp:232-268): elu needs the saved forward output */
int sgnn_activation_backward(sgnn_ctx ctx, int kind, int dtype, const void* grad_out,
                             const uint8_t* mask, const void* saved, int64_t count,
                             void* grad_in);
/* loss_mse (model.hpp): grad = 2 (out - target) / total, *loss (DEVICE double)
 * = sum (out - target)^2 / total over the count elements given; total is the
 * size of the whole prediction (== count unless the caller holds a block) */
int sgnn_loss_mse(sgnn_ctx ctx, int dtype, const void* out, const void* target, int64_t count,
                  int64_t total, void* grad, double* loss);
int sgnn_model_create(sgnn_ctx ctx, const sgnn_model_config* cfg, uint64_t seed, int dtype,
                      sgnn_model* out);
int sgnn_model_destroy(sgnn_model model);
/* param_tensors() (model.hpp:100-107, 208-218): count, then (device data,
 * element count, name) of tensor i */
int sgnn_model_num_params(sgnn_model model, int32_t* count);
int sgnn_model_param(sgnn_model model, int32_t i, void** data, int64_t* size, const char** name);
/* One training step (bench.hpp:193-219): forward, loss_mse(out, target),
 * backward.  adj for gcn2, pattern for gat2; out (optional) receives the
 * prediction; grads[i] receives the gradient of parameter i (device buffers,
 * param_tensors() order); d_input is required when cfg.input_grad; loss
 * (optional) is a DEVICE double receiving the mean squared error.
 * Stream-ordered, no host synchronisation. */
int sgnn_model_train_step(sgnn_ctx ctx, sgnn_model model, sgnn_adj adj, sgnn_pattern pattern,
                          const void* X, const void* target, void* out, void* const* grads,
                          void* d_input, double* loss);

/* ---- host-buffer layer steps (pipeline.cu) -------------------------------
 * One forward + backward step with HOST inputs and outputs, the shape of the
 * reference API (DenseMatrix in host memory, gcn.hpp:91-193 / gat.hpp:89-219)
 * and of its benchmark step (forward, then backward with a given output
 * gradient, bench.hpp:193-219).  Parameters stay device-resident; X and the
 * output gradient are copied in, the output and all gradients copied out.
 * Transfers run on internal copy streams, overlapped with compute and with
 * each other (output D2H while dX' is H2D).  Stream-ordered on the ctx
 * stream; host buffers should be pinned for the copies to be asynchronous.
 * h_d_input may be NULL when needs_feature_grad == 0. */
int sgnn_gcn_step_host(sgnn_ctx ctx, sgnn_adj adj, const void* hX, int32_t m, const void* theta,
                       const void* bias, int32_t k, const sgnn_scheme* scheme, const void* hG,
                       int needs_feature_grad, void* h_out, void* h_d_theta, void* h_d_bias,
                       void* h_d_input);
int sgnn_gat_step_host(sgnn_ctx ctx, sgnn_pattern p, const void* hX, int32_t m,
                       const void* theta, const void* a_src, const void* a_dst, const void* bias,
                       int32_t heads, int32_t k, double beta, int level, int dtype,
                       const void* hG, int needs_feature_grad, void* h_out, void* h_d_theta,
                       void* h_d_a_src, void* h_d_a_dst, void* h_d_bias, void* h_d_input);

#ifdef __cplusplus
}
#endif
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* SGNN_CUDA_H */
