/*
 * sgnn_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, single-threaded restatement of the reference `sgnn` CPU algorithms
 * on the GCN/GAT hot path (/root/reference/proj/include/sgnn/*.hpp).  It is
 * the parity checker for the sm_100a product path: only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline leg may load it.
 * The product library (libsgnn_cuda.so) never links or calls it.
 *
 * Every function restates the reference loop order exactly (same per-element
 * accumulation order, no FP contraction), so in float64 it is bit-identical
 * to the reference; that is pinned by tests/test_oracle_golden.py against the
 * golden vectors in tests/golden/ produced by the reference itself
 * (oracle/_ref, built from the reference headers by oracle/Makefile).
 *
 * Conventions: index arrays are int32 (ref common.hpp:16), counts int64
 * (common.hpp:17); dense matrices are row-major; edge values are head-major
 * h x q like the reference's EdgeValues (pattern.hpp:99-123).
 * Return codes: 0 ok, -1 invalid argument (the reference throws
 * std::invalid_argument at the same points).
 */
#ifndef SGNN_ORACLE_H
#define SGNN_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp ---------------------------------------------------------- */
void orc_random_uniform(int64_t rows, int64_t cols, uint64_t seed, double lo, double hi,
                        double* out);
void orc_random_uniform_f32(int64_t rows, int64_t cols, uint64_t seed, double lo, double hi,
                            float* out);
void orc_rng_u64(uint64_t seed, int64_t count, uint64_t* out);
void orc_rng_below(uint64_t seed, uint64_t bound, int64_t count, uint64_t* out);

/* ---- graph.hpp -------------------------------------------------------- */
int64_t orc_synthetic_graph_edges(int32_t n, double avg_degree);
int orc_synthetic_graph(int32_t n, double avg_degree, uint64_t seed, int32_t* src, int32_t* dst);

/* ---- sparse.hpp ------------------------------------------------------- */
/* returns deduplicated nnz, or -1 on out-of-range index */
int64_t orc_coo_canonicalize(int32_t n_rows, int32_t n_cols, int64_t nnz, const int32_t* rows,
                             const int32_t* cols, const double* vals, int32_t* out_rows,
                             int32_t* out_cols, double* out_vals);
void orc_coo_to_csr(int32_t n_rows, int64_t nnz, const int32_t* rows, int32_t* rowptr);
void orc_coo_to_csc(int32_t n_cols, int64_t nnz, const int32_t* rows, const int32_t* cols,
                    const double* vals, int32_t* colptr, int32_t* out_rows, double* out_vals,
                    int32_t* perm);
/* capacity of outputs must be nnz + n; returns new nnz, -1 if not square */
int64_t orc_add_self_loops(int32_t n, int64_t nnz, const int32_t* rows, const int32_t* cols,
                           const double* vals, int32_t* out_rows, int32_t* out_cols,
                           double* out_vals);
/* canonical COO in -> canonical normalized COO with self loops (cap nnz+n);
 * returns new nnz, -1 on negative weight */
int64_t orc_gcn_normalize(int32_t n, int64_t nnz, const int32_t* rows, const int32_t* cols,
                          const double* vals, int32_t* out_rows, int32_t* out_cols,
                          double* out_vals);
int64_t orc_gcn_normalize_f32(int32_t n, int64_t nnz, const int32_t* rows, const int32_t* cols,
                              const float* vals, int32_t* out_rows, int32_t* out_cols,
                              float* out_vals);

/* ---- pattern.hpp ------------------------------------------------------ */
int orc_pattern_build(int32_t n, const int32_t* rowptr, const int32_t* cols, int32_t* colptr,
                      int32_t* rows, int32_t* perm, int32_t* diag);

/* ---- kernels.hpp ------------------------------------------------------ */
void orc_spmm_csr(int32_t n_rows, const int32_t* rowptr, const int32_t* cols, const double* vals,
                  const double* B, int32_t f, double* C);
void orc_spmm_csr_f32(int32_t n_rows, const int32_t* rowptr, const int32_t* cols,
                      const float* vals, const float* B, int32_t f, float* C);
void orc_sddmm(int32_t n, const int32_t* rowptr, const int32_t* cols, const double* B,
               int32_t f, const double* C, int32_t ldc, double* out);
int orc_edge_softmax(int32_t n, const int32_t* rowptr, int64_t q, int32_t heads,
                     const double* w, double* alpha);
void orc_spmm_semibatched(int32_t n, const int32_t* rowptr, const int32_t* cols, int64_t q,
                          int32_t h, int32_t k, const double* alpha, const double* B, double* C);

/* ---- dense.hpp -------------------------------------------------------- */
/* C = op(A) op(B); A is ra x ca row-major, B is rb x cb row-major */
int orc_gemm(const double* A, int32_t ra, int32_t ca, const double* B, int32_t rb, int32_t cb,
             int trans_a, int trans_b, double* C);
void orc_column_sums(const double* X, int32_t rows, int32_t cols, double* out);
double orc_max_rel_diff(const double* a, const double* b, int64_t n);
double orc_max_rel_diff_f32(const float* a, const double* b, int64_t n);
/* kind: 0 relu, 2 elu (param alpha) */
void orc_activation(const double* X, int64_t n, int kind, double param, double* out,
                    uint8_t* mask);
void orc_activation_backward(const double* g, const uint8_t* mask, int64_t n, int kind,
                             double param, const double* saved, double* out);
double orc_loss_mse(const double* out, const double* target, int64_t n, double* grad);

/* ---- cost.hpp --------------------------------------------------------- */
/* format: 0 coo, 1 csr, 2 csc, 3 ellpack, 4 hybrid (sparse.hpp:22) */
int orc_spmm_cost(int fmt, int64_t n, int64_t q, int64_t p, int64_t f, int64_t sb, int64_t ib,
                  int64_t* flops, int64_t* bytes, double* oi);
int orc_sddmm_cost(int fmt, int64_t n, int64_t q, int64_t p, int64_t f, int64_t sb, int64_t ib,
                   int64_t* flops, int64_t* bytes, double* oi);
/* forward: 0 TF, 1 PF, 2 PF_cached; backward: 0 fused, 1 split, 2 split_cached */
int orc_gcn_select_scheme(int64_t m, int64_t k, int fg, int caching, int* fwd, int* bwd,
                          int* cached);
int orc_resolve_scheme(int policy, int64_t m, int64_t k, int fg, int caching, int* fwd,
                       int* bwd, int* cached);
int64_t orc_gcn_forward_flops(int s, int64_t n, int64_t m, int64_t k, int64_t q);
int64_t orc_gcn_backward_flops(int s, int64_t n, int64_t m, int64_t k, int64_t q, int fg);
int64_t orc_gcn_forward_transients(int s, int64_t n, int64_t m, int64_t k);
int64_t orc_gcn_backward_transients(int s, int64_t n, int64_t m, int64_t k, int fg);
int64_t orc_gat_cache_footprint(int level, int64_t n, int64_t h, int64_t k, int64_t q,
                                int64_t sb);

/* ---- gcn.hpp ---------------------------------------------------------- */
void orc_gcn_params_init(int32_t m, int32_t k, uint64_t seed, double* theta, double* bias);
/* A' given as CSR (forward) + CSC (backward view). P_out (n x m) written for PF schemes. */
int orc_gcn_forward(int32_t n, const int32_t* rowptr, const int32_t* cols, const double* vals,
                    const double* X, int32_t m, const double* theta, const double* bias,
                    int32_t k, int fwd_scheme, double* out, double* P_out);
/* saved = X for uncached schemes, P for split_cached */
int orc_gcn_backward(int32_t n, const int32_t* rowptr, const int32_t* cols, const double* vals,
                     const int32_t* colptr, const int32_t* crows, const double* cvals,
                     const double* d_out, const double* saved, int32_t m, const double* theta,
                     int32_t k, int bwd_scheme, int fg, double* d_theta, double* d_bias,
                     double* d_input);

/* ---- gat.hpp ---------------------------------------------------------- */
void orc_gat_params_init(int32_t m, int32_t h, int32_t k, uint64_t seed, double* theta,
                         double* a_src, double* a_dst, double* bias);
/* M (n x hk), s,d (n x h), alpha (h x q), mask (h x q) are outputs (may be NULL) */
int orc_gat_forward(int32_t n, const int32_t* rowptr, const int32_t* cols, const double* X,
                    int32_t m, const double* theta, const double* a_src, const double* a_dst,
                    const double* bias, int32_t h, int32_t k, double beta, double* out,
                    double* M_out, double* s_out, double* d_out_scores, double* alpha_out,
                    uint8_t* mask_out);
int orc_gat_backward(int32_t n, const int32_t* rowptr, const int32_t* cols,
                     const int32_t* colptr, const int32_t* crows, const int32_t* perm,
                     const double* G, const double* X, int32_t m, const double* theta,
                     const double* a_src, const double* a_dst, int32_t h, int32_t k,
                     double beta, int fg, double* d_theta, double* d_a_src, double* d_a_dst,
                     double* d_bias, double* d_input);

#ifdef __cplusplus
}
#endif
#endif
