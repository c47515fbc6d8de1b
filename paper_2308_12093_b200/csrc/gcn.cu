// gcn.cu -- GCN scheme engine (north-star subsystem 2; gcn.hpp:91-193).
//
//   transform_first          M = X Theta (tcgen05 GEMM), out = A'M + b (SpMM, bias epilogue)
//   propagate_first[_cached] P = A'X (SpMM), out = P Theta + b (GEMM, bias epilogue);
//                            the cached variant keeps P for backward
//   fused_propagate          S = A'^T dX', dTheta = X^T S, dX = S Theta^T
//   split_propagate          P = A'X, G = dX' Theta^T, dTheta = P^T dX', dX = A'^T G
//   split_propagate_cached   as split with P from the cache (no SpMM without dX)
// Transients come from the stream-ordered pool; A'^T products run the same
// CSR kernel over the CSC arrays (CSR of A'^T).
#include "common.cuh"
#include "internal.cuh"

using namespace sgnn;

namespace {

const LongRows* fwd_plan(sgnn_ctx ctx, sgnn_adj A) {
  return &long_rows(ctx, A->long_fwd, A->n_rows, A->rowptr.as<int32_t>());
}
const LongRows* bwd_plan(sgnn_ctx ctx, sgnn_adj A) {
  return &long_rows(ctx, A->long_bwd, A->n_cols, A->colptr.as<int32_t>());
}

inline void ok(int rc) {
  if (rc == SGNN_OK) return;
  if (rc == SGNN_EINVAL) throw invalid_argument(sgnn_last_error());
  throw std::runtime_error(sgnn_last_error());
}

template <class T>
constexpr int dt() {
  return sizeof(T) == 4 ? SGNN_F32 : SGNN_F64;
}

// SGNN_PRESPLIT=1: split Theta on the side stream during the forward SpMM
// (A/B knob, off by default: 4 us faster eager but 4 us slower under the
// CUDA-graph replay the step is timed with -- measured)
static bool presplit_on() {
  static const bool on = [] {
    const char* e = getenv("SGNN_PRESPLIT");
    return e && e[0] == '1';
  }();
  return on;
}

// out = A' X Theta + b, then (relu != nullptr) ReLU with its mask -- fused into
// the X.Theta / P.Theta epilogue when that GEMM runs on tcgen05
template <class T>
void gcn_forward_t(sgnn_ctx ctx, sgnn_adj A, const T* X, int32_t m, const T* theta,
                   const T* bias, int32_t k, const sgnn_scheme& s, T* out, sgnn_gcn_cache c,
                   uint8_t* relu = nullptr) {
  const int32_t n = A->n_rows;
  cudaStream_t st = ctx->stream;
  const int32_t* rp = A->rowptr.as<int32_t>();
  const int32_t* ci = A->cols.as<int32_t>();
  const T* av = A->vals.as<T>();
  if (s.forward == SGNN_TRANSFORM_FIRST) {
    DevBuf M((size_t)n * k * sizeof(T), st);
    M.track(kTransient, M.bytes());  // gcn.hpp:103-106
    gemm<T>(ctx, X, n, m, theta, m, k, false, false, M.as<T>());
    spmm_csr<T>(ctx, n, rp, ci, av, M.as<T>(), k, out, bias, A->nnz, fwd_plan(ctx, A),
                A->n_cols);
    if (relu) ok(sgnn_activation(ctx, 0, dt<T>(), out, (int64_t)n * k, out, relu));
    c->saved_input = X;
  } else {
    DevBuf P((size_t)n * m * sizeof(T), st);
    P.track(kTransient, P.bytes());  // gcn.hpp:114-117
    const LongRows* fp = fwd_plan(ctx, A);
    // float32: Theta's tf32 hi / lo split for the P.Theta GEMM on the side
    // stream, overlapped with the SpMM (off the step's critical path)
    DevBuf th_split;
    bool presplit = false;
    if constexpr (sizeof(T) == 4)
      presplit = gemm_uses_presplit((int64_t)m * k, n, m) && presplit_on();
    if (presplit) {
      th_split = DevBuf((size_t)m * k * 8, st);
      SideStream side(ctx);
      side.side();
      gemm_presplit_f32(ctx, reinterpret_cast<const float*>(theta), (int64_t)m * k,
                        th_split.as<float>(), th_split.as<float>() + (size_t)m * k);
      side.main();
      spmm_csr<T>(ctx, n, rp, ci, av, X, m, P.as<T>(), nullptr, A->nnz, fp, A->n_cols);
      side.join();
      ctx->split_src = reinterpret_cast<const float*>(theta);
      ctx->split_elems = (int64_t)m * k;
      ctx->split_hi = th_split.as<float>();
      ctx->split_lo = th_split.as<float>() + (size_t)m * k;
    } else {
      spmm_csr<T>(ctx, n, rp, ci, av, X, m, P.as<T>(), nullptr, A->nnz, fp, A->n_cols);
    }
    struct ClearHint {  // the hint covers this GEMM only (also on exceptions)
      sgnn_ctx c;
      ~ClearHint() { c->split_src = nullptr; c->split_elems = 0; }
    } clear_hint{ctx};
    bool fused = false;
    if constexpr (sizeof(T) == 4)
      if (relu) fused = gemm_relu_f32(ctx, P.as<T>(), n, m, theta, m, k, false, false, out, bias,
                                      relu, nullptr);
    if (!fused) {
      gemm<T>(ctx, P.as<T>(), n, m, theta, m, k, false, false, out, bias);
      if (relu) ok(sgnn_activation(ctx, 0, dt<T>(), out, (int64_t)n * k, out, relu));
    }
    if (s.forward == SGNN_PROPAGATE_FIRST_CACHED) {
      P.reclassify(kCache);  // reclassified into the cache (gcn.hpp:124)
      c->saved_propagated = std::move(P);
    }
    else
      c->saved_input = X;
  }
}

// d_input gets the ReLU backward of the previous layer applied when dmask is
// given (fused into the S.Theta^T epilogue on the fused_propagate scheme)
template <class T>
void gcn_backward_t(sgnn_ctx ctx, sgnn_adj A, const T* G, const T* theta, int32_t m, int32_t k,
                    sgnn_gcn_cache c, bool fg, T* d_theta, T* d_bias, T* d_input,
                    const uint8_t* dmask = nullptr) {
  auto relu_bwd = [&]() {
    if (dmask && fg)
      ok(sgnn_activation_backward(ctx, 0, dt<T>(), d_input, dmask, nullptr,
                                  (int64_t)A->n_cols * m, d_input));
  };
  const int32_t n = A->n_rows;
  cudaStream_t st = ctx->stream;
  const int32_t* rp = A->rowptr.as<int32_t>();
  const int32_t* ci = A->cols.as<int32_t>();
  const T* av = A->vals.as<T>();
  const int32_t* cp = A->colptr.as<int32_t>();
  const int32_t* cr = A->crows.as<int32_t>();
  const T* cv = A->cvals.as<T>();
  switch (c->scheme.backward) {
    case SGNN_FUSED_PROPAGATE: {
      const T* X = static_cast<const T*>(c->saved_input);
      DevBuf S((size_t)n * k * sizeof(T), st);
      S.track(kTransient, S.bytes());  // gcn.hpp:152-155
      const LongRows* bp = bwd_plan(ctx, A);
      SideStream side(ctx);  // d_bias on the side stream, during the SpMM
      side.side();
      column_sums<T>(ctx, G, n, k, d_bias);
      side.main();
      spmm_csr<T>(ctx, A->n_cols, cp, cr, cv, G, k, S.as<T>(), nullptr, A->nnz, bp, n);
      side.join();
      SideStream side2(ctx);  // dTheta = X^T S on the side stream, dX = S Theta^T here
      if (fg) side2.side();
      gemm<T>(ctx, X, n, m, S.as<T>(), n, k, true, false, d_theta);
      side2.main();
      if (fg) {
        bool fused = false;
        if constexpr (sizeof(T) == 4)
          if (dmask) fused = gemm_relu_f32(ctx, S.as<T>(), n, k, theta, m, k, false, true, d_input,
                                           nullptr, nullptr, dmask);
        if (!fused) {
          gemm<T>(ctx, S.as<T>(), n, k, theta, m, k, false, true, d_input);
          relu_bwd();
        }
      }
      break;
    }
    case SGNN_SPLIT_PROPAGATE: {
      const T* X = static_cast<const T*>(c->saved_input);
      DevBuf P((size_t)n * m * sizeof(T), st);
      P.track(kTransient, P.bytes());  // gcn.hpp:163-167
      const LongRows* fp = fwd_plan(ctx, A);
      const LongRows* bp = fg ? bwd_plan(ctx, A) : nullptr;
      // P = A'X -> dTheta (+ d_bias) on the side stream, G Theta^T -> A'^T G2
      // on the main stream: independent chains, overlapped
      SideStream side(ctx);
      if (fg) side.side();
      spmm_csr<T>(ctx, n, rp, ci, av, X, m, P.as<T>(), nullptr, A->nnz, fp, A->n_cols);
      gemm_tn_colsum<T>(ctx, P.as<T>(), n, m, G, n, k, d_theta, d_bias);
      side.main();
      if (fg) {
        DevBuf G2((size_t)n * m * sizeof(T), st);
        G2.track(kTransient, G2.bytes());
        gemm<T>(ctx, G, n, k, theta, m, k, false, true, G2.as<T>());
        spmm_csr<T>(ctx, A->n_cols, cp, cr, cv, G2.as<T>(), m, d_input, nullptr, A->nnz, bp, n);
        relu_bwd();
      }
      side.join();
      break;
    }
    case SGNN_SPLIT_PROPAGATE_CACHED: {
      const T* P = c->saved_propagated.as<T>();
      const LongRows* bp = fg ? bwd_plan(ctx, A) : nullptr;
      // dTheta (+ d_bias) = P^T G on the side stream, overlapped with
      // G Theta^T -> A'^T G2 on the main stream
      SideStream side(ctx);
      if (fg) side.side();
      gemm_tn_colsum<T>(ctx, P, n, m, G, n, k, d_theta, d_bias);
      side.main();
      if (fg) {
        DevBuf G2((size_t)n * m * sizeof(T), ctx->stream);
        G2.track(kTransient, G2.bytes());  // gcn.hpp:180-184
        gemm<T>(ctx, G, n, k, theta, m, k, false, true, G2.as<T>());
        spmm_csr<T>(ctx, A->n_cols, cp, cr, cv, G2.as<T>(), m, d_input, nullptr, A->nnz, bp, n);
        relu_bwd();
      }
      side.join();
      break;
    }
    default: throw invalid_argument("gcn_backward: unknown scheme");
  }
}

}  // namespace

extern "C" {

int sgnn_gcn_forward(sgnn_ctx ctx, sgnn_adj A, const void* X, int32_t m, const void* theta,
                     const void* bias, int32_t k, const sgnn_scheme* scheme, void* out,
                     sgnn_gcn_cache* cache) {
  return sgnn::gcn_forward_relu(ctx, A, X, m, theta, bias, k, scheme, out, cache, nullptr);
}

int sgnn_gcn_backward(sgnn_ctx ctx, sgnn_adj A, const void* d_out, const void* theta, int32_t m,
                      int32_t k, sgnn_gcn_cache c, int fg, void* d_theta, void* d_bias,
                      void* d_input) {
  return sgnn::gcn_backward_relu(ctx, A, d_out, theta, m, k, c, fg, d_theta, d_bias, d_input,
                                 nullptr);
}

}  // extern "C"

int sgnn::gcn_forward_relu(sgnn_ctx ctx, sgnn_adj A, const void* X, int32_t m,
                           const void* theta, const void* bias, int32_t k,
                           const sgnn_scheme* scheme, void* out, sgnn_gcn_cache* cache,
                           uint8_t* relu_mask) {
  SGNN_API_BEGIN
  require(A && scheme && cache, "gcn_forward: null argument");
  require(A->n_rows == A->n_cols, "gcn_forward: adjacency/input shape mismatch");
  require(m >= 1 && k >= 1, "gcn_forward: input width does not match theta");
  require(scheme->forward >= 0 && scheme->forward <= 2 && scheme->backward >= 0 &&
              scheme->backward <= 2,
          "gcn_forward: unknown scheme");
  auto* c = new sgnn_gcn_cache_s;
  c->scheme = *scheme;
  c->dtype = A->dtype;
  c->n = A->n_rows;
  c->m = m;
  c->saved_propagated.set_stream(ctx->stream);
  try {
    if (A->dtype == SGNN_F32)
      gcn_forward_t<float>(ctx, A, (const float*)X, m, (const float*)theta, (const float*)bias,
                           k, *scheme, (float*)out, c, relu_mask);
    else
      gcn_forward_t<double>(ctx, A, (const double*)X, m, (const double*)theta,
                            (const double*)bias, k, *scheme, (double*)out, c, relu_mask);
  } catch (...) {
    delete c;
    throw;
  }
  *cache = c;
  SGNN_API_END
}

int sgnn::gcn_backward_relu(sgnn_ctx ctx, sgnn_adj A, const void* d_out, const void* theta,
                            int32_t m, int32_t k, sgnn_gcn_cache c, int fg, void* d_theta,
                            void* d_bias, void* d_input, const uint8_t* relu_mask_in) {
  SGNN_API_BEGIN
  require(c != nullptr, "gcn_backward: missing saved input");
  require(!c->consumed, "gcn_backward: cache already consumed");
  c->consumed = true;  // gcn.hpp:137-138: consumed before any other validation
  require(A && c->m == m, "gcn_backward: gradient shape mismatch");
  const bool cached = c->scheme.backward == SGNN_SPLIT_PROPAGATE_CACHED;
  if (cached)
    require(c->saved_propagated.get() != nullptr,
            "gcn_backward: cached scheme without saved A'X");
  else
    require(c->saved_input != nullptr, "gcn_backward: missing saved input");
  require(!fg || d_input != nullptr, "gcn_backward: d_input required for feature gradients");
  if (A->dtype == SGNN_F32)
    gcn_backward_t<float>(ctx, A, (const float*)d_out, (const float*)theta, m, k, c, fg != 0,
                          (float*)d_theta, (float*)d_bias, (float*)d_input, relu_mask_in);
  else
    gcn_backward_t<double>(ctx, A, (const double*)d_out, (const double*)theta, m, k, c, fg != 0,
                           (double*)d_theta, (double*)d_bias, (double*)d_input, relu_mask_in);
  // the cached P is released once consumed (its lifetime ends with backward)
  c->saved_propagated.reset();
  SGNN_API_END
}

extern "C" {

int sgnn_gcn_cache_destroy(sgnn_gcn_cache c) {
  SGNN_API_BEGIN
  delete c;
  SGNN_API_END
}

// device arrays the cache retains: the borrowed X (uncached schemes) or the
// owned P = A'X (propagate_first_cached); the other is NULL
int sgnn_gcn_cache_arrays(sgnn_gcn_cache c, const void** saved_input,
                          const void** saved_propagated) {
  SGNN_API_BEGIN
  require(c != nullptr, "gcn cache: null handle");
  if (saved_input) *saved_input = c->saved_propagated.get() ? nullptr : c->saved_input;
  if (saved_propagated) *saved_propagated = c->saved_propagated.get();
  SGNN_API_END
}

int sgnn_gcn_cache_retained_bytes(sgnn_gcn_cache c, int64_t* out) {
  SGNN_API_BEGIN
  const int64_t sb = c->dtype == SGNN_F32 ? 4 : 8;
  *out = c->saved_propagated.get() ? (int64_t)c->saved_propagated.bytes()
                                   : (c->saved_input ? sb * c->n * c->m : 0);
  SGNN_API_END
}

}  // extern "C"
