#pragma once

// Drop-in replacement for the reference's sgnn/gcn.hpp (gcn.hpp:1-193): the
// same names, signatures, field names, require() messages and exception
// types, executed on B200 by libsgnn_cuda.so (sgnn_gcn_forward /
// sgnn_gcn_backward, include/sgnn_cuda.h).  The caller's own sgnn headers
// supply the host types (DenseMatrix, AdjacencyOp, SchemeChoice, MemTracker).
//
// Per call: the operator and dense inputs are uploaded, the layer runs on the
// device, results are downloaded into the reference's host containers.  The
// cache keeps its device state (the uploaded X, or P = A'X owned by the
// device cache) for the backward pass, and mirrors the reference's host
// fields: saved_input aliases X (gcn.hpp:111) and saved_propagated holds a
// host copy of P in the cache memory class (gcn.hpp:122-125), so
// retained_bytes() and the MemTracker classes read like the reference's.

#include <memory>
#include <optional>

#include "sgnn/b200.hpp"
#include "sgnn/cost.hpp"
#include "sgnn/kernels.hpp"

namespace sgnn {

enum class SchemePolicy { adaptive, force_transform_first, force_propagate_first };

inline const char* to_string(SchemePolicy p) {
  switch (p) {
    case SchemePolicy::adaptive: return "adaptive";
    case SchemePolicy::force_transform_first: return "transform-first";
    case SchemePolicy::force_propagate_first: return "propagate-first";
  }
  return "?";
}

// gcn.hpp:34-47 through sgnn_resolve_scheme (bit-identical selector)
inline SchemeChoice resolve_scheme(SchemePolicy policy, count_t m, count_t k,
                                   bool needs_feature_grad, bool caching) {
  sgnn_scheme s{};
  b200::check(sgnn_resolve_scheme(static_cast<int>(policy), m, k, needs_feature_grad ? 1 : 0,
                                  caching ? 1 : 0, &s));
  return {static_cast<GcnForward>(s.forward), static_cast<GcnBackward>(s.backward),
          s.caching != 0};
}

template <class S>
struct GcnParams {
  DenseMatrix<S> theta;  // m x k
  std::vector<S> bias;   // k

  // gcn.hpp:54-62 through the device generator (bit-identical splitmix64 draws)
  static GcnParams init(index_t in_features, index_t out_features, std::uint64_t seed) {
    GcnParams p;
    b200::Buf th(sizeof(S) * static_cast<std::size_t>(in_features) * out_features);
    b200::Buf b(sizeof(S) * static_cast<std::size_t>(out_features));
    b200::check(sgnn_gcn_params_init(b200::ctx(), in_features, out_features, seed,
                                     b200::dtype<S>(), th.get(), b.get()));
    b200::sync();
    p.theta = b200::download_matrix<S>(th.get(), in_features, out_features);
    p.bias.resize(static_cast<std::size_t>(out_features));
    b200::download(b.get(), p.bias.data(), p.bias.size());
    return p;
  }
};

namespace b200 {

// device operator of an AdjacencyOp: its canonical COO uploaded once per call
struct DeviceAdjacency {
  sgnn_adj h = nullptr;
  ~DeviceAdjacency() {
    if (h) sgnn_adj_destroy(h);
  }
};
template <class S>
std::shared_ptr<DeviceAdjacency> upload_adjacency(const AdjacencyOp<S>& A) {
  const CooMatrix<S> coo = to_coo(A.matrix());
  const std::size_t q = static_cast<std::size_t>(coo.nnz());
  auto r = upload(coo.rows.data(), q), c = upload(coo.cols.data(), q);
  auto v = upload(coo.vals.data(), q);
  auto out = std::make_shared<DeviceAdjacency>();
  check(sgnn_adj_create(ctx(), coo.n_rows, coo.n_cols, static_cast<int64_t>(q),
                        static_cast<const int32_t*>(r->get()), static_cast<const int32_t*>(c->get()),
                        v->get(), dtype<S>(), static_cast<int>(A.format()), &out->h));
  sync();
  return out;
}

struct GcnDeviceCache {
  sgnn_gcn_cache h = nullptr;
  BufPtr X;  // the device copy of X the cache borrows (uncached schemes)
  ~GcnDeviceCache() {
    if (h) sgnn_gcn_cache_destroy(h);
  }
};

}  // namespace b200

// Exactly one of saved_input / saved_propagated is retained.
template <class S>
struct GcnCache {
  SchemeChoice scheme;
  DenseMatrix<S> saved_input;       // X, for the uncached backward schemes
  DenseMatrix<S> saved_propagated;  // P = A'X, for the cached scheme
  bool consumed = false;
  std::shared_ptr<b200::GcnDeviceCache> device;  // the B200 engine's cache

  count_t retained_bytes() const {
    return static_cast<count_t>(saved_input.bytes() + saved_propagated.bytes());
  }
};

template <class S>
struct GcnGradients {
  DenseMatrix<S> d_theta;
  std::vector<S> d_bias;
  std::optional<DenseMatrix<S>> d_input;
};

template <class S>
struct GcnForwardResult {
  DenseMatrix<S> output;
  GcnCache<S> cache;
};

template <class S>
GcnForwardResult<S> gcn_forward(const DenseMatrix<S>& X, const AdjacencyOp<S>& A,
                                const GcnParams<S>& params, const SchemeChoice& scheme) {
  require(A.n_rows() == A.n_cols() && A.n_cols() == X.rows(),
          "gcn_forward: adjacency/input shape mismatch");
  require(X.cols() == params.theta.rows(), "gcn_forward: input width does not match theta");
  const index_t n = X.rows(), m = X.cols(), k = params.theta.cols();
  b200::TransientMirror mirror;
  auto adj = b200::upload_adjacency(A);
  auto dev = std::make_shared<b200::GcnDeviceCache>();
  dev->X = b200::upload(X);
  auto th = b200::upload(params.theta);
  auto b = b200::upload(params.bias.data(), params.bias.size());
  b200::Buf out(sizeof(S) * static_cast<std::size_t>(n) * k);
  const sgnn_scheme sc{static_cast<int32_t>(scheme.forward),
                       static_cast<int32_t>(scheme.backward), scheme.caching ? 1 : 0};
  b200::check(sgnn_gcn_forward(b200::ctx(), adj->h, dev->X->get(), m, th->get(), b->get(), k,
                               &sc, out.get(), &dev->h));
  mirror.replay();
  // the reference's FLOP model of the pass (cost.hpp:143-160)
  counters().gemm_flops += 2 * static_cast<count_t>(n) * m * k;
  counters().spmm_flops += 2 * static_cast<count_t>(A.nnz()) *
                           (scheme.forward == GcnForward::transform_first ? k : m);
  GcnForwardResult<S> r;
  r.cache.scheme = scheme;
  {
    ScopedMemClass o(MemClass::output);
    r.output = b200::download_matrix<S>(out.get(), n, k);
  }
  if (scheme.forward == GcnForward::propagate_first_cached) {
    const void* P = nullptr;
    b200::check(sgnn_gcn_cache_arrays(dev->h, nullptr, &P));
    ScopedMemClass c(MemClass::cache);
    r.cache.saved_propagated = b200::download_matrix<S>(P, n, m);
    dev->X.reset();  // the device cache owns P; X is not retained (gcn.hpp:122-125)
  } else {
    r.cache.saved_input = X;
  }
  r.cache.device = std::move(dev);
  return r;
}

template <class S>
GcnGradients<S> gcn_backward(const DenseMatrix<S>& d_output, const AdjacencyOp<S>& A,
                             const GcnParams<S>& params, GcnCache<S>& cache,
                             bool needs_feature_grad) {
  require(!cache.consumed, "gcn_backward: cache already consumed");
  cache.consumed = true;
  require(d_output.cols() == params.theta.cols() && d_output.rows() == A.n_rows(),
          "gcn_backward: gradient shape mismatch");
  const bool cached = cache.scheme.backward == GcnBackward::split_propagate_cached;
  if (cached)
    require(!cache.saved_propagated.empty(), "gcn_backward: cached scheme without saved A'X");
  else
    require(!cache.saved_input.empty(), "gcn_backward: missing saved input");
  require(cache.device && cache.device->h != nullptr,
          "gcn_backward: cache was not produced by gcn_forward on this device");
  const index_t n = d_output.rows(), m = params.theta.rows(), k = params.theta.cols();
  b200::TransientMirror mirror;
  auto adj = b200::upload_adjacency(A);
  auto G = b200::upload(d_output);
  auto th = b200::upload(params.theta);
  b200::Buf dth(sizeof(S) * static_cast<std::size_t>(m) * k), db(sizeof(S) * k);
  b200::Buf dx(needs_feature_grad ? sizeof(S) * static_cast<std::size_t>(n) * m : 0);
  b200::check(sgnn_gcn_backward(b200::ctx(), adj->h, G->get(), th->get(), m, k, cache.device->h,
                                needs_feature_grad ? 1 : 0, dth.get(), db.get(),
                                needs_feature_grad ? dx.get() : nullptr));
  mirror.replay();
  counters().gemm_flops += 2 * static_cast<count_t>(n) * m * k * (needs_feature_grad ? 2 : 1);
  counters().elementwise_flops += static_cast<count_t>(n) * k;
  GcnGradients<S> g;
  ScopedMemClass o(MemClass::output);
  g.d_theta = b200::download_matrix<S>(dth.get(), m, k);
  g.d_bias.resize(static_cast<std::size_t>(k));
  b200::download(db.get(), g.d_bias.data(), g.d_bias.size());
  if (needs_feature_grad) g.d_input = b200::download_matrix<S>(dx.get(), n, m);
  cache.device.reset();  // consumed: release the device cache
  return g;
}

}  // namespace sgnn
