#pragma once

// Drop-in replacement for the reference's sgnn/gat.hpp (gat.hpp:1-219): the
// same names, signatures, field names, require() messages and exception
// types, executed on B200 by libsgnn_cuda.so (sgnn_gat_forward /
// sgnn_gat_backward / sgnn_gat_cache_edge_values, include/sgnn_cuda.h).
//
// The cache keeps the device engine's cache (the level's retained buffers,
// charged to the device's cache class) and mirrors them into the reference's
// host fields -- M, scores, alpha / mask in the reference's head-major layout
// -- allocated in the cache memory class, so extra_bytes() and the caller's
// MemTracker see exactly gat_cache_footprint (cost.hpp:236-248).  The
// analytic operation counters are charged like the reference's kernels
// (kernels.hpp charge sites) for the work the device performs, including the
// stages a cache level lets the backward pass skip (gat.hpp:150-170).

#include <memory>
#include <optional>

#include "sgnn/b200.hpp"
#include "sgnn/cost.hpp"
#include "sgnn/kernels.hpp"

namespace sgnn {

template <class S>
struct GatParams {
  index_t heads = 1;
  index_t out_features = 0;  // k, per head
  DenseMatrix<S> theta;      // m x (h*k), per-head column blocks
  DenseMatrix<S> a_src;      // h x k
  DenseMatrix<S> a_dst;      // h x k
  std::vector<S> bias;       // h*k

  // gat.hpp:36-52 through the device generator (bit-identical draws)
  static GatParams init(index_t in_features, index_t heads, index_t out_features,
                        std::uint64_t seed) {
    require(heads >= 1, "GatParams: heads must be >= 1");
    GatParams p;
    p.heads = heads;
    p.out_features = out_features;
    const std::size_t hk = static_cast<std::size_t>(heads) * out_features;
    b200::Buf th(sizeof(S) * in_features * hk), as(sizeof(S) * hk), ad(sizeof(S) * hk),
        b(sizeof(S) * hk);
    b200::check(sgnn_gat_params_init(b200::ctx(), in_features, heads, out_features, seed,
                                     b200::dtype<S>(), th.get(), as.get(), ad.get(), b.get()));
    b200::sync();
    p.theta = b200::download_matrix<S>(th.get(), in_features, heads * out_features);
    p.a_src = b200::download_matrix<S>(as.get(), heads, out_features);
    p.a_dst = b200::download_matrix<S>(ad.get(), heads, out_features);
    p.bias.resize(hk);
    b200::download(b.get(), p.bias.data(), hk);
    return p;
  }
};

namespace b200 {

struct DevicePattern {
  sgnn_pattern h = nullptr;
  const SparsePattern* host = nullptr;
  ~DevicePattern() {
    if (h) sgnn_pattern_destroy(h);
  }
};
inline std::shared_ptr<DevicePattern> upload_pattern(const PatternPtr& p) {
  const std::size_t n = static_cast<std::size_t>(p->n()), q = static_cast<std::size_t>(p->nnz());
  auto rp = upload(p->rowptr(), n + 1), cl = upload(p->cols(), q);
  auto out = std::make_shared<DevicePattern>();
  out->host = p.get();
  check(sgnn_pattern_create(ctx(), p->n(), static_cast<int64_t>(q), static_cast<const int32_t*>(rp->get()),
                            static_cast<const int32_t*>(cl->get()), &out->h));
  sync();
  return out;
}

struct GatDeviceCache {
  sgnn_gat_cache h = nullptr;
  BufPtr X;                               // the device X the cache borrows
  std::shared_ptr<DevicePattern> pattern;  // the pattern it was built on
  ~GatDeviceCache() {
    if (h) sgnn_gat_cache_destroy(h);
  }
};

// kernels.hpp charge sites of the stages a level recomputes (gat.hpp:150-170)
inline void charge_recompute(GatCacheLevel level, count_t n, count_t m, count_t h, count_t k,
                             count_t q) {
  if (level < GatCacheLevel::features) counters().gemm_flops += 2 * n * m * h * k;  // X Theta
  if (level < GatCacheLevel::node_attention) counters().gemm_flops += 4 * n * h * k;  // scores
  if (level < GatCacheLevel::full) counters().edge_flops += 7 * h * q;  // scores, lrelu, softmax
}

}  // namespace b200

template <class S>
struct GatCache {
  GatCacheLevel level = GatCacheLevel::none;
  DenseMatrix<S> saved_input;  // always retained
  DenseMatrix<S> M;            // level >= features
  NodeScores<S> scores;        // level == node_attention
  EdgeValues<S> alpha;         // level == full
  EdgeMask mask;               // level == full
  bool consumed = false;
  std::shared_ptr<b200::GatDeviceCache> device;  // the B200 engine's cache

  // Bytes owned by the bundle beyond the retained input.
  count_t extra_bytes() const {
    count_t b = static_cast<count_t>(M.bytes());
    b += static_cast<count_t>(scores.src.bytes() + scores.dst.bytes());
    b += static_cast<count_t>(alpha.vals.bytes() + mask.bits.bytes());
    return b;
  }
};

template <class S>
struct GatGradients {
  DenseMatrix<S> d_theta;  // m x (h*k)
  DenseMatrix<S> d_a_src;  // h x k
  DenseMatrix<S> d_a_dst;  // h x k
  std::vector<S> d_bias;   // h*k
  std::optional<DenseMatrix<S>> d_input;
};

template <class S>
struct GatForwardResult {
  DenseMatrix<S> output;  // n x (h*k), heads concatenated
  GatCache<S> cache;
};

namespace b200 {
// head-major alpha / mask of a device cache (cached at level full, recomputed
// by the device otherwise) into the reference's containers
template <class S>
void edge_values(const PatternPtr& pattern, const GatParams<S>& params, GatDeviceCache& dev,
                 EdgeValues<S>& alpha, EdgeMask& mask) {
  const index_t h = params.heads;
  const std::size_t hq = static_cast<std::size_t>(h) * pattern->nnz();
  auto th = upload(params.theta), as = upload(params.a_src), ad = upload(params.a_dst);
  Buf a(sizeof(S) * hq), mk(hq);
  check(sgnn_gat_cache_edge_values(ctx(), dev.pattern->h, dev.h, th->get(), as->get(),
                                   ad->get(), a.get(), static_cast<uint8_t*>(mk.get())));
  sync();
  alpha = EdgeValues<S>::uninitialized(pattern, h);
  download(a.get(), alpha.vals.mutable_data(), hq);
  mask = EdgeMask::allocate(pattern, h);
  download(mk.get(), mask.bits.mutable_data(), hq);
}
}  // namespace b200

template <class S>
GatForwardResult<S> gat_forward(const DenseMatrix<S>& X, const PatternPtr& pattern,
                                const GatParams<S>& params, double beta,
                                GatCacheLevel level) {
  const index_t h = params.heads, k = params.out_features;
  require(pattern && pattern->has_all_self_loops(),
          "gat_forward: pattern must contain all self loops");
  require(pattern->n() == X.rows(), "gat_forward: node count mismatch");
  require(X.cols() == params.theta.rows(), "gat_forward: input width does not match theta");
  require(beta > 0, "gat_forward: beta must be positive");
  const index_t n = X.rows(), m = X.cols(), hk = h * k;
  const count_t q = pattern->nnz();

  auto dev = std::make_shared<b200::GatDeviceCache>();
  dev->pattern = b200::upload_pattern(pattern);
  dev->X = b200::upload(X);
  auto th = b200::upload(params.theta), as = b200::upload(params.a_src),
       ad = b200::upload(params.a_dst);
  auto b = b200::upload(params.bias.data(), params.bias.size());
  b200::Buf out(sizeof(S) * static_cast<std::size_t>(n) * hk);
  b200::TransientMirror mirror;
  b200::check(sgnn_gat_forward(b200::ctx(), dev->pattern->h, dev->X->get(), m, th->get(),
                               as->get(), ad->get(), b->get(), h, k, beta,
                               static_cast<int>(level), b200::dtype<S>(), out.get(), &dev->h));
  mirror.replay();
  // kernels.hpp / dense.hpp charge sites of gat.hpp:99-121
  b200::charge_recompute(GatCacheLevel::none, n, m, h, k, q);
  counters().spmm_flops += 2 * q * h * k;
  counters().elementwise_flops += static_cast<count_t>(n) * hk;

  GatForwardResult<S> r;
  r.cache.level = level;
  r.cache.saved_input = X;
  {
    ScopedMemClass o(MemClass::output);
    r.output = b200::download_matrix<S>(out.get(), n, hk);
  }
  const void *dM = nullptr, *ds = nullptr, *dd = nullptr;
  b200::check(sgnn_gat_cache_arrays(dev->h, &dM, &ds, &dd, nullptr, nullptr));
  ScopedMemClass c(MemClass::cache);  // the retained pieces (gat.hpp:123-137)
  if (level >= GatCacheLevel::features) r.cache.M = b200::download_matrix<S>(dM, n, hk);
  if (level == GatCacheLevel::node_attention) {
    r.cache.scores.src = b200::download_matrix<S>(ds, n, h);
    r.cache.scores.dst = b200::download_matrix<S>(dd, n, h);
  }
  if (level == GatCacheLevel::full)
    b200::edge_values(pattern, params, *dev, r.cache.alpha, r.cache.mask);
  r.cache.device = std::move(dev);
  return r;
}

// Everything the backward pass needs; cached pieces are shared, missing ones
// recomputed on the device with the same kernels and order as the forward pass.
template <class S>
struct GatIntermediates {
  DenseMatrix<S> M;
  EdgeValues<S> alpha;
  EdgeMask mask;
};

template <class S>
GatIntermediates<S> gat_recompute(const PatternPtr& pattern, const GatParams<S>& params,
                                  const GatCache<S>& cache, double beta) {
  (void)beta;  // the device cache carries the forward's slope
  require(cache.device && cache.device->h != nullptr,
          "gat_recompute: cache was not produced by gat_forward on this device");
  const index_t h = params.heads, k = params.out_features;
  const index_t n = cache.saved_input.rows(), m = cache.saved_input.cols();
  b200::charge_recompute(cache.level, n, m, h, k, pattern->nnz());
  GatIntermediates<S> r;
  if (cache.level >= GatCacheLevel::features) {
    r.M = cache.M;
  } else {  // the forward's feature GEMM, on the device
    auto th = b200::upload(params.theta);
    b200::Buf M(sizeof(S) * static_cast<std::size_t>(n) * h * k);
    b200::check(sgnn_gemm(b200::ctx(), b200::dtype<S>(), cache.device->X->get(), n, m,
                          th->get(), m, h * k, 0, 0, M.get()));
    b200::sync();
    r.M = b200::download_matrix<S>(M.get(), n, h * k);
  }
  if (cache.level == GatCacheLevel::full) {
    r.alpha = cache.alpha;
    r.mask = cache.mask;
    return r;
  }
  b200::edge_values(pattern, params, *cache.device, r.alpha, r.mask);
  return r;
}

template <class S>
GatGradients<S> gat_backward(const DenseMatrix<S>& d_output, const PatternPtr& pattern,
                             const GatParams<S>& params, GatCache<S>& cache, double beta,
                             bool needs_feature_grad) {
  (void)beta;  // the device cache carries the forward's slope (the reference passes the same)
  const index_t h = params.heads, k = params.out_features;
  require(!cache.consumed, "gat_backward: cache already consumed");
  cache.consumed = true;
  require(d_output.rows() == pattern->n() && d_output.cols() == h * k,
          "gat_backward: gradient shape mismatch");
  require(!cache.saved_input.empty(), "gat_backward: missing saved input");
  if (cache.level >= GatCacheLevel::features)
    require(!cache.M.empty(), "gat_backward: cache level promises M but it is absent");
  if (cache.level == GatCacheLevel::full)
    require(cache.alpha.heads == h && cache.mask.heads == h,
            "gat_backward: cache level promises alpha/mask but they are absent");
  require(cache.device && cache.device->h != nullptr,
          "gat_backward: cache was not produced by gat_forward on this device");
  const index_t n = d_output.rows(), m = params.theta.rows(), hk = h * k;
  const count_t q = pattern->nnz();
  auto& dev = *cache.device;
  if (dev.pattern->host != pattern.get()) dev.pattern = b200::upload_pattern(pattern);
  auto G = b200::upload(d_output);
  auto th = b200::upload(params.theta), as = b200::upload(params.a_src),
       ad = b200::upload(params.a_dst);
  b200::Buf dth(sizeof(S) * static_cast<std::size_t>(m) * hk), das(sizeof(S) * hk),
      dad(sizeof(S) * hk), db(sizeof(S) * hk),
      dx(needs_feature_grad ? sizeof(S) * static_cast<std::size_t>(n) * m : 0);
  b200::TransientMirror mirror;
  b200::check(sgnn_gat_backward(b200::ctx(), dev.pattern->h, G->get(), th->get(), as->get(),
                                ad->get(), m, h, k, beta, dev.h, needs_feature_grad ? 1 : 0,
                                dth.get(), das.get(), dad.get(), db.get(),
                                needs_feature_grad ? dx.get() : nullptr));
  mirror.replay();
  // kernels.hpp / dense.hpp charge sites of gat.hpp:184-217
  b200::charge_recompute(cache.level, n, m, h, k, q);
  counters().sddmm_flops += q * h * (2 * k + 1);
  counters().edge_flops += 7 * h * q;  // softmax bwd 4, lrelu bwd 1, row and column sums 1 + 1
  counters().spmm_flops += 2 * q * h * k;
  counters().elementwise_flops += 5 * static_cast<count_t>(n) * hk;
  counters().gemm_flops += 4 * static_cast<count_t>(n) * hk +
                           2 * static_cast<count_t>(n) * m * hk * (needs_feature_grad ? 2 : 1);

  GatGradients<S> g;
  ScopedMemClass o(MemClass::output);
  g.d_theta = b200::download_matrix<S>(dth.get(), m, hk);
  g.d_a_src = b200::download_matrix<S>(das.get(), h, k);
  g.d_a_dst = b200::download_matrix<S>(dad.get(), h, k);
  g.d_bias.resize(static_cast<std::size_t>(hk));
  b200::download(db.get(), g.d_bias.data(), g.d_bias.size());
  if (needs_feature_grad) g.d_input = b200::download_matrix<S>(dx.get(), n, m);
  cache.device.reset();  // consumed: release the device cache
  return g;
}

}  // namespace sgnn
