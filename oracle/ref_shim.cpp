// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference headers, compiled in place
// from /root/reference/proj/include by oracle/Makefile into
// oracle/_ref/libsgnn_ref.so (git-ignored, travels to the GPU box).
// Uses: (1) oracle/gen_golden.py produces tests/golden/*.npz with it, which
// pin the C restatement in oracle/sgnn_oracle.c; (2) bench.py's reference arm
// and cpu_baseline time the reference's own OpenMP CPU path through it.
// Nothing from the reference is copied here; this file only calls its API.
#include <chrono>
#include <cstring>
#include <functional>
#include <memory>
#include <optional>

#include "sgnn/bench.hpp"
#include "sgnn/cost.hpp"
#include "sgnn/gat.hpp"
#include "sgnn/gcn.hpp"
#include "sgnn/graph.hpp"
#include "sgnn/kernels.hpp"
#include "sgnn/model.hpp"

using namespace sgnn;

namespace {

template <class S>
DenseMatrix<S> mat(const S* p, index_t r, index_t c) {
  DenseMatrix<S> m(r, c);
  std::memcpy(m.mutable_data(), p, sizeof(S) * m.size());
  return m;
}
template <class S>
void out(const DenseMatrix<S>& m, S* p) {
  if (p) std::memcpy(p, m.data(), sizeof(S) * m.size());
}
template <class S>
CooMatrix<S> coo_of(index_t nr, index_t nc, long long nnz, const int* r, const int* c,
                    const S* v) {
  std::vector<Triplet<S>> ts(static_cast<std::size_t>(nnz));
  for (long long i = 0; i < nnz; ++i) ts[i] = {r[i], c[i], v[i]};
  return coo_from_triplets(nr, nc, std::move(ts));
}
thread_local std::string g_err;

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_num_threads() { return num_threads(); }
void ref_set_num_threads(int n) { set_num_threads(n); }

long long ref_synthetic_graph(int n, double deg, unsigned long long seed, int* src, int* dst) {
  Graph g = synthetic_graph(n, deg, seed);
  for (std::size_t i = 0; i < g.edges.size(); ++i) {
    if (src) src[i] = g.edges[i].src;
    if (dst) dst[i] = g.edges[i].dst;
  }
  return static_cast<long long>(g.edges.size());
}

// bench.hpp run_benchmark (BenchReport, schema_version 1) of one
// configuration with a minimal timing protocol (0 warmups, 1 block x 1 run):
// the report JSON (report_to_json) is written into `out` (cap bytes).
// Returns the JSON length, or -1 (text in ref_last_error()).
long long ref_bench_report_json(const char* dataset, int gat2, int fmt, int hidden, int heads,
                                int policy, int level, int fwdbwd, int fg, int f32,
                                int in_features, int classes, unsigned long long seed,
                                char* out, long long cap) {
  try {
    BenchConfig cfg;
    cfg.dataset = dataset;
    cfg.format = static_cast<SparseFormat>(fmt);
    cfg.pass = fwdbwd ? BenchPass::forward_backward : BenchPass::forward;
    cfg.warmups = 0;
    cfg.blocks = 1;
    cfg.runs_per_block = 1;
    cfg.seed = seed;
    cfg.f32 = f32 != 0;
    ModelConfig& mc = cfg.model;
    mc.kind = gat2 ? ModelKind::gat2 : ModelKind::gcn2;
    mc.in_features = in_features;
    mc.hidden = hidden;
    mc.out_features = classes;
    mc.heads = heads;
    mc.scheme = static_cast<SchemePolicy>(policy);
    mc.input_grad = fg != 0;
    if (gat2) mc.gat_level = static_cast<GatCacheLevel>(level);
    else mc.caching = level != 0;
    const std::string js = report_to_json(run_benchmark(cfg)).dump();
    if (static_cast<long long>(js.size()) + 1 > cap) {
      g_err = "ref_bench_report_json: buffer too small";
      return -1;
    }
    std::memcpy(out, js.c_str(), js.size() + 1);
    return static_cast<long long>(js.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// graph.hpp load_graph: returns the edge count (arrays filled when non-null,
// n in *n), or -1 with the runtime_error text in ref_last_error().
long long ref_load_graph(const char* path, int matrix_market, int* n, int* src, int* dst,
                         double* w) {
  try {
    Graph g = load_graph(path, matrix_market ? GraphFileFormat::matrix_market
                                             : GraphFileFormat::edge_list);
    *n = g.n;
    for (std::size_t i = 0; i < g.edges.size(); ++i) {
      if (src) src[i] = g.edges[i].src;
      if (dst) dst[i] = g.edges[i].dst;
      if (w) w[i] = g.edges[i].weight;
    }
    return static_cast<long long>(g.edges.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

void ref_random_uniform(int rows, int cols, unsigned long long seed, double lo, double hi,
                        double* o) {
  out(DenseMatrix<double>::random_uniform(rows, cols, seed, lo, hi), o);
}

long long ref_coo_canonicalize(int nr, int nc, long long nnz, const int* r, const int* c,
                               const double* v, int* ro, int* co, double* vo) {
  try {
    auto m = coo_of<double>(nr, nc, nnz, r, c, v);
    for (index_t e = 0; e < m.nnz(); ++e) {
      ro[e] = m.rows[e];
      co[e] = m.cols[e];
      vo[e] = m.vals[e];
    }
    return m.nnz();
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

// COO -> canonical normalized COO (python gcn_normalize, bindings.cpp:121-136)
long long ref_gcn_normalize(int n, long long nnz, const int* r, const int* c, const double* v,
                            int* ro, int* co, double* vo) {
  try {
    auto coo = to_coo(gcn_normalize(SparseMatrix<double>{coo_of<double>(n, n, nnz, r, c, v)}));
    for (index_t e = 0; e < coo.nnz(); ++e) {
      ro[e] = coo.rows[e];
      co[e] = coo.cols[e];
      vo[e] = coo.vals[e];
    }
    return coo.nnz();
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}
long long ref_gcn_normalize_f32(int n, long long nnz, const int* r, const int* c,
                                const float* v, int* ro, int* co, float* vo) {
  try {
    auto coo = to_coo(gcn_normalize(SparseMatrix<float>{coo_of<float>(n, n, nnz, r, c, v)}));
    for (index_t e = 0; e < coo.nnz(); ++e) {
      ro[e] = coo.rows[e];
      co[e] = coo.cols[e];
      vo[e] = coo.vals[e];
    }
    return coo.nnz();
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

// canonical CSR + CSC arrays for a canonical COO (sparse.hpp:151-218)
void ref_csr_csc(int n_rows, int n_cols, long long nnz, const int* r, const int* c,
                 const double* v, int* rowptr, int* colptr, int* crows, double* cvals) {
  auto coo = coo_of<double>(n_rows, n_cols, nnz, r, c, v);
  auto csr = coo_to_csr(coo);
  auto csc = coo_to_csc(coo);
  for (index_t i = 0; i <= n_rows; ++i) rowptr[i] = csr.rowptr[i];
  for (index_t j = 0; j <= n_cols; ++j) colptr[j] = csc.colptr[j];
  for (index_t e = 0; e < csc.nnz(); ++e) {
    crows[e] = csc.rows[e];
    cvals[e] = csc.vals[e];
  }
}

// SparsePattern arrays (pattern.hpp:19-59); returns all-self-loops flag
int ref_pattern(int n, const int* rowptr, const int* cols, int* colptr, int* rows, int* perm,
                int* diag) {
  auto p = SparsePattern::build(n, rowptr, cols);
  for (index_t j = 0; j <= n; ++j) colptr[j] = p->colptr()[j];
  for (index_t e = 0; e < p->nnz(); ++e) {
    rows[e] = p->rows()[e];
    perm[e] = p->perm()[e];
  }
  for (index_t i = 0; i < n; ++i) diag[i] = p->diag_index(i);
  return p->has_all_self_loops() ? 1 : 0;
}

// python spmm (bindings.cpp:138-148); fmt 0 coo 1 csr 2 csc 3 ellpack 4 hybrid
int ref_spmm(int fmt, int nr, int nc, long long nnz, const int* r, const int* c,
             const double* v, const double* B, int f, double* C) {
  try {
    auto A = convert(SparseMatrix<double>{coo_of<double>(nr, nc, nnz, r, c, v)},
                     static_cast<SparseFormat>(fmt));
    out(spmm(A, mat(B, nc, f)), C);
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}
int ref_spmm_f32(int fmt, int nr, int nc, long long nnz, const int* r, const int* c,
                 const float* v, const float* B, int f, float* C) {
  try {
    auto A = convert(SparseMatrix<float>{coo_of<float>(nr, nc, nnz, r, c, v)},
                     static_cast<SparseFormat>(fmt));
    out(spmm(A, mat(B, nc, f)), C);
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

// python sddmm (bindings.cpp:150-171): values in canonical pattern order
long long ref_sddmm(int n, long long nnz, const int* r, const int* c, const double* B, int f,
                    const double* C, double* vals_out) {
  std::vector<double> ones(static_cast<std::size_t>(nnz), 1.0);
  auto csr = coo_to_csr(coo_of<double>(n, n, nnz, r, c, ones.data()));
  auto pattern = SparsePattern::from_csr(csr);
  auto o = sddmm<double>(pattern, nullptr, mat(B, n, f), mat(C, f, n));
  std::memcpy(vals_out, o.vals.data(), sizeof(double) * pattern->nnz());
  return pattern->nnz();
}

// python edge_softmax (bindings.cpp:173-193)
int ref_edge_softmax(int n, long long nnz, const int* r, const int* c, const double* scores,
                     double* alpha) {
  try {
    std::vector<double> ones(static_cast<std::size_t>(nnz), 1.0);
    auto csr = coo_to_csr(coo_of<double>(n, n, nnz, r, c, ones.data()));
    auto pattern = SparsePattern::from_csr(csr);
    EdgeValues<double> w;
    w.pattern = pattern;
    w.heads = 1;
    w.vals = mat(scores, 1, pattern->nnz());
    out(edge_softmax(w).vals, alpha);
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

int ref_select_scheme(int policy, long long m, long long k, int fg, int caching, int* fwd,
                      int* bwd, int* cached) {
  try {
    auto s = resolve_scheme(static_cast<SchemePolicy>(policy), m, k, fg != 0, caching != 0);
    *fwd = static_cast<int>(s.forward);
    *bwd = static_cast<int>(s.backward);
    *cached = s.caching ? 1 : 0;
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

int ref_spmm_cost(int fmt, long long n, long long q, long long p, long long f, long long sb,
                  long long ib, long long* flops, long long* bytes, double* oi) {
  try {
    auto c = spmm_cost(static_cast<SparseFormat>(fmt), n, q, p, f, sb, ib);
    *flops = c.flops;
    *bytes = c.bytes;
    *oi = c.operational_intensity;
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}
int ref_sddmm_cost(int fmt, long long n, long long q, long long p, long long f, long long sb,
                   long long ib, long long* flops, long long* bytes, double* oi) {
  try {
    auto c = sddmm_cost(static_cast<SparseFormat>(fmt), n, q, p, f, sb, ib);
    *flops = c.flops;
    *bytes = c.bytes;
    *oi = c.operational_intensity;
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

void ref_gcn_params(int m, int k, unsigned long long seed, double* theta, double* bias) {
  auto p = GcnParams<double>::init(m, k, seed);
  out(p.theta, theta);
  std::memcpy(bias, p.bias.data(), sizeof(double) * k);
}
void ref_gat_params(int m, int h, int k, unsigned long long seed, double* theta, double* as,
                    double* ad, double* bias) {
  auto p = GatParams<double>::init(m, h, k, seed);
  out(p.theta, theta);
  out(p.a_src, as);
  out(p.a_dst, ad);
  std::memcpy(bias, p.bias.data(), sizeof(double) * h * k);
}

// One GCN layer fwd + bwd over a canonical normalized COO stored in `fmt`.
int ref_gcn_layer(int n, long long nnz, const int* r, const int* c, const double* v, int fmt,
                  const double* X, int m, const double* theta, const double* bias, int k,
                  int fwd, int bwd, int caching, const double* G, int fg, double* o,
                  double* dtheta, double* dbias, double* dinput) {
  try {
    AdjacencyOp<double> A(convert(SparseMatrix<double>{coo_of<double>(n, n, nnz, r, c, v)},
                                  static_cast<SparseFormat>(fmt)));
    GcnParams<double> p;
    p.theta = mat(theta, m, k);
    p.bias.assign(bias, bias + k);
    SchemeChoice s{static_cast<GcnForward>(fwd), static_cast<GcnBackward>(bwd), caching != 0};
    auto res = gcn_forward(mat(X, n, m), A, p, s);
    out(res.output, o);
    if (G) {
      auto g = gcn_backward(mat(G, n, k), A, p, res.cache, fg != 0);
      out(g.d_theta, dtheta);
      std::memcpy(dbias, g.d_bias.data(), sizeof(double) * k);
      if (fg && dinput) out(*g.d_input, dinput);
    }
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

// One GAT layer fwd + bwd over a CSR pattern (must hold all self loops).
// alpha/mask are written head-major h x q (pattern.hpp:99-141) when non-null.
int ref_gat_layer(int n, const int* rowptr, const int* cols, const double* X, int m,
                  const double* theta, const double* as, const double* ad, const double* bias,
                  int h, int k, double beta, int level, const double* G, int fg, double* o,
                  double* alpha, unsigned char* mask, double* dtheta, double* das, double* dad,
                  double* dbias, double* dinput) {
  try {
    auto pattern = SparsePattern::build(n, rowptr, cols);
    GatParams<double> p;
    p.heads = h;
    p.out_features = k;
    p.theta = mat(theta, m, h * k);
    p.a_src = mat(as, h, k);
    p.a_dst = mat(ad, h, k);
    p.bias.assign(bias, bias + h * k);
    auto res = gat_forward(mat(X, n, m), pattern, p, beta, static_cast<GatCacheLevel>(level));
    out(res.output, o);
    if (alpha || mask) {
      auto im = gat_recompute(pattern, p, res.cache, beta);
      out(im.alpha.vals, alpha);
      if (mask) std::memcpy(mask, im.mask.bits.data(), im.mask.bits.size());
    }
    if (G) {
      auto g = gat_backward(mat(G, n, h * k), pattern, p, res.cache, beta, fg != 0);
      out(g.d_theta, dtheta);
      out(g.d_a_src, das);
      out(g.d_a_dst, dad);
      std::memcpy(dbias, g.d_bias.data(), sizeof(double) * h * k);
      if (fg && dinput) out(*g.d_input, dinput);
    }
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

// One training step of Gcn2Model (kind 0) / Gat2Model (kind 1) in double on
// the workload of run_benchmark_typed (bench.hpp:160-219): graph from
// synthetic_graph(n, deg, seed), X seed+11, target seed+12, model seed+13.
// Writes the loss, the prediction and the gradients flattened in
// param_tensors() order (grad_vectors, model.hpp:109-115 / 220-228).
int ref_model_step(int kind, int n, double deg, unsigned long long seed, int m, int hidden,
                   int out_f, int heads, int policy, int caching, int level, int input_grad,
                   double* loss, double* pred, double* grads) {
  try {
    Graph g = synthetic_graph(n, deg, seed);
    ModelConfig mc;
    mc.kind = kind == 0 ? ModelKind::gcn2 : ModelKind::gat2;
    mc.in_features = m;
    mc.hidden = hidden;
    mc.out_features = out_f;
    mc.heads = heads;
    mc.scheme = static_cast<SchemePolicy>(policy);
    mc.caching = caching != 0;
    mc.gat_level = static_cast<GatCacheLevel>(level);
    mc.input_grad = input_grad != 0;
    auto X = DenseMatrix<double>::random_uniform(n, m, seed + 11);
    const index_t ow = kind == 0 ? out_f : heads * out_f;
    auto target = DenseMatrix<double>::random_uniform(n, ow, seed + 12);
    std::vector<std::vector<double>> gv;
    if (kind == 0) {
      Gcn2Model<double> model(mc, seed + 13);
      AdjacencyOp<double> adj(
          convert(gcn_normalize(SparseMatrix<double>{adjacency<double>(g)}), SparseFormat::csc));
      typename Gcn2Model<double>::Caches caches;
      auto o = model.forward(X, adj, caches);
      auto l = loss_mse(o, target);
      *loss = l.value;
      out(o, pred);
      gv = Gcn2Model<double>::grad_vectors(model.backward(l.grad, adj, caches));
    } else {
      Gat2Model<double> model(mc, seed + 13);
      auto csr = coo_to_csr(to_coo(add_self_loops(SparseMatrix<double>{adjacency<double>(g)})));
      auto pattern = SparsePattern::from_csr(csr);
      typename Gat2Model<double>::Caches caches;
      auto o = model.forward(X, pattern, caches);
      auto l = loss_mse(o, target);
      *loss = l.value;
      out(o, pred);
      gv = Gat2Model<double>::grad_vectors(model.backward(l.grad, pattern, caches));
    }
    std::size_t off = 0;
    for (const auto& v : gv) {
      std::memcpy(grads + off, v.data(), sizeof(double) * v.size());
      off += v.size();
    }
    return 0;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return -1;
  }
}

// ---------------------------------------------------------------------------
// CPU timing harness for bench.py (reference arm and cpu_baseline): builds the
// workload exactly like run_benchmark_typed (bench.hpp:160-219) -- X from
// seed+11, dX' from seed+12, params from seed+13 -- then times single steps.
// kind: 0 GCN layer fwd+bwd, 1 GAT layer fwd+bwd, 2/3 Gcn2/Gat2 training step
// (k = hidden, level packs the GAT level | out_features << 8). f32 timing.
// ---------------------------------------------------------------------------
struct RefBench {
  std::function<void()> step;
  long long q = 0;
  // owned state
  std::optional<AdjacencyOp<float>> adj;
  PatternPtr pattern;
  DenseMatrix<float> X, G;
  GcnParams<float> gp;
  GatParams<float> ap;
  std::optional<Gcn2Model<float>> gcn2;
  std::optional<Gat2Model<float>> gat2;
  DenseMatrix<float> target;
};

void* ref_bench_create(int kind, int n, double deg, unsigned long long seed, int m, int k,
                       int heads, int fg, int policy, int caching, int level, int fmt) {
  try {
    auto* b = new RefBench;
    Graph g = synthetic_graph(n, deg, seed);
    b->X = DenseMatrix<float>::random_uniform(n, m, seed + 11);
    if (kind == 0) {
      b->adj.emplace(convert(gcn_normalize(SparseMatrix<float>{adjacency<float>(g)}),
                             static_cast<SparseFormat>(fmt)));
      b->q = b->adj->nnz();
      b->G = DenseMatrix<float>::random_uniform(n, k, seed + 12);
      b->gp = GcnParams<float>::init(m, k, seed + 13);
      SchemeChoice s = resolve_scheme(static_cast<SchemePolicy>(policy), m, k, fg != 0,
                                      caching != 0);
      b->step = [b, s, fg] {
        auto r = gcn_forward(b->X, *b->adj, b->gp, s);
        auto gr = gcn_backward(b->G, *b->adj, b->gp, r.cache, fg != 0);
        (void)gr;
      };
    } else if (kind >= 2) {
      // 2-layer model training step (bench.hpp:193-219): m -> hidden (k) -> out,
      // MSE against random_uniform(seed + 12); kind 2 gcn2, kind 3 gat2 (heads)
      const int out_f = level >> 8;  // packed: level | out_features << 8
      ModelConfig mc;
      mc.kind = kind == 2 ? ModelKind::gcn2 : ModelKind::gat2;
      mc.in_features = m;
      mc.hidden = k;
      mc.out_features = out_f;
      mc.heads = heads;
      mc.scheme = static_cast<SchemePolicy>(policy);
      mc.caching = caching != 0;
      mc.gat_level = static_cast<GatCacheLevel>(level & 255);
      mc.input_grad = fg != 0;
      if (kind == 2) {
        b->adj.emplace(convert(gcn_normalize(SparseMatrix<float>{adjacency<float>(g)}),
                               static_cast<SparseFormat>(fmt)));
        b->q = b->adj->nnz();
        b->gcn2.emplace(mc, seed + 13);
        b->target = DenseMatrix<float>::random_uniform(n, out_f, seed + 12);
        b->step = [b] {
          typename Gcn2Model<float>::Caches caches;
          auto o = b->gcn2->forward(b->X, *b->adj, caches);
          auto l = loss_mse(o, b->target);
          auto gr = b->gcn2->backward(l.grad, *b->adj, caches);
          (void)gr;
        };
      } else {
        auto csr = coo_to_csr(to_coo(add_self_loops(SparseMatrix<float>{adjacency<float>(g)})));
        b->pattern = SparsePattern::from_csr(csr);
        b->q = b->pattern->nnz();
        b->gat2.emplace(mc, seed + 13);
        b->target = DenseMatrix<float>::random_uniform(n, heads * out_f, seed + 12);
        b->step = [b] {
          typename Gat2Model<float>::Caches caches;
          auto o = b->gat2->forward(b->X, b->pattern, caches);
          auto l = loss_mse(o, b->target);
          auto gr = b->gat2->backward(l.grad, b->pattern, caches);
          (void)gr;
        };
      }
    } else {
      auto csr = coo_to_csr(to_coo(add_self_loops(SparseMatrix<float>{adjacency<float>(g)})));
      b->pattern = SparsePattern::from_csr(csr);
      b->q = b->pattern->nnz();
      b->G = DenseMatrix<float>::random_uniform(n, heads * k, seed + 12);
      b->ap = GatParams<float>::init(m, heads, k, seed + 13);
      const auto lv = static_cast<GatCacheLevel>(level);
      b->step = [b, lv, fg] {
        auto r = gat_forward(b->X, b->pattern, b->ap, 0.2, lv);
        auto gr = gat_backward(b->G, b->pattern, b->ap, r.cache, 0.2, fg != 0);
        (void)gr;
      };
    }
    return b;
  } catch (const std::exception& ex) {
    g_err = ex.what();
    return nullptr;
  }
}
long long ref_bench_nnz(void* h) { return static_cast<RefBench*>(h)->q; }
double ref_bench_step(void* h) {
  auto t0 = std::chrono::steady_clock::now();
  static_cast<RefBench*>(h)->step();
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count();
}
void ref_bench_destroy(void* h) { delete static_cast<RefBench*>(h); }

}  // extern "C"
