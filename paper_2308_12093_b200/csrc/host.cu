// host.cu -- host-pure entry points: error state, context, the adaptive
// scheme selector and the analytic FLOP/byte model (cost.hpp), and the seeded
// synthetic graph generator (graph.hpp).  No device work here except the
// context's stream/pool setup.
#include <algorithm>
#include <mutex>
#include <unordered_set>
#include <vector>

#include "common.cuh"
#include "internal.cuh"

namespace sgnn {
static thread_local std::string g_last_error;
void set_last_error(const std::string& s) { g_last_error = s; }

// ---- device memory accounting (memtrack.hpp:19-94) --------------------------
namespace {
struct MemCat {
  int64_t live = 0, peak = 0, total = 0;
};
std::mutex g_mem_mu;
MemCat g_mem[4], g_mem_all;
}  // namespace

MemTrack& MemTrack::get() {
  static MemTrack t;
  return t;
}
void MemTrack::on_alloc(int c, size_t b) {
  std::lock_guard<std::mutex> lock(g_mem_mu);
  for (MemCat* k : {&g_mem[c], &g_mem_all}) {
    k->live += (int64_t)b;
    k->total += (int64_t)b;
    k->peak = std::max(k->peak, k->live);
  }
}
void MemTrack::on_free(int c, size_t b) {
  std::lock_guard<std::mutex> lock(g_mem_mu);
  g_mem[c].live -= (int64_t)b;
  g_mem_all.live -= (int64_t)b;
}
void MemTrack::on_reclass(int from, int to, size_t b) {
  std::lock_guard<std::mutex> lock(g_mem_mu);
  g_mem[from].live -= (int64_t)b;
  MemCat& k = g_mem[to];
  k.live += (int64_t)b;
  k.total += (int64_t)b;
  k.peak = std::max(k.peak, k.live);
}
void MemTrack::stats(int c, int64_t* live, int64_t* peak, int64_t* total) {
  std::lock_guard<std::mutex> lock(g_mem_mu);
  const MemCat& k = c == 4 ? g_mem_all : g_mem[c];
  if (live) *live = k.live;
  if (peak) *peak = k.peak;
  if (total) *total = k.total;
}
void MemTrack::reset_peaks() {  // peaks restart from the live level (memtrack.hpp:79-87)
  std::lock_guard<std::mutex> lock(g_mem_mu);
  for (MemCat* k : {&g_mem[0], &g_mem[1], &g_mem[2], &g_mem[3], &g_mem_all}) {
    k->peak = k->live;
    k->total = 0;
  }
}

SideStream::SideStream(sgnn_ctx ctx) : ctx_(ctx), main_(ctx->stream) {
  static const bool off = getenv("SGNN_NO_FORK") != nullptr;
  if (off) return;
  if (!ctx->aux) {
    SGNN_CUDA(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
    SGNN_CUDA(cudaEventCreateWithFlags(&ctx->fork_ev, cudaEventDisableTiming));
    SGNN_CUDA(cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
  }
  SGNN_CUDA(cudaEventRecord(ctx->fork_ev, main_));
  SGNN_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->fork_ev, 0));
  active_ = true;
}

void SideStream::join() {
  ctx_->stream = main_;
  if (!active_) return;
  active_ = false;
  cudaEventRecord(ctx_->join_ev, ctx_->aux);
  cudaStreamWaitEvent(main_, ctx_->join_ev, 0);
}
}  // namespace sgnn

using namespace sgnn;

extern "C" {

const char* sgnn_last_error(void) { return g_last_error.c_str(); }
const char* sgnn_version(void) { return "sgnn-b200 0.1 (sm_100a)"; }

int sgnn_mem_stats(int mem_class, int64_t* live, int64_t* peak, int64_t* total) {
  SGNN_API_BEGIN
  require(mem_class >= 0 && mem_class <= 4, "sgnn_mem_stats: class must be 0..4");
  MemTrack::get().stats(mem_class, live, peak, total);
  SGNN_API_END
}

int sgnn_mem_reset_peaks(void) {
  SGNN_API_BEGIN
  MemTrack::get().reset_peaks();
  SGNN_API_END
}

int sgnn_ctx_create(int device, void* stream, sgnn_ctx* out) {
  SGNN_API_BEGIN
  require(out != nullptr, "sgnn_ctx_create: null output");
  auto* c = new sgnn_ctx_s;
  c->device = device;
  SGNN_CUDA(cudaSetDevice(device));
  SGNN_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  // NULL is CUDA's default stream (torch's default stream reports handle 0),
  // so work stays ordered with the caller's allocations and copies.
  c->stream = static_cast<cudaStream_t>(stream);
  // Keep freed transients pooled: the stream-ordered allocator then never
  // returns memory to the driver between layer calls.
  cudaMemPool_t pool;
  SGNN_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = UINT64_MAX;
  SGNN_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  *out = c;
  SGNN_API_END
}

int sgnn_ctx_destroy(sgnn_ctx ctx) {
  SGNN_API_BEGIN
  if (!ctx) return SGNN_OK;
  if (ctx->aux) {
    cudaStreamSynchronize(ctx->aux);
    cudaStreamDestroy(ctx->aux);
    cudaEventDestroy(ctx->fork_ev);
    cudaEventDestroy(ctx->join_ev);
  }
  if (ctx->pipe) {
    cudaStreamSynchronize(ctx->stream);
    destroy_pipe(ctx);
  }
  if (ctx->own_stream) {
    cudaStreamSynchronize(ctx->stream);
    cudaStreamDestroy(ctx->stream);
  }
  delete ctx;
  SGNN_API_END
}

int sgnn_ctx_set_stream(sgnn_ctx ctx, void* stream) {
  SGNN_API_BEGIN
  require(ctx != nullptr, "sgnn_ctx_set_stream: null context");
  if (ctx->own_stream) {
    cudaStreamSynchronize(ctx->stream);
    cudaStreamDestroy(ctx->stream);
    ctx->own_stream = false;
  }
  ctx->stream = static_cast<cudaStream_t>(stream);
  SGNN_API_END
}

int sgnn_ctx_synchronize(sgnn_ctx ctx) {
  SGNN_API_BEGIN
  SGNN_CUDA(cudaStreamSynchronize(ctx->stream));
  SGNN_API_END
}

int sgnn_ctx_launch_count(sgnn_ctx ctx, int64_t* out) {
  SGNN_API_BEGIN
  *out = ctx->launches;
  SGNN_API_END
}

// ---------------------------------------------------------------------------
// cost.hpp:199-223 gcn_select_scheme -- argmin of the FLOP model with ties to
// the propagate/split side; must make the reference's choice bit for bit.
// ---------------------------------------------------------------------------
int sgnn_gcn_select_scheme(int64_t m, int64_t k, int fg, int caching, sgnn_scheme* out) {
  SGNN_API_BEGIN
  require(m >= 1 && k >= 1, "gcn_select_scheme: m and k must be >= 1");
  sgnn_scheme c{};
  if (!caching) {
    c.forward = k < m ? SGNN_TRANSFORM_FIRST : SGNN_PROPAGATE_FIRST;
    const bool fused = fg ? (k < 2 * m) : (k < m);
    c.backward = fused ? SGNN_FUSED_PROPAGATE : SGNN_SPLIT_PROPAGATE;
    c.caching = 0;
  } else {
    const bool transform = fg ? (k < m) : (2 * k < m);
    if (transform) {
      c.forward = SGNN_TRANSFORM_FIRST;
      c.backward = SGNN_FUSED_PROPAGATE;
      c.caching = 0;
    } else {
      c.forward = SGNN_PROPAGATE_FIRST_CACHED;
      c.backward = SGNN_SPLIT_PROPAGATE_CACHED;
      c.caching = 1;
    }
  }
  *out = c;
  SGNN_API_END
}

// gcn.hpp:34-47 resolve_scheme
int sgnn_resolve_scheme(int policy, int64_t m, int64_t k, int fg, int caching,
                        sgnn_scheme* out) {
  if (policy == SGNN_POLICY_ADAPTIVE) return sgnn_gcn_select_scheme(m, k, fg, caching, out);
  SGNN_API_BEGIN
  if (policy == SGNN_POLICY_TRANSFORM_FIRST) {
    *out = {SGNN_TRANSFORM_FIRST, SGNN_FUSED_PROPAGATE, 0};
  } else if (policy == SGNN_POLICY_PROPAGATE_FIRST) {
    *out = caching ? sgnn_scheme{SGNN_PROPAGATE_FIRST_CACHED, SGNN_SPLIT_PROPAGATE_CACHED, 1}
                   : sgnn_scheme{SGNN_PROPAGATE_FIRST, SGNN_SPLIT_PROPAGATE, 0};
  } else {
    throw invalid_argument("unknown scheme");
  }
  SGNN_API_END
}

int64_t sgnn_gcn_forward_flops(int s, int64_t n, int64_t m, int64_t k, int64_t q) {
  return s == SGNN_TRANSFORM_FIRST ? 2 * (n * m * k + q * k) : 2 * (n * m * k + q * m);
}
int64_t sgnn_gcn_backward_flops(int s, int64_t n, int64_t m, int64_t k, int64_t q, int fg) {
  switch (s) {
    case SGNN_FUSED_PROPAGATE: return 2 * q * k + 2 * n * m * k + (fg ? 2 * n * m * k : 0);
    case SGNN_SPLIT_PROPAGATE:
      return 2 * q * m + 2 * n * m * k + (fg ? 2 * n * m * k + 2 * q * m : 0);
    case SGNN_SPLIT_PROPAGATE_CACHED: return 2 * n * m * k + (fg ? 2 * n * m * k + 2 * q * m : 0);
  }
  return 0;
}
int64_t sgnn_gcn_forward_transients(int s, int64_t n, int64_t m, int64_t k) {
  return s == SGNN_TRANSFORM_FIRST ? n * k : n * m;
}
int64_t sgnn_gcn_backward_transients(int s, int64_t n, int64_t m, int64_t k, int fg) {
  switch (s) {
    case SGNN_FUSED_PROPAGATE: return n * k;
    case SGNN_SPLIT_PROPAGATE: return fg ? 2 * n * m : n * m;
    case SGNN_SPLIT_PROPAGATE_CACHED: return fg ? n * m : 0;
  }
  return 0;
}

static int64_t sparse_bytes(int fmt, int64_t n, int64_t q, int64_t p, int64_t sb, int64_t ib) {
  switch (fmt) {  // cost.hpp:44-60
    case SGNN_CSR:
    case SGNN_CSC: return ib * (q + n + 1) + sb * q;
    case SGNN_COO: return ib * 2 * q + sb * q;
    case SGNN_ELLPACK:
      require(p > 0, "cost: ELLPACK width p is required");
      return (ib + sb) * n * p;
    case SGNN_HYBRID:
      throw invalid_argument("cost: hybrid needs the per-part split, use the *_hybrid overload");
  }
  throw invalid_argument("unknown format");
}

int sgnn_spmm_cost(int fmt, int64_t n, int64_t q, int64_t p, int64_t f, int64_t sb, int64_t ib,
                   int64_t* flops, int64_t* bytes, double* oi) {
  SGNN_API_BEGIN
  const int64_t fl = 2 * q * f;
  const int64_t by = sparse_bytes(fmt, n, q, p, sb, ib) + 3 * sb * n * f;
  *flops = fl;
  *bytes = by;
  *oi = by > 0 ? (double)fl / (double)by : 0.0;
  SGNN_API_END
}

int sgnn_sddmm_cost(int fmt, int64_t n, int64_t q, int64_t p, int64_t f, int64_t sb,
                    int64_t ib, int64_t* flops, int64_t* bytes, double* oi) {
  SGNN_API_BEGIN
  const int64_t fl = q * (2 * f + 1);
  int64_t by = sb * q * f;  // cost.hpp:81-101
  switch (fmt) {
    case SGNN_CSR:
    case SGNN_CSC: by += ib * (q + n + 1) + 2 * sb * q; break;
    case SGNN_COO: by += ib * 2 * q + 2 * sb * q; break;
    case SGNN_ELLPACK:
      require(p > 0, "cost: ELLPACK width p is required");
      by += ib * n * p + 2 * sb * q;
      break;
    case SGNN_HYBRID:
      throw invalid_argument("cost: hybrid needs the per-part split, use the *_hybrid overload");
    default: throw invalid_argument("unknown format");
  }
  *flops = fl;
  *bytes = by;
  *oi = by > 0 ? (double)fl / (double)by : 0.0;
  SGNN_API_END
}

int64_t sgnn_gat_cache_footprint(int level, int64_t n, int64_t h, int64_t k, int64_t q,
                                 int64_t sb) {
  switch (level) {  // cost.hpp:243-252
    case SGNN_GAT_NONE: return 0;
    case SGNN_GAT_FEATURES: return sb * n * h * k;
    case SGNN_GAT_NODE_ATTENTION: return sb * n * h * (k + 2);
    case SGNN_GAT_FULL: return sb * n * h * k + (sb + 1) * q * h;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// graph.hpp:160-190 synthetic_graph: sequential rejection sampler over the
// splitmix64 stream (inherently serial -- stays on the host), then the
// canonical (src, dst) order of dedup_edges (graph.hpp:42-55).
// ---------------------------------------------------------------------------
namespace {
struct HostRng {
  uint64_t s;
  explicit HostRng(uint64_t seed) : s(seed + 0x9E3779B97F4A7C15ull) {}
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  uint64_t below(uint64_t bound) {
    if (bound <= 1) return 0;
    const uint64_t limit = bound * ((~uint64_t{0}) / bound);
    uint64_t x = next();
    while (x >= limit) x = next();
    return x % bound;
  }
};
}  // namespace

int64_t sgnn_synthetic_graph_edges(int32_t n, double avg_degree) {
  return 2 * (int64_t)(uint64_t)(avg_degree * (double)n / 2.0 + 0.5);
}

int sgnn_synthetic_graph(int32_t n, double avg_degree, uint64_t seed, int32_t* src,
                         int32_t* dst) {
  SGNN_API_BEGIN
  require(n >= 1, "synthetic_graph: n must be >= 1");
  require(avg_degree >= 0, "synthetic_graph: avg_degree must be >= 0");
  require(avg_degree < (double)n, "synthetic_graph: avg_degree must be < n");
  const uint64_t target = (uint64_t)(avg_degree * (double)n / 2.0 + 0.5);
  if (target == 0) return SGNN_OK;
  std::unordered_set<uint64_t> used;
  used.reserve(target * 2);
  std::vector<uint64_t> keys;
  keys.reserve(target * 2);
  HostRng rng(seed);
  while (used.size() < target) {
    const int32_t a = (int32_t)rng.below((uint64_t)n);
    const int32_t b = (int32_t)rng.below((uint64_t)n);
    if (a == b) continue;
    const int32_t lo = std::min(a, b), hi = std::max(a, b);
    const uint64_t key = ((uint64_t)lo << 32) | (uint32_t)hi;
    if (!used.insert(key).second) continue;
    keys.push_back(key);
    keys.push_back(((uint64_t)hi << 32) | (uint32_t)lo);
  }
  std::sort(keys.begin(), keys.end());
  for (size_t i = 0; i < keys.size(); ++i) {
    src[i] = (int32_t)(keys[i] >> 32);
    dst[i] = (int32_t)(keys[i] & 0xffffffffu);
  }
  SGNN_API_END
}

}  // extern "C"
