// model.cu -- the two evaluation networks of the reference (model.hpp:16-245):
// Gcn2 = GCN -> ReLU -> GCN and Gat2 = GAT -> ELU(1) -> GAT, with the MSE loss
// (model.hpp loss_mse) and the activation kernels (dense.hpp:190-270), all on
// the device.  A model owns its parameters (initialised on the device with
// the reference's seeds: layer 2 from seed+101 / seed+201, model.hpp:46-49,
// 126-130); a training step is the benchmark's step (bench.hpp:193-219):
// forward, loss_mse against a target, backward, gradients in param_tensors()
// order (model.hpp:100-107, 208-218).
#include <cmath>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.cuh"

struct sgnn_model_s {
  sgnn_model_config cfg{};
  int dtype = SGNN_F32;
  std::vector<sgnn::DevBuf> params;  // param_tensors() order
  std::vector<int64_t> sizes;
  std::vector<std::string> names;
};

namespace sgnn {
namespace {

// activation (dense.hpp:197-228): out = f(x), mask = x > 0.  kind 0 relu, 2 elu
template <class T>
__global__ void k_act_fwd(int64_t n, int kind, T alpha, const T* __restrict__ x,
                          T* __restrict__ out, uint8_t* __restrict__ mask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T v = x[i];
    const bool pos = v > T(0);
    mask[i] = pos ? 1 : 0;
    out[i] = pos ? v : (kind == 0 ? T(0) : mul_rn(alpha, T(exp(v)) - T(1)));
  }
}

// activation_backward (dense.hpp:232-268): elu uses the saved forward output
template <class T>
__global__ void k_act_bwd(int64_t n, int kind, T alpha, const T* __restrict__ g,
                          const uint8_t* __restrict__ mask, const T* __restrict__ saved,
                          T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T gv = g[i];
    out[i] = mask[i] ? gv : (kind == 0 ? T(0) : mul_rn(saved[i] + alpha, gv));
  }
}

// loss_mse (model.hpp loss_mse): grad = S(2 d / size) with d in double, the
// loss = sum d^2 / size in double (block partials, fixed-order final sum)
template <class T>
__global__ void __launch_bounds__(256) k_mse(int64_t n, const T* __restrict__ out,
                                             const T* __restrict__ target, double inv,
                                             T* __restrict__ grad, double* __restrict__ part) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double d = (double)out[i] - (double)target[i];
    acc += d * d;
    grad[i] = (T)(2.0 * d * inv);
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void k_mse_final(int nb, const double* __restrict__ part, double inv,
                            double* __restrict__ loss) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) acc += part[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = sh[0] * inv;
}

template <class T>
void act_fwd(sgnn_ctx ctx, int kind, int64_t n, const T* x, T* out, uint8_t* mask) {
  k_act_fwd<T><<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(n, kind, T(1), x, out, mask);
  launched(ctx);
}
template <class T>
void act_bwd(sgnn_ctx ctx, int kind, int64_t n, const T* g, const uint8_t* mask, const T* saved,
             T* out) {
  k_act_bwd<T><<<grid_for(ctx, n, 256), 256, 0, ctx->stream>>>(n, kind, T(1), g, mask, saved,
                                                                out);
  launched(ctx);
}
// total: the element count of the whole prediction (row-partitioned callers
// hold a block of it); the loss written is the block's sum of squares / total
template <class T>
void mse(sgnn_ctx ctx, int64_t n, const T* out, const T* target, T* grad, double* loss,
         int64_t total = 0) {
  const int nb = grid_for(ctx, n > 0 ? n : 1, 256);
  DevBuf part((size_t)nb * sizeof(double), ctx->stream);
  const double inv = 1.0 / (double)(total > 0 ? total : n);
  k_mse<T><<<nb, 256, 0, ctx->stream>>>(n, out, target, inv, grad, part.as<double>());
  launched(ctx);
  k_mse_final<<<1, 256, 0, ctx->stream>>>(nb, part.as<double>(), inv, loss);
  launched(ctx);
}

// SGNN_NO_ACT_FUSION=1: run the activations as separate passes (tests compare
// the fused and unfused steps bit for bit); read per call so it can be toggled
inline bool act_fusion() {
  const char* e = getenv("SGNN_NO_ACT_FUSION");
  return !(e && e[0] == '1');
}

inline void ok(int rc) {
  if (rc == SGNN_OK) return;
  if (rc == SGNN_EINVAL) throw invalid_argument(sgnn_last_error());
  throw std::runtime_error(sgnn_last_error());
}

struct GcnCacheGuard {
  sgnn_gcn_cache c = nullptr;
  ~GcnCacheGuard() {
    if (c) sgnn_gcn_cache_destroy(c);
  }
};
struct GatCacheGuard {
  sgnn_gat_cache c = nullptr;
  ~GatCacheGuard() {
    if (c) sgnn_gat_cache_destroy(c);
  }
};

template <class T>
void gcn2_step(sgnn_ctx ctx, sgnn_model md, sgnn_adj A, const T* X, const T* target, T* out,
               void* const* grads, T* d_input, double* loss) {
  const auto& cf = md->cfg;
  const int32_t n = A->n_rows, m = cf.in_features, hid = cf.hidden, k = cf.out_features;
  cudaStream_t st = ctx->stream;
  sgnn_scheme s1, s2;
  ok(sgnn_resolve_scheme(cf.scheme_policy, m, hid, cf.input_grad, cf.caching, &s1));
  // the hidden layer always needs its input gradient (model.hpp:61-62)
  ok(sgnn_resolve_scheme(cf.scheme_policy, hid, k, 1, cf.caching, &s2));
  const T* th1 = md->params[0].as<T>();
  const T* b1 = md->params[1].as<T>();
  const T* th2 = md->params[2].as<T>();
  const T* b2 = md->params[3].as<T>();
  DevBuf h((size_t)n * hid * sizeof(T), st), mask((size_t)n * hid, st);
  DevBuf o2;
  if (!out) o2 = DevBuf((size_t)n * k * sizeof(T), st);
  T* o = out ? out : o2.as<T>();
  GcnCacheGuard c1, c2;
  // layer 1 with its ReLU (fused into the P.Theta / X.Theta epilogue when possible)
  ok(gcn_forward_relu(ctx, A, X, m, th1, b1, hid, &s1, h.get(), &c1.c, mask.as<uint8_t>()));
  ok(sgnn_gcn_forward(ctx, A, h.get(), hid, th2, b2, k, &s2, o, &c2.c));
  DevBuf g((size_t)n * k * sizeof(T), st), dl(sizeof(double), st);
  mse<T>(ctx, (int64_t)n * k, o, target, g.as<T>(), loss ? loss : dl.as<double>());
  DevBuf dh((size_t)n * hid * sizeof(T), st);
  // layer 2 backward with the ReLU backward applied to its input gradient
  ok(gcn_backward_relu(ctx, A, g.get(), th2, hid, k, c2.c, 1, grads[2], grads[3], dh.get(),
                       mask.as<uint8_t>()));
  ok(sgnn_gcn_backward(ctx, A, dh.get(), th1, m, hid, c1.c, cf.input_grad, grads[0], grads[1],
                       cf.input_grad ? d_input : nullptr));
}

template <class T>
void gat2_step(sgnn_ctx ctx, sgnn_model md, sgnn_pattern P, const T* X, const T* target, T* out,
               void* const* grads, T* d_input, double* loss) {
  const auto& cf = md->cfg;
  const int32_t n = P->n, m = cf.in_features, hd = cf.heads, hid = cf.hidden,
                k = cf.out_features;
  const int32_t w1 = hd * hid, w2 = hd * k;
  cudaStream_t st = ctx->stream;
  const double beta = cf.leaky_slope;
  auto prm = [&](int i) { return md->params[i].get(); };
  DevBuf h((size_t)n * w1 * sizeof(T), st), mask((size_t)n * w1, st);
  DevBuf o2;
  if (!out) o2 = DevBuf((size_t)n * w2 * sizeof(T), st);
  T* o = out ? out : o2.as<T>();
  GatCacheGuard c1, c2;
  // layer 1 with its ELU(1) fused into the aggregation epilogue when possible,
  // else applied in place: h is also the saved value the ELU backward needs
  bool fused = false;
  ok(gat_forward_elu(ctx, P, X, m, prm(0), prm(1), prm(2), prm(3), hd, hid, beta, cf.gat_level,
                     md->dtype, h.get(), &c1.c, act_fusion() ? mask.as<uint8_t>() : nullptr,
                     &fused, true));
  if (!fused) act_fwd<T>(ctx, 2, (int64_t)n * w1, h.as<T>(), h.as<T>(), mask.as<uint8_t>());
  // both layers may run operator-reordered (wide heads, k > m): the model
  // keeps its caches private, so only its outputs and gradients are visible
  ok(sgnn_gat_forward_ex(ctx, P, h.get(), w1, prm(4), prm(5), prm(6), prm(7), hd, k, beta,
                         cf.gat_level, md->dtype, o, &c2.c, SGNN_GAT_REORDER));
  DevBuf g((size_t)n * w2 * sizeof(T), st), dl(sizeof(double), st);
  mse<T>(ctx, (int64_t)n * w2, o, target, g.as<T>(), loss ? loss : dl.as<double>());
  DevBuf dh((size_t)n * w1 * sizeof(T), st);
  // layer 2 backward with the ELU backward fused into its d_input GEMM epilogue
  ok(gat_backward_elu(ctx, P, g.get(), prm(4), prm(5), prm(6), w1, hd, k, c2.c, 1, grads[4],
                      grads[5], grads[6], grads[7], dh.get(),
                      act_fusion() ? mask.as<uint8_t>() : nullptr, h.get(), &fused));
  if (!fused)
    act_bwd<T>(ctx, 2, (int64_t)n * w1, dh.as<T>(), mask.as<uint8_t>(), h.as<T>(), dh.as<T>());
  ok(sgnn_gat_backward(ctx, P, dh.get(), prm(0), prm(1), prm(2), m, hd, hid, beta, c1.c,
                       cf.input_grad, grads[0], grads[1], grads[2], grads[3],
                       cf.input_grad ? d_input : nullptr));
}

}  // namespace
}  // namespace sgnn

using namespace sgnn;

extern "C" {

int sgnn_model_create(sgnn_ctx ctx, const sgnn_model_config* cfg, uint64_t seed, int dtype,
                      sgnn_model* out) {
  SGNN_API_BEGIN
  require(ctx && cfg && out, "model: null argument");
  require(cfg->kind == 0 || cfg->kind == 1, "model: unknown kind");
  require(cfg->in_features >= 1 && cfg->hidden >= 1 && cfg->out_features >= 1,
          "model: feature sizes must be positive");
  require(cfg->kind == 0 || cfg->heads >= 1, "model: heads must be positive");
  const size_t sb = dtype_size(dtype);
  auto* md = new sgnn_model_s;
  md->cfg = *cfg;
  md->dtype = dtype;
  auto add = [&](const char* name, int64_t size) {
    md->params.emplace_back((size_t)size * sb, ctx->stream);
    md->sizes.push_back(size);
    md->names.push_back(name);
  };
  try {
    const int32_t m = cfg->in_features, hid = cfg->hidden, k = cfg->out_features;
    if (cfg->kind == 0) {  // Gcn2Model (model.hpp:43-49)
      add("l1.theta", (int64_t)m * hid);
      add("l1.bias", hid);
      add("l2.theta", (int64_t)hid * k);
      add("l2.bias", k);
      int rc = sgnn_gcn_params_init(ctx, m, hid, seed, dtype, md->params[0].get(),
                                    md->params[1].get());
      if (rc == SGNN_OK)
        rc = sgnn_gcn_params_init(ctx, hid, k, seed + 101, dtype, md->params[2].get(),
                                  md->params[3].get());
      ok(rc);
    } else {  // Gat2Model (model.hpp:123-130)
      const int32_t hd = cfg->heads;
      add("l1.theta", (int64_t)m * hd * hid);
      add("l1.a_src", (int64_t)hd * hid);
      add("l1.a_dst", (int64_t)hd * hid);
      add("l1.bias", (int64_t)hd * hid);
      add("l2.theta", (int64_t)hd * hid * hd * k);
      add("l2.a_src", (int64_t)hd * k);
      add("l2.a_dst", (int64_t)hd * k);
      add("l2.bias", (int64_t)hd * k);
      int rc = sgnn_gat_params_init(ctx, m, hd, hid, seed, dtype, md->params[0].get(),
                                    md->params[1].get(), md->params[2].get(),
                                    md->params[3].get());
      if (rc == SGNN_OK)
        rc = sgnn_gat_params_init(ctx, hd * hid, hd, k, seed + 201, dtype, md->params[4].get(),
                                  md->params[5].get(), md->params[6].get(),
                                  md->params[7].get());
      ok(rc);
    }
  } catch (...) {
    delete md;
    throw;
  }
  *out = md;
  SGNN_API_END
}

int sgnn_activation(sgnn_ctx ctx, int kind, int dtype, const void* x, int64_t count, void* out,
                    uint8_t* mask) {
  SGNN_API_BEGIN
  require(kind == 0 || kind == 2, "activation: relu (0) or elu (2)");
  if (count == 0) return SGNN_OK;
  if (dtype == SGNN_F32)
    act_fwd<float>(ctx, kind, count, (const float*)x, (float*)out, mask);
  else
    act_fwd<double>(ctx, kind, count, (const double*)x, (double*)out, mask);
  SGNN_API_END
}

int sgnn_activation_backward(sgnn_ctx ctx, int kind, int dtype, const void* grad_out,
                             const uint8_t* mask, const void* saved, int64_t count,
                             void* grad_in) {
  SGNN_API_BEGIN
  require(kind == 0 || kind == 2, "activation: relu (0) or elu (2)");
  require(kind != 2 || saved != nullptr,
          "activation_backward: elu requires the saved forward output");
  if (count == 0) return SGNN_OK;
  if (dtype == SGNN_F32)
    act_bwd<float>(ctx, kind, count, (const float*)grad_out, mask, (const float*)saved,
                   (float*)grad_in);
  else
    act_bwd<double>(ctx, kind, count, (const double*)grad_out, mask, (const double*)saved,
                    (double*)grad_in);
  SGNN_API_END
}

int sgnn_loss_mse(sgnn_ctx ctx, int dtype, const void* out, const void* target, int64_t count,
                  int64_t total, void* grad, double* loss) {
  SGNN_API_BEGIN
  require(count >= 0 && total >= count && total > 0, "loss_mse: target shape mismatch");
  if (dtype == SGNN_F32)
    mse<float>(ctx, count, (const float*)out, (const float*)target, (float*)grad, loss, total);
  else
    mse<double>(ctx, count, (const double*)out, (const double*)target, (double*)grad, loss,
                total);
  SGNN_API_END
}

int sgnn_model_destroy(sgnn_model md) {
  SGNN_API_BEGIN
  delete md;
  SGNN_API_END
}

int sgnn_model_num_params(sgnn_model md, int32_t* count) {
  SGNN_API_BEGIN
  require(md && count, "model: null argument");
  *count = (int32_t)md->params.size();
  SGNN_API_END
}

int sgnn_model_param(sgnn_model md, int32_t i, void** data, int64_t* size, const char** name) {
  SGNN_API_BEGIN
  require(md && i >= 0 && i < (int32_t)md->params.size(), "model: parameter index out of range");
  if (data) *data = md->params[i].get();
  if (size) *size = md->sizes[i];
  if (name) *name = md->names[i].c_str();
  SGNN_API_END
}

int sgnn_model_train_step(sgnn_ctx ctx, sgnn_model md, sgnn_adj adj, sgnn_pattern pattern,
                          const void* X, const void* target, void* out, void* const* grads,
                          void* d_input, double* loss) {
  SGNN_API_BEGIN
  require(ctx && md && X && target && grads, "model: null argument");
  require(!md->cfg.input_grad || d_input, "model: d_input required for input_grad");
  if (md->cfg.kind == 0) {
    require(adj != nullptr, "model: gcn2 needs an adjacency operator");
    require(adj->dtype == md->dtype, "model: dtype mismatch");
    if (md->dtype == SGNN_F32)
      gcn2_step<float>(ctx, md, adj, (const float*)X, (const float*)target, (float*)out, grads,
                       (float*)d_input, loss);
    else
      gcn2_step<double>(ctx, md, adj, (const double*)X, (const double*)target, (double*)out,
                        grads, (double*)d_input, loss);
  } else {
    require(pattern != nullptr, "model: gat2 needs a sparse pattern");
    if (md->dtype == SGNN_F32)
      gat2_step<float>(ctx, md, pattern, (const float*)X, (const float*)target, (float*)out,
                       grads, (float*)d_input, loss);
    else
      gat2_step<double>(ctx, md, pattern, (const double*)X, (const double*)target,
                        (double*)out, grads, (double*)d_input, loss);
  }
  SGNN_API_END
}

}  // extern "C"
