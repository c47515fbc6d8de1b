// pipeline.cu -- host-buffer layer steps: the reference's API takes and
// returns host matrices (gcn.hpp:91-193, gat.hpp:89-219 on DenseMatrix), and
// its benchmark step is forward + backward with a given output gradient
// (bench.hpp:193-219).  These entry points run that step from HOST buffers
// with the PCIe transfers overlapped with compute and with each other:
//
//   h2d stream : X ----------> dX' ------------------>
//   compute    :      [fwd] ............ [bwd]
//   d2h stream :           out ---------------> grads, dX
//
// The output of the forward travels device->host while the output gradient
// travels host->device (PCIe is full duplex), so a step costs about
// |X| + max(|dX'|, |out|) + |dX| of link time instead of the sum of all four.
// Device staging buffers live in the context (grown on demand, reused), all
// work is ordered after prior work on the context stream and the context
// stream waits for the last copy, so the call is stream-ordered like every
// other entry point.
#include "common.cuh"
#include "internal.cuh"

namespace sgnn {

Pipe::~Pipe() {
  for (auto& p : ws)
    if (p) cudaFree(p);
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  if (h2d) cudaStreamDestroy(h2d);
  if (d2h) cudaStreamDestroy(d2h);
}

void* Pipe::buf(int slot, size_t bytes) {
  if (cap[slot] < bytes) {
    if (ws[slot]) {
      SGNN_CUDA(cudaDeviceSynchronize());  // growth only: in-flight users may hold it
      SGNN_CUDA(cudaFree(ws[slot]));
      ws[slot] = nullptr;
    }
    SGNN_CUDA(cudaMalloc(&ws[slot], bytes));
    cap[slot] = bytes;
  }
  return ws[slot];
}

Pipe& pipe(sgnn_ctx ctx) {
  if (!ctx->pipe) {
    auto* p = new Pipe;
    SGNN_CUDA(cudaStreamCreateWithFlags(&p->h2d, cudaStreamNonBlocking));
    SGNN_CUDA(cudaStreamCreateWithFlags(&p->d2h, cudaStreamNonBlocking));
    for (auto& e : p->ev) SGNN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->pipe = p;
  }
  return *ctx->pipe;
}

void destroy_pipe(sgnn_ctx ctx) {
  delete ctx->pipe;
  ctx->pipe = nullptr;
}

}  // namespace sgnn

using namespace sgnn;

namespace {

enum { EV_START, EV_X, EV_G, EV_OUT, EV_BWD, EV_DONE };

struct Fence {  // orders the copy streams after prior work on the context stream
  Fence(sgnn_ctx ctx, Pipe& p) {
    SGNN_CUDA(cudaEventRecord(p.ev[EV_START], ctx->stream));
    SGNN_CUDA(cudaStreamWaitEvent(p.h2d, p.ev[EV_START], 0));
    SGNN_CUDA(cudaStreamWaitEvent(p.d2h, p.ev[EV_START], 0));
  }
};

void h2d(Pipe& p, void* dst, const void* src, size_t bytes) {
  if (bytes) SGNN_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, p.h2d));
}
void d2h(Pipe& p, void* dst, const void* src, size_t bytes) {
  if (bytes && dst) SGNN_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, p.d2h));
}

}  // namespace

extern "C" {

int sgnn_gcn_step_host(sgnn_ctx ctx, sgnn_adj A, const void* hX, int32_t m, const void* theta,
                       const void* bias, int32_t k, const sgnn_scheme* scheme, const void* hG,
                       int needs_feature_grad, void* h_out, void* h_d_theta, void* h_d_bias,
                       void* h_d_input) {
  SGNN_API_BEGIN
  require(ctx && A && scheme && hX && hG, "gcn_step_host: null argument");
  require(m >= 1 && k >= 1, "gcn_forward: input width does not match theta");
  const size_t sb = dtype_size(A->dtype);
  const size_t n = (size_t)A->n_rows;
  const bool fg = needs_feature_grad != 0;
  require(!fg || h_d_input != nullptr, "gcn_backward: d_input required for feature gradients");
  Pipe& p = pipe(ctx);
  void* X = p.buf(0, n * m * sb);
  void* G = p.buf(1, n * k * sb);
  void* out = p.buf(2, n * k * sb);
  void* dth = p.buf(3, (size_t)m * k * sb);
  void* db = p.buf(4, (size_t)k * sb);
  void* dx = fg ? p.buf(5, n * m * sb) : nullptr;
  Fence f(ctx, p);
  h2d(p, X, hX, n * m * sb);
  SGNN_CUDA(cudaEventRecord(p.ev[EV_X], p.h2d));
  h2d(p, G, hG, n * k * sb);
  SGNN_CUDA(cudaEventRecord(p.ev[EV_G], p.h2d));

  SGNN_CUDA(cudaStreamWaitEvent(ctx->stream, p.ev[EV_X], 0));
  sgnn_gcn_cache cache = nullptr;
  int rc = sgnn_gcn_forward(ctx, A, X, m, theta, bias, k, scheme, out, &cache);
  if (rc != SGNN_OK) return rc;
  SGNN_CUDA(cudaEventRecord(p.ev[EV_OUT], ctx->stream));
  SGNN_CUDA(cudaStreamWaitEvent(p.d2h, p.ev[EV_OUT], 0));
  d2h(p, h_out, out, n * k * sb);

  SGNN_CUDA(cudaStreamWaitEvent(ctx->stream, p.ev[EV_G], 0));
  rc = sgnn_gcn_backward(ctx, A, G, theta, m, k, cache, fg ? 1 : 0, dth, db, dx);
  sgnn_gcn_cache_destroy(cache);
  if (rc != SGNN_OK) return rc;
  SGNN_CUDA(cudaEventRecord(p.ev[EV_BWD], ctx->stream));
  SGNN_CUDA(cudaStreamWaitEvent(p.d2h, p.ev[EV_BWD], 0));
  d2h(p, h_d_theta, dth, (size_t)m * k * sb);
  d2h(p, h_d_bias, db, (size_t)k * sb);
  if (fg) d2h(p, h_d_input, dx, n * m * sb);
  SGNN_CUDA(cudaEventRecord(p.ev[EV_DONE], p.d2h));
  SGNN_CUDA(cudaStreamWaitEvent(ctx->stream, p.ev[EV_DONE], 0));
  SGNN_API_END
}

int sgnn_gat_step_host(sgnn_ctx ctx, sgnn_pattern P, const void* hX, int32_t m,
                       const void* theta, const void* a_src, const void* a_dst, const void* bias,
                       int32_t heads, int32_t k, double beta, int level, int dtype,
                       const void* hG, int needs_feature_grad, void* h_out, void* h_d_theta,
                       void* h_d_a_src, void* h_d_a_dst, void* h_d_bias, void* h_d_input) {
  SGNN_API_BEGIN
  require(ctx && P && hX && hG, "gat_step_host: null argument");
  require(m >= 1 && heads >= 1 && k >= 1, "gat_forward: input width does not match theta");
  require(!needs_feature_grad || h_d_input != nullptr,
          "gat_backward: d_input required for feature gradients");
  const size_t sb = dtype_size(dtype);
  const size_t n = (size_t)P->n, hk = (size_t)heads * k;
  const bool fg = needs_feature_grad != 0;
  Pipe& p = pipe(ctx);
  void* X = p.buf(0, n * m * sb);
  void* G = p.buf(1, n * hk * sb);
  void* out = p.buf(2, n * hk * sb);
  void* dth = p.buf(3, (size_t)m * hk * sb + 3 * hk * sb);
  char* small = static_cast<char*>(dth) + (size_t)m * hk * sb;  // d_a_src | d_a_dst | d_bias
  void* dx = fg ? p.buf(5, n * m * sb) : nullptr;
  Fence f(ctx, p);
  h2d(p, X, hX, n * m * sb);
  SGNN_CUDA(cudaEventRecord(p.ev[EV_X], p.h2d));
  h2d(p, G, hG, n * hk * sb);
  SGNN_CUDA(cudaEventRecord(p.ev[EV_G], p.h2d));

  SGNN_CUDA(cudaStreamWaitEvent(ctx->stream, p.ev[EV_X], 0));
  sgnn_gat_cache cache = nullptr;
  int rc = sgnn_gat_forward(ctx, P, X, m, theta, a_src, a_dst, bias, heads, k, beta, level,
                            dtype, out, &cache);
  if (rc != SGNN_OK) return rc;
  SGNN_CUDA(cudaEventRecord(p.ev[EV_OUT], ctx->stream));
  SGNN_CUDA(cudaStreamWaitEvent(p.d2h, p.ev[EV_OUT], 0));
  d2h(p, h_out, out, n * hk * sb);

  SGNN_CUDA(cudaStreamWaitEvent(ctx->stream, p.ev[EV_G], 0));
  rc = sgnn_gat_backward(ctx, P, G, theta, a_src, a_dst, m, heads, k, beta, cache, fg ? 1 : 0,
                         dth, small, small + hk * sb, small + 2 * hk * sb, dx);
  sgnn_gat_cache_destroy(cache);
  if (rc != SGNN_OK) return rc;
  SGNN_CUDA(cudaEventRecord(p.ev[EV_BWD], ctx->stream));
  SGNN_CUDA(cudaStreamWaitEvent(p.d2h, p.ev[EV_BWD], 0));
  d2h(p, h_d_theta, dth, (size_t)m * hk * sb);
  d2h(p, h_d_a_src, small, hk * sb);
  d2h(p, h_d_a_dst, small + hk * sb, hk * sb);
  d2h(p, h_d_bias, small + 2 * hk * sb, hk * sb);
  if (fg) d2h(p, h_d_input, dx, n * m * sb);
  SGNN_CUDA(cudaEventRecord(p.ev[EV_DONE], p.d2h));
  SGNN_CUDA(cudaStreamWaitEvent(ctx->stream, p.ev[EV_DONE], 0));
  SGNN_API_END
}

}  // extern "C"
