// common.cuh -- shared plumbing of libsgnn_cuda.so: error model, context,
// stream-ordered device buffers, launch accounting, warp helpers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <utility>
#include <stdexcept>
#include <string>

#include "../../include/sgnn_cuda.h"

namespace sgnn {

// require() throws invalid_argument exactly where the reference does
// (common.hpp:37-43); the C-ABI maps it to SGNN_EINVAL + message.
struct invalid_argument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void require(bool cond, const char* msg) {
  if (!cond) throw invalid_argument(msg);
}

#define SGNN_CUDA(call)                                                              \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      throw ::sgnn::cuda_error(std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

void set_last_error(const std::string& s);

// C-ABI wrapper: exceptions -> status codes
#define SGNN_API_BEGIN try {
#define SGNN_API_END                                \
  return SGNN_OK;                                   \
  }                                                 \
  catch (const ::sgnn::invalid_argument& e) {       \
    ::sgnn::set_last_error(e.what());               \
    return SGNN_EINVAL;                             \
  }                                                 \
  catch (const ::sgnn::cuda_error& e) {             \
    ::sgnn::set_last_error(e.what());               \
    return SGNN_ECUDA;                              \
  }                                                 \
  catch (const std::exception& e) {                 \
    ::sgnn::set_last_error(e.what());               \
    return SGNN_ERUNTIME;                           \
  }

struct Pipe;  // host-buffer step staging (pipeline.cu)

}  // namespace sgnn

struct sgnn_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  int64_t launches = 0;
  sgnn::Pipe* pipe = nullptr;  // lazily created copy streams + staging buffers
  // side stream for independent work inside one layer call (fork / join by
  // events; captured into CUDA graphs with the main stream)
  cudaStream_t aux = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  // tcgen05 GEMM B operand already split into tf32 hi / lo by the caller (on
  // the side stream, overlapped with earlier work): used by the next GEMM
  // whose contiguous B is `split_src` with `split_elems` elements
  const float* split_src = nullptr;
  int64_t split_elems = 0;
  const float* split_hi = nullptr;
  const float* split_lo = nullptr;
};

namespace sgnn {

// After every kernel launch: count it, surface launch errors immediately.
inline void launched(sgnn_ctx ctx) {
  ctx->launches++;
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) throw cuda_error(std::string("kernel launch: ") + cudaGetErrorString(e));
}

// Device memory accounting by class (memtrack.hpp:19-94 MemTracker on the
// device): live / peak / total bytes of the layer intermediates the reference
// classifies as transient, cache or output.  Buffers are charged with their
// LOGICAL size (what the reference's Array would hold: n x k scalars, 1-byte
// masks) when a layer tags them; kernel scratch (split-K partials, hub-row
// partials, sort temporaries) stays untracked like the reference's
// untracked class.  Process-wide and mutex-protected, like the reference's.
enum MemCls : int { kUntracked = 0, kTransient = 1, kCache = 2, kOutput = 3 };

class MemTrack {
 public:
  static MemTrack& get();
  void on_alloc(int c, size_t b);
  void on_free(int c, size_t b);
  void on_reclass(int from, int to, size_t b);
  void stats(int c, int64_t* live, int64_t* peak, int64_t* total);  // c == 4: all classes
  void reset_peaks();
};

// Independent work inside one layer call on the context's side stream.  The
// constructor forks (the side stream waits for the main stream's work so
// far); side() / main() switch ctx->stream, so launches and stream-ordered
// allocations go to that stream (the context is single-writer, so the swap is
// safe); join() -- also run by the destructor -- makes the main stream wait
// for the side stream.  Fork and join are events, so a captured step keeps
// the concurrency in its CUDA graph.  SGNN_NO_FORK=1 keeps everything on the
// main stream (same kernels, issue order).
class SideStream {
 public:
  explicit SideStream(sgnn_ctx ctx);
  ~SideStream() { join(); }
  void side() {
    if (active_) ctx_->stream = ctx_->aux;
  }
  void main() { ctx_->stream = main_; }
  void join();

 private:
  sgnn_ctx ctx_;
  cudaStream_t main_ = nullptr;
  bool active_ = false;
};

// Stream-ordered device buffer (cudaMallocAsync from the pooled default mem
// pool: transients cost no cudaMalloc/cudaFree round trips on the hot path).
class DevBuf {
 public:
  DevBuf() = default;
  DevBuf(size_t bytes, cudaStream_t s) : bytes_(bytes), stream_(s) {
    if (bytes_) SGNN_CUDA(cudaMallocAsync(&p_, bytes_, stream_));
  }
  ~DevBuf() { reset(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      p_ = o.p_;
      bytes_ = o.bytes_;
      stream_ = o.stream_;
      cls_ = o.cls_;
      charged_ = o.charged_;
      o.p_ = nullptr;
      o.bytes_ = 0;
      o.charged_ = 0;
    }
    return *this;
  }
  void reset() {
    if (charged_) MemTrack::get().on_free(cls_, charged_);
    charged_ = 0;
    if (p_) cudaFreeAsync(p_, stream_);
    p_ = nullptr;
    bytes_ = 0;
  }
  // charge `logical` bytes of this buffer to class `cls` (memory accounting)
  DevBuf& track(int cls, size_t logical) {
    if (charged_) MemTrack::get().on_free(cls_, charged_);
    cls_ = cls;
    charged_ = logical;
    if (charged_) MemTrack::get().on_alloc(cls_, charged_);
    return *this;
  }
  // ScopedMemClass / Array::reclassify (memtrack.hpp:176-181)
  void reclassify(int to) {
    if (charged_ && to != cls_) MemTrack::get().on_reclass(cls_, to, charged_);
    cls_ = to;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p_);
  }
  void* get() const { return p_; }
  size_t bytes() const { return bytes_; }
  void set_stream(cudaStream_t s) { stream_ = s; }

 private:
  void* p_ = nullptr;
  size_t bytes_ = 0;
  cudaStream_t stream_ = nullptr;
  int cls_ = kUntracked;
  size_t charged_ = 0;
};

inline size_t dtype_size(int dtype) {
  require(dtype == SGNN_F32 || dtype == SGNN_F64, "unknown dtype");
  return dtype == SGNN_F32 ? 4 : 8;
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Grid for grid-stride kernels: a multiple of the SM count.
inline int grid_for(sgnn_ctx ctx, int64_t work, int block, int per_sm = 8) {
  int64_t g = ceil_div(work, block);
  int64_t cap = (int64_t)ctx->num_sms * per_sm;
  if (g > cap) g = cap;
  return g < 1 ? 1 : (int)g;
}

// ---- device helpers --------------------------------------------------------
// Unfused multiply-add in the reference order (`acc += a * b` compiled without
// contraction, kernels.hpp:50): keeps SpMM/SDDMM bit-identical to the reference.
__device__ __forceinline__ float madd(float acc, float a, float b) {
  return __fadd_rn(acc, __fmul_rn(a, b));
}
__device__ __forceinline__ double madd(double acc, double a, double b) {
  return __dadd_rn(acc, __dmul_rn(a, b));
}
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }

template <class T>
struct Vec;  // 16-byte vector of T
template <>
struct Vec<float> {
  using type = float4;
  static constexpr int N = 4;
};
template <>
struct Vec<double> {
  using type = double2;
  static constexpr int N = 2;
};

}  // namespace sgnn
