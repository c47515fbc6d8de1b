#pragma once

// B200 runtime glue of the drop-in layer headers (include/dropin/sgnn/gcn.hpp,
// gat.hpp): the reference's C++ layer API (namespace sgnn, its host types
// DenseMatrix / AdjacencyOp / SparsePattern from the caller's own sgnn
// headers) executed by libsgnn_cuda.so through the C-ABI (include/sgnn_cuda.h).
//
//  * errors: a failing C-ABI call rethrows the reference's exception type with
//    the same message (SGNN_EINVAL -> std::invalid_argument, common.hpp:37-43;
//    anything else -> std::runtime_error);
//  * one process-wide sgnn_ctx on device $SGNN_DEVICE (default 0), legacy
//    default stream: every facade call is synchronous like the reference's;
//  * memory accounting: the device engine's transient peak of each call is
//    replayed into the caller's MemTracker (memtrack.hpp:19-94), so the
//    reference's instrumented-peak checks see the device's intermediates;
//  * operation counters: the analytic costs the reference charges per kernel
//    (counters.hpp, kernels.hpp / dense.hpp charge sites) are charged for the
//    work the device performs.
//
// Build with -I include/dropin -I include ahead of the reference's include
// directory and link libsgnn_cuda.so; the replacement headers shadow only
// sgnn/gcn.hpp and sgnn/gat.hpp.

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sgnn/common.hpp"
#include "sgnn/counters.hpp"
#include "sgnn/dense.hpp"
#include "sgnn/memtrack.hpp"
#include "sgnn_cuda.h"

namespace sgnn::b200 {

inline void check(int status) {
  if (status == SGNN_OK) return;
  const std::string msg = sgnn_last_error();
  if (status == SGNN_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

inline sgnn_ctx ctx() {
  static const std::unique_ptr<sgnn_ctx_s, int (*)(sgnn_ctx)> c = [] {
    const char* env = std::getenv("SGNN_DEVICE");
    sgnn_ctx h = nullptr;
    check(sgnn_ctx_create(env ? std::atoi(env) : 0, nullptr, &h));
    return std::unique_ptr<sgnn_ctx_s, int (*)(sgnn_ctx)>(h, sgnn_ctx_destroy);
  }();
  return c.get();
}

template <class S>
constexpr int dtype() {
  static_assert(sizeof(S) == 4 || sizeof(S) == 8, "float or double");
  return sizeof(S) == 4 ? SGNN_F32 : SGNN_F64;
}

// owning device buffer
class Buf {
 public:
  Buf() = default;
  explicit Buf(std::size_t bytes) : bytes_(bytes) {
    if (bytes_) cuda_check(cudaMalloc(&p_, bytes_), "cudaMalloc");
  }
  ~Buf() {
    if (p_) cudaFree(p_);
  }
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  void* get() const { return p_; }
  template <class T>
  T* as() const {
    return static_cast<T*>(p_);
  }
  std::size_t bytes() const { return bytes_; }

 private:
  void* p_ = nullptr;
  std::size_t bytes_ = 0;
};
using BufPtr = std::shared_ptr<Buf>;

template <class T>
BufPtr upload(const T* host, std::size_t n) {
  auto b = std::make_shared<Buf>(n * sizeof(T));
  if (n) cuda_check(cudaMemcpy(b->get(), host, n * sizeof(T), cudaMemcpyHostToDevice), "H2D");
  return b;
}
template <class S>
BufPtr upload(const DenseMatrix<S>& m) {
  return upload(m.data(), m.size());
}
template <class T>
void download(const void* dev, T* host, std::size_t n) {
  if (n) cuda_check(cudaMemcpy(host, dev, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
}
template <class S>
DenseMatrix<S> download_matrix(const void* dev, index_t rows, index_t cols) {
  DenseMatrix<S> m(rows, cols);
  download(dev, m.mutable_data(), m.size());
  return m;
}
inline void sync() { check(sgnn_ctx_synchronize(ctx())); }

// Device transient peak of one facade call -> the caller's MemTracker: the
// reference's tracker then sees the same peak as if the intermediates were
// its own Arrays (on_alloc + on_free of the peak raise the transient peak by
// exactly that amount and leave the live count unchanged).
class TransientMirror {
 public:
  TransientMirror() {
    check(sgnn_mem_stats(SGNN_MEM_TRANSIENT, &live0_, nullptr, nullptr));
    check(sgnn_mem_reset_peaks());
  }
  void replay() {
    sync();
    int64_t peak = 0;
    check(sgnn_mem_stats(SGNN_MEM_TRANSIENT, nullptr, &peak, nullptr));
    const int64_t extra = peak - live0_;
    if (extra > 0) {
      MemTracker::instance().on_alloc(MemClass::transient, static_cast<std::size_t>(extra));
      MemTracker::instance().on_free(MemClass::transient, static_cast<std::size_t>(extra));
    }
  }

 private:
  int64_t live0_ = 0;
};

}  // namespace sgnn::b200
