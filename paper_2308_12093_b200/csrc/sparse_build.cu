// sparse_build.cu -- the sparse-format layer on the device (north-star
// subsystem 1): canonical COO (stable sort + keep-last dedup), CSR/CSC build,
// self loops, symmetric degree normalization, SparsePattern, AdjacencyOp.
// Every output is bit-identical to the reference's host code
// (sparse.hpp:110-218,457-495; pattern.hpp:19-59): CUB's LSD radix sort is
// stable, so equal keys keep input order exactly like std::stable_sort and the
// counting sorts of the reference.
#include <cub/cub.cuh>

#include "common.cuh"
#include "internal.cuh"

namespace sgnn {

static int bits_for(uint64_t maxval) {
  int b = 0;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b < 1 ? 1 : b;
}

// ---- kernels ---------------------------------------------------------------
__global__ void k_range_keys(int64_t nnz, const int32_t* rows, const int32_t* cols, int32_t nr,
                             int32_t nc, uint64_t* keys, int32_t* idx, int* bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = rows[e], c = cols[e];
    if (r < 0 || r >= nr || c < 0 || c >= nc) {
      *bad = 1;
      keys[e] = 0;
    } else {
      keys[e] = (uint64_t)r * (uint64_t)nc + (uint64_t)c;
    }
    idx[e] = (int32_t)e;
  }
}

__global__ void k_last_of_run(int64_t nnz, const uint64_t* keys, int32_t* flag) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    flag[e] = (e == nnz - 1 || keys[e] != keys[e + 1]) ? 1 : 0;
}

template <class T>
__global__ void k_scatter_kept(int64_t nnz, const int32_t* flag, const int32_t* pos,
                               const int32_t* idx, const int32_t* rows, const int32_t* cols,
                               const T* vals, int32_t* orow, int32_t* ocol, T* oval) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[e]) continue;
    const int32_t src = idx[e];  // last occurrence of the key (stable sort)
    const int32_t at = pos[e];
    orow[at] = rows[src];
    ocol[at] = cols[src];
    if (vals) oval[at] = vals[src];
  }
}

// ptr[r] = first e with sorted_ids[e] >= r, for r in [0, n]
__global__ void k_ptr_from_sorted(int64_t nnz, const int32_t* ids, int32_t n, int32_t* ptr) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e <= nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t prev = e == 0 ? -1 : ids[e - 1];
    const int32_t cur = e == nnz ? n : ids[e];
    for (int32_t r = prev + 1; r <= cur; ++r) ptr[r] = (int32_t)e;
  }
}

template <class T>
__global__ void k_gather_csc(int64_t nnz, const int32_t* perm, const int32_t* rows,
                             const T* vals, int32_t* orows, T* ovals) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e = perm[p];
    if (orows) orows[p] = rows[e];
    if (ovals) ovals[p] = vals[e];
  }
}

__global__ void k_iota(int64_t n, int32_t* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] = (int32_t)e;
}

__global__ void k_row_ids(int32_t n, const int32_t* rowptr, int32_t* rid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) rid[e] = (int32_t)i;
}

// diagonal position of row i (first e with col == i), pattern.hpp:46-57
__device__ __forceinline__ int32_t find_diag(const int32_t* rowptr, const int32_t* cols,
                                             int32_t i) {
  int32_t lo = rowptr[i], hi = rowptr[i + 1];
  while (lo < hi) {  // columns ascend within a canonical row
    const int32_t mid = (lo + hi) >> 1;
    if (cols[mid] < i) lo = mid + 1;
    else hi = mid;
  }
  return (lo < rowptr[i + 1] && cols[lo] == i) ? lo : -1;
}

__global__ void k_diag(int32_t n, const int32_t* rowptr, const int32_t* cols, int32_t* diag,
                       int32_t* missing) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d = find_diag(rowptr, cols, (int32_t)i);
    if (diag) diag[i] = d;
    missing[i] = d < 0 ? 1 : 0;
  }
}

// new row length = old + missing diagonal
__global__ void k_loop_lengths(int32_t n, const int32_t* rowptr, const int32_t* missing,
                               int32_t* len) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    len[i] = rowptr[i + 1] - rowptr[i] + missing[i];
}

// sparse.hpp:457-472: insert (i,i,1) in canonical position where missing
template <class T>
__global__ void k_insert_loops(int32_t n, const int32_t* rowptr, const int32_t* cols,
                               const T* vals, const int32_t* missing, const int32_t* newptr,
                               int32_t* orow, int32_t* ocol, T* oval) {
  for (int64_t ii = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ii < n;
       ii += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = (int32_t)ii;
    int32_t w = newptr[i];
    int32_t e = rowptr[i];
    const int32_t end = rowptr[i + 1];
    for (; e < end && cols[e] < i; ++e, ++w) {
      orow[w] = i; ocol[w] = cols[e]; oval[w] = vals[e];
    }
    if (missing[i]) {
      orow[w] = i; ocol[w] = i; oval[w] = T(1); ++w;
    }
    for (; e < end; ++e, ++w) {
      orow[w] = i; ocol[w] = cols[e]; oval[w] = vals[e];
    }
  }
}

// sparse.hpp:479-484: deg_i = sum over row i of A+I in double, canonical order
template <class T>
__global__ void k_degrees(int32_t n, const int32_t* rowptr, const T* vals, double* deg,
                          int* negative) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double d = 0.0;
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {
      const T v = vals[e];
      if (v < T(0)) *negative = 1;
      d = __dadd_rn(d, (double)v);
    }
    deg[i] = d;
  }
}

// sparse.hpp:486-491: v <- S(double(v) / sqrt(d_i * d_j)), IEEE-rounded ops
template <class T>
__global__ void k_normalize(int64_t q, const int32_t* rows, const int32_t* cols,
                            const double* deg, T* vals) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < q;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double s = __dsqrt_rn(__dmul_rn(deg[rows[e]], deg[cols[e]]));
    vals[e] = (T)__ddiv_rn((double)vals[e], s);
  }
}

__global__ void k_any(int64_t n, const int32_t* flags, int* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    if (flags[e]) *out = 1;
}

// ---- host helpers ------------------------------------------------------------
template <class K, class V>
static void radix_sort_pairs(sgnn_ctx ctx, const K* kin, K* kout, const V* vin, V* vout,
                             int64_t n, int end_bit) {
  if (n == 0) return;
  size_t tmp = 0;
  SGNN_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, (int)n, 0,
                                            end_bit, ctx->stream));
  DevBuf t(tmp, ctx->stream);
  SGNN_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, kin, kout, vin, vout, (int)n, 0,
                                            end_bit, ctx->stream));
  ctx->launches += 4;
}

static void exclusive_scan(sgnn_ctx ctx, const int32_t* in, int32_t* out, int64_t n) {
  if (n == 0) return;
  size_t tmp = 0;
  SGNN_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, (int)n, ctx->stream));
  DevBuf t(tmp, ctx->stream);
  SGNN_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, in, out, (int)n, ctx->stream));
  ctx->launches += 2;
}

template <class T>
static T read_back(sgnn_ctx ctx, const T* dev) {
  T h{};
  SGNN_CUDA(cudaMemcpyAsync(&h, dev, sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  SGNN_CUDA(cudaStreamSynchronize(ctx->stream));
  return h;
}

void build_ptr(sgnn_ctx ctx, const int32_t* sorted_ids, int64_t nnz, int32_t n, int32_t* ptr) {
  k_ptr_from_sorted<<<grid_for(ctx, nnz + 1, 256), 256, 0, ctx->stream>>>(nnz, sorted_ids, n,
                                                                          ptr);
  launched(ctx);
}

template <class T>
int64_t canonicalize(sgnn_ctx ctx, int32_t nr, int32_t nc, int64_t nnz, const int32_t* rows,
                     const int32_t* cols, const T* vals, int32_t* orow, int32_t* ocol, T* oval) {
  require(nr >= 0 && nc >= 0 && nnz >= 0, "coo_from_triplets: bad sizes");
  require(nnz < (int64_t)INT32_MAX, "coo_from_triplets: nnz exceeds int32 indices");
  if (nnz == 0) return 0;
  cudaStream_t s = ctx->stream;
  DevBuf keys(nnz * 8, s), skeys(nnz * 8, s), idx(nnz * 4, s), sidx(nnz * 4, s);
  DevBuf flag(nnz * 4, s), pos(nnz * 4, s), bad(sizeof(int), s);
  SGNN_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
  const int g = grid_for(ctx, nnz, 256);
  k_range_keys<<<g, 256, 0, s>>>(nnz, rows, cols, nr, nc, keys.as<uint64_t>(),
                                 idx.as<int32_t>(), bad.as<int>());
  launched(ctx);
  require(read_back(ctx, bad.as<int>()) == 0, "coo_from_triplets: index out of range");
  radix_sort_pairs(ctx, keys.as<uint64_t>(), skeys.as<uint64_t>(), idx.as<int32_t>(),
                   sidx.as<int32_t>(), nnz, bits_for((uint64_t)nr * (uint64_t)nc));
  k_last_of_run<<<g, 256, 0, s>>>(nnz, skeys.as<uint64_t>(), flag.as<int32_t>());
  launched(ctx);
  exclusive_scan(ctx, flag.as<int32_t>(), pos.as<int32_t>(), nnz);
  const int32_t last_pos = read_back(ctx, pos.as<int32_t>() + nnz - 1);
  const int32_t last_flag = read_back(ctx, flag.as<int32_t>() + nnz - 1);
  k_scatter_kept<T><<<g, 256, 0, s>>>(nnz, flag.as<int32_t>(), pos.as<int32_t>(),
                                      sidx.as<int32_t>(), rows, cols, vals, orow, ocol, oval);
  launched(ctx);
  return (int64_t)last_pos + last_flag;
}

// CSC of a canonical COO: stable sort by column (rows stay ascending)
template <class T>
void csc_from_coo(sgnn_ctx ctx, int32_t nc, int64_t nnz, const int32_t* rows,
                  const int32_t* cols, const T* vals, int32_t* colptr, int32_t* orows, T* ovals,
                  int32_t* perm_out) {
  cudaStream_t s = ctx->stream;
  DevBuf scols(nnz * 4 + 4, s), iota(nnz * 4 + 4, s), permb;
  int32_t* perm = perm_out;
  if (!perm) {
    permb = DevBuf(nnz * 4 + 4, s);
    perm = permb.as<int32_t>();
  }
  if (nnz > 0) {
    k_iota<<<grid_for(ctx, nnz, 256), 256, 0, s>>>(nnz, iota.as<int32_t>());
    launched(ctx);
    radix_sort_pairs(ctx, cols, scols.as<int32_t>(), iota.as<int32_t>(), perm, nnz,
                     bits_for((uint64_t)(nc > 0 ? nc : 1)));
  }
  build_ptr(ctx, scols.as<int32_t>(), nnz, nc, colptr);
  if (nnz > 0 && (orows || ovals)) {
    k_gather_csc<T><<<grid_for(ctx, nnz, 256), 256, 0, s>>>(nnz, perm, rows, vals, orows,
                                                            ovals);
    launched(ctx);
  }
}

template <class T>
int64_t add_self_loops(sgnn_ctx ctx, int32_t n, int64_t nnz, const int32_t* rows,
                       const int32_t* cols, const T* vals, int32_t* orow, int32_t* ocol,
                       T* oval) {
  cudaStream_t s = ctx->stream;
  DevBuf rowptr((n + 1) * 4, s), missing((n + 1) * 4, s), len((n + 1) * 4, s),
      newptr((n + 1) * 4, s);
  build_ptr(ctx, rows, nnz, n, rowptr.as<int32_t>());
  const int g = grid_for(ctx, n, 256);
  k_diag<<<g, 256, 0, s>>>(n, rowptr.as<int32_t>(), cols, nullptr, missing.as<int32_t>());
  launched(ctx);
  k_loop_lengths<<<g, 256, 0, s>>>(n, rowptr.as<int32_t>(), missing.as<int32_t>(),
                                   len.as<int32_t>());
  launched(ctx);
  SGNN_CUDA(cudaMemsetAsync(len.as<int32_t>() + n, 0, 4, s));
  exclusive_scan(ctx, len.as<int32_t>(), newptr.as<int32_t>(), n + 1);
  k_insert_loops<T><<<g, 256, 0, s>>>(n, rowptr.as<int32_t>(), cols, vals,
                                      missing.as<int32_t>(), newptr.as<int32_t>(), orow, ocol,
                                      oval);
  launched(ctx);
  return read_back(ctx, newptr.as<int32_t>() + n);
}

template <class T>
int64_t gcn_normalize(sgnn_ctx ctx, int32_t n, int64_t nnz, const int32_t* rows,
                      const int32_t* cols, const T* vals, int32_t* orow, int32_t* ocol,
                      T* oval) {
  cudaStream_t s = ctx->stream;
  const int64_t q = add_self_loops<T>(ctx, n, nnz, rows, cols, vals, orow, ocol, oval);
  DevBuf rowptr((n + 1) * 4, s), deg((n + 1) * 8, s), neg(sizeof(int), s);
  SGNN_CUDA(cudaMemsetAsync(neg.get(), 0, sizeof(int), s));
  build_ptr(ctx, orow, q, n, rowptr.as<int32_t>());
  k_degrees<T><<<grid_for(ctx, n, 256), 256, 0, s>>>(n, rowptr.as<int32_t>(), oval,
                                                     deg.as<double>(), neg.as<int>());
  launched(ctx);
  require(read_back(ctx, neg.as<int>()) == 0, "gcn_normalize: negative edge weight");
  k_normalize<T><<<grid_for(ctx, q, 256), 256, 0, s>>>(q, orow, ocol, deg.as<double>(), oval);
  launched(ctx);
  return q;
}

template int64_t canonicalize<float>(sgnn_ctx, int32_t, int32_t, int64_t, const int32_t*,
                                     const int32_t*, const float*, int32_t*, int32_t*, float*);
template int64_t canonicalize<double>(sgnn_ctx, int32_t, int32_t, int64_t, const int32_t*,
                                      const int32_t*, const double*, int32_t*, int32_t*,
                                      double*);

}  // namespace sgnn

// ---------------------------------------------------------------------------
// AdjacencyOp and SparsePattern handles
// ---------------------------------------------------------------------------
using namespace sgnn;

sgnn_adj_s::~sgnn_adj_s() {}
sgnn_pattern_s::~sgnn_pattern_s() {}

#define DISPATCH_T(dtype, ...)                   \
  do {                                           \
    if ((dtype) == SGNN_F32) {                   \
      using T = float;                           \
      __VA_ARGS__;                               \
    } else if ((dtype) == SGNN_F64) {            \
      using T = double;                          \
      __VA_ARGS__;                               \
    } else {                                     \
      throw invalid_argument("unknown dtype");   \
    }                                            \
  } while (0)

extern "C" {

int sgnn_coo_canonicalize(sgnn_ctx ctx, int32_t nr, int32_t nc, int64_t nnz,
                          const int32_t* rows, const int32_t* cols, const void* vals, int dtype,
                          int32_t* orow, int32_t* ocol, void* oval, int64_t* out_nnz) {
  SGNN_API_BEGIN
  DISPATCH_T(dtype, *out_nnz = canonicalize<T>(ctx, nr, nc, nnz, rows, cols,
                                               static_cast<const T*>(vals), orow, ocol,
                                               static_cast<T*>(oval)));
  SGNN_API_END
}

int sgnn_csr_from_coo(sgnn_ctx ctx, int32_t nr, int64_t nnz, const int32_t* rows,
                      int32_t* rowptr) {
  SGNN_API_BEGIN
  build_ptr(ctx, rows, nnz, nr, rowptr);
  SGNN_API_END
}

int sgnn_csc_from_coo(sgnn_ctx ctx, int32_t nc, int64_t nnz, const int32_t* rows,
                      const int32_t* cols, const void* vals, int dtype, int32_t* colptr,
                      int32_t* orows, void* ovals, int32_t* perm) {
  SGNN_API_BEGIN
  DISPATCH_T(dtype, csc_from_coo<T>(ctx, nc, nnz, rows, cols, static_cast<const T*>(vals),
                                    colptr, orows, static_cast<T*>(ovals), perm));
  SGNN_API_END
}

int sgnn_add_self_loops(sgnn_ctx ctx, int32_t n, int64_t nnz, const int32_t* rows,
                        const int32_t* cols, const void* vals, int dtype, int32_t* orow,
                        int32_t* ocol, void* oval, int64_t* out_nnz) {
  SGNN_API_BEGIN
  DISPATCH_T(dtype, *out_nnz = add_self_loops<T>(ctx, n, nnz, rows, cols,
                                                 static_cast<const T*>(vals), orow, ocol,
                                                 static_cast<T*>(oval)));
  SGNN_API_END
}

int sgnn_gcn_normalize(sgnn_ctx ctx, int32_t n, int64_t nnz, const int32_t* rows,
                       const int32_t* cols, const void* vals, int dtype, int32_t* orow,
                       int32_t* ocol, void* oval, int64_t* out_nnz) {
  SGNN_API_BEGIN
  DISPATCH_T(dtype, *out_nnz = gcn_normalize<T>(ctx, n, nnz, rows, cols,
                                                static_cast<const T*>(vals), orow, ocol,
                                                static_cast<T*>(oval)));
  SGNN_API_END
}

int sgnn_adj_create(sgnn_ctx ctx, int32_t nr, int32_t nc, int64_t nnz, const int32_t* rows,
                    const int32_t* cols, const void* vals, int dtype, int format,
                    sgnn_adj* out) {
  SGNN_API_BEGIN
  require(format >= SGNN_COO && format <= SGNN_HYBRID, "unknown format");
  require(nnz < (int64_t)INT32_MAX, "adjacency: nnz exceeds int32 indices");
  const size_t sb = dtype_size(dtype);
  cudaStream_t s = ctx->stream;
  auto* a = new sgnn_adj_s;
  a->n_rows = nr;
  a->n_cols = nc;
  a->nnz = nnz;
  a->dtype = dtype;
  a->format = format;
  a->rowptr = DevBuf((size_t)(nr + 1) * 4, s);
  a->cols = DevBuf(nnz * 4 + 4, s);
  a->vals = DevBuf(nnz * sb + 8, s);
  a->colptr = DevBuf((size_t)(nc + 1) * 4, s);
  a->crows = DevBuf(nnz * 4 + 4, s);
  a->cvals = DevBuf(nnz * sb + 8, s);
  try {
    build_ptr(ctx, rows, nnz, nr, a->rowptr.as<int32_t>());
    if (nnz) {
      SGNN_CUDA(cudaMemcpyAsync(a->cols.get(), cols, nnz * 4, cudaMemcpyDeviceToDevice, s));
      SGNN_CUDA(cudaMemcpyAsync(a->vals.get(), vals, nnz * sb, cudaMemcpyDeviceToDevice, s));
    }
    DISPATCH_T(dtype, csc_from_coo<T>(ctx, nc, nnz, rows, cols, static_cast<const T*>(vals),
                                      a->colptr.as<int32_t>(), a->crows.as<int32_t>(),
                                      a->cvals.as<T>(), nullptr));
  } catch (...) {
    delete a;
    throw;
  }
  *out = a;
  SGNN_API_END
}

int sgnn_adj_destroy(sgnn_adj a) {
  SGNN_API_BEGIN
  delete a;
  SGNN_API_END
}

int sgnn_adj_info(sgnn_adj a, int32_t* nr, int32_t* nc, int64_t* nnz, int* dtype) {
  SGNN_API_BEGIN
  if (nr) *nr = a->n_rows;
  if (nc) *nc = a->n_cols;
  if (nnz) *nnz = a->nnz;
  if (dtype) *dtype = a->dtype;
  SGNN_API_END
}

int sgnn_adj_arrays(sgnn_adj a, const int32_t** rowptr, const int32_t** cols, const void** vals,
                    const int32_t** colptr, const int32_t** crows, const void** cvals) {
  SGNN_API_BEGIN
  if (rowptr) *rowptr = a->rowptr.as<int32_t>();
  if (cols) *cols = a->cols.as<int32_t>();
  if (vals) *vals = a->vals.get();
  if (colptr) *colptr = a->colptr.as<int32_t>();
  if (crows) *crows = a->crows.as<int32_t>();
  if (cvals) *cvals = a->cvals.get();
  SGNN_API_END
}

int sgnn_pattern_create(sgnn_ctx ctx, int32_t n, int64_t nnz, const int32_t* rowptr,
                        const int32_t* cols, sgnn_pattern* out) {
  SGNN_API_BEGIN
  require(nnz < (int64_t)INT32_MAX, "SparsePattern: nnz exceeds int32 indices");
  cudaStream_t s = ctx->stream;
  auto* p = new sgnn_pattern_s;
  p->n = n;
  p->nnz = nnz;
  p->rowptr = DevBuf((size_t)(n + 1) * 4, s);
  p->cols = DevBuf(nnz * 4 + 4, s);
  p->colptr = DevBuf((size_t)(n + 1) * 4, s);
  p->rows = DevBuf(nnz * 4 + 4, s);
  p->perm = DevBuf(nnz * 4 + 4, s);
  p->diag = DevBuf((size_t)n * 4 + 4, s);
  try {
    SGNN_CUDA(cudaMemcpyAsync(p->rowptr.get(), rowptr, (size_t)(n + 1) * 4,
                              cudaMemcpyDeviceToDevice, s));
    if (nnz) SGNN_CUDA(cudaMemcpyAsync(p->cols.get(), cols, nnz * 4, cudaMemcpyDeviceToDevice, s));
    DevBuf rid(nnz * 4 + 4, s), missing((size_t)n * 4 + 4, s), any(sizeof(int), s);
    k_row_ids<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, rowptr, rid.as<int32_t>());
    launched(ctx);
    csc_from_coo<int32_t>(ctx, n, nnz, rid.as<int32_t>(), cols, nullptr,
                          p->colptr.as<int32_t>(), p->rows.as<int32_t>(), nullptr,
                          p->perm.as<int32_t>());
    k_diag<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, rowptr, cols, p->diag.as<int32_t>(),
                                                 missing.as<int32_t>());
    launched(ctx);
    SGNN_CUDA(cudaMemsetAsync(any.get(), 0, sizeof(int), s));
    k_any<<<grid_for(ctx, n, 256), 256, 0, s>>>(n, missing.as<int32_t>(), any.as<int>());
    launched(ctx);
    p->all_self_loops = read_back(ctx, any.as<int>()) == 0;
  } catch (...) {
    delete p;
    throw;
  }
  *out = p;
  SGNN_API_END
}

int sgnn_pattern_destroy(sgnn_pattern p) {
  SGNN_API_BEGIN
  delete p;
  SGNN_API_END
}

int sgnn_pattern_info(sgnn_pattern p, int32_t* n, int64_t* nnz, int* all) {
  SGNN_API_BEGIN
  if (n) *n = p->n;
  if (nnz) *nnz = p->nnz;
  if (all) *all = p->all_self_loops ? 1 : 0;
  SGNN_API_END
}

int sgnn_pattern_arrays(sgnn_pattern p, const int32_t** rowptr, const int32_t** cols,
                        const int32_t** colptr, const int32_t** rows, const int32_t** perm,
                        const int32_t** diag) {
  SGNN_API_BEGIN
  if (rowptr) *rowptr = p->rowptr.as<int32_t>();
  if (cols) *cols = p->cols.as<int32_t>();
  if (colptr) *colptr = p->colptr.as<int32_t>();
  if (rows) *rows = p->rows.as<int32_t>();
  if (perm) *perm = p->perm.as<int32_t>();
  if (diag) *diag = p->diag.as<int32_t>();
  SGNN_API_END
}

}  // extern "C"
