// gemm_tc.cu -- tcgen05 (5th-generation tensor core) GEMM for the float32
// dense transforms of the path: X.Theta / P.Theta (forward), X^T S / P^T dX'
// (dTheta, split-K over the n-long reduction) and S.Theta^T / dX'.Theta^T (dX).
//
// Accuracy: the north star requires fp32 results within 1e-4 of the float64
// reference; plain TF32 misses that.  Each fp32 operand tile is
// split in shared memory into hi = tf32(x) (low 13 mantissa bits cleared) and
// lo = x - hi, and the tile product is hi.hi + hi.lo + lo.hi ("3xTF32"),
// accumulated in fp32 in TMEM -- ~2^-21 relative error per product.
//
// Structure (one 128 x BN output tile per CTA, K pipelined in BK=32 stages):
//   warp 0      TMA producer (cp.async.bulk.tensor, SWIZZLE_128B, mbarrier tx)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (kind::tf32,
//               M=128, N=BN, K=8), tcgen05.commit frees smem stages
//   warps 2..5  split converters (raw -> hi in place, lo to a twin buffer,
//               fence.proxy.async) during the main loop, then the epilogue
//               (tcgen05.ld 32x32b.x32 -> registers -> +bias -> global)
// Operands may be K-major or MN-major (UMMA transpose bits), so X^T . S reads
// X and S in place -- no transposed copies.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "internal.cuh"

namespace sgnn {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per 128-byte swizzle row
constexpr int NUM_THREADS = 320;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0,
                                             int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// UMMA shared-memory descriptor, version 1.  Layout type 2 = SWIZZLE_128B
// (16-byte chunks, K-major tiles); 1 = SWIZZLE_128B_BASE32B (32-byte chunks,
// 4-row period) -- the only layout UMMA accepts for MN-major tf32 operands.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  d |= (uint64_t)layout << 61;
  return d;
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, M=128, N=n, majors
__host__ __device__ constexpr uint32_t instr_desc(int n, bool a_mn, bool b_mn) {
  return (1u << 4)                      // c_format F32
         | (2u << 7)                    // a_format TF32
         | (2u << 10)                   // b_format TF32
         | ((a_mn ? 1u : 0u) << 15)     // a_major
         | ((b_mn ? 1u : 0u) << 16)     // b_major
         | ((uint32_t)(n >> 3) << 17)   // N >> 3
         | ((uint32_t)(BM >> 4) << 24); // M >> 4
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// tcgen05.ld without the wait: the registers are written asynchronously until
// tmem_wait32 on the same array, whose "+r" operands keep every use after it
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait32(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),
                 "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]),
                 "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]),
                 "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]),
                 "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]),
                 "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

__device__ __forceinline__ void tmem_ld8_async(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait8(uint32_t (&r)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),
                 "+r"(r[6]), "+r"(r[7])
               :
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.b32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// explicit shared-space accesses (the 1024-aligned smem base is computed
// through an integer, so plain dereferences compile to generic LD / ST)
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float4 lds_f32x4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
__device__ __forceinline__ void sts_f32x4(uint32_t a, const float4& v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

__device__ __forceinline__ uint32_t tf32_hi(float x) { return __float_as_uint(x) & 0xFFFFE000u; }

// Split a raw fp32 smem tile in place into hi (tf32-exact) and write lo.
__device__ __forceinline__ void split_tile(float4* raw, float4* lo, int n4, int tid, int nthr) {
  for (int i = tid; i < n4; i += nthr) {
    float4 v = raw[i];
    float4 h, l;
    h.x = __uint_as_float(tf32_hi(v.x));
    h.y = __uint_as_float(tf32_hi(v.y));
    h.z = __uint_as_float(tf32_hi(v.z));
    h.w = __uint_as_float(tf32_hi(v.w));
    l.x = __fsub_rn(v.x, h.x);
    l.y = __fsub_rn(v.y, h.y);
    l.z = __fsub_rn(v.z, h.z);
    l.w = __fsub_rn(v.w, h.w);
    raw[i] = h;
    lo[i] = l;
  }
}

__global__ void k_split_global(int64_t n, const float* __restrict__ x, float* __restrict__ hi,
                               float* __restrict__ lo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    const float h = __uint_as_float(tf32_hi(v));
    hi[i] = h;
    lo[i] = __fsub_rn(v, h);
  }
}

// the same for a rows x cols block of a matrix with row pitch ld (contiguous out)
__global__ void k_split_global2d(int32_t rows, int32_t cols, const float* __restrict__ x,
                                 int32_t ld, float* __restrict__ hi, float* __restrict__ lo) {
  const int64_t n = (int64_t)rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[(i / cols) * ld + i % cols];
    const float h = __uint_as_float(tf32_hi(v));
    hi[i] = h;
    lo[i] = __fsub_rn(v, h);
  }
}

// optional epilogue: GAT node scores s = M a_src^T, d = M a_dst^T per head
// (kernels.hpp:385-423) from the output tile while it is in registers
struct EpiScores {
  const float* a_src = nullptr;
  const float* a_dst = nullptr;
  float* s = nullptr;
  float* d = nullptr;
  int h = 0, k = 0;
  // fused ReLU (dense.hpp:197-228 activation / :232-268 backward), row-major
  // n x N byte masks: relu_out -> out = max(out + bias, 0) and mask = (x > 0);
  // mask_in -> out = mask ? out : 0 (the activation's backward)
  uint8_t* relu_out = nullptr;
  const uint8_t* mask_in = nullptr;
  // ELU(1) backward (dense.hpp:232-268) with mask_in: out = mask ? out :
  // (saved + 1) * out, saved = the activation's forward output (row-major n x N)
  const float* elu_saved = nullptr;
  // with relu_out: ELU(1) forward instead of ReLU -- out = x > 0 ? x : exp(x) - 1
  // and mask = (x > 0), the expressions of the separate activation pass (EPI bit 5)
  bool elu = false;
  // k-block drain mode (K > 256, BN <= 128): every k-block is accumulated
  // afresh in one of three TMEM accumulators and added into fp32 registers
  // by the epilogue (round-to-nearest), instead of ~12 truncating tensor-core
  // accumulations per k-block into one growing sum (5e-6 relative bias at
  // K = 500, measured); the final sum goes back to TMEM for the epilogue
  bool drain = false;
  // k-blocks per drained partial (1, or 2 for unsplit GEMMs of moderate K:
  // the drain's TMEM read -- 64 B/clk -- costs 8 BN cycles per partial
  // against 6 BN cycles of MMAs per k-block, so draining every k-block made
  // the K = 320 Gat2 d_input GEMM epilogue-bound)
  int drain_group = 1;
  // row pitch of C in elements (0: N) -- column blocks of a wider matrix
  int ldc = 0;
};

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 4;  // 16 KB raw A tile
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE_BYTES = A_BYTES + 2 * B_BYTES;  // A raw | B hi | B lo
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES >= 4 ? 4 : (200 * 1024) / STAGE_BYTES;
  static constexpr int EPI_BYTES = 4 * 2 * 4096;  // 4 epilogue warps x 2 x (32 x 32 fp32)
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int NA = 2;                                // TMEM A buffers (hi|lo, 64 cols)
  // accumulators: 3 when BN <= 128 (the k-block drain mode rotates three),
  // else 2 (the tile double buffer)
  static constexpr int NACC = BN <= 128 ? 3 : 2;
  static constexpr uint32_t USED = NACC * BN + NA * 64;       // accumulators + A buffers
  static constexpr uint32_t TMEM_COLS = USED <= 256 ? 256 : 512;
};

// Persistent, warp-specialized: CTA b processes tiles b, b+grid, ... where a
// tile is (split z, m-tile, n-tile), n fastest so the CTAs sharing an A tile
// run concurrently (A read from HBM once).  Roles:
//   warp 0      TMA producer over a continuous smem stage ring (A raw, B hi/lo
//               -- B pre-split in global when small, else raw + split here)
//   warp 1      TMEM alloc + MMA issuer: A (hi, lo) from TMEM, B from smem,
//               D in one of two TMEM accumulators (tile & 1)
//   warps 2..5  converters: thread = one A row = one TMEM lane; reads its row
//               from smem, splits hi/lo in registers and tcgen05.st's both into
//               a TMEM A buffer (no smem write-back); splits B in smem if needed
//   warps 6..9  epilogue: TMEM -> registers -> (+bias) -> global, overlapping
//               the next tile's MMAs
// EPI: compile-time epilogue extras (the plain GEMM pays nothing for them):
// bit 0 node scores, bit 1 ReLU + mask out, bit 2 ReLU backward (mask in),
// bit 3 node scores for head widths k % 32 != 0 (k % 4 == 0), bit 4 (with
// bit 2) ELU backward
template <bool A_MN, bool B_MN, int BN, bool B_PRE, int EPI>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmBlo, const __grid_constant__ CUtensorMap tmC,
              int M, int N, int K, int kchunk, int splits, float* __restrict__ C, int ldc,
              const float* __restrict__ bias, float* __restrict__ part, int tma_store,
              double* __restrict__ cs_part, const EpiScores sc) {
  using CF = Cfg<BN>;
  constexpr int S = CF::STAGES;
  constexpr int NA = CF::NA;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* epi = smem + S * CF::STAGE_BYTES;  // 1024-aligned (STAGE_BYTES % 1024 == 0)
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + CF::EPI_BYTES);
  uint64_t* empty = full + S;
  uint64_t* afull = empty + S;    // [NA] converters -> MMA
  uint64_t* aempty = afull + NA;  // [NA] MMA -> converters
  uint64_t* tfull = aempty + NA;  // [3]
  uint64_t* tempty = tfull + 3;   // [3]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 3);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN;
  const int tiles = num_m * num_n * splits;

  auto a_raw = [&](int s) { return smem + s * CF::STAGE_BYTES; };
  auto b_hi = [&](int s) { return smem + s * CF::STAGE_BYTES + CF::A_BYTES; };
  auto b_lo = [&](int s) { return smem + s * CF::STAGE_BYTES + CF::A_BYTES + CF::B_BYTES; };
  auto tile_of = [&](int t, int& z, int& m0, int& n0, int& kb, int& nk) {
    const int nt = t % num_n;
    const int rest = t / num_n;
    // m-tiles last to first: an A operand just written in row order by the
    // preceding kernel (the propagate-first SpMM) still has its tail rows in
    // L2 when the GEMM starts (Arxiv GCN step -2 us, measured)
#ifndef GEMM_FWD_M
    const int mt = num_m - 1 - rest % num_m;
#else
    const int mt = rest % num_m;
#endif
    z = rest / num_m;
    m0 = mt * BM;
    n0 = nt * BN;
    kb = z * kchunk;
    const int ke = min(K, kb + kchunk);
    nk = (ke - kb + BK - 1) / BK;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NA; ++a) {
      mbar_init(&afull[a], 4);
      mbar_init(&aempty[a], 1);
    }
    for (int a = 0; a < 3; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(CF::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform
  const uint32_t tmem_a = tmem + CF::NACC * BN;  // A buffers after the accumulators

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int z, m0, n0, kb, nk;
        tile_of(t, z, m0, n0, kb, nk);
        for (int ks = 0; ks < nk; ++ks, ++it) {
          const int s = it % S;
          const uint32_t ph = (it / S) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], CF::A_BYTES + (B_PRE ? 2 : 1) * CF::B_BYTES);
          const int kc = kb + ks * BK;
          if (A_MN) {  // A stored K x M: boxes of 32 M-elements x 32 K-rows
#pragma unroll
            for (int b = 0; b < BM / 32; ++b)
              tma_load_2d(a_raw(s) + b * 4096, &tmA, &full[s], m0 + 32 * b, kc);
          } else {  // A stored M x K: one box of 32 K x 128 rows
            tma_load_2d(a_raw(s), &tmA, &full[s], kc, m0);
          }
          if (B_MN) {  // B stored K x N
#pragma unroll
            for (int b = 0; b < BN / 32; ++b) {
              tma_load_2d(b_hi(s) + b * 4096, &tmB, &full[s], n0 + 32 * b, kc);
              if (B_PRE) tma_load_2d(b_lo(s) + b * 4096, &tmBlo, &full[s], n0 + 32 * b, kc);
            }
          } else {  // B stored N x K
            tma_load_2d(b_hi(s), &tmB, &full[s], kc, n0);
            if (B_PRE) tma_load_2d(b_lo(s), &tmBlo, &full[s], kc, n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // the whole warp walks the loop, so the MMA operands are warp-uniform
    // values the compiler keeps in uniform registers (issued from one lane
    // inside the loop it wrapped every tcgen05.mma in an ELECT / R2UR
    // uniformization loop: 8 instructions per MMA; X.Theta 72 -> 66 us,
    // G.Theta^T 68 -> 60 us measured); one elected lane issues MMAs / commits
    {
      const bool leader = elect_one();
      constexpr uint32_t idesc = instr_desc(BN, false, B_MN);  // A from TMEM is K-major
      int it = 0, tl = 0, dr = 0;
      const bool kdrain = sc.drain;  // per-k-block(-group) accumulators (three)
      const int nacc = 3;
      // one k-block into accumulator tacc (fresh: its first MMA overwrites)
      auto kblock = [&](uint32_t tacc, bool fresh) {
        const int s = it % S, a = it % NA;
        mbar_wait(&afull[a], (it / NA) & 1);  // implies full[s] (converters waited on it)
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ta = tmem_a + (uint32_t)(a * 64);
        const uint32_t bh = smem_u32(b_hi(s)), bl = smem_u32(b_lo(s));
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          // B K-major (SW128): +32 B inside the swizzled row, SBO 1024.
          // B MN-major (SW128_BASE32B): +1024 B per 8 K-rows, LBO 4096, SBO 512.
          const uint32_t boff = B_MN ? kk * 1024 : kk * 32;
          const uint32_t blb = B_MN ? 4096 : 16, bsb = B_MN ? 512 : 1024, blt = B_MN ? 1 : 2;
          const uint64_t dbh = smem_desc(bh + boff, blb, bsb, blt);
          const uint64_t dbl = smem_desc(bl + boff, blb, bsb, blt);
          const uint32_t acc = (!fresh || kk > 0) ? 1u : 0u;
          if (leader) {
            mma_tf32_ts(tacc, ta + kk * 8, dbh, idesc, acc);       // hi . hi
            mma_tf32_ts(tacc, ta + kk * 8, dbl, idesc, 1u);        // hi . lo
            mma_tf32_ts(tacc, ta + 32 + kk * 8, dbh, idesc, 1u);   // lo . hi
          }
        }
        if (leader) {
          umma_commit(&empty[s]);   // smem stage free
          umma_commit(&aempty[a]);  // TMEM A buffer free
        }
        __syncwarp();
        ++it;
      };
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++tl) {
        int z, m0, n0, kb, nk;
        tile_of(t, z, m0, n0, kb, nk);
        if (!kdrain) {  // the tile's accumulator: one of two, by tile parity
          const int abuf = tl & 1;
          const uint32_t tacc = tmem + (uint32_t)(abuf * BN);
          mbar_wait(&tempty[abuf], ((tl >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          for (int ks = 0; ks < nk; ++ks) kblock(tacc, ks == 0);
          if (leader) umma_commit(&tfull[abuf]);  // accumulator ready for the epilogue
          __syncwarp();
        } else {  // every group of 1-2 k-blocks into the next of three accumulators
          const int gm = sc.drain_group - 1;
          uint32_t tacc = 0;
          int abuf = 0;
          for (int ks = 0; ks < nk; ++ks) {
            const bool gfirst = (ks & gm) == 0, glast = (ks & gm) == gm || ks + 1 == nk;
            if (gfirst) {
              abuf = dr % nacc;
              tacc = tmem + (uint32_t)(abuf * BN);
              mbar_wait(&tempty[abuf], ((dr / nacc) & 1) ^ 1);
              asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
            kblock(tacc, gfirst);
            if (glast) {
              if (leader) umma_commit(&tfull[abuf]);  // this group's partial ready for the drain
              __syncwarp();
              ++dr;
            }
          }
        }
      }
    }
  } else if (warp < 6) {
    // ---------------- converters: one A row per thread -> TMEM lane ----------------
    const int q = warp & 3;
    const int r = q * 32 + lane;  // tile row == TMEM lane
    const int ctid = threadIdx.x - 64;
    // column sums of an MN-major B over K (d_bias = 1^T dX' fused into
    // dTheta = P^T dX'): thread ctid always sees the same 4 columns of every
    // 32-column box of a stage (chunk i = ctid + 128 j -> box j/2, K-row
    // ctid/8 + 16 (j&1), 32 B atom ((ctid&7)>>1) ^ ((ctid>>3)&3), see split_tile)
    constexpr int NB = BN / 32;
    const bool want_cs = (cs_part != nullptr) && B_MN && !B_PRE;
    // float32 within 8 k-blocks (16 rows per thread), then float64: one
    // float32 running sum over a split's thousands of rows drifts past the
    // 1e-4 bar on columns whose total cancels to O(1) (measured), and a
    // float64 add per element costs the converters 20 us on dTheta
    double cs[NB][4];
    float cf[NB][4];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      cs[b][0] = cs[b][1] = cs[b][2] = cs[b][3] = 0.0;
      cf[b][0] = cf[b][1] = cf[b][2] = cf[b][3] = 0.f;
    }
    auto fold_cs = [&] {
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          cs[b][e] += (double)cf[b][e];
          cf[b][e] = 0.f;
        }
    };
    int it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      int z, m0, n0, kb, nk;
      tile_of(t, z, m0, n0, kb, nk);
      const bool cs_tile = want_cs && m0 == 0;
      for (int ks = 0; ks < nk; ++ks, ++it) {
        const int s = it % S, a = it % NA;
        mbar_wait(&full[s], (it / S) & 1);
        if (!B_PRE) {
          if (B_MN && cs_tile) {
            float4* raw = reinterpret_cast<float4*>(b_hi(s));
            float4* lo = reinterpret_cast<float4*>(b_lo(s));
#pragma unroll
            for (int j = 0; j < CF::B_BYTES / 16 / 128; ++j) {
              const int i = ctid + 128 * j;
              float4 v = raw[i];
              cf[j >> 1][0] += v.x;
              cf[j >> 1][1] += v.y;
              cf[j >> 1][2] += v.z;
              cf[j >> 1][3] += v.w;
              float4 h, l;
              h.x = __uint_as_float(tf32_hi(v.x));
              h.y = __uint_as_float(tf32_hi(v.y));
              h.z = __uint_as_float(tf32_hi(v.z));
              h.w = __uint_as_float(tf32_hi(v.w));
              l.x = __fsub_rn(v.x, h.x);
              l.y = __fsub_rn(v.y, h.y);
              l.z = __fsub_rn(v.z, h.z);
              l.w = __fsub_rn(v.w, h.w);
              raw[i] = h;
              lo[i] = l;
            }
            if ((ks & 7) == 7 || ks + 1 == nk) fold_cs();
          } else {
            split_tile(reinterpret_cast<float4*>(b_hi(s)), reinterpret_cast<float4*>(b_lo(s)),
                       CF::B_BYTES / 16, ctid, 128);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        float v[32];
        const uint8_t* base = a_raw(s);
        if (A_MN) {
          // 4 boxes of 32 M x 32 K-rows; 32 B chunks swizzled with (K-row % 4)
          const uint8_t* bx = base + (r >> 5) * 4096;
          const int p = r & 31, c32 = p >> 3, e = p & 7;
#pragma unroll
          for (int kr = 0; kr < 32; ++kr)
            v[kr] = lds_f32(smem_u32(bx) + kr * 128 + ((c32 ^ (kr & 3)) << 5) + e * 4);
        } else {
          // row r: 128 B, 16 B chunks swizzled with (row % 8)
          const uint8_t* row = base + r * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 x = lds_f32x4(smem_u32(row) + ((c ^ (r & 7)) << 4));
            v[4 * c] = x.x;
            v[4 * c + 1] = x.y;
            v[4 * c + 2] = x.z;
            v[4 * c + 3] = x.w;
          }
        }
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          hi[j] = tf32_hi(v[j]);
          lo[j] = __float_as_uint(__fsub_rn(v[j], __uint_as_float(hi[j])));
        }
        mbar_wait(&aempty[a], ((it / NA) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ta = tmem_a + (uint32_t)(a * 64) + ((uint32_t)(q * 32) << 16);
        tmem_st32(ta, hi);
        tmem_st32(ta + 32, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[a]);
      }
      if (cs_tile) {
        // combine the 4 lanes holding the same logical 32 B atom (fixed order),
        // one lane per atom writes this warp's partial: cs_part[z][warp][n]
        const int half = lane & 1, kr3 = (lane >> 3) & 3;
        const int c32 = ((lane & 7) >> 1) ^ kr3;
        double* dst = cs_part + ((int64_t)z * 4 + q) * N;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            double sum = 0.0;
#pragma unroll
            for (int r3 = 0; r3 < 4; ++r3) {
              const int src = ((((c32 ^ r3) << 1) | half)) + 8 * r3;
              sum += __shfl_sync(0xffffffffu, cs[b][e], src);
            }
            cs[b][e] = 0.0;
            const int n = n0 + b * 32 + c32 * 8 + half * 4 + e;
            if (kr3 == 0 && n < N) dst[n] = sum;
          }
        }
      }
    }
  } else {
    // ---------------- epilogue: warp w reads TMEM lanes 32*(w%4) .. +31 ----------------
    const int q = warp & 3;
    const bool vec = ((ldc & 3) == 0) && ((N & 3) == 0);
    int tl = 0, ecnt = 0, dr = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++tl) {
      int z, m0, n0, kb, nk;
      tile_of(t, z, m0, n0, kb, nk);
      int abuf = tl & 1;
      const int row = m0 + q * 32 + lane;
      // activation-backward inputs of this row's next 32 columns (mask bytes,
      // saved ELU outputs): fetched one chunk ahead -- the first while the
      // accumulator is still being produced -- so their latency overlaps the
      // TMEM loads and stores instead of stalling every chunk
      constexpr int NSV = (EPI & 16) ? 8 : 1;
      uint4 mk_n[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
      float4 sv_n[NSV];
      auto fetch = [&](int cc) {
        const int col = n0 + cc;
        const bool ok = row < M && col < N;
        if (EPI & 4) {
          const uint4* mp = reinterpret_cast<const uint4*>(sc.mask_in + (int64_t)row * sc.ldc + col);
          mk_n[0] = ok ? __ldg(mp) : make_uint4(0, 0, 0, 0);
          mk_n[1] = ok ? __ldg(mp + 1) : make_uint4(0, 0, 0, 0);
        }
        if (EPI & 16) {
          const float4* sp = reinterpret_cast<const float4*>(sc.elu_saved + (int64_t)row * sc.ldc + col);
#pragma unroll
          for (int j = 0; j < NSV; ++j) sv_n[j] = ok ? __ldg(sp + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      };
      bool drained = false;
      if constexpr (BN <= 128) {
        if (sc.drain) {
          // k-block drain: sum the per-k-block partials in fp32 registers
          // (round-to-nearest, fixed order), then put the tile's sum back in
          // the last k-block's accumulator for the epilogue below
          float sum[BN];
#pragma unroll
          for (int j = 0; j < BN; ++j) sum[j] = 0.f;
          const int ng = sc.drain_group == 1 ? nk : (nk + 1) >> 1;
          for (int ks = 0; ks < ng; ++ks, ++dr) {
            const int b = dr % 3;
            mbar_wait(&tfull[b], (dr / 3) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * BN);
            // two-deep pipeline: the 8-column load c + 8 is in flight while
            // columns c are added (same adds, same order; 8-wide keeps the
            // BN sums plus both buffers inside the register budget)
            uint32_t ra[8], rb[8];
            tmem_ld8_async(ta, ra);
#pragma unroll
            for (int c = 0; c < BN; c += 16) {
              tmem_wait8(ra);
              tmem_ld8_async(ta + c + 8, rb);
#pragma unroll
              for (int j = 0; j < 8; ++j)
                sum[c + j] = __fadd_rn(sum[c + j], __uint_as_float(ra[j]));
              tmem_wait8(rb);
              if (c + 16 < BN) tmem_ld8_async(ta + c + 16, ra);
#pragma unroll
              for (int j = 0; j < 8; ++j)
                sum[c + 8 + j] = __fadd_rn(sum[c + 8 + j], __uint_as_float(rb[j]));
            }
            if (ks + 1 < ng) {
              asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
              __syncwarp();
              if (lane == 0) mbar_arrive(&tempty[b]);
            } else {
              abuf = b;
#pragma unroll
              for (int c = 0; c < BN; c += 32) {
                uint32_t r[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(sum[c + j]);
                tmem_st32(ta + c, r);
              }
              asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
          }
          drained = true;
        }
      }
      if (!drained) {
        if (EPI & 20) fetch(0);  // overlaps the wait for the accumulator
        mbar_wait(&tfull[abuf], (tl >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      } else if (EPI & 20) {
        fetch(0);  // after the drain: its registers are free again
      }
      float ss = 0.f, sd = 0.f;  // fused node scores of the current head
      int hrem = sc.k >> 2, head = (EPI & 8) ? n0 / sc.k : 0;
      // k = 32 with 4 heads per 128-wide tile (h % 4 == 0): a row's four
      // head scores leave as one 16-byte store per array at the tile's end
      const bool vsc = (EPI & 1) && !(EPI & 8) && BN == 128 && sc.k == 32 &&
                       (sc.h & 3) == 0 && (N & 127) == 0 &&
                       ((reinterpret_cast<uintptr_t>(sc.s) | reinterpret_cast<uintptr_t>(sc.d)) & 15) == 0;
      float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f), d4 = s4;
      // software pipeline over the 32-column chunks: the TMEM load of chunk
      // c + 32 (and lane j's bias of its column j) is in flight while chunk c
      // is processed, and the accumulator goes back to the MMA warp as soon as
      // its last chunk is in registers
      const uint32_t tacc = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(abuf * BN);
      // Only the ELU forward epilogue (exp per element) gains from it:
      // measured, the plain / bias / ReLU epilogues are 4 us slower with it
      // (X.Theta 80 -> 84 us), the ELU one 131 -> 96 us faster
      constexpr bool PIPE = (EPI & 32) != 0;
      const float* bsh = (PIPE && tma_store && !part) ? bias : nullptr;  // bias by shuffle
      uint32_t rn[32];
      if constexpr (PIPE) tmem_ld32_async(tacc, rn);
      float bnx = (bsh && n0 + lane < N) ? __ldg(bsh + n0 + lane) : 0.f;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        uint4 mk[2];
        float4 sv[NSV];
        if constexpr (PIPE) {
          tmem_wait32(rn);
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = rn[j];
        } else {
          tmem_ld32(tacc + c, r);
        }
        const float bcur = bnx;
        if (c + 32 < BN) {
          if constexpr (PIPE) tmem_ld32_async(tacc + c + 32, rn);
          if (bsh) bnx = (n0 + c + 32 + lane < N) ? __ldg(bsh + n0 + c + 32 + lane) : 0.f;
        } else {
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[abuf]);
        }
        if (EPI & 20) {
          mk[0] = mk_n[0];
          mk[1] = mk_n[1];
#pragma unroll
          for (int j = 0; j < NSV; ++j) sv[j] = sv_n[j];
          if (c + 32 < BN) fetch(c + 32);
        }
        if ((EPI & 1) && n0 + c < N) {
          // s[i,t] = sum_c a_src[t,c] M[i,tk+c] (kernels.hpp:385-423): a_src is h x k
          // row-major, so its flat index is the output column; k % 4 == 0 and
          // BN % k == 0, so a head is whole within this tile and ends on a
          // float4 boundary (hrem counts the head's float4 groups still to come)
          const int col0 = n0 + c;
          const float4* as4 = reinterpret_cast<const float4*>(sc.a_src + col0);
          const float4* ad4 = reinterpret_cast<const float4*>(sc.a_dst + col0);
          if (!(EPI & 8)) {  // k % 32 == 0: heads of whole 32-column chunks, one flush per chunk
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // warp-uniform 16-byte loads (L1 broadcast)
              const float4 as = __ldg(as4 + j), ad = __ldg(ad4 + j);
              const float m0 = __uint_as_float(r[4 * j]), m1 = __uint_as_float(r[4 * j + 1]);
              const float m2 = __uint_as_float(r[4 * j + 2]), m3 = __uint_as_float(r[4 * j + 3]);
              ss = fmaf(m3, as.w, fmaf(m2, as.z, fmaf(m1, as.y, fmaf(m0, as.x, ss))));
              sd = fmaf(m3, ad.w, fmaf(m2, ad.z, fmaf(m1, ad.y, fmaf(m0, ad.x, sd))));
            }
            if (vsc) {  // shift the head's scores in; store after the 4th head
              s4 = make_float4(s4.y, s4.z, s4.w, ss);
              d4 = make_float4(d4.y, d4.z, d4.w, sd);
              if (c + 32 == BN && row < M) {
                *reinterpret_cast<float4*>(sc.s + (int64_t)row * sc.h + n0 / 32) = s4;
                *reinterpret_cast<float4*>(sc.d + (int64_t)row * sc.h + n0 / 32) = d4;
              }
              ss = sd = 0.f;
            } else if ((col0 + 32) % sc.k == 0) {
              if (row < M) {
                sc.s[(int64_t)row * sc.h + col0 / sc.k] = ss;
                sc.d[(int64_t)row * sc.h + col0 / sc.k] = sd;
              }
              ss = sd = 0.f;
            }
          } else {  // EPI bit 3, k % 4 == 0: a head may end at any float4 of the chunk
            const int jn = min(8, (N - col0) >> 2);  // float4 groups inside N
            // all loads first (the flush stores below could alias them, so the
            // compiler would not hoist them); clamped, so always in bounds --
            // groups past N only feed a sum that is never stored
            float4 as[8], ad[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              as[j] = __ldg(as4 + min(j, jn - 1));
              ad[j] = __ldg(ad4 + min(j, jn - 1));
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float m0 = __uint_as_float(r[4 * j]), m1 = __uint_as_float(r[4 * j + 1]);
              const float m2 = __uint_as_float(r[4 * j + 2]), m3 = __uint_as_float(r[4 * j + 3]);
              ss = fmaf(m3, as[j].w, fmaf(m2, as[j].z, fmaf(m1, as[j].y, fmaf(m0, as[j].x, ss))));
              sd = fmaf(m3, ad[j].w, fmaf(m2, ad[j].z, fmaf(m1, ad[j].y, fmaf(m0, ad[j].x, sd))));
              if (j < jn && --hrem == 0) {
                if (row < M) {
                  sc.s[(int64_t)row * sc.h + head] = ss;
                  sc.d[(int64_t)row * sc.h + head] = sd;
                }
                ss = sd = 0.f;
                hrem = sc.k >> 2;
                ++head;
              }
            }
          }
        }
        if (tma_store) {
          // stage the 32 x 32 block in smem (SWIZZLE_128B: 16 B chunk j of row
          // `lane` at chunk j ^ (lane & 7), conflict-free) and let TMA write
          // full 128 B row segments (clipped at M, N)
          uint8_t* buf = epi + q * 8192 + (ecnt & 1) * 4096;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
          const int col0 = n0 + c;
          const bool mrow = row < M && col0 < N;  // masks need N % 32 == 0 (host)
          uint32_t mo[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 v = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                   __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
            if (!bsh && bias && col0 + 4 * j < N) {
              const float4 b = __ldg(reinterpret_cast<const float4*>(bias + col0 + 4 * j));
              v.x = __fadd_rn(v.x, b.x);
              v.y = __fadd_rn(v.y, b.y);
              v.z = __fadd_rn(v.z, b.z);
              v.w = __fadd_rn(v.w, b.w);
            }
            if (bsh) {  // columns past N add lane 0's 0.f and are clipped by TMA
              const float4 b = make_float4(__shfl_sync(0xffffffffu, bcur, 4 * j),
                                           __shfl_sync(0xffffffffu, bcur, 4 * j + 1),
                                           __shfl_sync(0xffffffffu, bcur, 4 * j + 2),
                                           __shfl_sync(0xffffffffu, bcur, 4 * j + 3));
              v.x = __fadd_rn(v.x, b.x);
              v.y = __fadd_rn(v.y, b.y);
              v.z = __fadd_rn(v.z, b.z);
              v.w = __fadd_rn(v.w, b.w);
            }
            if (EPI & 2) {
              mo[j] = (v.x > 0.f ? 1u : 0u) | (v.y > 0.f ? 1u : 0u) << 8 |
                      (v.z > 0.f ? 1u : 0u) << 16 | (v.w > 0.f ? 1u : 0u) << 24;
              if constexpr ((EPI & 32) != 0) {  // ELU(1), as k_act_fwd
                // exp for every element, then a select: a branch around each
                // expf serialises the chunk (3x slower epilogue, measured)
                const float ex = expf(v.x) - 1.f, ey = expf(v.y) - 1.f;
                const float ez = expf(v.z) - 1.f, ew = expf(v.w) - 1.f;
                v.x = v.x > 0.f ? v.x : ex;
                v.y = v.y > 0.f ? v.y : ey;
                v.z = v.z > 0.f ? v.z : ez;
                v.w = v.w > 0.f ? v.w : ew;
              } else {
                v.x = v.x > 0.f ? v.x : 0.f;
                v.y = v.y > 0.f ? v.y : 0.f;
                v.z = v.z > 0.f ? v.z : 0.f;
                v.w = v.w > 0.f ? v.w : 0.f;
              }
            }
            if ((EPI & 4) && !(EPI & 16)) {
              const uint32_t w = (&mk[j >> 2].x)[j & 3];
              v.x = (w & 0xffu) ? v.x : 0.f;
              v.y = (w & 0xff00u) ? v.y : 0.f;
              v.z = (w & 0xff0000u) ? v.z : 0.f;
              v.w = (w & 0xff000000u) ? v.w : 0.f;
            }
            if constexpr ((EPI & 16) != 0) {  // same rounding as the separate pass
              const uint32_t w = (&mk[j >> 2].x)[j & 3];
              const float4 e = sv[j];
              v.x = (w & 0xffu) ? v.x : __fmul_rn(__fadd_rn(e.x, 1.f), v.x);
              v.y = (w & 0xff00u) ? v.y : __fmul_rn(__fadd_rn(e.y, 1.f), v.y);
              v.z = (w & 0xff0000u) ? v.z : __fmul_rn(__fadd_rn(e.z, 1.f), v.z);
              v.w = (w & 0xff000000u) ? v.w : __fmul_rn(__fadd_rn(e.w, 1.f), v.w);
            }
            sts_f32x4(smem_u32(buf) + lane * 128 + ((j ^ (lane & 7)) << 4), v);
          }
          if ((EPI & 2) && mrow) {
            uint4* mp = reinterpret_cast<uint4*>(sc.relu_out + (int64_t)row * sc.ldc + col0);
            mp[0] = make_uint4(mo[0], mo[1], mo[2], mo[3]);
            mp[1] = make_uint4(mo[4], mo[5], mo[6], mo[7]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) tma_store_2d(&tmC, buf, col0, m0 + q * 32);
          ++ecnt;
          continue;
        }
        if (row >= M) continue;
        const int col0 = n0 + c;
        float* dst = part ? part + ((int64_t)z * M + row) * N : C + (int64_t)row * ldc;
        const float* bb = part ? nullptr : bias;
        if (vec && col0 + 32 <= N) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 v = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                   __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
            if (bb) {
              const float4 b = __ldg(reinterpret_cast<const float4*>(bb + col0 + j));
              v.x = __fadd_rn(v.x, b.x);
              v.y = __fadd_rn(v.y, b.y);
              v.z = __fadd_rn(v.z, b.z);
              v.w = __fadd_rn(v.w, b.w);
            }
            *reinterpret_cast<float4*>(dst + col0 + j) = v;
          }
        } else {
          for (int j = 0; j < 32; ++j)
            if (col0 + j < N)
              dst[col0 + j] = bb ? __fadd_rn(__uint_as_float(r[j]), bb[col0 + j])
                                 : __uint_as_float(r[j]);
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(CF::TMEM_COLS));
  }
}

// C = sum over split partials (+ bias).  Block = 32 consecutive outputs x 8
// split groups; each thread folds every 8th split in float64, then a fixed
// smem tree -- deterministic, and 8x the memory parallelism of one thread per
// output (the split count is ~num_sms / tiles, ~74 for dTheta).
__global__ void __launch_bounds__(256) k_reduce_splits(int splits, int64_t MN, int N,
                                                       const float* __restrict__ part,
                                                       float* __restrict__ C, int ldc,
                                                       const float* __restrict__ bias,
                                                       int cs_parts = 0,
                                                       const double* __restrict__ cs_part = nullptr,
                                                       float* __restrict__ cs_out = nullptr) {
  __shared__ double sh[8][33];
  const int g = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int64_t nbc = (MN + 31) / 32;
  if (blockIdx.x >= nbc) {  // the fused column sums (d_bias) of the same GEMM
    const int n = (int)((blockIdx.x - nbc) * 32 + l);
    double s = 0.0;
    if (n < N)
      for (int p = g; p < cs_parts; p += 8) s += cs_part[(int64_t)p * N + n];
    sh[g][l] = s;
    __syncthreads();
    if (g == 0 && n < N) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) t += sh[k][l];
      cs_out[n] = (float)t;
    }
    return;
  }
  const int64_t x = blockIdx.x * 32LL + l;
  double s = 0.0;
  if (x < MN) {
#pragma unroll 4
    for (int z = g; z < splits; z += 8) s += (double)part[(int64_t)z * MN + x];
  }
  sh[g][l] = s;
  __syncthreads();
  if (g == 0 && x < MN) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sh[k][l];
    const int64_t row = x / N, col = x % N;
    float v = (float)t;
    if (bias) v = __fadd_rn(v, bias[col]);
    C[row * ldc + col] = v;
  }
}

// out[n] = sum over (z, warp) of the converters' column-sum partials: one
// block per column, threads stride the partials, then a fixed-order smem tree
// (deterministic; a few L2 round trips instead of parts / 32 dependent ones)
__global__ void __launch_bounds__(256) k_colsum_parts(int parts, int N,
                                                      const double* __restrict__ cs_part,
                                                      float* __restrict__ out) {
  __shared__ double sh[256];
  const int n = blockIdx.x;
  double s = 0.0;
  for (int p = threadIdx.x; p < parts; p += 256) s += cs_part[(int64_t)p * N + n];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = (float)sh[0];
}

// ---- host side -------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D fp32 tensor map over a row-major [outer][inner] array with leading
// dimension ld (elements), box {32, box_outer}, 128-byte swizzle, OOB -> 0
static bool make_map(CUtensorMap* m, const float* base, int64_t inner, int64_t outer, int64_t ld,
                     int box_outer, bool mn_major) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {32u, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

struct Maps {
  CUtensorMap a, b, blo, c;
};

template <bool A_MN, bool B_MN, int BN, bool B_PRE, int EPI>
static void launch(sgnn_ctx ctx, const Maps& mp, int M, int N, int K, int splits, int kchunk,
                   float* C, const float* bias, float* part, int tma_store, double* cs_part,
                   const EpiScores& sc) {
  auto kern = k_gemm_tc<A_MN, B_MN, BN, B_PRE, EPI>;
  const int smem = Cfg<BN>::SMEM;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    SGNN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set = true;
  }
  const int64_t tiles = ceil_div(N, BN) * ceil_div(M, BM) * splits;
  const int grid = (int)std::min<int64_t>(tiles, ctx->num_sms);
  kern<<<grid, NUM_THREADS, smem, ctx->stream>>>(mp.a, mp.b, mp.blo, mp.c, M, N, K, kchunk,
                                                  splits, C, sc.ldc ? sc.ldc : N, bias, part,
                                                  tma_store, cs_part, sc);
  launched(ctx);
}

template <int BN>
static void dispatch(sgnn_ctx ctx, bool a_mn, bool b_mn, bool pre, const Maps& mp, int M, int N,
                     int K, int splits, int kchunk, float* C, const float* bias, float* part,
                     int tma_store, double* cs_part, const EpiScores& sc) {
#define L(AM, BM_, PR) \
  launch<AM, BM_, BN, PR, 0>(ctx, mp, M, N, K, splits, kchunk, C, bias, part, tma_store, cs_part, sc)
  // epilogue extras: only the shapes that use them are instantiated (the
  // caller checked a_mn == false and pre == true)
  if (sc.a_src && sc.k % 32 == 0) {
    if (b_mn) launch<false, true, BN, true, 1>(ctx, mp, M, N, K, splits, kchunk, C, bias, part, tma_store, cs_part, sc);
    else launch<false, false, BN, true, 1>(ctx, mp, M, N, K, splits, kchunk, C, bias, part, tma_store, cs_part, sc);
    return;
  }
  if (sc.a_src) {
    if (b_mn) launch<false, true, BN, true, 9>(ctx, mp, M, N, K, splits, kchunk, C, bias, part, tma_store, cs_part, sc);
    else launch<false, false, BN, true, 9>(ctx, mp, M, N, K, splits, kchunk, C, bias, part, tma_store, cs_part, sc);
    return;
  }
  if (sc.relu_out && sc.elu) {
    if (b_mn) launch<false, true, BN, true, 34>(ctx, mp, M, N, K, splits, kchunk, C, bias, part, tma_store, cs_part, sc);
    else launch<false, false, BN, true, 34>(ctx, mp, M, N, K, splits, kchunk, C, bias, part, tma_store, cs_part, sc);
    return;
  }
  if (sc.relu_out) {
    if (b_mn) launch<false, true, BN, true, 2>(ctx, mp, M, N, K, splits, kchunk, C, bias, part, tma_store, cs_part, sc);
    else launch<false, false, BN, true, 2>(ctx, mp, M, N, K, splits, kchunk, C, bias, part, tma_store, cs_part, sc);
    return;
  }
  if (sc.mask_in && sc.elu_saved) {
    if (b_mn) launch<false, true, BN, true, 20>(ctx, mp, M, N, K, splits, kchunk, C, bias, part, tma_store, cs_part, sc);
    else launch<false, false, BN, true, 20>(ctx, mp, M, N, K, splits, kchunk, C, bias, part, tma_store, cs_part, sc);
    return;
  }
  if (sc.mask_in) {
    if (b_mn) launch<false, true, BN, true, 4>(ctx, mp, M, N, K, splits, kchunk, C, bias, part, tma_store, cs_part, sc);
    else launch<false, false, BN, true, 4>(ctx, mp, M, N, K, splits, kchunk, C, bias, part, tma_store, cs_part, sc);
    return;
  }
  if (pre) {
    if (a_mn && b_mn) L(true, true, true);
    else if (a_mn) L(true, false, true);
    else if (b_mn) L(false, true, true);
    else L(false, false, true);
  } else {
    if (a_mn && b_mn) L(true, true, false);
    else if (a_mn) L(true, false, false);
    else if (b_mn) L(false, true, false);
    else L(false, false, false);
  }
#undef L
}

}  // namespace tc

static bool tc_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SGNN_DISABLE_TCGEN05");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

bool gemm_tc_available() { return !tc_disabled(); }

// Zero-padded copy of a rows x cols row-major matrix (pitch ld) into an
// orows x ocols one: TMA needs 16-byte row pitches, so operands whose stored
// width is not a multiple of 4 floats (Cora's 1433 input features) are staged
// with zero columns (and zero K rows) -- the extra products are exact zeros.
__global__ void k_pad2d(int32_t rows, int32_t cols, const float* __restrict__ src, int32_t ld,
                        int32_t orows, int32_t ocols, float* __restrict__ dst) {
  // a warp per output row (grid-stride), lanes over columns: coalesced
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < orows;
       r += nw) {
    const float* s = src + r * ld;
    float* d = dst + r * ocols;
    if (r < rows) {
      for (int32_t c = lane; c < ocols; c += 32) d[c] = c < cols ? __ldg(s + c) : 0.f;
    } else {
      for (int32_t c = lane; c < ocols; c += 32) d[c] = 0.f;
    }
  }
}

static int32_t round4(int32_t x) { return (x + 3) & ~3; }

// dst (rows x ocols) = src (rows x cols, pitch ld) + bias, dropping padding
__global__ void k_unpad2d(int32_t rows, int32_t ocols, const float* __restrict__ src, int32_t ld,
                          const float* __restrict__ bias, float* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
       r += nw)
    for (int32_t c = lane; c < ocols; c += 32) {
      const float v = __ldg(src + r * ld + c);
      dst[r * ocols + c] = bias ? v + __ldg(bias + c) : v;
    }
}

void pad_rows_f32(sgnn_ctx ctx, int32_t rows, int32_t cols, const float* src, int32_t ld,
                  int32_t ocols, float* dst) {
  k_pad2d<<<grid_for(ctx, (int64_t)rows * 32, 256), 256, 0, ctx->stream>>>(rows, cols, src, ld,
                                                                            rows, ocols, dst);
  launched(ctx);
}

void unpad_rows_f32(sgnn_ctx ctx, int32_t rows, int32_t ocols, const float* src, int32_t ld,
                    const float* bias, float* dst) {
  k_unpad2d<<<grid_for(ctx, (int64_t)rows * 32, 256), 256, 0, ctx->stream>>>(rows, ocols, src, ld,
                                                                              bias, dst);
  launched(ctx);
}

bool gemm_tc_f32(sgnn_ctx ctx, const float* A, int32_t ra, int32_t ca, const float* B,
                 int32_t rb, int32_t cb, bool ta, bool tb, float* C, const float* bias,
                 float* colsum_b, const float* att_src, const float* att_dst, float* s_out,
                 float* d_out, int heads, uint8_t* relu_out, const uint8_t* mask_in,
                 const float* elu_saved);

void gemm_presplit_f32(sgnn_ctx ctx, const float* B, int64_t elems, float* hi, float* lo) {
  tc::k_split_global<<<grid_for(ctx, elems, 256), 256, 0, ctx->stream>>>(elems, B, hi, lo);
  launched(ctx);
}
bool gemm_uses_presplit(int64_t elems, int32_t ra, int32_t ca) {
  return elems * 8 <= (int64_t)ra * ca;  // = `pre` in the launcher below
}

// Operands with stored widths that are not multiples of 4: stage padded
// copies (K padded with zeros on both operands, M / N padded as stored
// widths), run the tcgen05 GEMM on them and copy the M x N block back.
static bool gemm_tc_f32_padded(sgnn_ctx ctx, const float* A, int32_t ra, int32_t ca,
                               const float* B, int32_t rb, int32_t cb, bool ta, bool tb,
                               float* C, const float* bias, float* colsum_b,
                               const float* att_src, const float* att_dst, float* s_out,
                               float* d_out, int heads, uint8_t* relu_out,
                               const uint8_t* mask_in, const float* elu_saved) {
  const int32_t M = ta ? ca : ra, K = ta ? ra : ca, N = tb ? rb : cb;
  const int32_t K4 = round4(K), M2 = ta ? round4(M) : M, N2 = tb ? N : round4(N);
  const bool same_out = M2 == M && N2 == N;
  if (!same_out && (att_src || relu_out || mask_in || elu_saved)) return false;
  const int32_t ra2 = ta ? K4 : M, ca2 = ta ? M2 : K4, rb2 = tb ? N : K4, cb2 = tb ? K4 : N2;
  cudaStream_t st = ctx->stream;
  DevBuf a2((size_t)ra2 * ca2 * 4, st), b2((size_t)rb2 * cb2 * 4, st);
  k_pad2d<<<grid_for(ctx, (int64_t)ra2 * ca2, 256), 256, 0, st>>>(ra, ca, A, ca, ra2, ca2,
                                                                   a2.as<float>());
  launched(ctx);
  k_pad2d<<<grid_for(ctx, (int64_t)rb2 * cb2, 256), 256, 0, st>>>(rb, cb, B, cb, rb2, cb2,
                                                                   b2.as<float>());
  launched(ctx);
  DevBuf c2, bias2, cs2;
  float* Cp = C;
  const float* bp = bias;
  float* csp = colsum_b;
  if (!same_out) {
    c2 = DevBuf((size_t)M2 * N2 * 4, st);
    Cp = c2.as<float>();
    if (bias && N2 != N) {
      bias2 = DevBuf((size_t)N2 * 4, st);
      k_pad2d<<<1, 256, 0, st>>>(1, N, bias, N, 1, N2, bias2.as<float>());
      launched(ctx);
      bp = bias2.as<float>();
    }
    if (colsum_b && N2 != N) {
      cs2 = DevBuf((size_t)N2 * 4, st);
      csp = cs2.as<float>();
    }
  }
  if (!gemm_tc_f32(ctx, a2.as<float>(), ra2, ca2, b2.as<float>(), rb2, cb2, ta, tb, Cp, bp, csp,
                   att_src, att_dst, s_out, d_out, heads, relu_out, mask_in, elu_saved))
    return false;
  if (!same_out) {
    SGNN_CUDA(cudaMemcpy2DAsync(C, (size_t)N * 4, Cp, (size_t)N2 * 4, (size_t)N * 4, M,
                                cudaMemcpyDeviceToDevice, st));
    if (colsum_b && csp != colsum_b)
      SGNN_CUDA(cudaMemcpyAsync(colsum_b, csp, (size_t)N * 4, cudaMemcpyDeviceToDevice, st));
  }
  return true;
}

// Returns false (caller falls back to the SIMT kernel) when the shape or the
// operand alignment does not fit the TMA/UMMA path.  colsum_b (optional, only
// for C = A^T B with B read MN-major and split in the kernel): also writes the
// column sums of B over its K rows -- d_bias = 1^T dX' fused into the dTheta
// GEMM, so dX' is read once.  Returns false without doing anything if the
// fused form does not apply (the caller then runs the two ops separately).
static bool gemm_tc_f32_impl(sgnn_ctx ctx, const float* A, int32_t ra, int32_t ca, int32_t lda,
                             const float* B, int32_t rb, int32_t cb, int32_t ldb, bool ta, bool tb,
                             float* C, int32_t ldc, const float* bias, float* colsum_b,
                             const float* att_src, const float* att_dst, float* s_out,
                             float* d_out, int heads, uint8_t* relu_out, const uint8_t* mask_in,
                             const float* elu_saved, bool elu_out = false);

bool gemm_tc_f32(sgnn_ctx ctx, const float* A, int32_t ra, int32_t ca, const float* B,
                 int32_t rb, int32_t cb, bool ta, bool tb, float* C, const float* bias,
                 float* colsum_b, const float* att_src, const float* att_dst, float* s_out,
                 float* d_out, int heads, uint8_t* relu_out, const uint8_t* mask_in,
                 const float* elu_saved) {
  return gemm_tc_f32_impl(ctx, A, ra, ca, ca, B, rb, cb, cb, ta, tb, C, 0, bias, colsum_b,
                          att_src, att_dst, s_out, d_out, heads, relu_out, mask_in, elu_saved);
}

// C = op(A) op(B) (+ bias) on blocks of wider matrices: A, B, C with row
// pitches lda, ldb, ldc (elements, multiples of 4); e.g. one head's column
// block of an n x (h k) slab.  false (nothing launched) if not supported.
bool gemm_tc_f32_pitched(sgnn_ctx ctx, const float* A, int32_t ra, int32_t ca, int32_t lda,
                         const float* B, int32_t rb, int32_t cb, int32_t ldb, bool ta, bool tb,
                         float* C, int32_t ldc, const float* bias, float* colsum_b,
                         uint8_t* elu_mask) {
  if ((lda & 3) || (ldb & 3) || (ldc & 3)) return false;
  return gemm_tc_f32_impl(ctx, A, ra, ca, lda, B, rb, cb, ldb, ta, tb, C, ldc, bias, colsum_b,
                          nullptr, nullptr, nullptr, nullptr, 0, elu_mask, nullptr, nullptr,
                          elu_mask != nullptr);
}

static bool gemm_tc_f32_impl(sgnn_ctx ctx, const float* A, int32_t ra, int32_t ca, int32_t lda,
                             const float* B, int32_t rb, int32_t cb, int32_t ldb, bool ta, bool tb,
                             float* C, int32_t ldc, const float* bias, float* colsum_b,
                             const float* att_src, const float* att_dst, float* s_out,
                             float* d_out, int heads, uint8_t* relu_out, const uint8_t* mask_in,
                             const float* elu_saved, bool elu_out) {
  using namespace tc;
  if (tc_disabled()) return false;
  const int M = ta ? ca : ra, K = ta ? ra : ca, N = tb ? rb : cb;
  if (M <= 0 || N <= 0 || K <= 0) return false;
  const bool pitched = lda != ca || ldb != cb || (ldc != 0 && ldc != N);
  // tiny: SIMT is fine (pitched operands have no SIMT path)
  if (!pitched && (int64_t)M * N * K < (int64_t)1 << 20) return false;
  if (ldc <= 0) ldc = N;
  // pitched: output masks / column sums are fine, the fused scores and the
  // activation backward read row-major n x N side arrays
  if (pitched && (att_src || mask_in || elu_saved)) return false;
  if (elu_out && !relu_out) return false;
  static const bool no_pad = getenv("SGNN_NO_PAD") != nullptr;  // dev switch
  if (!pitched && ((ca & 3) || (cb & 3))) {  // 16-byte row pitches for TMA: stage padded operands
    if (no_pad) return false;
    return gemm_tc_f32_padded(ctx, A, ra, ca, B, rb, cb, ta, tb, C, bias, colsum_b, att_src,
                              att_dst, s_out, d_out, heads, relu_out, mask_in, elu_saved);
  }
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15)) return false;
  if ((reinterpret_cast<uintptr_t>(C) & 15) || (bias && (reinterpret_cast<uintptr_t>(bias) & 15)))
    return false;
  // 128 or 160 columns per tile, whichever pads N less (N = 320, the GAT
  // 8 x 40 slab: two exact 160-wide tiles instead of three 128-wide ones)
  int BN = N <= 32 ? 32
           : N <= 64 ? 64
           : (ceil_div(N, 160) * 160 < ceil_div(N, 128) * 128 ? 160 : 128);
  const bool a_mn = ta, b_mn = !tb;
  // K > 256 (every split-K GEMM included, e.g. dTheta = X^T dX' over K = n):
  // k-block drain mode (EpiScores::drain).  It keeps three accumulators in
  // TMEM and BN fp32 sums per thread, so BN <= 128; 160-wide tiles (N = 320,
  // the Gat2 8 x 40 slab, K = 2048) keep one accumulator per tile -- their
  // fused node scores need whole 40-wide heads per tile, and the model step
  // stays at 1.4e-5 of the float64 reference (tests/test_gpu_fullsize.py).
  const int ksteps = (int)ceil_div(K, BK);
  const bool drain = ksteps > 8 && BN <= 128;
  auto split_count = [&](int bn) {
    const int tl = (int)(ceil_div(M, BM) * ceil_div(N, bn));
    int sp = 1;
    if (tl < ctx->num_sms && ksteps >= 16) {
      // one wave: tiles * splits <= num_sms (a 149th tile would double the time)
      sp = (int)std::min<int64_t>(ctx->num_sms / tl, ksteps / 8);
      if (sp < 1) sp = 1;
    }
    // accuracy: a split sums its k-block results in float32 registers (drain
    // mode), so its rounding error grows with its k-block count.  Above
    // kMaxDrainBlocks per split (K > ~4k rows per split: config 5's dTheta
    // over n = 2.45M rows) use more splits -- several waves -- so the float32
    // part stays as short as at Arxiv and the splits combine in float64.
    static const int kMaxDrainBlocks = [] {  // dev knob SGNN_DRAIN_MAX (default 128)
      const char* e = getenv("SGNN_DRAIN_MAX");
      return e ? atoi(e) : 128;
    }();
    if (drain && ksteps > (int64_t)kMaxDrainBlocks * sp)
      sp = (int)ceil_div(ksteps, kMaxDrainBlocks);
    return sp;
  };
  // Small B (the parameter matrix Theta): split hi/lo once in global memory so
  // the kernel streams both halves with TMA and spends no smem bandwidth on it.
  const int64_t belems = (int64_t)rb * cb;
  const bool pre = belems * 8 <= (int64_t)ra * ca;
  if (colsum_b && (pre || !b_mn)) return false;
  DevBuf bsplit;
  const float* Bhi = B;
  const float* Blo = B;
  Maps mp;
  // A: ta -> stored K x M (MN-major), else M x K (K-major)
  const bool okA = a_mn ? make_map(&mp.a, A, M, K, lda, BK, true)
                        : make_map(&mp.a, A, K, M, lda, BM, false);
  if (!okA) return false;
  // the caller split B already (gemm_presplit_f32 on its side stream)
  const bool hinted = pre && ldb == cb && ctx->split_src == B && ctx->split_elems == belems;
  if (hinted) {
    Bhi = ctx->split_hi;
    Blo = ctx->split_lo;
  } else if (pre) {
    bsplit = DevBuf((size_t)belems * 8, ctx->stream);
    Bhi = bsplit.as<float>();
    Blo = bsplit.as<float>() + belems;
  }
  // B: tb -> stored N x K (K-major), else K x N (MN-major)
  const int32_t bld = pre ? cb : ldb;  // the pre-split copies are contiguous
  bool okB = b_mn ? make_map(&mp.b, Bhi, N, K, bld, BK, true)
                  : make_map(&mp.b, Bhi, K, N, bld, BN, false);
  okB = okB && (b_mn ? make_map(&mp.blo, Blo, N, K, bld, BK, true)
                     : make_map(&mp.blo, Blo, K, N, bld, BN, false));
  if (!okB) return false;
  int splits = split_count(BN);
  int kchunk = (int)ceil_div(ceil_div(K, splits), BK) * BK;
  {  // dev knob (accuracy experiments): force the split-K chunk length
    static const int forced = [] {
      const char* e = getenv("SGNN_GEMM_KCHUNK");
      return e ? atoi(e) : 0;
    }();
    if (forced > 0 && splits > 1) kchunk = (int)ceil_div(forced, BK) * BK;
  }
  splits = (int)ceil_div(K, kchunk);
  EpiScores sc;
  if (att_src) {  // fused node scores: whole heads per tile, no split-K, no bias
    const int hk = heads > 0 ? N / heads : 0;
    if (splits != 1 || bias || heads <= 0 || hk * heads != N || hk % 4 != 0 || BN % hk != 0 ||
        (reinterpret_cast<uintptr_t>(att_src) & 15) || (reinterpret_cast<uintptr_t>(att_dst) & 15))
      return false;
    sc.a_src = att_src;
    sc.a_dst = att_dst;
    sc.s = s_out;
    sc.d = d_out;
    sc.h = heads;
    sc.k = hk;
  }
  sc.relu_out = relu_out;
  sc.elu = elu_out;
  sc.mask_in = mask_in;
  sc.elu_saved = elu_saved;
  sc.drain = drain;
  {
    static const int kGroupMax = [] {  // dev knob SGNN_DRAIN_GROUP (default 2)
      const char* e = getenv("SGNN_DRAIN_GROUP");
      return (e && atoi(e) <= 1) ? 1 : 2;
    }();
    // split-K partials (dTheta over K = n: long, cancelling sums) keep
    // one k-block per partial; unsplit GEMMs up to K = 2048 group
    sc.drain_group = (drain && splits == 1 && K <= 2048) ? kGroupMax : 1;
  }
  if (elu_saved && (!mask_in || (reinterpret_cast<uintptr_t>(elu_saved) & 15))) return false;
  if ((sc.a_src || relu_out || mask_in) && (a_mn || !pre)) return false;
  // TMA-store epilogue for the final output (row pitch N*4 must be 16 B aligned)
  sc.ldc = ldc;
  const int tma_store = (splits == 1 && (N & 3) == 0 && (ldc & 3) == 0 &&
                         make_map(&mp.c, C, N, M, ldc, 32, false));
  if (!tma_store) mp.c = mp.a;  // unused
  if (relu_out || mask_in) {  // fused ReLU / ReLU backward: TMA-store epilogue, whole 32-col chunks
    if (!tma_store || (N & 31) != 0 || (reinterpret_cast<uintptr_t>(relu_out) & 15) ||
        (reinterpret_cast<uintptr_t>(mask_in) & 15))
      return false;
  }
  if (pre && !hinted) {
    if (ldb == cb)
      k_split_global<<<grid_for(ctx, belems, 256), 256, 0, ctx->stream>>>(
          belems, B, bsplit.as<float>(), bsplit.as<float>() + belems);
    else
      k_split_global2d<<<grid_for(ctx, belems, 256), 256, 0, ctx->stream>>>(
          rb, cb, B, ldb, bsplit.as<float>(), bsplit.as<float>() + belems);
    launched(ctx);
  }
  DevBuf part, csp;
  float* pp = nullptr;
  if (splits > 1) {
    part = DevBuf((size_t)splits * M * N * sizeof(float), ctx->stream);
    pp = part.as<float>();
  }
  double* cs = nullptr;
  if (colsum_b) {
    csp = DevBuf((size_t)splits * 4 * N * sizeof(double), ctx->stream);
    cs = csp.as<double>();
  }
  switch (BN) {
    case 32: dispatch<32>(ctx, a_mn, b_mn, pre, mp, M, N, K, splits, kchunk, C, bias, pp, tma_store, cs, sc); break;
    case 64: dispatch<64>(ctx, a_mn, b_mn, pre, mp, M, N, K, splits, kchunk, C, bias, pp, tma_store, cs, sc); break;
    case 160: dispatch<160>(ctx, a_mn, b_mn, pre, mp, M, N, K, splits, kchunk, C, bias, pp, tma_store, cs, sc); break;
    default: dispatch<128>(ctx, a_mn, b_mn, pre, mp, M, N, K, splits, kchunk, C, bias, pp, tma_store, cs, sc); break;
  }
  if (splits > 1) {
    const int64_t MN = (int64_t)M * N;
    // split-K partials -> C, and the fused column sums in the same launch
    const unsigned ncs = colsum_b ? (unsigned)ceil_div(N, 32) : 0u;
    k_reduce_splits<<<(unsigned)ceil_div(MN, 32) + ncs, 256, 0, ctx->stream>>>(
        splits, MN, N, pp, C, ldc, bias, splits * 4, cs, colsum_b);
    launched(ctx);
  } else if (colsum_b) {
    k_colsum_parts<<<(unsigned)N, 256, 0, ctx->stream>>>(splits * 4, N, cs, colsum_b);
    launched(ctx);
  }
  return true;
}

}  // namespace sgnn
