// tcgen05 3xTF32 GEMM on pre-split operands (contract in tc_gemm.cuh).
//
// One launch runs up to four independent problems (a dependency level of an
// intersect class). The flattened grid enumerates (problem, 128x80 tile,
// K-split); the S CTAs of a tile form a (S,1,1) thread-block cluster, each
// streams its K range through a 3-stage cp.async ring into 128B-swizzled
// K-major tiles, one thread issues the UMMAs, and the leader reduces the
// peers' fp32 partials over DSMEM in rank order (deterministic). Each K chunk
// accumulates in a fresh TMEM buffer and is folded into fp32 registers, which
// keeps the contraction at fp32 accuracy (the tensor core's accumulator loses
// precision over long runs). The epilogue stages the tile through shared
// memory so global reads/writes of C are row-coalesced.
//
// Two mainloops share that contract and epilogue:
//  * tc_gemm_tma_kernel (used whenever every operand row stride is a multiple
//    of 16 bytes): warp-specialised. Warp 0 streams hi/lo tiles of A and B with
//    TMA (cp.async.bulk.tensor, 128B swizzle, out-of-bounds rows / K zero-filled
//    by the copy engine) into a 4-stage mbarrier ring; warp 1's elected lane
//    issues the 12 UMMAs of a K chunk into one of two TMEM buffers and commits
//    to the stage's "empty" and the buffer's "full" barriers; warps 2-5 drain a
//    full buffer (tcgen05.ld), free it, and fold the chunk into fp32 registers
//    while the tensor core already works on the next chunk. The per-chunk fold
//    keeps the arithmetic (and the results) identical to the cp.async kernel.
//  * tc_gemm_kernel: all threads stream with cp.async (any row stride).
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "tc_gemm.cuh"

namespace ngdb_dev {
namespace {
// 0: split-K chosen per launch to fill the GPU; S > 0: every GEMM uses S (with
// S = 1 a row's result no longer depends on how many rows share the launch —
// the operator microbench verifies batched == per-op loop bit for bit)
std::atomic<int> g_split_override{0};
}  // namespace

namespace {

constexpr int BM = 128, BN = 80, BK = 32;
constexpr int kThreads = 256;   // 8 warps; warps w and w+4 share TMEM lane quarter w%4
constexpr int kStages = 2;      // smem operand ring; 104 KB -> two CTAs per SM
constexpr int kTmemCols = 256;  // 2 accumulator buffers of BN columns (power of two)
constexpr int kHalfCols = BN / 2;
constexpr int kMaxProblems = 4;

constexpr int A_TILE = BM * BK * 4;  // 16 KB (128 rows x 128 B)
constexpr int B_TILE = BN * BK * 4;  // 10 KB
constexpr int STAGE = 2 * A_TILE + 2 * B_TILE;  // A_hi, A_lo, B_hi, B_lo
constexpr int SMEM_BYTES = kStages * STAGE + 64;
// epilogue staging tile [BM][BN+4]: 16-byte aligned rows; float4 stores of a
// quarter-warp (8 consecutive rows) and float4 reads along a row are
// bank-conflict free
constexpr int kTileStride = BN + 4;

struct TcGemmBatch {
  TcGemmArgs p[kMaxProblems];
  int tile_begin[kMaxProblems + 1];
  int n;
  int S;  // K-split factor == cluster size
};

// UMMA instruction descriptor: D=f32, A=B=tf32, both K-major, M=128, N=80.
constexpr uint32_t kInstrDesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major operand tile, 128B swizzle, 8-row atoms of 1024 B (SBO = 1024 B).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3fff) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}

// MN-major operand tile (tf32 admits only the 128B swizzle with 32-byte
// atoms, UMMA layout type SWIZZLE_128B_BASE32B = 1, Swizzle<2,5,2>): per
// 32-row block (4096 B, one TMA box {32 rows, 32 K} with
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) a 128-byte line holds 32 consecutive
// rows at one k, 4-line (4-k) atoms of 512 B. LBO = 4096 B (next 32-row
// block), SBO = 512 B (next 4-k atom); one tf32 UMMA (k = 8) spans two atoms.
__device__ __forceinline__ uint64_t umma_desc_mn(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3fff) | (static_cast<uint64_t>(4096 >> 4) << 16) |
         (static_cast<uint64_t>(512 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(1) << 61);
}
constexpr int kMnBlock = 32 * BK * 4;  // bytes of one 32-row MN-major block (4096)

// byte offset of the 16-byte chunk (row r, k4 = k/4) in a swizzled K-major tile
__device__ __forceinline__ uint32_t swz16(int r, int k4) {
  return static_cast<uint32_t>(r * 128 + ((k4 ^ (r & 7)) << 4));
}

__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);  // round to 10-bit mantissa
  lo = x - hi;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity));
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kInstrDesc), "r"(acc));
}

// Per-thread copy slots: every chunk this thread copies the same (row, k4)
// 16-byte pieces — 4 rows of A and up to 3 rows of B, each for hi and lo.
struct CopyPlan {
  int64_t a_off[4], b_off[3];  // element offsets of (row, 4*k4) in the hi/lo arrays
  uint32_t a_dst[4], b_dst[3];
  bool a_ok[4], b_ok[3];
  int kk;                      // 4*k4
};

__device__ __forceinline__ void make_copy_plan(const TcGemmArgs& g, int m0, int n0, CopyPlan& cp) {
  const int k4 = threadIdx.x & 7, r0 = threadIdx.x >> 3;
  cp.kk = 4 * k4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + 32 * i;
    cp.a_ok[i] = (m0 + r) < g.M;
    cp.a_off[i] = (int64_t)(m0 + r) * g.A.ld + cp.kk;
    cp.a_dst[i] = swz16(r, k4);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int r = r0 + 32 * i;
    cp.b_ok[i] = r < BN && (n0 + r) < g.N;
    cp.b_off[i] = (int64_t)(n0 + r) * g.B.ld + cp.kk;
    cp.b_dst[i] = swz16(r < BN ? r : 0, k4);
  }
}

__device__ __forceinline__ void load_chunk(const TcGemmArgs& g, const CopyPlan& cp, int kc,
                                           uint32_t st) {
  const int k0 = kc * BK;
  const bool kok = (k0 + cp.kk) < g.K;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool ok = cp.a_ok[i] && kok;
    cp_async16(st + cp.a_dst[i], ok ? g.A.hi + cp.a_off[i] + k0 : g.A.hi, ok);
    cp_async16(st + A_TILE + cp.a_dst[i], ok ? g.A.lo + cp.a_off[i] + k0 : g.A.lo, ok);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    if (threadIdx.x + 256 * i >= BN * 8) break;  // rows beyond the 80-row tile
    const bool ok = cp.b_ok[i] && kok;
    cp_async16(st + 2 * A_TILE + cp.b_dst[i], ok ? g.B.hi + cp.b_off[i] + k0 : g.B.hi, ok);
    cp_async16(st + 2 * A_TILE + B_TILE + cp.b_dst[i], ok ? g.B.lo + cp.b_off[i] + k0 : g.B.lo, ok);
  }
}

// acc[0..39] += this thread's 40 accumulator columns of TMEM buffer `buf`
__device__ __forceinline__ void drain(uint32_t tmem, int buf, float* acc) {
  const int warp = threadIdx.x / 32;
  const uint32_t base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + buf * BN +
                        (warp >> 2) * kHalfCols;
  uint32_t r[kHalfCols];
#pragma unroll
  for (int j = 0; j < kHalfCols; j += 8)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[j]), "=r"(r[j + 1]), "=r"(r[j + 2]), "=r"(r[j + 3]), "=r"(r[j + 4]),
                   "=r"(r[j + 5]), "=r"(r[j + 6]), "=r"(r[j + 7])
                 : "r"(base + j));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
  for (int j = 0; j < kHalfCols; ++j) acc[j] += __uint_as_float(r[j]);
}

// Split-K reduce-scatter over distributed shared memory plus the epilogue:
// CTA `rank` owns rows [r_beg, r_end) of the tile, sums them over the S
// partial tiles in rank order (deterministic) and writes them out (bias, ReLU
// mask, accumulate, row scatter, chained split).
template <int TBN = BN>
__device__ __forceinline__ void store_tile(const TcGemmArgs& g, float* tile_s, int m0, int n0,
                                           int r_beg, int r_end, int rank, int S, int nthreads) {
  constexpr int kTileStride = TBN + 4;
  const int warp = threadIdx.x / 32;
  const uint32_t local = smem_u32(tile_s);
  if (((g.N | g.ldc) & 3) == 0) {
    // float4 epilogue: thread t takes 16-byte column groups of the CTA's rows;
    // the S partial loads are all issued before they are summed
    constexpr int kQ = TBN / 4;
    const int n_items = (r_end - r_beg) * kQ;
    for (int it = threadIdx.x; it < n_items; it += nthreads) {
      const int r = r_beg + it / kQ, cq = (it % kQ) * 4;
      const int row = m0 + r, n = n0 + cq;
      if (row >= g.M || n >= g.N) continue;
      const uint32_t off = static_cast<uint32_t>((r * kTileStride + cq) * 4);
      float4 part[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        if (p >= S) break;
        if (p == rank) {
          part[p] = *reinterpret_cast<const float4*>(&tile_s[r * kTileStride + cq]);
        } else {
          uint32_t remote;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local + off), "r"(p));
          asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
                       : "=f"(part[p].x), "=f"(part[p].y), "=f"(part[p].z), "=f"(part[p].w)
                       : "r"(remote));
        }
      }
      float4 v = part[0];
#pragma unroll
      for (int p = 1; p < 8; ++p) {
        if (p >= S) break;
        v.x += part[p].x; v.y += part[p].y; v.z += part[p].z; v.w += part[p].w;
      }
      float* crow =
          g.c_rowoff ? g.C + g.c_rowoff[(int64_t)row * g.c_stride] : g.C + (int64_t)row * g.ldc;
      if (g.bias) {
        const float4 b = *reinterpret_cast<const float4*>(g.bias + n);
        v.x += b.x; v.y += b.y; v.z += b.z; v.w += b.w;
      }
      if (g.mask) {
        const float4 mk = *reinterpret_cast<const float4*>(g.mask + (int64_t)row * g.ldc + n);
        if (!(mk.x > 0.f)) v.x = 0.f;
        if (!(mk.y > 0.f)) v.y = 0.f;
        if (!(mk.z > 0.f)) v.z = 0.f;
        if (!(mk.w > 0.f)) v.w = 0.f;
      }
      if (g.accumulate) {
        const float4 c0 = *reinterpret_cast<const float4*>(crow + n);
        v.x += c0.x; v.y += c0.y; v.z += c0.z; v.w += c0.w;
      }
      if (g.sigmoid) {
        v.x = sigmoidf(v.x); v.y = sigmoidf(v.y); v.z = sigmoidf(v.z); v.w = sigmoidf(v.w);
      }
      *reinterpret_cast<float4*>(crow + n) = v;
      if (g.s_hi) {
        float4 h, l;
        const float4 u = g.s_relu ? make_float4(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f), fmaxf(v.z, 0.f),
                                                fmaxf(v.w, 0.f))
                                  : v;
        split_tf32(u.x, h.x, l.x);
        split_tf32(u.y, h.y, l.y);
        split_tf32(u.z, h.z, l.z);
        split_tf32(u.w, h.w, l.w);
        *reinterpret_cast<float4*>(g.s_hi + (int64_t)row * g.ldc + n) = h;
        *reinterpret_cast<float4*>(g.s_lo + (int64_t)row * g.ldc + n) = l;
      }
    }
  } else {
    const int lane = threadIdx.x & 31;
    for (int r = r_beg + warp; r < r_end; r += nthreads / 32) {
      const int row = m0 + r;
      if (row >= g.M) break;
      float* crow =
          g.c_rowoff ? g.C + g.c_rowoff[(int64_t)row * g.c_stride] : g.C + (int64_t)row * g.ldc;
      for (int cc = lane; cc < TBN; cc += 32) {
        const int n = n0 + cc;
        if (n >= g.N) break;
        float v = 0.f;
        const uint32_t off = static_cast<uint32_t>((r * kTileStride + cc) * 4);
        for (int p = 0; p < S; ++p) {
          if (p == rank) {
            v += tile_s[r * kTileStride + cc];
          } else {
            uint32_t remote;
            float pv;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local + off), "r"(p));
            asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(pv) : "r"(remote));
            v += pv;
          }
        }
        if (g.bias) v += g.bias[n];
        if (g.mask && !(g.mask[(int64_t)row * g.ldc + n] > 0.f)) v = 0.f;
        if (g.accumulate) v += crow[n];
        if (g.sigmoid) v = sigmoidf(v);
        crow[n] = v;
        if (g.s_hi) {
          float h, l;
          split_tf32(g.s_relu ? fmaxf(v, 0.f) : v, h, l);
          g.s_hi[(int64_t)row * g.ldc + n] = h;
          g.s_lo[(int64_t)row * g.ldc + n] = l;
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads, 2) tc_gemm_kernel(const __grid_constant__ TcGemmBatch batch) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t s_base = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * STAGE);  // [kStages]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kStages);

  // flattened grid -> (problem, tile, K-split rank)
  const int S = batch.S;
  const int tile = blockIdx.x / S, rank = blockIdx.x % S;
  int pi = 0;
  while (pi + 1 < batch.n && tile >= batch.tile_begin[pi + 1]) ++pi;
  const TcGemmArgs& g = batch.p[pi];
  const int lt = tile - batch.tile_begin[pi];
  const int n_tiles_n = (g.N + BN - 1) / BN;
  const int m0 = (lt / n_tiles_n) * BM, n0 = (lt % n_tiles_n) * BN;
  const int warp = threadIdx.x / 32;
  const int total_chunks = (g.K + BK - 1) / BK;
  const int c_beg = rank * total_chunks / S;
  const int n_chunks = (rank + 1) * total_chunks / S - c_beg;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(smem_u32(&bars[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  CopyPlan cp;
  make_copy_plan(g, m0, n0, cp);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  // barrier init, TMEM allocation and copy planning overlap the previous kernel
  pdl_start();
  float acc[kHalfCols];
#pragma unroll
  for (int j = 0; j < kHalfCols; ++j) acc[j] = 0.f;

  for (int c = 0; c < kStages - 1; ++c) {
    if (c < n_chunks) load_chunk(g, cp, c_beg + c, s_base + c * STAGE);
    asm volatile("cp.async.commit_group;");
  }
  for (int c = 0; c < n_chunks; ++c) {
    const int st = c % kStages;
    asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 2));  // chunk c has landed
    asm volatile("fence.proxy.async.shared::cta;");             // cp.async -> tensor-core proxy
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a_hi = s_base + st * STAGE, a_lo = a_hi + A_TILE;
      const uint32_t b_hi = a_hi + 2 * A_TILE, b_lo = b_hi + B_TILE;
      const uint32_t d = tmem + (c & 1) * BN;
#pragma unroll
      for (int ks = 0; ks < BK / 8; ++ks) {  // UMMA K = 8 tf32 = 32 bytes; small terms first
        const uint32_t off = ks * 32;
        umma_tf32(d, umma_desc(a_lo + off), umma_desc(b_hi + off), ks == 0 ? 0u : 1u);
        umma_tf32(d, umma_desc(a_hi + off), umma_desc(b_lo + off), 1u);
        umma_tf32(d, umma_desc(a_hi + off), umma_desc(b_hi + off), 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(&bars[st])));
    }
    // fold chunk c-1 (its MMAs ran while chunk c was landing): frees its ring
    // stage and TMEM buffer
    if (c >= 1) {
      const int pc = c - 1;
      mbar_wait(smem_u32(&bars[pc % kStages]), (pc / kStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      drain(tmem, pc & 1, acc);
      asm volatile("tcgen05.fence::before_thread_sync;");
    }
    const int nc = c + kStages - 1;
    if (nc < n_chunks) load_chunk(g, cp, c_beg + nc, s_base + (nc % kStages) * STAGE);
    asm volatile("cp.async.commit_group;");
  }
  if (n_chunks > 0) {
    const int pc = n_chunks - 1;
    mbar_wait(smem_u32(&bars[pc % kStages]), (pc / kStages) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
    drain(tmem, pc & 1, acc);
  }
  asm volatile("cp.async.wait_group 0;");

  // Stage this CTA's (partial) tile row-major in its own shared memory.
  float* tile_s = reinterpret_cast<float*>(smem);
  {
    const int r = (warp & 3) * 32 + (threadIdx.x & 31), cb = (warp >> 2) * kHalfCols;
#pragma unroll
    for (int j = 0; j < kHalfCols; j += 4)
      *reinterpret_cast<float4*>(&tile_s[r * kTileStride + cb + j]) =
          make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
  }
  // Split-K reduce-scatter over distributed shared memory: CTA `rank` owns rows
  // [r_beg, r_end) of the tile, sums them over the S partial tiles in rank
  // order (deterministic) and writes them out; all S CTAs share the work.
  const int r_beg = rank * BM / S, r_end = (rank + 1) * BM / S;
  if (S > 1) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  else __syncthreads();
  store_tile(g, tile_s, m0, n0, r_beg, r_end, rank, S, kThreads);
  // peers' partial tiles must stay resident until every slice has been read
  if (S > 1) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(kTmemCols));
}


// ---------------------------------------------------------------------------
// TMA + warp-specialised mainloop (see the file comment). Two tile widths:
// BN = 80 (4 stages, 4 drain warps; small problems, where split-K fills the
// GPU) and BN = 208 (2 stages, 8 drain warps — two per TMEM lane quarter, each
// folding half the columns; problems with enough tiles to fill the GPU without
// split-K). The wide tile reads A once per 208 output columns instead of per
// 80: the large GEMMs (FuseSemantic, BetaE projections) are bound by the L2 ->
// SMEM operand stream (hi + lo operands re-read per N tile), not by the MMA.
template <int TBN, int TG = (TBN <= 80 ? 1 : 2)>
struct TmaCfg {
  static constexpr int kBN = TBN;
  static constexpr int kBTile = TBN * BK * 4;
  static constexpr int kStage = 2 * A_TILE + 2 * kBTile;
  static constexpr int kStages = TBN <= 80 ? 4 : (227 * 1024 - 1024 - 256) / kStage;
  static constexpr int kGroups = TG;  // drain warps per TMEM lane quarter
  static constexpr int kCols = TBN / kGroups;        // accumulator columns per drain thread
  static constexpr int kThreads = 64 + 128 * kGroups;
  static constexpr int kTmem = 2 * TBN <= 256 ? 256 : 512;
  static constexpr int kSmem = kStages * kStage + 1024 + 256;
  static constexpr uint32_t kInstr = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TBN >> 3) << 17) |
                                     ((uint32_t)(BM >> 4) << 24);
  static_assert(kStages >= 2, "operand ring");
  static_assert(kCols % 8 == 0 && TBN % 16 == 0 && TBN <= 256, "UMMA N");
  static_assert(BM * (TBN + 4) * 4 <= kStages * kStage, "epilogue tile fits the ring");
};
constexpr int kWideBN = 208;

struct TmaProblem {
  CUtensorMap a_hi, a_lo, b_hi, b_lo;  // 2-D {K, rows} fp32 maps, box {32, BM | BN}
};
struct TcGemmTmaBatch {
  TmaProblem maps[kMaxProblems];
  TcGemmArgs p[kMaxProblems];
  int tile_begin[kMaxProblems + 1];
  int n;
  int S;
  int fold;  // K chunks per fresh TMEM accumulation folded into the fp32 registers
};

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void umma_tf32_n(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int TBN, int TG = (TBN <= 80 ? 1 : 2)>
__global__ void __launch_bounds__(TmaCfg<TBN, TG>::kThreads, 1)
    tc_gemm_tma_kernel(const __grid_constant__ TcGemmTmaBatch batch) {
  using Cfg = TmaCfg<TBN, TG>;
  constexpr int kSt = Cfg::kStages, kStageB = Cfg::kStage, kBT = Cfg::kBTile, kNC = Cfg::kCols;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 128B-swizzled tiles need 1024-byte aligned stage bases
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const uint32_t s_base = smem_u32(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSt * kStageB);
  uint64_t* empty = full + kSt;
  uint64_t* tfull = empty + kSt;   // [2] TMEM buffer holds a finished chunk
  uint64_t* tempty = tfull + 2;    // [2] TMEM buffer drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int S = batch.S;
  const int tile = blockIdx.x / S, rank = blockIdx.x % S;
  int pi = 0;
  while (pi + 1 < batch.n && tile >= batch.tile_begin[pi + 1]) ++pi;
  const TcGemmArgs& g = batch.p[pi];
  const TmaProblem& mp = batch.maps[pi];
  const int lt = tile - batch.tile_begin[pi];
  const int n_tiles_n = (g.N + TBN - 1) / TBN;
  const int m0 = (lt / n_tiles_n) * BM, n0 = (lt % n_tiles_n) * TBN;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int total_chunks = (g.K + BK - 1) / BK;
  const int c_beg = rank * total_chunks / S;
  const int n_chunks = (rank + 1) * total_chunks / S - c_beg;
  const int F = batch.fold;
  const int n_groups = (n_chunks + F - 1) / F;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kSt; ++i) {
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&tfull[i]), 1);
      mbar_init(smem_u32(&tempty[i]), 4 * Cfg::kGroups);  // one arrive per drain warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mp.a_hi)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mp.a_lo)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mp.b_hi)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mp.b_lo)));
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(Cfg::kTmem));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  pdl_start();  // everything above overlapped the previous kernel's tail

  float acc[kNC];
  const int quarter = warp & 3, group = warp >= 2 ? (warp - 2) / 4 : 0;
  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      for (int c = 0; c < n_chunks; ++c) {
        const int st = c % kSt, ph = (c / kSt) & 1;
        mbar_wait(smem_u32(&empty[st]), ph ^ 1);
        const uint32_t bar = smem_u32(&full[st]), dst = s_base + st * kStageB;
        mbar_expect_tx(bar, kStageB);
        const int k0 = (c_beg + c) * BK;
        if (g.A.mn) {  // MN-major: {rows, K} map, one box per 32-row block
#pragma unroll
          for (int blk = 0; blk < BM / 32; ++blk) {
            tma_load_2d(dst + blk * kMnBlock, &mp.a_hi, bar, m0 + 32 * blk, k0);
            tma_load_2d(dst + A_TILE + blk * kMnBlock, &mp.a_lo, bar, m0 + 32 * blk, k0);
          }
        } else {
          tma_load_2d(dst, &mp.a_hi, bar, k0, m0);
          tma_load_2d(dst + A_TILE, &mp.a_lo, bar, k0, m0);
        }
        if constexpr (TBN % 32 == 0) {
          if (g.B.mn) {
#pragma unroll
            for (int blk = 0; blk < TBN / 32; ++blk) {
              tma_load_2d(dst + 2 * A_TILE + blk * kMnBlock, &mp.b_hi, bar, n0 + 32 * blk, k0);
              tma_load_2d(dst + 2 * A_TILE + kBT + blk * kMnBlock, &mp.b_lo, bar, n0 + 32 * blk, k0);
            }
            continue;
          }
        }
        tma_load_2d(dst + 2 * A_TILE, &mp.b_hi, bar, k0, n0);
        tma_load_2d(dst + 2 * A_TILE + kBT, &mp.b_lo, bar, k0, n0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      // operand majors (instruction descriptor bits 15 / 16) and the k-step
      // advance: 32 B along a K-major 128-byte line, or one 1024-byte 8-k atom
      const uint32_t idesc = Cfg::kInstr | (g.A.mn ? 1u << 15 : 0u) | (g.B.mn ? 1u << 16 : 0u);
      const uint32_t a_step = g.A.mn ? 1024u : 32u, b_step = g.B.mn ? 1024u : 32u;
      auto desc_a = [&](uint32_t addr) { return g.A.mn ? umma_desc_mn(addr) : umma_desc(addr); };
      auto desc_b = [&](uint32_t addr) { return g.B.mn ? umma_desc_mn(addr) : umma_desc(addr); };
      for (int c = 0; c < n_chunks; ++c) {
        const int st = c % kSt, ph = (c / kSt) & 1;
        const int gi = c / F, buf = gi & 1, bph = (gi >> 1) & 1;
        const bool fresh = c % F == 0, last = c % F == F - 1 || c == n_chunks - 1;
        if (fresh) mbar_wait(smem_u32(&tempty[buf]), bph ^ 1);
        mbar_wait(smem_u32(&full[st]), ph);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t a_hi = s_base + st * kStageB, a_lo = a_hi + A_TILE;
        const uint32_t b_hi = a_hi + 2 * A_TILE, b_lo = b_hi + kBT;
        const uint32_t d = tmem + buf * TBN;
#pragma unroll
        for (int ks = 0; ks < BK / 8; ++ks) {  // small terms first, fresh accumulator per chunk
          const uint32_t ao = ks * a_step, bo = ks * b_step;
          umma_tf32_n(d, desc_a(a_lo + ao), desc_b(b_hi + bo), idesc, (ks == 0 && fresh) ? 0u : 1u);
          umma_tf32_n(d, desc_a(a_hi + ao), desc_b(b_lo + bo), idesc, 1u);
          umma_tf32_n(d, desc_a(a_hi + ao), desc_b(b_hi + bo), idesc, 1u);
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&empty[st])));
        if (last)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              smem_u32(&tfull[buf])));
      }
    }
    __syncwarp();
  } else {  // ---- drain warps: TMEM lane quarter (warp % 4), column group, one row per thread
#pragma unroll
    for (int j = 0; j < kNC; ++j) acc[j] = 0.f;
    const uint32_t lanes = (static_cast<uint32_t>(quarter * 32) << 16) + group * kNC;
    constexpr int kPiece = kNC <= 80 ? kNC : 32;  // columns in flight per tcgen05.wait
    for (int c = 0; c < n_groups; ++c) {
      const int buf = c & 1, bph = (c >> 1) & 1;
      mbar_wait(smem_u32(&tfull[buf]), bph);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int p0 = 0; p0 < kNC; p0 += kPiece) {
        uint32_t r[kPiece];
#pragma unroll
        for (int j = 0; j < kPiece; j += 8)
          if (p0 + j < kNC)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[j]), "=r"(r[j + 1]), "=r"(r[j + 2]), "=r"(r[j + 3]), "=r"(r[j + 4]),
                           "=r"(r[j + 5]), "=r"(r[j + 6]), "=r"(r[j + 7])
                         : "r"(tmem + lanes + buf * TBN + p0 + j));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int j = 0; j < kPiece; ++j)
          if (p0 + j < kNC) acc[p0 + j] += __uint_as_float(r[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&tempty[buf]));
    }
  }
  // every chunk has been consumed by the tensor core and drained: the ring is free
  __syncthreads();
  constexpr int kStride = TBN + 4;
  float* tile_s = reinterpret_cast<float*>(smem);
  if (warp >= 2) {
    const int r = quarter * 32 + lane;
#pragma unroll
    for (int j = 0; j < kNC; j += 4)
      *reinterpret_cast<float4*>(&tile_s[r * kStride + group * kNC + j]) =
          make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
  }
  const int r_beg = rank * BM / S, r_end = (rank + 1) * BM / S;
  if (S > 1) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  else __syncthreads();
  store_tile<TBN>(g, tile_s, m0, n0, r_beg, r_end, rank, S, Cfg::kThreads);
  if (S > 1) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(Cfg::kTmem));
}

// --- operand split / transpose ------------------------------------------------
__global__ void split_kernel(const float* src, int rows, int cols, int ld, int relu, float* hi,
                             float* lo) {
  pdl_start();
  const int64_t n = (int64_t)rows * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / cols), c = (int)(i % cols);
    float v = src[(int64_t)r * ld + c];
    if (relu) v = fmaxf(v, 0.f);
    float h, l;
    split_tf32(v, h, l);
    hi[i] = h;
    lo[i] = l;
  }
}

// dst[c][r] (row stride pad4(rows), zero padded) = split(op(src[r][c]))
__global__ void split_t_multi_kernel(SplitJobs jobs) {
  pdl_start();
  __shared__ float tile[32][33];
  const SplitJob& j = jobs.job[blockIdx.z];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  if (r0 >= j.rows || c0 >= j.cols) return;  // grid sized for the largest job
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int r = r0 + y, c = c0 + threadIdx.x;
    float v = 0.f;
    if (r < j.rows && c < j.cols) {
      if (j.node_grad) {  // computed source (see SplitJob)
        const int node = r < j.n1 * j.k1 ? r / j.k1 : j.n1 + (r - j.n1 * j.k1) / j.k2;
        const int k = r < j.n1 * j.k1 ? j.k1 : j.k2;
        const int64_t o = (int64_t)r * j.ld + c;
        v = j.mask[o] > 0.f ? j.node_grad[(int64_t)node * j.cols + c] / static_cast<float>(k) : 0.f;
        float h, l;
        split_tf32(v, h, l);
        j.plain[o] = v;
        j.rhi[o] = h;
        j.rlo[o] = l;
      } else {
        v = j.src[(int64_t)r * j.ld + c];
      }
    }
    tile[y][threadIdx.x] = j.relu ? fmaxf(v, 0.f) : v;
  }
  __syncthreads();
  if (!j.hi) return;  // computed source written row-major only (MN-major consumer)
  const int ldp = (j.rows + 3) & ~3;  // 16-byte aligned rows for cp.async; zero padded
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int c = c0 + y, r = r0 + threadIdx.x;
    if (c < j.cols && r < ldp) {
      float h = 0.f, l = 0.f;
      if (r < j.rows) split_tf32(tile[threadIdx.x][y], h, l);
      j.hi[(int64_t)c * ldp + r] = h;
      j.lo[(int64_t)c * ldp + r] = l;
    }
  }
}

}  // namespace

// Opt the kernels into > 48 KB dynamic shared memory (once per process, before
// any launch or stream capture).
void tc_gemm_init() {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    cudaFuncSetAttribute(tc_gemm_tma_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         TmaCfg<BN>::kSmem);
    cudaFuncSetAttribute(tc_gemm_tma_kernel<kWideBN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         TmaCfg<kWideBN>::kSmem);
    cudaFuncSetAttribute(tc_gemm_tma_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         TmaCfg<128>::kSmem);
    cudaFuncSetAttribute(tc_gemm_tma_kernel<160>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         TmaCfg<160>::kSmem);
    configured = true;
  }
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// TMA needs 16-byte aligned bases and row strides
bool tma_ok(const SplitOperand& o) {
  return (o.ld & 3) == 0 && ((reinterpret_cast<uintptr_t>(o.hi) | reinterpret_cast<uintptr_t>(o.lo)) & 15) == 0;
}

// {K, rows} fp32, box {32, box_rows}, 128B swizzle (the UMMA K-major layout),
// out-of-bounds elements read as zero
bool encode(CUtensorMap* m, const float* base, int rows, int K, int ld, int box_rows) {
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  return tensor_map_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// MN-major operand [K][rows] (row stride ld): {rows, K} map, box {32, 32}
// (one 4096-byte block per box, 32-byte-atom 128B swizzle; rows / K beyond
// the matrix zero)
bool encode_mn(CUtensorMap* m, const float* base, int rows, int K, int ld) {
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(K)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  const cuuint32_t box[2] = {32, static_cast<cuuint32_t>(BK)};
  const cuuint32_t estr[2] = {1, 1};
  return tensor_map_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
bool encode_op(CUtensorMap* m, const float* base, const SplitOperand& o, int rows, int K, int box_rows) {
  return o.mn ? encode_mn(m, base, rows, K, o.ld) : encode(m, base, rows, K, o.ld, box_rows);
}
}  // namespace

int tc_gemm_batch(const TcGemmArgs* probs, int n, cudaStream_t s) {
  tc_gemm_init();
  TcGemmBatch b{};
  int max_chunks = 0, tiles = 0;
  bool any_mn = false, b_mn = false;
  for (int i = 0; i < n && i < kMaxProblems; ++i) {
    any_mn = any_mn || probs[i].A.mn || probs[i].B.mn;
    b_mn = b_mn || probs[i].B.mn;
  }
  // MN-major operands exist only in the TMA mainloop (the cp.async knob is ignored)
  bool tma = tensor_map_encoder() != nullptr && (any_mn || !std::getenv("NGDB_GEMM_CPASYNC"));
  b.n = 0;
  for (int i = 0; i < n && b.n < kMaxProblems; ++i) {
    const TcGemmArgs& g = probs[i];
    if (g.M <= 0 || g.N <= 0) continue;
    b.p[b.n] = g;
    b.tile_begin[b.n] = tiles;
    tiles += ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN);
    max_chunks = std::max(max_chunks, (g.K + BK - 1) / BK);
    tma = tma && tma_ok(g.A) && tma_ok(g.B) && g.K > 0;
    ++b.n;
  }
  if (b.n == 0) return 0;
  b.tile_begin[b.n] = tiles;
  int num_sms = 148;
  cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, 0);
  if (tma) {
    // Tile width per launch (UMMA N = 80 / 160 / 208), from the measured table
    // profiles/r02/gemm_variants.txt: the operand stream from L2 (hi + lo
    // tiles, A re-read once per N tile, B once per M tile) bounds the large
    // shapes, so wider tiles win where there are enough of them to fill the
    // GPU; narrow tiles + split-K win on the small ones.
    //   big M (>= 4096 rows) ............................. 208  (14.5k x 400 x 768: 85 -> 65 us)
    //   K = rows weight gradients, both sides <= 512 ...... 160  (400 x 400 x 14.5k: 97 -> 57 us)
    //   mid M (>= 1024 rows), N >= 640 ................... 160  (1434 x 800 x 1200: 31 -> 24 us)
    //   K >= 1024, M and N >= 640 ........................ 208  (800 x 1200 x 1434: 36 -> 26 us)
    //   otherwise (C2's 731-row MLPs, ...) ................ 80
    // The class of the launch's largest problem decides; NGDB_GEMM_BN forces one.
    static const int forced_bn = [] {
      const char* e = std::getenv("NGDB_GEMM_BN");
      return e ? std::atoi(e) : 0;
    }();
    int min_n = 1 << 30, big = 0;
    double big_flops = -1.0;
    for (int i = 0; i < b.n; ++i) {
      min_n = std::min(min_n, b.p[i].N);
      const double fl = double(b.p[i].M) * b.p[i].N * b.p[i].K;
      if (fl > big_flops) {
        big_flops = fl;
        big = i;
      }
    }
    auto pick = [&](const TcGemmArgs& g) {
      if (min_n < 192) return BN;
      if (g.M >= 4096) return kWideBN;
      if (g.K >= 8 * std::max(g.M, g.N)) return (g.M <= 512 && g.N <= 512) ? 160 : BN;
      if (g.M >= 1024 && g.N >= 640) return 160;
      if (g.K >= 1024 && g.M >= 640 && g.N >= 640) return kWideBN;
      return BN;
    };
    int tbn = pick(b.p[big]);
    if (forced_bn == 80 || forced_bn == 128 || forced_bn == 160 || forced_bn == kWideBN) tbn = forced_bn;
    if (g_split_override.load(std::memory_order_relaxed)) tbn = BN;
    // an MN-major B is loaded in 32-row blocks: the tile width is a multiple of 32
    if (b_mn && tbn % 32 != 0) tbn = 160;
    TcGemmTmaBatch t{};  // ~2.6 KB of kernel parameters (4 tensor maps per problem)
    int tiles_t = 0;
    for (int i = 0; i < b.n && tma; ++i) {
      const TcGemmArgs& g = b.p[i];
      t.p[i] = g;
      tma = encode_op(&t.maps[i].a_hi, g.A.hi, g.A, g.M, g.K, BM) &&
            encode_op(&t.maps[i].a_lo, g.A.lo, g.A, g.M, g.K, BM) &&
            encode_op(&t.maps[i].b_hi, g.B.hi, g.B, g.N, g.K, tbn) &&
            encode_op(&t.maps[i].b_lo, g.B.lo, g.B, g.N, g.K, tbn);
      t.tile_begin[i] = tiles_t;
      tiles_t += ((g.M + BM - 1) / BM) * ((g.N + tbn - 1) / tbn);
    }
    if (tma) {
      t.tile_begin[b.n] = tiles_t;
      t.n = b.n;
      // one CTA per SM (~210 KB ring): split-K so the launch fills about one
      // wave, at most 8 CTAs per cluster and at least 2 chunks per CTA
      t.S = std::max(1, std::min({8, num_sms / std::max(tiles_t, 1), max_chunks / 2}));
      if (const int o = g_split_override.load(std::memory_order_relaxed)) t.S = std::min(o, std::max(1, max_chunks));
      // K chunks per fresh TMEM accumulation: 1 keeps every contraction at fp32
      // accuracy (2 measured 2-5 % faster but moved BetaE projection weight
      // gradients, K = rows, past the 1e-4 parity bar); NGDB_GEMM_FOLD overrides
      static const int fold_env = [] {
        const char* e = std::getenv("NGDB_GEMM_FOLD");
        return e ? std::max(1, std::atoi(e)) : 1;
      }();
      t.fold = fold_env;
      static const bool log_shapes = std::getenv("NGDB_GEMM_LOG") != nullptr;
      if (log_shapes) {  // one line per launch (diagnostics)
        std::fprintf(stderr, "gemm bn=%d S=%d tiles=%d", tbn, t.S, tiles_t);
        for (int i = 0; i < b.n; ++i)
          std::fprintf(stderr, " [%dx%dx%d%s%s]", b.p[i].M, b.p[i].N, b.p[i].K, b.p[i].A.mn ? " A:mn" : "",
                       b.p[i].B.mn ? " B:mn" : "");
        std::fprintf(stderr, "\n");
      }
      auto go = [&](auto kernel, int threads, int smem) {
        launch_pdl(kernel, dim3(tiles_t * t.S), dim3(threads), smem, s, t.S, t);
      };
      switch (tbn) {
        case kWideBN: go(tc_gemm_tma_kernel<kWideBN>, TmaCfg<kWideBN>::kThreads, TmaCfg<kWideBN>::kSmem); break;
        case 160: go(tc_gemm_tma_kernel<160>, TmaCfg<160>::kThreads, TmaCfg<160>::kSmem); break;
        case 128: go(tc_gemm_tma_kernel<128>, TmaCfg<128>::kThreads, TmaCfg<128>::kSmem); break;
        default:
          go(tc_gemm_tma_kernel<BN>, TmaCfg<BN>::kThreads, TmaCfg<BN>::kSmem);
      }
      return 1;
    }
  }
  if (any_mn) {  // no cp.async form of an MN-major operand: fail loudly
    std::fprintf(stderr, "ngdb: tc_gemm_batch: MN-major operand needs the TMA mainloop "
                         "(16-byte aligned hi/lo, ld %% 4 == 0)\n");
    std::abort();
  }
  // split-K so the launch fills about one wave (2 CTAs per SM), at most 8 CTAs
  // per cluster (portable size) and at least 2 chunks per CTA
  b.S = std::max(1, std::min({8, (2 * num_sms) / std::max(tiles, 1), max_chunks / 2}));
  if (const int o = g_split_override.load(std::memory_order_relaxed)) b.S = std::min(o, std::max(1, max_chunks));
  launch_pdl(tc_gemm_kernel, dim3(tiles * b.S), dim3(kThreads), SMEM_BYTES, s, b.S, b);
  return 1;
}

int tc_gemm(const TcGemmArgs& g, cudaStream_t s) { return tc_gemm_batch(&g, 1, s); }

void set_gemm_split_override(int s) { g_split_override.store(s, std::memory_order_relaxed); }

int split_transposed(const SplitJobs& jobs, cudaStream_t s) {
  if (jobs.n <= 0) return 0;
  int mr = 0, mc = 0;
  for (int i = 0; i < jobs.n; ++i) {
    mr = std::max(mr, jobs.job[i].rows);
    mc = std::max(mc, jobs.job[i].cols);
  }
  if (mr <= 0 || mc <= 0) return 0;
  dim3 grid((mc + 31) / 32, (mr + 31) / 32, jobs.n);
  launch_pdl(split_t_multi_kernel, dim3(grid), dim3(dim3(32, 8)), 0, s, 1, jobs);
  return 1;
}

int split_matrix(const float* src, int rows, int cols, int ld_src, int transpose, int relu,
                 float* dst_hi, float* dst_lo, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return 0;
  if (!transpose) {
    const int64_t n = (int64_t)rows * cols;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    launch_pdl(split_kernel, dim3(blocks), dim3(256), 0, s, 1, src, rows, cols, ld_src, relu, dst_hi, dst_lo);
    return 1;
  }
  SplitJobs jobs{};
  jobs.job[0] = {src, rows, cols, ld_src, relu, dst_hi, dst_lo};
  jobs.n = 1;
  return split_transposed(jobs, s);
}

int split_weight(const float* w, int rows, int cols, float* dst, cudaStream_t s) {
  const int64_t n = (int64_t)rows * cols;
  split_matrix(w, rows, cols, cols, 0, 0, dst, dst + n, s);
  split_matrix(w, rows, cols, cols, 1, 0, dst + 2 * n, dst + 3 * n, s);
  return 2;
}

}  // namespace ngdb_dev

// Debug entry point for the GEMM unit test (host pointers, synchronous):
// C = op_a(A) op_b(B)^T with A [M][K] (a_major 0) or [K][M] (1), B [N][K] (0)
// or [K][N] (1); ops bit0 = relu(A), bit1 = relu(B), bit2 = route [K][rows]
// operands through the transposing split (K-major) instead of reading them
// MN-major in place (the two must agree bit for bit).
extern "C" int ngdb_debug_tc_gemm(int M, int N, int K, int a_major, int b_major, int ops,
                                  const float* A, int lda, const float* B, int ldb, float* C,
                                  int ldc, const float* bias, int accumulate) {
  using namespace ngdb_dev;
  const int64_t nc = (int64_t)M * ldc;
  // [K][rows] operands with 16-byte rows go MN-major (non-transposing split,
  // dense [K][rows]); everything else goes K-major through the transposing
  // split (which pads rows to a multiple of 4 floats): K-major inputs are
  // transposed on the host first.
  const bool legacy = (ops & 4) != 0;
  const bool a_mn = a_major == 1 && (M & 3) == 0 && !legacy;
  const bool b_mn = b_major == 1 && (N & 3) == 0 && !legacy;
  std::vector<float> At, Bt;
  if (a_major == 0) {
    At.resize((size_t)K * M);
    for (int m = 0; m < M; ++m)
      for (int k = 0; k < K; ++k) At[(size_t)k * M + m] = A[(size_t)m * lda + k];
    A = At.data();
    lda = M;
  }
  if (b_major == 0) {
    Bt.resize((size_t)K * N);
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) Bt[(size_t)k * N + n] = B[(size_t)n * ldb + k];
    B = Bt.data();
    ldb = N;
  }
  const int64_t na2 = (int64_t)K * lda, nb2 = (int64_t)K * ldb;
  const int KP = (K + 3) & ~3;
  const int64_t sa = std::max<int64_t>((int64_t)M * KP, (int64_t)K * M);
  const int64_t sb = std::max<int64_t>((int64_t)N * KP, (int64_t)K * N);
  float *dA, *dB, *dC, *dbias = nullptr, *sp;
  if (cudaMalloc(&dA, na2 * 4) || cudaMalloc(&dB, nb2 * 4) || cudaMalloc(&dC, nc * 4)) return 8;
  if (cudaMalloc(&sp, (sa + sb) * 2 * 4)) return 8;
  cudaMemcpy(dA, A, na2 * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B, nb2 * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dC, C, nc * 4, cudaMemcpyHostToDevice);
  if (bias) {
    cudaMalloc(&dbias, N * 4);
    cudaMemcpy(dbias, bias, N * 4, cudaMemcpyHostToDevice);
  }
  float *ahi = sp, *alo = ahi + sa, *bhi = alo + sa, *blo = bhi + sb;
  TcGemmArgs g{};
  g.M = M; g.N = N; g.K = K;
  if (a_mn) {
    split_matrix(dA, K, M, lda, 0, ops & 1, ahi, alo, 0);
    g.A = {ahi, alo, M, 1};
  } else {
    split_matrix(dA, K, M, lda, 1, ops & 1, ahi, alo, 0);
    g.A = {ahi, alo, KP, 0};
  }
  if (b_mn) {
    split_matrix(dB, K, N, ldb, 0, (ops >> 1) & 1, bhi, blo, 0);
    g.B = {bhi, blo, N, 1};
  } else {
    split_matrix(dB, K, N, ldb, 1, (ops >> 1) & 1, bhi, blo, 0);
    g.B = {bhi, blo, KP, 0};
  }
  g.C = dC; g.ldc = ldc;
  g.bias = dbias; g.accumulate = accumulate;
  tc_gemm(g, 0);
  cudaError_t e = cudaGetLastError();  // launch-configuration errors
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) std::fprintf(stderr, "ngdb_debug_tc_gemm: %s\n", cudaGetErrorString(e));
  cudaMemcpy(C, dC, nc * 4, cudaMemcpyDeviceToHost);
  cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(sp);
  if (dbias) cudaFree(dbias);
  return e == cudaSuccess ? 0 : 8;
}

// Timing entry point (tools/gemm_bench.py): `reps` back-to-back launches of one
// M x N x K problem (or `batch` independent copies in one grouped launch) on
// random pre-split operands; returns the mean CUDA-event time per launch.
extern "C" int ngdb_debug_tc_gemm_time(int M, int N, int K, int batch, int reps, float* ms_out) {
  using namespace ngdb_dev;
  const int KP = (K + 3) & ~3;
  batch = std::max(1, std::min(batch, 4));
  const int64_t na = (int64_t)M * KP, nb = (int64_t)N * KP, nc = (int64_t)M * N;
  float* buf = nullptr;
  const int64_t per = 2 * na + 2 * nb + nc;
  if (cudaMalloc(&buf, per * batch * 4)) return 8;
  std::vector<float> host(per);
  uint32_t x = 12345;
  for (auto& v : host) {
    x = x * 1664525u + 1013904223u;
    v = ((x >> 8) * (1.0f / 16777216.0f) - 0.5f) * 0.1f;
  }
  TcGemmArgs gs[4];
  for (int i = 0; i < batch; ++i) {
    float* p = buf + i * per;
    cudaMemcpy(p, host.data(), per * 4, cudaMemcpyHostToDevice);
    TcGemmArgs g{};
    g.M = M; g.N = N; g.K = K;
    g.A = {p, p + na, KP};
    g.B = {p + 2 * na, p + 2 * na + nb, KP};
    g.C = p + 2 * na + 2 * nb; g.ldc = N;
    gs[i] = g;
  }
  cudaStream_t s;
  cudaStreamCreate(&s);
  tc_gemm_batch(gs, batch, s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int r = 0; r < reps; ++r) tc_gemm_batch(gs, batch, s);
  cudaEventRecord(b, s);
  cudaError_t e = cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  *ms_out = ms / reps;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaStreamDestroy(s);
  cudaFree(buf);
  return e == cudaSuccess ? 0 : 8;
}
