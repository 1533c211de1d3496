// OptimizerStep (Alg. 1 l.21): sorted-segment gradient reduce fused with a
// touched-rows-only Adam (SPEC.md:550-558 adam_step; north_star "fused Adam
// update applied only to touched rows"; lazy semantics, SURVEY A-9), and the
// dense Adam for MLP weights.
//
// Entity rows receive two kinds of contributions, listed per row in a host-
// planned CSR (rows ascending, so the reduction order is fixed and the result
// deterministic):
//   anchor   (code < 0): an explicit gradient row from EmbedAnchor's mirror
//   candidate(code >= 0): coef_j * d dist(v, q_s) / dv, recomputed here from the
//            score slot's query copy (L2-resident) and the row itself, which
//            this kernel reads anyway for the update. The 66k x 1600 B candidate
//            gradient rows of a step are therefore never written to HBM.
// HBM traffic per touched row: read theta, m, v; write theta, m, v (6 w bytes).
//
// Adam's bias corrections bc = (1 - b1^t, 1 - b2^t) are read from device
// memory so a captured CUDA graph of the step replays with the current t.
#include <algorithm>

#include "adam.cuh"
#include "common.cuh"

namespace ngdb_dev {
namespace {

constexpr int kWarps = 8;

// coef * d dist / dv, branch-free: copysign of the magnitude, 0 at delta == 0
// (ca = coef * alpha, hoisted out of the element loop)
template <int BB>
__device__ __forceinline__ float cand_grad(float v, float qc, float qo, float coef, float ca) {
  const float delta = v - qc;
  float mag = coef;
  if (BB == NGDB_Q2B) mag = fabsf(delta) > qo ? coef : ca;
  const float s = __int_as_float((__float_as_int(mag) ^ (__float_as_int(delta) & 0x80000000)));
  return delta != 0.f ? s : 0.f;
}

// Touched-row entity Adam, TMA-staged: each CTA owns a contiguous range of
// touched rows; a producer warp streams every row's theta, m and v (3 x w
// bytes) into a shared-memory ring with bulk copies (cp.async.bulk +
// mbarrier complete_tx), so kAdamRing rows per CTA are always in flight
// regardless of what the consumers are doing. Consumer warps take rows
// round-robin: the gradient is summed along the row's CSR contributions
// (codes and coefficients fetched lane-parallel, then broadcast), Adam runs in
// registers and theta, m, v are stored straight back to HBM.
constexpr int kAdamConsumers = 8;
constexpr int kAdamThreads = 32 * (kAdamConsumers + 1);
constexpr int kAdamRing = 8;  // a multiple of kAdamConsumers (see the score ring)

inline size_t adam_smem_bytes(int width) {
  return static_cast<size_t>(kAdamRing) * 3 * width * sizeof(float) + 2 * kAdamRing * sizeof(uint64_t);
}

template <int BB, int NCH>
__global__ void __launch_bounds__(kAdamThreads, 4) entity_adam_kernel(DevArgs a, SparseTable t,
                                                                   AdamHyper hp, const float* bc,
                                                                   int rows_per_cta) {
  extern __shared__ __align__(128) float smem[];
  const int W = t.width;
  float* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kAdamRing * 3 * W);
  uint64_t* empty = full + kAdamRing;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kAdamRing; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  // The producer streams theta, m, v before waiting on the previous kernel:
  // they are written only by this kernel (plus the row ids: plan data), so
  // the reads overlap the tail of the step's last pool. The consumers wait
  // before they read any gradient input or write a row.
  pdl_launch();
  const int r_beg = blockIdx.x * rows_per_cta;
  const int n_mine = max(0, min(t.n_rows, r_beg + rows_per_cta) - r_beg);
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == kAdamConsumers) {  // producer warp: row ids staged 32 at a time, lane 0 issues
    __shared__ int32_t rows_s[32];
    const uint32_t bytes = static_cast<uint32_t>(W * sizeof(float));
    for (int u0 = 0; u0 < n_mine; u0 += 32) {
      if (u0 + lane < n_mine) rows_s[lane] = __ldg(t.rows + r_beg + u0 + lane);
      __syncwarp();
      const int cnt = min(32, n_mine - u0);
      if (lane == 0)
        for (int r = 0; r < cnt; ++r) {
          const int u = u0 + r;
          const int64_t row = rows_s[r];
          const int slot = u % kAdamRing, round = u / kAdamRing;
          if (round > 0) mbar_wait_parity(&empty[slot], (round - 1) & 1);
          float* dst = ring + slot * 3 * W;
          mbar_arrive_expect_tx(&full[slot], 3 * bytes);
          bulk_g2s(dst, t.w + row * W, bytes, &full[slot]);
          bulk_g2s(dst + W, t.m + row * W, bytes, &full[slot]);
          bulk_g2s(dst + 2 * W, t.v + row * W, bytes, &full[slot]);
        }
      __syncwarp();  // rows_s is reused by the next chunk
    }
    return;
  }
  pdl_wait();
  const int w4 = W / 4;
  const AdamK k = adam_consts(hp, bc);
  for (int u = warp; u < n_mine; u += kAdamConsumers) {
    const int slot = u % kAdamRing, round = u / kAdamRing;
    const int row_idx = r_beg + u;
    const int64_t row = __ldg(t.rows + row_idx);
    const int beg = __ldg(t.seg + row_idx), end = __ldg(t.seg + row_idx + 1);
    // contribution codes / coefficients of the row's first 32 contributions
    // are fetched before waiting for the row itself
    int32_t my_code = 0;
    float my_coef = 0.f;
    if (lane < end - beg) {
      my_code = __ldg(t.contrib + beg + lane);
      if (my_code >= 0) my_coef = __ldg(a.coefbuf + my_code);
    }
    const float* ws = ring + slot * 3 * W;  // theta, m, v stay in shared memory
    mbar_wait_parity(&full[slot], round & 1);
    float4 g[NCH];
#pragma unroll
    for (int i = 0; i < NCH; ++i) g[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k0 = beg; k0 < end; k0 += 32) {
      const int nk = min(32, end - k0);
      if (k0 > beg) {
        my_code = 0;
        my_coef = 0.f;
        if (lane < nk) {
          my_code = __ldg(t.contrib + k0 + lane);
          if (my_code >= 0) my_coef = __ldg(a.coefbuf + my_code);
        }
      }
      for (int j = 0; j < nk; ++j) {
        const int32_t code = __shfl_sync(0xffffffffu, my_code, j);
        const float coef = __shfl_sync(0xffffffffu, my_coef, j);
        if (code < 0) {
          const float* r = a.agbuf + static_cast<int64_t>(-code - 1) * W;
#pragma unroll
          for (int i = 0; i < NCH; ++i) {
            const int c = lane + 32 * i;
            if (c < w4) {
              const float4 x = ld4(r + 4 * c);
              g[i].x += x.x; g[i].y += x.y; g[i].z += x.z; g[i].w += x.w;
            }
          }
        } else {
          const float* q = a.qbuf + static_cast<int64_t>(code / a.ncand) * a.wq;
          const float ca = coef * a.alpha_box;
#pragma unroll
          for (int i = 0; i < NCH; ++i) {
            const int c = lane + 32 * i;
            if (c < w4) {
              const float4 qc = ld4(q + 4 * c);
              float4 qo = make_float4(0.f, 0.f, 0.f, 0.f);
              if (BB == NGDB_Q2B) qo = ld4(q + a.dim + 4 * c);
              const float4 w = ld4(ws + 4 * c);
              g[i].x += cand_grad<BB>(w.x, qc.x, qo.x, coef, ca);
              g[i].y += cand_grad<BB>(w.y, qc.y, qo.y, coef, ca);
              g[i].z += cand_grad<BB>(w.z, qc.z, qo.z, coef, ca);
              g[i].w += cand_grad<BB>(w.w, qc.w, qo.w, coef, ca);
            }
          }
        }
      }
    }
    float* wp = t.w + row * W;
    float* mp = t.m + row * W;
    float* vp = t.v + row * W;
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      const int c = lane + 32 * i;
      if (c < w4) {
        if (t.dbg_g) st4(t.dbg_g + row * W + 4 * c, g[i]);
        float4 m = ld4(ws + W + 4 * c), v = ld4(ws + 2 * W + 4 * c);
        const float4 nw = adam4(ld4(ws + 4 * c), m, v, g[i], k);
        st4(wp + 4 * c, nw);
        st4(mp + 4 * c, m);
        st4(vp + 4 * c, v);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);  // slot's smem fully read
  }
}

// Relation rows: few rows (|R| <= a few hundred) with many contributions each
// (every Project node of the step), so one THREAD per (row, float4 chunk): the
// contribution loads of a chunk are independent and issued 4 at a time, and
// the whole table is covered by ~|R| * w/4 threads instead of |R| warps.
__global__ void __launch_bounds__(256) relation_adam_kernel(DevArgs a, SparseTable t,
                                                           AdamHyper hp, const float* bc) {
  pdl_start();
  const int w4 = t.width / 4;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (item >= static_cast<int64_t>(t.n_rows) * w4) return;
  const int row_idx = static_cast<int>(item / w4), c = static_cast<int>(item % w4);
  const AdamK k = adam_consts(hp, bc);
  const int64_t row = t.rows[row_idx];
  const int beg = t.seg[row_idx], end = t.seg[row_idx + 1];
  float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
  int kk = beg;
  for (; kk + 4 <= end; kk += 4) {
    float4 r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      r[u] = ld4(a.rgbuf + static_cast<int64_t>(__ldg(t.contrib + kk + u)) * t.width + 4 * c);
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // contribution order kept (deterministic)
      g.x += r[u].x; g.y += r[u].y; g.z += r[u].z; g.w += r[u].w;
    }
  }
  for (; kk < end; ++kk) {
    const float4 r = ld4(a.rgbuf + static_cast<int64_t>(__ldg(t.contrib + kk)) * t.width + 4 * c);
    g.x += r.x; g.y += r.y; g.z += r.z; g.w += r.w;
  }
  float* wp = t.w + row * t.width;
  float* mp = t.m + row * t.width;
  float* vp = t.v + row * t.width;
  if (t.dbg_g) st4(t.dbg_g + row * t.width + 4 * c, g);
  float4 w = ld4(wp + 4 * c), m = ld4(mp + 4 * c), v = ld4(vp + 4 * c);
  w = adam4(w, m, v, g, k);
  st4(wp + 4 * c, w);
  st4(mp + 4 * c, m);
  st4(vp + 4 * c, v);
}

__global__ void dense_adam_kernel(float* w, float* m, float* v, const float* g, int64_t n,
                                  AdamHyper hp, const float* bc) {
  pdl_start();
  const AdamK k = adam_consts(hp, bc);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float wi = w[i], mi = m[i], vi = v[i];
    adam_update(wi, mi, vi, g[i], k);
    w[i] = wi;
    m[i] = mi;
    v[i] = vi;
  }
}

// Dense Adam fused with the 3xTF32 operand refresh of the MLP weights: one
// 32x32 tile per CTA updates theta, m, v and writes W_hi, W_lo and, through a
// shared-memory transpose, (W^T)_hi, (W^T)_lo — the split layout wop()
// reads (mlp_util.cuh). Replaces one Adam launch + two split launches per
// weight matrix.
__device__ __forceinline__ void split_hi_lo(float x, float& hi, float& lo) {
  hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
  lo = x - hi;
}

__global__ void __launch_bounds__(256) dense_adam_split_kernel(float* w, float* m, float* v,
                                                               const float* g, float* wsplit,
                                                               DenseJobs jobs, AdamHyper hp,
                                                               const float* bc) {
  pdl_start();
  __shared__ float tile[32][33];
  const int t = blockIdx.x;
  int j = 0;
  while (j + 1 < jobs.n && t >= jobs.job[j + 1].tile_begin) ++j;
  const DenseJob& J = jobs.job[j];
  const int lt = t - J.tile_begin;
  const int tiles_c = (J.cols + 31) / 32;
  const int r0 = (lt / tiles_c) * 32, c0 = (lt % tiles_c) * 32;
  const AdamK k = adam_consts(hp, bc);
  const int tx = threadIdx.x & 31, ty = threadIdx.x / 32;
  const int64_t n = static_cast<int64_t>(J.rows) * J.cols;
  for (int y = ty; y < 32; y += 8) {
    const int r = r0 + y, c = c0 + tx;
    if (r < J.rows && c < J.cols) {
      const int64_t i = J.off + static_cast<int64_t>(r) * J.cols + c;
      float wi = w[i], mi = m[i], vi = v[i];
      adam_update(wi, mi, vi, g[i], k);
      w[i] = wi;
      m[i] = mi;
      v[i] = vi;
      if (J.split_off >= 0) {
        float hi, lo;
        split_hi_lo(wi, hi, lo);
        wsplit[J.split_off + static_cast<int64_t>(r) * J.cols + c] = hi;
        wsplit[J.split_off + n + static_cast<int64_t>(r) * J.cols + c] = lo;
      }
      tile[y][tx] = wi;
    }
  }
  if (J.split_off < 0) return;  // uniform per CTA
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    const int c = c0 + y, r = r0 + tx;  // W^T [cols][rows]
    if (r < J.rows && c < J.cols) {
      float hi, lo;
      split_hi_lo(tile[tx][y], hi, lo);
      wsplit[J.split_off + 2 * n + static_cast<int64_t>(c) * J.rows + r] = hi;
      wsplit[J.split_off + 3 * n + static_cast<int64_t>(c) * J.rows + r] = lo;
    }
  }
}

}  // namespace

int launch_dense_adam_split(float* w, float* m, float* v, const float* g, float* wsplit,
                            const DenseJobs& jobs, const AdamHyper& hp, const float* bc,
                            const LaunchCtx& lc) {
  if (jobs.n <= 0 || jobs.tiles <= 0) return 0;
  launch_pdl(dense_adam_split_kernel, dim3(jobs.tiles), dim3(256), 0, lc.stream, 1, w, m, v, g,
             wsplit, jobs, hp, bc);
  return 1;
}

int launch_sparse_adam_entity(const DevArgs& a, const SparseTable& t, const AdamHyper& hp,
                              const float* bc, const LaunchCtx& lc) {
  if (t.n_rows <= 0) return 0;
  if (a.backbone == NGDB_BETAE) return launch_beta_entity_adam(a, t, hp, bc, lc);
  const size_t smem = adam_smem_bytes(t.width);
  // persistent-style grid: 4 CTAs per SM (56 registers, 38 KB rings), contiguous row ranges
  const int ctas = std::max(1, std::min(t.n_rows, 4 * lc.num_sms));
  const int rows_per_cta = (t.n_rows + ctas - 1) / ctas;
  const int grid = (t.n_rows + rows_per_cta - 1) / rows_per_cta;
  auto go = [&](auto kernel) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(kernel, dim3(grid), dim3(kAdamThreads), smem, lc.stream, 1, a, t, hp, bc,
               rows_per_cta);
  };
  if (t.width <= 512) {
    if (a.backbone == NGDB_GQE) go(entity_adam_kernel<NGDB_GQE, 4>);
    else go(entity_adam_kernel<NGDB_Q2B, 4>);
  } else {
    if (a.backbone == NGDB_GQE) go(entity_adam_kernel<NGDB_GQE, 8>);
    else go(entity_adam_kernel<NGDB_Q2B, 8>);
  }
  return 1;
}

int launch_sparse_adam_relation(const DevArgs& a, const SparseTable& t, const AdamHyper& hp,
                                const float* bc, const LaunchCtx& lc) {
  if (t.n_rows <= 0) return 0;
  const int64_t items = static_cast<int64_t>(t.n_rows) * (t.width / 4);
  launch_pdl(relation_adam_kernel, dim3(static_cast<int>((items + 255) / 256)), dim3(256), 0,
             lc.stream, 1, a, t, hp, bc);
  return 1;
}

int launch_dense_adam(float* w, float* m, float* v, float* g, int64_t n, const AdamHyper& hp,
                      const float* bc, const LaunchCtx& lc) {
  if (n <= 0) return 0;
  const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, lc.num_sms * 8));
  launch_pdl(dense_adam_kernel, dim3(blocks), dim3(256), 0, lc.stream, 1, w, m, v, g, n, hp, bc);
  return 1;
}

}  // namespace ngdb_dev
