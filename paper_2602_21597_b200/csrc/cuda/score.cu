// Fused negative-sample scoring + loss (SPEC.md:541-549 compute_loss, Eq. 6
// PAPER.md:259-263) and the union-branch Score operator.
//
// A cluster of S CTAs per scoring node, each taking a contiguous range of its
// candidates. Candidate rows are staged in shared memory by the bulk-copy (TMA
// 1-D) engine: a producer warp keeps a ring of ~48 KB of rows in flight
// (cp.async.bulk + mbarrier complete_tx), four consumer warps take rows
// round-robin, read them with 128-bit shared loads, reduce the distance with
// shuffles and — because the loss is a sum of per-candidate terms, so dL/dd_j
// depends on d_j alone — fold coef_j * dd_j/dq into per-lane registers in the
// same pass. Loads never wait on math: the ring decouples HBM latency from the
// per-row work. Every candidate row is read exactly once. Candidate-row
// gradients are NOT materialised: the
// optimizer recomputes coef_j * dd_j/dv from (q, coef) while it updates each
// touched row.
//
//   psi_pos = -log sigma(gamma - d_pos) = softplus(d_pos - gamma)
//   psi_neg = -log sigma(d_neg - gamma) = softplus(gamma - d_neg), mean over K
//   GQE distance: ||v - q||_1                                     (SURVEY A-7)
//   Q2B distance: ||max(0,|v-c|-o)||_1 + alpha ||min(|v-c|,o)||_1
//   BetaE:        sum_dims KL(entity || query) = lnB(q) + etab_c[r] + <q, etab[r]>
//                 over the per-step entity table of beta.cu;
//                 dL/dq = sum_j coef_j etab[r_j] + (sum_j coef_j) [psi(A)-psi(A+B) | psi(B)-psi(A+B)]
#include <algorithm>
#include <cstdio>
#include <map>

#include "common.cuh"
#include "dist.cuh"
#include "special.cuh"

namespace ngdb_dev {
namespace {

constexpr int kCWarps = 8;                // consumer warps
constexpr int kThreads = 32 * (kCWarps + 1);  // + one producer warp
constexpr int kWarps = kThreads / 32;
// Shared-memory ring of candidate rows: `depth` slots of ent_w floats +
// barriers; ~48 KB of rows in flight per CTA (8..32 rows).
__host__ __device__ inline int ring_depth(int width) {
  const int d = 49152 / (width * 4);
  return d < 8 ? 8 : (d > 32 ? 32 : d);
}
struct Ring {
  float* rows;
  uint64_t* full;
  uint64_t* empty;
  int width;  // floats per row
  int depth;  // slots
};
inline size_t ring_bytes(int width) {
  const int depth = ring_depth(width);
  return static_cast<size_t>(depth) * width * sizeof(float) + 2 * depth * sizeof(uint64_t);
}
__device__ __forceinline__ Ring make_ring(float* smem, int width) {
  Ring r;
  r.depth = ring_depth(width);
  r.rows = smem;
  r.full = reinterpret_cast<uint64_t*>(smem + r.depth * width);
  r.empty = r.full + r.depth;
  r.width = width;
  if (threadIdx.x == 0) {
    for (int i = 0; i < r.depth; ++i) {
      mbar_init(&r.full[i], 1);
      mbar_init(&r.empty[i], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  return r;
}

__device__ __forceinline__ float4 f4(float x) { return make_float4(x, x, x, x); }

template <int BB, int kMaxChunks>
struct Lane {
  // this lane's slice of q: chunks c = lane + 32*i  (float4 units)
  float4 qc[kMaxChunks], qo[kMaxChunks];
  float4 gc[kMaxChunks], go[kMaxChunks];
  int nch;

  __device__ void load_q(const float* q, int dim, int lane) {
    const int d4 = dim / 4;
    nch = 0;
#pragma unroll
    for (int i = 0; i < kMaxChunks; ++i) {
      const int c = lane + 32 * i;
      if (c < d4) {
        qc[i] = ld4(q + 4 * c);
        qo[i] = BB != NGDB_GQE ? ld4(q + dim + 4 * c) : f4(0.f);
        nch = i + 1;
      }
      gc[i] = f4(0.f);
      go[i] = f4(0.f);
    }
  }
};

// Candidate rows of one scoring node: rows base + idx[j] * ent_w (the entity
// table, or for BetaE the step's entity table indexed by CSR row, whose
// per-row constant cbias[idx[j]] and the query constant qbias complete d_j).
struct Cands {
  const float* base;
  const int32_t* idx;
  const float* cbias;
  float qbias;
};

// Walk candidates [j_beg, j_end) of the node: the producer warp streams their
// rows into the ring, consumer warp w takes local rows w, w+4, ... For every
// candidate: d_j -> coef_of(j, d_j) returns coef_j -> dq accumulation.
template <int BB, int kMaxChunks, bool kGrad, class CoefOp>
__device__ __forceinline__ void sweep(const DevArgs& a, const Cands& cs, Lane<BB, kMaxChunks>& L,
                                      const Ring& ring, CoefOp&& coef_of, int part_idx = 0,
                                      int n_parts = 1) {
  constexpr bool kBeta = BB == NGDB_BETAE;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int d4 = a.dim / 4;
  const int j_beg = part_idx * a.ncand / n_parts, j_end = (part_idx + 1) * a.ncand / n_parts;
  const int n_mine = j_end - j_beg;
  if (warp == kCWarps) {  // producer
    if (lane == 0) {
      const uint32_t bytes = static_cast<uint32_t>(ring.width * sizeof(float));
      for (int t = 0; t < n_mine; ++t) {
        const int slot = t % ring.depth, round = t / ring.depth;
        if (round > 0) mbar_wait_parity(&ring.empty[slot], (round - 1) & 1);
        const float* src = cs.base + static_cast<int64_t>(__ldg(cs.idx + j_beg + t)) * a.ent_w;
        mbar_arrive_expect_tx(&ring.full[slot], bytes);
        bulk_g2s(ring.rows + slot * ring.width, src, bytes, &ring.full[slot]);
      }
    }
    return;
  }
  for (int t = warp; t < n_mine; t += kCWarps) {
    const int slot = t % ring.depth, round = t / ring.depth, j = j_beg + t;
    const float* row = ring.rows + slot * ring.width;
    mbar_wait_parity(&ring.full[slot], round & 1);
    float4 v[kMaxChunks];
    float4 v2[kBeta ? kMaxChunks : 1];
#pragma unroll
    for (int i = 0; i < kMaxChunks; ++i) {
      const int c = lane + 32 * i;
      if (i < L.nch && c < d4) {
        v[i] = ld4(row + 4 * c);
        if constexpr (kBeta) v2[i] = ld4(row + a.dim + 4 * c);
      } else {
        v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        if constexpr (kBeta) v2[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring.empty[slot]);  // row is in registers: slot free
    float sx = 0.f, sy = 0.f, sz = 0.f, sw = 0.f;  // independent chains (ILP)
#pragma unroll
    for (int i = 0; i < kMaxChunks; ++i) {
      const int c = lane + 32 * i;
      if (i < L.nch && c < d4) {
        if constexpr (kBeta) {
          sx += Dist<BB>::term(v[i].x, v2[i].x, L.qc[i].x, L.qo[i].x);
          sy += Dist<BB>::term(v[i].y, v2[i].y, L.qc[i].y, L.qo[i].y);
          sz += Dist<BB>::term(v[i].z, v2[i].z, L.qc[i].z, L.qo[i].z);
          sw += Dist<BB>::term(v[i].w, v2[i].w, L.qc[i].w, L.qo[i].w);
        } else {
          sx += Dist<BB>::term(v[i].x, L.qc[i].x, L.qo[i].x, a.alpha_box);
          sy += Dist<BB>::term(v[i].y, L.qc[i].y, L.qo[i].y, a.alpha_box);
          sz += Dist<BB>::term(v[i].z, L.qc[i].z, L.qo[i].z, a.alpha_box);
          sw += Dist<BB>::term(v[i].w, L.qc[i].w, L.qo[i].w, a.alpha_box);
        }
      }
    }
    float dj = warp_sum((sx + sy) + (sz + sw));
    if constexpr (kBeta) dj += cs.qbias + __ldg(cs.cbias + __ldg(cs.idx + j));
    const float coef = coef_of(j, dj);
    if (!kGrad) continue;
#pragma unroll
    for (int i = 0; i < kMaxChunks; ++i) {
      const int c = lane + 32 * i;
      if (i < L.nch && c < d4) {
        if constexpr (kBeta) {
          L.gc[i].x += coef * v[i].x; L.go[i].x += coef * v2[i].x;
          L.gc[i].y += coef * v[i].y; L.go[i].y += coef * v2[i].y;
          L.gc[i].z += coef * v[i].z; L.go[i].z += coef * v2[i].z;
          L.gc[i].w += coef * v[i].w; L.go[i].w += coef * v2[i].w;
        } else {
          Dist<BB>::grad(v[i].x, L.qc[i].x, L.qo[i].x, coef, a.alpha_box, L.gc[i].x, L.go[i].x);
          Dist<BB>::grad(v[i].y, L.qc[i].y, L.qo[i].y, coef, a.alpha_box, L.gc[i].y, L.go[i].y);
          Dist<BB>::grad(v[i].z, L.qc[i].z, L.qo[i].z, coef, a.alpha_box, L.gc[i].z, L.go[i].z);
          Dist<BB>::grad(v[i].w, L.qc[i].w, L.qo[i].w, coef, a.alpha_box, L.gc[i].w, L.go[i].w);
        }
      }
    }
  }
}

// Cross-warp sum of the per-lane dq accumulators: every consumer warp stores
// its partial (and its loss / coefficient-sum partials) in its own shared row,
// one barrier, then the block sums the kCWarps rows in warp order
// (deterministic) into part[0]; lred[kLossTot] / lred[kCsumTot] receive the
// loss and coefficient sums. Ends with a barrier.
constexpr int kMaxWq = 1024;
constexpr int kLossTot = 2 * kCWarps, kCsumTot = 2 * kCWarps + 1, kLred = 2 * kCWarps + 2;
template <int BB, int kMaxChunks>
__device__ void reduce_partials(const DevArgs& a, const Lane<BB, kMaxChunks>& L, float (*part)[kMaxWq],
                                float* lred, float loss, float csum) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int d4 = a.dim / 4;
  if (warp < kCWarps) {
#pragma unroll
    for (int i = 0; i < kMaxChunks; ++i) {
      const int c = lane + 32 * i;
      if (i < L.nch && c < d4) {
        st4(part[warp] + 4 * c, L.gc[i]);
        if (BB != NGDB_GQE) st4(part[warp] + a.dim + 4 * c, L.go[i]);
      }
    }
    if (lane == 0) {
      lred[2 * warp] = loss;
      lred[2 * warp + 1] = csum;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x * 4; e < a.wq; e += kThreads * 4) {
    float4 t = ld4(part[0] + e);
#pragma unroll
    for (int w = 1; w < kCWarps; ++w) {
      const float4 u = ld4(part[w] + e);
      t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
    }
    st4(part[0] + e, t);
  }
  if (threadIdx.x == 0) {
    float l = 0.f, cs = 0.f;
    for (int w = 0; w < kCWarps; ++w) {
      l += lred[2 * w];
      cs += lred[2 * w + 1];
    }
    lred[kLossTot] = l;
    lred[kCsumTot] = cs;
  }
  __syncthreads();
}

__device__ float block_sum(float v, float* red) {
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  if (threadIdx.x == 0)
    for (int i = 0; i < kWarps; ++i) t += red[i];
  return t;  // thread 0
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
}
__device__ __forceinline__ float ld_peer(const float* local, uint32_t peer) {
  uint32_t remote;
  float v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(remote)
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(local))), "r"(peer));
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote));
  return v;
}

// Candidate set of a scoring node. BetaE also needs lnB(query) summed over the
// dims (block-wide; every thread gets the value).
template <int BB>
__device__ Cands node_cands(const DevArgs& a, const ngdb_node_desc& d, const float* q, float* lred) {
  if constexpr (BB == NGDB_BETAE) {
    __shared__ float qb;
    float t = 0.f;
    for (int e = threadIdx.x; e < a.dim; e += kThreads) t += dg_lbeta(q[e], q[a.dim + e]);
    t = block_sum(warp_sum(t), lred);
    if (threadIdx.x == 0) qb = t;
    __syncthreads();
    return Cands{a.etab, a.cand_local + static_cast<int64_t>(d.aux) * a.ncand, a.etab_c, qb};
  } else {
    if (a.fused)  // FuseSemantic: candidate rows are the step's fused rows
      return Cands{a.etab, a.cand_local + static_cast<int64_t>(d.aux) * a.ncand, nullptr, 0.f};
    return Cands{a.ent, a.cand + static_cast<int64_t>(d.id) * a.ncand, nullptr, 0.f};
  }
}
// BetaE query-side part of dKL/dq (per unit coefficient): psi(A) - psi(A+B) for
// the alpha half, psi(B) - psi(A+B) for the beta half
__device__ __forceinline__ float beta_qterm(const DevArgs& a, const float* q, int e) {
  const int D = a.dim;
  const int i = e < D ? e : e - D;
  const float A = q[i], B = q[D + i];
  return dg_digamma(e < D ? A : B) - dg_digamma(A + B);
}

// Fused score + loss, persistent and streaming. Work items are (Loss node,
// part): the S parts of a node split its candidates into contiguous ranges.
// Each CTA walks items blockIdx.x, +gridDim.x, ...; its producer warp streams
// the query row of every item (double-buffered) and the candidate rows of
// every item (ring) ahead of the consumers without ever draining between
// items, so HBM stays busy through the per-item reductions. An item's dL/dq
// and loss partials are combined in part order by the last CTA to finish the
// node (global partials + arrival counter: deterministic, no cluster needed).
constexpr int kConsumerThreads = kCWarps * 32;
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumerThreads) : "memory");
}

struct LossSmem {  // dynamic shared memory of loss_stream_kernel, after the ring
  float* q[2];     // query rows of the current / next item
  uint64_t* qfull;
  uint64_t* qempty;
};
inline size_t loss_smem_bytes(int ent_w, int wq) {
  return ring_bytes(ent_w) + 2 * static_cast<size_t>(wq) * sizeof(float) + 4 * sizeof(uint64_t);
}

template <int BB, int NCH>
__global__ void __launch_bounds__(kThreads, 2) loss_stream_kernel(DevArgs a, int first, int n,
                                                                  int S) {
  extern __shared__ __align__(128) float ring_smem[];
  __shared__ __align__(16) float parts[kCWarps][kMaxWq];
  __shared__ float lred[kLred];
  __shared__ int last_flag;
  __shared__ float qbias_s;
  constexpr bool kBeta = BB == NGDB_BETAE;
  LossSmem ls;
  const int depth = ring_depth(a.ent_w);
  ls.q[0] = ring_smem + depth * a.ent_w + 4 * depth;  // after rows + 2*depth barriers
  ls.q[1] = ls.q[0] + a.wq;
  ls.qfull = reinterpret_cast<uint64_t*>(ls.q[1] + a.wq);
  ls.qempty = ls.qfull + 2;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&ls.qfull[i], 1);
      mbar_init(&ls.qempty[i], 1);
    }
  }
  const Ring ring = make_ring(ring_smem, a.ent_w);  // inits its barriers + fence + __syncthreads
  pdl_start();
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int n_items = S * n;
  auto cand_index = [&](const ngdb_node_desc& d) -> const int32_t* {
    if (kBeta || a.fused) return a.cand_local + static_cast<int64_t>(d.aux) * a.ncand;
    return a.cand + static_cast<int64_t>(d.id) * a.ncand;
  };
  const float* rows_base = (kBeta || a.fused) ? a.etab : a.ent;

  if (warp == kCWarps) {  // ---- producer ----
    if (lane != 0) return;
    const uint32_t row_bytes = static_cast<uint32_t>(a.ent_w * sizeof(float));
    const uint32_t q_bytes = static_cast<uint32_t>(a.wq * sizeof(float));
    int pos = 0, qi = 0;
    for (int t = blockIdx.x; t < n_items; t += gridDim.x) {
      const int node = t / S, part = t % S;
      const ngdb_node_desc d = a.nodes[first + node];
      if (d.aux < 0) continue;  // union query: no candidate rows
      const int qs = qi & 1;
      if (qi >= 2) mbar_wait_parity(&ls.qempty[qs], ((qi >> 1) - 1) & 1);
      mbar_arrive_expect_tx(&ls.qfull[qs], q_bytes);
      bulk_g2s(ls.q[qs], a.arena + d.in[0], q_bytes, &ls.qfull[qs]);
      ++qi;
      const int32_t* idx = cand_index(d);
      const int j_beg = part * a.ncand / S, j_end = (part + 1) * a.ncand / S;
      for (int j = j_beg; j < j_end; ++j, ++pos) {
        const int slot = pos % ring.depth, round = pos / ring.depth;
        if (round > 0) mbar_wait_parity(&ring.empty[slot], (round - 1) & 1);
        mbar_arrive_expect_tx(&ring.full[slot], row_bytes);
        bulk_g2s(ring.rows + slot * ring.width,
                 rows_base + static_cast<int64_t>(__ldg(idx + j)) * a.ent_w, row_bytes,
                 &ring.full[slot]);
      }
    }
    return;
  }

  // ---- consumers (kCWarps warps) ----
  const int ctid = threadIdx.x;  // < kConsumerThreads
  const int d4 = a.dim / 4;
  int pos = 0, qi = 0;
  for (int t = blockIdx.x; t < n_items; t += gridDim.x) {
    const int node = t / S, part = t % S;
    const ngdb_node_desc d = a.nodes[first + node];
    const int qid = d.id;
    if (d.aux < 0) {
      // union query: the input already holds min-over-branch distances; part 0
      // computes the whole loss, the other parts have nothing to do
      if (part == 0) {
        float loss = 0.f;
        for (int j = ctid; j < a.ncand; j += kConsumerThreads) {
          const float c = loss_coef(a, j, a.arena[d.in[0] + j], loss);
          a.ddbuf[static_cast<int64_t>(qid) * a.ncand + j] = c;
        }
        loss = warp_sum(loss);
        if (lane == 0) lred[warp] = loss;
        consumers_sync();
        if (ctid == 0) {
          float total = 0.f;
          for (int w = 0; w < kCWarps; ++w) total += lred[w];
          a.loss_out[qid] = total;
          a.arena[d.out] = total;
          if (!isfinite(total)) atomicOr(&a.flags[0], 1);
        }
        consumers_sync();
      }
      continue;
    }
    const int qs = qi & 1;
    mbar_wait_parity(&ls.qfull[qs], (qi >> 1) & 1);
    const float* q = ls.q[qs];
    Lane<BB, NCH> L;
    L.load_q(q, a.dim, lane);
    if (part == 0) {
      float* qcopy = a.qbuf + static_cast<int64_t>(d.aux) * a.wq;
      for (int e = ctid * 4; e < a.wq; e += kConsumerThreads * 4) st4(qcopy + e, ld4(q + e));
    }
    float qbias = 0.f;
    if constexpr (kBeta) {  // lnB(query) summed over the dims
      float tq = 0.f;
      for (int e = ctid; e < a.dim; e += kConsumerThreads) tq += dg_lbeta(q[e], q[a.dim + e]);
      tq = warp_sum(tq);
      if (lane == 0) lred[warp] = tq;
      consumers_sync();
      if (ctid == 0) {
        float tt = 0.f;
        for (int w = 0; w < kCWarps; ++w) tt += lred[w];
        qbias_s = tt;
      }
      consumers_sync();
      qbias = qbias_s;
    }
    const int32_t* idx = cand_index(d);
    const int j_beg = part * a.ncand / S, j_end = (part + 1) * a.ncand / S;
    const int n_mine = j_end - j_beg;
    float* coefs = a.coefbuf + static_cast<int64_t>(d.aux) * a.ncand;
    float loss = 0.f, csum = 0.f;  // identical in every lane of a warp
    for (int u = warp; u < n_mine; u += kCWarps) {
      const int p = pos + u, slot = p % ring.depth, j = j_beg + u;
      const float* row = ring.rows + slot * ring.width;
      mbar_wait_parity(&ring.full[slot], (p / ring.depth) & 1);
      float4 v[NCH];
      float4 v2[kBeta ? NCH : 1];
#pragma unroll
      for (int i = 0; i < NCH; ++i) {
        const int c = lane + 32 * i;
        if (i < L.nch && c < d4) {
          v[i] = ld4(row + 4 * c);
          if constexpr (kBeta) v2[i] = ld4(row + a.dim + 4 * c);
        } else {
          v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
          if constexpr (kBeta) v2[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&ring.empty[slot]);
      float sx = 0.f, sy = 0.f, sz = 0.f, sw = 0.f;
#pragma unroll
      for (int i = 0; i < NCH; ++i) {
        const int c = lane + 32 * i;
        if (i < L.nch && c < d4) {
          if constexpr (kBeta) {
            sx += Dist<BB>::term(v[i].x, v2[i].x, L.qc[i].x, L.qo[i].x);
            sy += Dist<BB>::term(v[i].y, v2[i].y, L.qc[i].y, L.qo[i].y);
            sz += Dist<BB>::term(v[i].z, v2[i].z, L.qc[i].z, L.qo[i].z);
            sw += Dist<BB>::term(v[i].w, v2[i].w, L.qc[i].w, L.qo[i].w);
          } else {
            sx += Dist<BB>::term(v[i].x, L.qc[i].x, L.qo[i].x, a.alpha_box);
            sy += Dist<BB>::term(v[i].y, L.qc[i].y, L.qo[i].y, a.alpha_box);
            sz += Dist<BB>::term(v[i].z, L.qc[i].z, L.qo[i].z, a.alpha_box);
            sw += Dist<BB>::term(v[i].w, L.qc[i].w, L.qo[i].w, a.alpha_box);
          }
        }
      }
      float dj = warp_sum((sx + sy) + (sz + sw));
      if constexpr (kBeta) dj += qbias + __ldg(a.etab_c + __ldg(idx + j));
      const float coef = loss_coef(a, j, dj, loss);
      csum += coef;
      if (lane == 0) coefs[j] = coef;
#pragma unroll
      for (int i = 0; i < NCH; ++i) {
        const int c = lane + 32 * i;
        if (i < L.nch && c < d4) {
          if constexpr (kBeta) {
            L.gc[i].x += coef * v[i].x; L.go[i].x += coef * v2[i].x;
            L.gc[i].y += coef * v[i].y; L.go[i].y += coef * v2[i].y;
            L.gc[i].z += coef * v[i].z; L.go[i].z += coef * v2[i].z;
            L.gc[i].w += coef * v[i].w; L.go[i].w += coef * v2[i].w;
          } else {
            Dist<BB>::grad(v[i].x, L.qc[i].x, L.qo[i].x, coef, a.alpha_box, L.gc[i].x, L.go[i].x);
            Dist<BB>::grad(v[i].y, L.qc[i].y, L.qo[i].y, coef, a.alpha_box, L.gc[i].y, L.go[i].y);
            Dist<BB>::grad(v[i].z, L.qc[i].z, L.qo[i].z, coef, a.alpha_box, L.gc[i].z, L.go[i].z);
            Dist<BB>::grad(v[i].w, L.qc[i].w, L.qo[i].w, coef, a.alpha_box, L.gc[i].w, L.go[i].w);
          }
        }
      }
    }
    pos += n_mine;
    // cross-warp partials (consumer threads only): every warp stores its
    // row, one consumer barrier, then the rows are summed in warp order
    if (lane == 0) {
      lred[2 * warp] = loss;
      lred[2 * warp + 1] = csum;
    }
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      const int c = lane + 32 * i;
      if (i < L.nch && c < d4) {
        st4(parts[warp] + 4 * c, L.gc[i]);
        if (BB != NGDB_GQE) st4(parts[warp] + a.dim + 4 * c, L.go[i]);
      }
    }
    consumers_sync();
    if (ctid == 0) mbar_arrive(&ls.qempty[qs]);  // every consumer is done with q
    ++qi;
    float* dst = S == 1 ? a.dqbuf + static_cast<int64_t>(d.aux) * a.wq
                        : a.lpart + static_cast<int64_t>(t) * a.wq;
    for (int e = ctid * 4; e < a.wq; e += kConsumerThreads * 4) {
      float4 s4 = ld4(parts[0] + e);
#pragma unroll
      for (int w = 1; w < kCWarps; ++w) {
        const float4 u4 = ld4(parts[w] + e);
        s4.x += u4.x; s4.y += u4.y; s4.z += u4.z; s4.w += u4.w;
      }
      st4(dst + e, s4);
    }
    float l_item = 0.f, c_item = 0.f;
    if (ctid == 0)
      for (int w = 0; w < kCWarps; ++w) {
        l_item += lred[2 * w];
        c_item += lred[2 * w + 1];
      }
    if (S > 1) {
      if (ctid == 0) {
        a.lpart_scalar[2 * t] = l_item;
        a.lpart_scalar[2 * t + 1] = c_item;
      }
      __threadfence();
      consumers_sync();
      if (ctid == 0) last_flag = atomicAdd(&a.lcount[node], 1) == S - 1;
      consumers_sync();
      if (!last_flag) continue;
      __threadfence();  // the other parts' partials are visible
      // the last part of the node combines all S partials in part order
      float* out = a.dqbuf + static_cast<int64_t>(d.aux) * a.wq;
      const float* base = a.lpart + static_cast<int64_t>(node) * S * a.wq;
      for (int e = ctid * 4; e < a.wq; e += kConsumerThreads * 4) {
        float4 s4 = ld4(base + e);
        for (int p2 = 1; p2 < S; ++p2) {
          const float4 u4 = ld4(base + static_cast<int64_t>(p2) * a.wq + e);
          s4.x += u4.x; s4.y += u4.y; s4.z += u4.z; s4.w += u4.w;
        }
        st4(out + e, s4);
      }
      if (ctid == 0) {
        l_item = c_item = 0.f;
        for (int p2 = 0; p2 < S; ++p2) {
          l_item += a.lpart_scalar[2 * (node * S + p2)];
          c_item += a.lpart_scalar[2 * (node * S + p2) + 1];
        }
        a.lcount[node] = 0;  // ready for the next launch
      }
    }
    if constexpr (kBeta) {
      // dL/dq += (sum_j coef_j) [psi(A)-psi(A+B) | psi(B)-psi(A+B)] (query term)
      consumers_sync();
      if (ctid == 0) qbias_s = c_item;
      consumers_sync();
      const float sc = qbias_s;
      float* out = a.dqbuf + static_cast<int64_t>(d.aux) * a.wq;
      const float* qq = a.arena + d.in[0];
      for (int e = ctid; e < a.wq; e += kConsumerThreads) out[e] += sc * beta_qterm(a, qq, e);
    }
    if (ctid == 0) {
      a.loss_out[qid] = l_item;
      a.arena[d.out] = l_item;
      if (!isfinite(l_item)) atomicOr(&a.flags[0], 1);
    }
    consumers_sync();  // parts[] / lred reused by the next item
  }
}

// Union branch Score, a (S,1,1) cluster per node like the Loss kernel: fwd
// writes the distance vector; bwd turns the routed dL/dd into coef (for the
// optimizer) and dL/dq (its G slot), the S partials of dL/dq reduce-scattered
// over DSMEM in rank order.
template <int BB, int NCH>
__global__ void __launch_bounds__(kThreads, 2) score_kernel(DevArgs a, int dir, int first, int S) {
  extern __shared__ __align__(128) float ring_smem[];
  __shared__ __align__(16) float parts[kCWarps][kMaxWq];
  __shared__ float lred[kLred];
  const Ring ring = make_ring(ring_smem, a.ent_w);
  pdl_start();
  const int part = blockIdx.x % S;
  const ngdb_node_desc d = a.nodes[first + blockIdx.x / S];
  const float* q = a.arena + d.in[0];
  const int lane = threadIdx.x & 31;
  Lane<BB, NCH> L;
  L.load_q(q, a.dim, lane);
  const Cands cs = node_cands<BB>(a, d, q, lred);
  if (dir == 0) {
    if (part == 0) {
      float* qcopy = a.qbuf + static_cast<int64_t>(d.aux) * a.wq;
      for (int e = threadIdx.x * 4; e < a.wq; e += kThreads * 4) st4(qcopy + e, ld4(q + e));
    }
    float* out = a.arena + d.out;
    sweep<BB, NCH, false>(
        a, cs, L, ring,
        [&](int j, float dj) {
          if (lane == 0) out[j] = dj;
          return 0.f;
        },
        part, S);
    return;
  }
  const float* g = a.arena + d.grad;
  if (part == 0) {
    float* coefs = a.coefbuf + static_cast<int64_t>(d.aux) * a.ncand;
    for (int j = threadIdx.x; j < a.ncand; j += kThreads) coefs[j] = g[j];
  }
  float csum = 0.f;  // Σ_j g[j] over this CTA's candidates (BetaE query term)
  sweep<BB, NCH, true>(
      a, cs, L, ring,
      [&](int j, float) {
        csum += g[j];
        return g[j];
      },
      part, S);
  reduce_partials<BB, NCH>(a, L, parts, lred, 0.f, csum);
  const float* red = parts[0];
  cluster_sync_all();
  float sc = 0.f;
  if constexpr (BB == NGDB_BETAE)  // over all S parts, in rank order
    for (int p = 0; p < S; ++p) sc += (p == part) ? lred[kCsumTot] : ld_peer(lred + kCsumTot, p);
  float* dst = a.arena + d.out;
  const int e0 = part * a.wq / S, e1 = (part + 1) * a.wq / S;
  for (int e = e0 + threadIdx.x; e < e1; e += kThreads) {
    float v = 0.f;
    for (int p = 0; p < S; ++p) v += (p == part) ? red[e] : ld_peer(red + e, p);
    if constexpr (BB == NGDB_BETAE) v += sc * beta_qterm(a, q, e);
    dst[e] = v;
  }
  cluster_sync_all();  // partials stay resident until every slice was read
}

}  // namespace

// Launch geometry of a ring kernel for a given dynamic smem size: CTAs
// resident at once and the largest cluster the device can co-schedule. The
// function's max-dynamic-smem attribute is set to exactly `smem` before each
// launch whose size differs from the last one: cluster launches are validated
// against that attribute, not against the bytes actually requested.
struct RingGeom {
  int resident = 0, max_cluster = 1;
};
template <class K>
RingGeom ring_geometry(K kernel, size_t smem, int num_sms) {
  RingGeom g;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem);
  g.resident = std::max(1, per_sm) * num_sms;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(8 * 64);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  int mc = 1;
  if (cudaOccupancyMaxPotentialClusterSize(&mc, kernel, &cfg) != cudaSuccess) mc = 1;
  g.max_cluster = std::max(1, std::min(8, mc));
  cudaGetLastError();  // a failed query must not leak into the launch checks
  return g;
}
// parts per node (cluster size): as many as fit in ONE wave, so no CTA waits
// for a second wave
inline int parts_for(int n, const RingGeom& g) {
  // >= 2 keeps every launch a real cluster (the kernels use cluster barriers)
  return std::max(std::min(2, g.max_cluster), std::min(g.max_cluster, g.resident / std::max(n, 1)));
}

// A kernel's max-dynamic-smem attribute must cover every launch, and cluster
// launches are validated against the attribute itself: keep it equal to the
// size of the launch at hand (set only when it changes).
template <class K>
void ensure_smem_attr(K kernel, size_t smem) {
  static std::map<const void*, size_t> attr;  // kernel -> value last set
  const void* key = reinterpret_cast<const void*>(kernel);
  auto it = attr.find(key);
  if (it == attr.end() || it->second != smem) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr[key] = smem;
  }
}

template <class K>
void launch_ring_kernel(K kernel, int ent_w, int n, cudaStream_t s, const DevArgs& a, int x,
                        int first) {
  const size_t smem = ring_bytes(ent_w);
  static std::map<std::pair<const void*, size_t>, RingGeom> cache;  // (kernel, smem) -> geometry
  const void* key = reinterpret_cast<const void*>(kernel);
  ensure_smem_attr(kernel, smem);
  RingGeom& g = cache[{key, smem}];
  if (!g.resident) g = ring_geometry(kernel, smem, 148);
  const int S = parts_for(n, g);
  launch_pdl(kernel, dim3(S * n), dim3(kThreads), smem, s, S, a, x, first, S);
}

template <int NCH>
void launch_loss_nch(const DevArgs& a, int first, int n, cudaStream_t s) {
  auto go = [&](auto kernel) {
    const size_t smem = loss_smem_bytes(a.ent_w, a.wq);
    static std::map<std::pair<const void*, size_t>, int> cache;  // -> resident CTAs
    int& resident = cache[{reinterpret_cast<const void*>(kernel), smem}];
    ensure_smem_attr(kernel, smem);
    if (!resident) {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem);
      resident = std::max(1, per_sm) * 148;
    }
    // parts per node: enough items for every resident CTA, within the
    // partial-buffer capacity (a.lpart_items)
    int S = std::max(1, std::min(8, (resident + n - 1) / n));
    while (S > 1 && S * n > a.lpart_items) --S;
    const int grid = std::min(resident, S * n);
    launch_pdl(kernel, dim3(grid), dim3(kThreads), smem, s, 1, a, first, n, S);
  };
  if (a.backbone == NGDB_GQE) go(loss_stream_kernel<NGDB_GQE, NCH>);
  else if (a.backbone == NGDB_BETAE) go(loss_stream_kernel<NGDB_BETAE, NCH>);
  else go(loss_stream_kernel<NGDB_Q2B, NCH>);
}
template <int NCH>
void launch_score_nch(const DevArgs& a, int dir, int first, int n, cudaStream_t s) {
  if (a.backbone == NGDB_GQE) launch_ring_kernel(score_kernel<NGDB_GQE, NCH>, a.ent_w, n, s, a, dir, first);
  else if (a.backbone == NGDB_BETAE) launch_ring_kernel(score_kernel<NGDB_BETAE, NCH>, a.ent_w, n, s, a, dir, first);
  else launch_ring_kernel(score_kernel<NGDB_Q2B, NCH>, a.ent_w, n, s, a, dir, first);
}

int launch_loss_fwd(const DevArgs& a, int first, int n, const LaunchCtx& lc) {
  if (n <= 0) return 0;
  // rows of d floats are d/4 float4 chunks spread over 32 lanes
  if (a.dim <= 512) launch_loss_nch<4>(a, first, n, lc.stream);
  else launch_loss_nch<8>(a, first, n, lc.stream);
  return 1;
}

int launch_score(const DevArgs& a, int dir, int first, int n, const LaunchCtx& lc) {
  if (n <= 0) return 0;
  if (a.dim <= 512) launch_score_nch<4>(a, dir, first, n, lc.stream);
  else launch_score_nch<8>(a, dir, first, n, lc.stream);
  return 1;
}

}  // namespace ngdb_dev
