// Fused negative-sample scoring + loss (SPEC.md:541-549 compute_loss, Eq. 6
// PAPER.md:259-263) and the union-branch Score operator.
//
// One CTA per scoring node, 4 warps. Each warp owns candidates j = 4*warp + 16*t
// (+0..3): it issues the 128-bit loads of FOUR candidate rows at once (16 loads in
// flight per lane), reduces the four distances with shuffles, and — because the
// loss is a sum of per-candidate terms, so dL/dd_j depends on d_j alone — folds
// coef_j * dd_j/dq into per-lane registers in the same pass. Every candidate row
// is read exactly once. Candidate-row gradients are NOT materialised: the
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

#include "common.cuh"
#include "dist.cuh"
#include "special.cuh"

namespace ngdb_dev {
namespace {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kRows = 4;          // candidate rows in flight per warp

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

// Walk all candidates of the node with one warp per 4-row group. For every
// candidate: d_j -> coef_of(j, d_j) returns coef_j -> dq accumulation.
template <int BB, int kMaxChunks, bool kGrad, class CoefOp>
__device__ __forceinline__ void sweep(const DevArgs& a, const Cands& cs, Lane<BB, kMaxChunks>& L,
                                      CoefOp&& coef_of, int part_idx = 0, int n_parts = 1) {
  constexpr bool kBeta = BB == NGDB_BETAE;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int d4 = a.dim / 4;
  // candidate groups are dealt round-robin over (part, warp)
  for (int j0 = (part_idx * kWarps + warp) * kRows; j0 < a.ncand;
       j0 += n_parts * kWarps * kRows) {
    float4 v[kRows][kMaxChunks];
    float4 v2[kBeta ? kRows : 1][kBeta ? kMaxChunks : 1];
    float part[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const int j = min(j0 + r, a.ncand - 1);
      const float* row = cs.base + static_cast<int64_t>(__ldg(cs.idx + j)) * a.ent_w;
#pragma unroll
      for (int i = 0; i < kMaxChunks; ++i) {
        const int c = lane + 32 * i;
        if (i < L.nch && c < d4) {
          v[r][i] = ldg4(row + 4 * c);
          if constexpr (kBeta) v2[r][i] = ldg4(row + a.dim + 4 * c);
        } else {
          v[r][i] = make_float4(0.f, 0.f, 0.f, 0.f);
          if constexpr (kBeta) v2[r][i] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < kMaxChunks; ++i) {
        const int c = lane + 32 * i;
        if (i < L.nch && c < d4) {
          if constexpr (kBeta) {
            s += Dist<BB>::term(v[r][i].x, v2[r][i].x, L.qc[i].x, L.qo[i].x);
            s += Dist<BB>::term(v[r][i].y, v2[r][i].y, L.qc[i].y, L.qo[i].y);
            s += Dist<BB>::term(v[r][i].z, v2[r][i].z, L.qc[i].z, L.qo[i].z);
            s += Dist<BB>::term(v[r][i].w, v2[r][i].w, L.qc[i].w, L.qo[i].w);
          } else {
            s += Dist<BB>::term(v[r][i].x, L.qc[i].x, L.qo[i].x, a.alpha_box);
            s += Dist<BB>::term(v[r][i].y, L.qc[i].y, L.qo[i].y, a.alpha_box);
            s += Dist<BB>::term(v[r][i].z, L.qc[i].z, L.qo[i].z, a.alpha_box);
            s += Dist<BB>::term(v[r][i].w, L.qc[i].w, L.qo[i].w, a.alpha_box);
          }
        }
      }
      part[r] = warp_sum(s);
      if constexpr (kBeta) {
        const int j = min(j0 + r, a.ncand - 1);
        part[r] += cs.qbias + __ldg(cs.cbias + __ldg(cs.idx + j));
      }
    }
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const int j = j0 + r;
      if (j >= a.ncand) break;
      const float coef = coef_of(j, part[r]);
      if (!kGrad) continue;
#pragma unroll
      for (int i = 0; i < kMaxChunks; ++i) {
        const int c = lane + 32 * i;
        if (i < L.nch && c < d4) {
          if constexpr (kBeta) {
            L.gc[i].x += coef * v[r][i].x; L.go[i].x += coef * v2[r][i].x;
            L.gc[i].y += coef * v[r][i].y; L.go[i].y += coef * v2[r][i].y;
            L.gc[i].z += coef * v[r][i].z; L.go[i].z += coef * v2[r][i].z;
            L.gc[i].w += coef * v[r][i].w; L.go[i].w += coef * v2[r][i].w;
          } else {
            Dist<BB>::grad(v[r][i].x, L.qc[i].x, L.qo[i].x, coef, a.alpha_box, L.gc[i].x, L.go[i].x);
            Dist<BB>::grad(v[r][i].y, L.qc[i].y, L.qo[i].y, coef, a.alpha_box, L.gc[i].y, L.go[i].y);
            Dist<BB>::grad(v[r][i].z, L.qc[i].z, L.qo[i].z, coef, a.alpha_box, L.gc[i].z, L.go[i].z);
            Dist<BB>::grad(v[r][i].w, L.qc[i].w, L.qo[i].w, coef, a.alpha_box, L.gc[i].w, L.go[i].w);
          }
        }
      }
    }
  }
}

// Cross-warp sum of the per-lane dq accumulators into dst (wq floats).
template <int BB, int kMaxChunks>
__device__ void reduce_dq(const DevArgs& a, Lane<BB, kMaxChunks>& L, float* red, float* dst) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int d4 = a.dim / 4;
  for (int w = 0; w < kWarps; ++w) {
    if (warp == w) {
#pragma unroll
      for (int i = 0; i < kMaxChunks; ++i) {
        const int c = lane + 32 * i;
        if (i < L.nch && c < d4) {
          float4* rc = reinterpret_cast<float4*>(red + 4 * c);
          float4* ro = reinterpret_cast<float4*>(red + a.dim + 4 * c);
          if (w == 0) {
            *rc = L.gc[i];
            if (BB != NGDB_GQE) *ro = L.go[i];
          } else {
            float4 t = *rc;
            *rc = make_float4(t.x + L.gc[i].x, t.y + L.gc[i].y, t.z + L.gc[i].z, t.w + L.gc[i].w);
            if (BB != NGDB_GQE) {
              t = *ro;
              *ro = make_float4(t.x + L.go[i].x, t.y + L.go[i].y, t.z + L.go[i].z, t.w + L.go[i].w);
            }
          }
        }
      }
    }
    __syncthreads();
  }
  if (dst)
    for (int e = threadIdx.x * 4; e < a.wq; e += kThreads * 4) st4(dst + e, ld4(red + e));
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

// A (S,1,1) cluster per Loss node (S = 2..8, chosen so a pop fills the GPU):
// the CTAs take candidate groups round-robin, then reduce-scatter their dL/dq
// partials over DSMEM — CTA p sums dims [p*wq/S, (p+1)*wq/S) over all S
// partials in rank order (deterministic); CTA 0 sums the loss partials.
template <int BB, int NCH>
__global__ void __launch_bounds__(kThreads) loss_fwd_kernel(DevArgs a, int first, int S) {
  pdl_start();
  __shared__ __align__(16) float red[2 * 1024];
  __shared__ float lred[kWarps + 2];
  const int part = blockIdx.x % S;
  const ngdb_node_desc d = a.nodes[first + blockIdx.x / S];
  const int qi = d.id;
  if (d.aux < 0) {
    // union query: the input already holds min-over-branch distances
    if (part == 0) {
      float loss = 0.f;
      for (int j = threadIdx.x; j < a.ncand; j += kThreads) {
        const float c = loss_coef(a, j, a.arena[d.in[0] + j], loss);
        a.ddbuf[static_cast<int64_t>(qi) * a.ncand + j] = c;
      }
      loss = block_sum(warp_sum(loss), lred);
      if (threadIdx.x == 0) {
        a.loss_out[qi] = loss;
        a.arena[d.out] = loss;
        if (!isfinite(loss)) atomicOr(&a.flags[0], 1);
      }
    }
    cluster_sync_all();  // barrier count is uniform across both paths
    cluster_sync_all();
    return;
  }
  const float* q = a.arena + d.in[0];
  if (part == 0) {
    float* qcopy = a.qbuf + static_cast<int64_t>(d.aux) * a.wq;
    for (int e = threadIdx.x * 4; e < a.wq; e += kThreads * 4) st4(qcopy + e, ld4(q + e));
  }
  Lane<BB, NCH> L;
  L.load_q(q, a.dim, threadIdx.x & 31);
  const Cands cs = node_cands<BB>(a, d, q, lred);
  float loss = 0.f, csum = 0.f;  // identical in every lane of a warp
  float* coefs = a.coefbuf + static_cast<int64_t>(d.aux) * a.ncand;
  const int lane = threadIdx.x & 31;
  sweep<BB, NCH, true>(
      a, cs, L,
      [&](int j, float dj) {
        const float c = loss_coef(a, j, dj, loss);
        csum += c;
        if (lane == 0) coefs[j] = c;
        return c;
      },
      part, S);
  loss = block_sum(lane == 0 ? loss : 0.f, lred);
  if (threadIdx.x == 0) lred[kWarps] = loss;
  if constexpr (BB == NGDB_BETAE) {
    csum = block_sum(lane == 0 ? csum : 0.f, lred);
    if (threadIdx.x == 0) lred[kWarps + 1] = csum;
  }
  reduce_dq<BB, NCH>(a, L, red, nullptr);
  cluster_sync_all();
  {
    float* dst = a.dqbuf + static_cast<int64_t>(d.aux) * a.wq;
    const int e0 = part * a.wq / S, e1 = (part + 1) * a.wq / S;
    float sc = 0.f;
    if constexpr (BB == NGDB_BETAE)
      for (int p = 0; p < S; ++p) sc += (p == part) ? lred[kWarps + 1] : ld_peer(lred + kWarps + 1, p);
    for (int e = e0 + threadIdx.x; e < e1; e += kThreads) {
      float v = 0.f;
      for (int p = 0; p < S; ++p) v += (p == part) ? red[e] : ld_peer(red + e, p);
      if constexpr (BB == NGDB_BETAE) v += sc * beta_qterm(a, q, e);
      dst[e] = v;
    }
    if (part == 0 && threadIdx.x == 0) {
      float total = 0.f;
      for (int p = 0; p < S; ++p) total += (p == 0) ? lred[kWarps] : ld_peer(lred + kWarps, p);
      a.loss_out[qi] = total;
      a.arena[d.out] = total;
      if (!isfinite(total)) atomicOr(&a.flags[0], 1);
    }
  }
  cluster_sync_all();  // partial tiles stay resident until every slice was read
}

// Union branch Score: fwd writes the distance vector; bwd turns the routed
// dL/dd into coef (for the optimizer) and dL/dq (its G slot).
template <int BB, int NCH>
__global__ void __launch_bounds__(kThreads) score_kernel(DevArgs a, int dir, int first) {
  pdl_start();
  __shared__ __align__(16) float red[2 * 1024];
  __shared__ float lred[kWarps + 1];
  const ngdb_node_desc d = a.nodes[first + blockIdx.x];
  const float* q = a.arena + d.in[0];
  const int lane = threadIdx.x & 31;
  Lane<BB, NCH> L;
  L.load_q(q, a.dim, lane);
  const Cands cs = node_cands<BB>(a, d, q, lred);
  if (dir == 0) {
    float* qcopy = a.qbuf + static_cast<int64_t>(d.aux) * a.wq;
    for (int e = threadIdx.x * 4; e < a.wq; e += kThreads * 4) st4(qcopy + e, ld4(q + e));
    float* out = a.arena + d.out;
    sweep<BB, NCH, false>(a, cs, L, [&](int j, float dj) {
      if (lane == 0) out[j] = dj;
      return 0.f;
    });
    return;
  }
  const float* g = a.arena + d.grad;
  float* coefs = a.coefbuf + static_cast<int64_t>(d.aux) * a.ncand;
  for (int j = threadIdx.x; j < a.ncand; j += kThreads) coefs[j] = g[j];
  sweep<BB, NCH, true>(a, cs, L, [&](int j, float) { return g[j]; });
  if constexpr (BB == NGDB_BETAE) {
    reduce_dq<BB, NCH>(a, L, red, nullptr);
    float t = 0.f;
    for (int j = threadIdx.x; j < a.ncand; j += kThreads) t += g[j];
    t = block_sum(warp_sum(t), lred);
    if (threadIdx.x == 0) lred[kWarps] = t;
    __syncthreads();
    const float sc = lred[kWarps];
    float* dst = a.arena + d.out;
    for (int e = threadIdx.x; e < a.wq; e += kThreads) dst[e] = red[e] + sc * beta_qterm(a, q, e);
  } else {
    reduce_dq<BB, NCH>(a, L, red, a.arena + d.out);
  }
}

}  // namespace

template <int NCH>
void launch_loss_nch(const DevArgs& a, int first, int n, cudaStream_t s) {
  // cluster size: enough CTAs for ~4 per SM, 2..8 per node (portable limit)
  const int S = std::max(2, std::min(8, (4 * 148 + n - 1) / std::max(n, 1)));
  if (a.backbone == NGDB_GQE)
    launch_pdl(loss_fwd_kernel<NGDB_GQE, NCH>, dim3(S * n), dim3(kThreads), 0, s, S, a, first, S);
  else if (a.backbone == NGDB_BETAE)
    launch_pdl(loss_fwd_kernel<NGDB_BETAE, NCH>, dim3(S * n), dim3(kThreads), 0, s, S, a, first, S);
  else
    launch_pdl(loss_fwd_kernel<NGDB_Q2B, NCH>, dim3(S * n), dim3(kThreads), 0, s, S, a, first, S);
}
template <int NCH>
void launch_score_nch(const DevArgs& a, int dir, int first, int n, cudaStream_t s) {
  if (a.backbone == NGDB_GQE) launch_pdl(score_kernel<NGDB_GQE, NCH>, dim3(n), dim3(kThreads), 0, s, 1, a, dir, first);
  else if (a.backbone == NGDB_BETAE) launch_pdl(score_kernel<NGDB_BETAE, NCH>, dim3(n), dim3(kThreads), 0, s, 1, a, dir, first);
  else launch_pdl(score_kernel<NGDB_Q2B, NCH>, dim3(n), dim3(kThreads), 0, s, 1, a, dir, first);
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
