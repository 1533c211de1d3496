// Row-sharded step kernels (BASELINE.json configs[4]).
//
// Entity e lives on rank e mod G at local row e div G. Scoring ships queries,
// not rows: after the score-slot query vectors are all-gathered, every rank
// evaluates the loss terms of the candidates it OWNS for every rank's queries
// (the loss is a sum of per-candidate terms and coef_j depends on d_j alone;
// a union's min/argmin is per candidate too), writes coef for its own
// optimizer, and emits partial dL/dq + partial losses that a reduce-scatter
// returns to the query's rank. The collectives themselves run between the
// stages (ngdb_shard_run), on the framework's NCCL communicator.
#include <algorithm>

#include "common.cuh"
#include "dist.cuh"
#include "special.cuh"

namespace ngdb_dev {
namespace {

constexpr int kThreads = 128;  // pack / elementwise kernels
constexpr int kWarps = kThreads / 32;
constexpr int kScoreThreads = 256;  // owner scoring: 8 warps per unit
constexpr int kScoreWarps = kScoreThreads / 32;

// lookup send: the owned rows every rank asked for, requester-major
// (send[p] = local row send_rows[p]; FuseSemantic: the row's fused vector from
// the step table — BetaE: its Psi_theta row — at CSR row anchor_local[p]);
// one warp per row
__global__ void shard_anchor_pack_kernel(DevArgs a, ShardDev sd, float* send) {
  pdl_start();
  const int64_t p = static_cast<int64_t>(blockIdx.x) * 4 + threadIdx.x / 32;
  if (p >= sd.n_send) return;
  const float* src = a.fused ? (a.ytab ? a.ytab : a.etab) + static_cast<int64_t>(a.anchor_local[p]) * a.ent_w
                             : a.ent + static_cast<int64_t>(sd.send_rows[p]) * a.ent_w;
  float* dst = send + p * a.ent_w;
  for (int c = threadIdx.x & 31; c < a.ent_w / 4; c += 32) st4(dst + 4 * c, ld4(src + 4 * c));
}

// query tensors of a Score / Loss pool -> query_mine[slot]
__global__ void shard_query_pack_kernel(DevArgs a, int first, float* dst) {
  pdl_start();
  const ngdb_node_desc d = a.nodes[first + blockIdx.x];
  if (d.aux < 0) return;  // union Loss: its branches are the Score nodes
  const float* q = a.arena + d.in[0];
  float* o = dst + static_cast<int64_t>(d.aux) * a.wq;
  for (int e = threadIdx.x * 4; e < a.wq; e += blockDim.x * 4) st4(o + e, ld4(q + e));
}

// One CTA per scoring unit (rank q, query i) of ANY rank: the owned candidates'
// distances to the unit's 1..3 score-slot queries, union min/argmin (ties ->
// lowest branch), loss terms, coef (routed to the argmin branch), and the
// partial dL/dq of each branch slot. Shared: queries [3][wq], per-warp partial
// dq [kScoreWarps][3][wq] summed in warp order (deterministic).
//
// BetaE (linearised KL, beta.cu): the owned candidate's row is its step-table
// row etab[cand_local[code]] (computed once per owned row by beta_prep over the
// shard CSR), d = lnB(q) + etab_c + <q, etab>, and the query-side term
// (sum of this rank's coefs) [psi(A)-psi(A+B) | psi(B)-psi(A+B)] joins the
// partial dL/dq — linear in the coefficients, so the reduce-scatter's sum over
// owners is the full gradient.
template <int BB>
__device__ __forceinline__ float chunk_dist(const float4& v, const float* qc, int c, int D,
                                            float alpha) {
  const float4 cc = ld4(qc + 4 * c);
  if constexpr (BB == NGDB_BETAE) {
    return v.x * cc.x + v.y * cc.y + v.z * cc.z + v.w * cc.w;
  } else {
    const float4 oo = BB == NGDB_Q2B ? ld4(qc + D + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
    return Dist<BB>::term(v.x, cc.x, oo.x, alpha) + Dist<BB>::term(v.y, cc.y, oo.y, alpha) +
           Dist<BB>::term(v.z, cc.z, oo.z, alpha) + Dist<BB>::term(v.w, cc.w, oo.w, alpha);
  }
}
template <int BB>
__device__ __forceinline__ void chunk_grad(const float4& v, const float* qc, int c, int D,
                                           float coef, float alpha, float4& gc, float4& go) {
  if constexpr (BB == NGDB_BETAE) {
    gc.x += coef * v.x; gc.y += coef * v.y; gc.z += coef * v.z; gc.w += coef * v.w;
  } else {
    const float4 cc = ld4(qc + 4 * c);
    const float4 oo = BB == NGDB_Q2B ? ld4(qc + D + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
    Dist<BB>::grad(v.x, cc.x, oo.x, coef, alpha, gc.x, go.x);
    Dist<BB>::grad(v.y, cc.y, oo.y, coef, alpha, gc.y, go.y);
    Dist<BB>::grad(v.z, cc.z, oo.z, coef, alpha, gc.z, go.z);
    Dist<BB>::grad(v.w, cc.w, oo.w, coef, alpha, gc.w, go.w);
  }
}

template <int BB, int NCH>
__global__ void __launch_bounds__(kScoreThreads) shard_score_kernel(DevArgs a, ShardDev sd) {
  pdl_start();
  constexpr bool kBeta = BB == NGDB_BETAE;
  extern __shared__ __align__(16) float sm[];
  __shared__ float lred[kScoreWarps];
  __shared__ float csred[kScoreWarps][3];  // BetaE: per-warp coefficient sums per branch
  __shared__ float qbias[3];               // BetaE: lnB(q_b) summed over the dims
  const int u = blockIdx.x;
  const int q = u / sd.batch, i = u % sd.batch;
  const int k = sd.unit_k[u];
  const int wq = a.wq, D = a.dim;
  const int nch = kBeta ? wq / 4 : D / 4;  // float4 chunks of a candidate row
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  float* qs = sm;              // [3][wq]
  float* part = sm + 3 * wq;   // [kScoreWarps][3][wq]
  int gslot[3];
  for (int b = 0; b < 3; ++b)
    gslot[b] = b < k ? q * sd.max_slots + sd.unit_slots[static_cast<int64_t>(u) * 3 + b] : 0;
  float* dq_blk = sd.dq_part + static_cast<int64_t>(q) * sd.dq_block;  // rank q's block
  for (int b = 0; b < k; ++b)
    for (int e = threadIdx.x; e < wq; e += kScoreThreads)
      qs[b * wq + e] = sd.query_all[static_cast<int64_t>(gslot[b]) * wq + e];
  for (int e = threadIdx.x; e < kScoreWarps * 3 * wq; e += kScoreThreads) part[e] = 0.f;
  __syncthreads();
  if constexpr (kBeta) {
    for (int b = 0; b < k; ++b) {
      float t = 0.f;
      for (int e = threadIdx.x; e < D; e += kScoreThreads) t += dg_lbeta(qs[b * wq + e], qs[b * wq + D + e]);
      t = warp_sum(t);
      if (lane == 0) lred[warp] = t;
      __syncthreads();
      if (threadIdx.x == 0) {
        float tt = 0.f;
        for (int w = 0; w < kScoreWarps; ++w) tt += lred[w];
        qbias[b] = tt;
      }
      __syncthreads();
    }
  }
  float loss = 0.f;                  // identical in all lanes of a warp
  float csum[3] = {0.f, 0.f, 0.f};   // BetaE: coefficient sums per branch
  const int32_t* cand = sd.cand + static_cast<int64_t>(u) * a.ncand;
  const int t_end = sd.unit_off[u + 1];
  // candidate rows into registers one step ahead: two rows of loads in
  // flight per warp while the current one is reduced
  auto load_row = [&](int t, float4* v, float& cst) {
    const int j = sd.owned[t];
    const float* row;
    if constexpr (kBeta) {
      const int r = __ldg(a.cand_local + static_cast<int64_t>(gslot[0]) * a.ncand + j);
      row = a.etab + static_cast<int64_t>(r) * a.ent_w;
      cst = __ldg(a.etab_c + r);
    } else {
      // FuseSemantic: the owned row's fused vector in the step table
      row = a.fused ? a.etab + static_cast<int64_t>(__ldg(a.cand_local + static_cast<int64_t>(gslot[0]) * a.ncand + j)) * a.ent_w
                    : a.ent + static_cast<int64_t>(cand[j] / sd.world) * a.ent_w;
      cst = 0.f;
    }
#pragma unroll
    for (int c4 = 0; c4 < NCH; ++c4) {
      const int c = lane + 32 * c4;
      v[c4] = c < nch ? ld4(row + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  float4 v[NCH], vn[NCH];
  float cst = 0.f, cstn = 0.f;
  int t = sd.unit_off[u] + warp;
  if (t < t_end) load_row(t, v, cst);
  if (k == 1) {
    // one score slot (every pattern but the unions): dL/dq accumulates in
    // registers across the warp's rows, one shared-memory write at the end
    float4 gcs[NCH], gos[NCH];
#pragma unroll
    for (int c4 = 0; c4 < NCH; ++c4) gcs[c4] = gos[c4] = make_float4(0.f, 0.f, 0.f, 0.f);
    const float qb = kBeta ? qbias[0] : 0.f;
    for (; t < t_end; t += kScoreWarps) {
      const int j = sd.owned[t];
      if (t + kScoreWarps < t_end) load_row(t + kScoreWarps, vn, cstn);
      float s = 0.f;
#pragma unroll
      for (int c4 = 0; c4 < NCH; ++c4) {
        const int c = lane + 32 * c4;
        if (c < nch) s += chunk_dist<BB>(v[c4], qs, c, D, a.alpha_box);
      }
      float dj = warp_sum(s);
      if constexpr (kBeta) dj += qb + cst;
      const float coef = loss_coef(a, j, dj, loss);
      csum[0] += coef;
      if (lane == 0) sd.coef_all[static_cast<int64_t>(gslot[0]) * a.ncand + j] = coef;
#pragma unroll
      for (int c4 = 0; c4 < NCH; ++c4) {
        const int c = lane + 32 * c4;
        if (c < nch) chunk_grad<BB>(v[c4], qs, c, D, coef, a.alpha_box, gcs[c4], gos[c4]);
      }
#pragma unroll
      for (int c4 = 0; c4 < NCH; ++c4) v[c4] = vn[c4];
      cst = cstn;
    }
    float* pw = part + (warp * 3) * wq;
#pragma unroll
    for (int c4 = 0; c4 < NCH; ++c4) {
      const int c = lane + 32 * c4;
      if (c < nch) {
        st4(pw + 4 * c, gcs[c4]);
        if (BB == NGDB_Q2B) st4(pw + D + 4 * c, gos[c4]);
      }
    }
  }
  for (; k > 1 && t < t_end; t += kScoreWarps) {  // union branches: smem partials per branch
    const int j = sd.owned[t];
    if (t + kScoreWarps < t_end) load_row(t + kScoreWarps, vn, cstn);
    float dist[3];
    for (int b = 0; b < k; ++b) {
      const float* qc = qs + b * wq;
      float s = 0.f;
#pragma unroll
      for (int c4 = 0; c4 < NCH; ++c4) {
        const int c = lane + 32 * c4;
        if (c < nch) s += chunk_dist<BB>(v[c4], qc, c, D, a.alpha_box);
      }
      dist[b] = warp_sum(s);
      if constexpr (kBeta) dist[b] += qbias[b] + cst;
    }
    int bm = 0;
    for (int b = 1; b < k; ++b)
      if (dist[b] < dist[bm]) bm = b;  // min distance == max score; ties -> lowest branch
    const float coef = loss_coef(a, j, dist[bm], loss);
    for (int b = 0; b < k; ++b) csum[b] += b == bm ? coef : 0.f;
    if (lane == 0)
      for (int b = 0; b < k; ++b)
        sd.coef_all[static_cast<int64_t>(gslot[b]) * a.ncand + j] = b == bm ? coef : 0.f;
    const float* qc = qs + bm * wq;
    float* pw = part + (warp * 3 + bm) * wq;
#pragma unroll
    for (int c4 = 0; c4 < NCH; ++c4) {
      const int c = lane + 32 * c4;
      if (c < nch) {
        float4 gc = make_float4(0.f, 0.f, 0.f, 0.f), go = gc;
        chunk_grad<BB>(v[c4], qc, c, D, coef, a.alpha_box, gc, go);
        float4 p = ld4(pw + 4 * c);
        st4(pw + 4 * c, make_float4(p.x + gc.x, p.y + gc.y, p.z + gc.z, p.w + gc.w));
        if (BB == NGDB_Q2B) {
          p = ld4(pw + D + 4 * c);
          st4(pw + D + 4 * c, make_float4(p.x + go.x, p.y + go.y, p.z + go.z, p.w + go.w));
        }
      }
    }
#pragma unroll
    for (int c4 = 0; c4 < NCH; ++c4) v[c4] = vn[c4];
    cst = cstn;
  }
  if (lane == 0) {
    lred[warp] = loss;
    for (int b = 0; b < 3; ++b) csred[warp][b] = csum[b];
  }
  __syncthreads();
  for (int b = 0; b < k; ++b) {
    float cb = 0.f;
    if constexpr (kBeta)
      for (int w = 0; w < kScoreWarps; ++w) cb += csred[w][b];
    const float* qb = qs + b * wq;
    for (int e = threadIdx.x; e < wq; e += kScoreThreads) {
      float acc = 0.f;
      for (int w = 0; w < kScoreWarps; ++w) acc += part[(w * 3 + b) * wq + e];
      if constexpr (kBeta) {  // query-side term of dKL/dq
        const int ii = e < D ? e : e - D;
        const float A = qb[ii], B = qb[D + ii];
        acc += cb * (dg_digamma(e < D ? A : B) - dg_digamma(A + B));
      }
      dq_blk[static_cast<int64_t>(gslot[b] - q * sd.max_slots) * wq + e] = acc;
    }
  }
  if (threadIdx.x == 0) {
    float tl = 0.f;
    for (int w = 0; w < kScoreWarps; ++w) tl += lred[w];
    dq_blk[static_cast<int64_t>(sd.max_slots) * wq + i] = tl;
  }
}

// this rank's results: dqbuf <- dq_mine, loss_out <- loss_mine
__global__ void shard_score_done_kernel(DevArgs a, const float* dq_mine, int64_t n_dq,
                                        const float* loss_mine, int nq) {
  pdl_start();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_dq;
       e += (int64_t)gridDim.x * blockDim.x) {
    a.dqbuf[e] = dq_mine[e];
    if (e < nq) {
      a.loss_out[e] = loss_mine[e];
      if (!isfinite(loss_mine[e])) atomicOr(&a.flags[0], 1);
    }
  }
}

// gradient return: my anchors' gradient rows in receive order (owner-major),
// send[p] = agbuf[recv_slot[p]]; one warp per row
__global__ void shard_grad_pack_kernel(DevArgs a, ShardDev sd, float* send) {
  pdl_start();
  const int64_t p = static_cast<int64_t>(blockIdx.x) * 4 + threadIdx.x / 32;
  if (p >= sd.n_recv) return;
  const float* g = a.agbuf + static_cast<int64_t>(sd.recv_slot[p]) * a.ent_w;
  float* dst = send + p * a.ent_w;
  for (int c = threadIdx.x & 31; c < a.ent_w / 4; c += 32) st4(dst + 4 * c, ld4(g + 4 * c));
}

// relation CSR rows -> dense relation gradient rows + touched flags
__global__ void shard_rel_pack_kernel(DevArgs a, SparseTable t, float* rel_g, float* touched) {
  pdl_start();
  const int r = blockIdx.x;
  if (r >= t.n_rows) return;
  const int64_t row = t.rows[r];
  for (int e = threadIdx.x; e < t.width; e += blockDim.x) {
    float s = 0.f;
    for (int kk = t.seg[r]; kk < t.seg[r + 1]; ++kk)
      s += a.rgbuf[static_cast<int64_t>(t.contrib[kk]) * t.width + e];
    rel_g[row * t.width + e] = s;
  }
  if (threadIdx.x == 0) touched[row] = 1.f;
}

// lazy Adam on the rows any rank touched, from all-reduced dense rows
__global__ void masked_rows_adam_kernel(float* w, float* m, float* v, float* dbg, const float* g,
                                        const float* touched, int rows, int width, AdamHyper hp,
                                        const float* bc) {
  pdl_start();
  const int r = blockIdx.x;
  if (r >= rows || !(touched[r] > 0.f)) return;
  const float ibc1 = 1.f / bc[0], ibc2 = 1.f / bc[1];  // bias corrections as reciprocals
  for (int e = threadIdx.x; e < width; e += blockDim.x) {
    const int64_t o = static_cast<int64_t>(r) * width + e;
    const float gi = g[o];
    if (dbg) dbg[o] = gi;
    const float mi = hp.b1 * m[o] + (1.f - hp.b1) * gi;
    const float vi = hp.b2 * v[o] + (1.f - hp.b2) * gi * gi;
    m[o] = mi;
    v[o] = vi;
    w[o] -= hp.lr * (mi * ibc1) / (sqrtf(vi * ibc2) + hp.eps);
  }
}

}  // namespace

int launch_shard_anchor_pack(const DevArgs& a, const ShardDev& sd, float* send, const LaunchCtx& lc) {
  if (sd.n_send <= 0) return 0;
  launch_pdl(shard_anchor_pack_kernel, dim3((sd.n_send + 3) / 4), dim3(128), 0, lc.stream, 1, a,
             sd, send);
  return 1;
}

int launch_shard_query_pack(const DevArgs& a, int first, int n, float* dst, const LaunchCtx& lc) {
  if (n <= 0) return 0;
  launch_pdl(shard_query_pack_kernel, dim3(n), dim3(128), 0, lc.stream, 1, a, first, dst);
  return 1;
}

int launch_shard_score(const DevArgs& a, const ShardDev& sd, const LaunchCtx& lc) {
  const int units = sd.world * sd.batch;
  if (units <= 0) return 0;
  const size_t smem = static_cast<size_t>(3 + kScoreWarps * 3) * a.wq * sizeof(float);
  auto go = [&](auto kernel) {
    static bool configured = false;  // per instantiation
    if (!configured) {
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      configured = true;
    }
    launch_pdl(kernel, dim3(units), dim3(kScoreThreads), smem, lc.stream, 1, a, sd);
  };
  if (a.backbone == NGDB_BETAE) {  // rows are 2d wide (validate_shard: d <= 512)
    if (a.dim <= 256) go(shard_score_kernel<NGDB_BETAE, 4>);
    else go(shard_score_kernel<NGDB_BETAE, 8>);
  } else if (a.dim <= 512) {
    if (a.backbone == NGDB_GQE) go(shard_score_kernel<NGDB_GQE, 4>);
    else go(shard_score_kernel<NGDB_Q2B, 4>);
  } else {
    if (a.backbone == NGDB_GQE) go(shard_score_kernel<NGDB_GQE, 8>);
    else go(shard_score_kernel<NGDB_Q2B, 8>);
  }
  return 1;
}

int launch_shard_score_done(const DevArgs& a, const float* dq_mine, int64_t n_dq,
                            const float* loss_mine, int nq, const LaunchCtx& lc) {
  const int blocks = static_cast<int>(std::min<int64_t>((n_dq + 255) / 256, lc.num_sms * 4));
  launch_pdl(shard_score_done_kernel, dim3(std::max(blocks, 1)), dim3(256), 0, lc.stream, 1, a,
             dq_mine, n_dq, loss_mine, nq);
  return 1;
}

int launch_shard_grad_pack(const DevArgs& a, const ShardDev& sd, float* send, const LaunchCtx& lc) {
  if (sd.n_recv <= 0) return 0;
  launch_pdl(shard_grad_pack_kernel, dim3((sd.n_recv + 3) / 4), dim3(128), 0, lc.stream, 1, a,
             sd, send);
  return 1;
}

int launch_shard_rel_pack(const DevArgs& a, const SparseTable& t, float* rel_g, float* touched,
                          const LaunchCtx& lc) {
  if (t.n_rows <= 0) return 0;
  launch_pdl(shard_rel_pack_kernel, dim3(t.n_rows), dim3(128), 0, lc.stream, 1, a, t, rel_g, touched);
  return 1;
}

int launch_masked_rows_adam(float* w, float* m, float* v, float* dbg, const float* g,
                            const float* touched, int rows, int width, const AdamHyper& hp,
                            const float* bc, const LaunchCtx& lc) {
  if (rows <= 0) return 0;
  launch_pdl(masked_rows_adam_kernel, dim3(rows), dim3(128), 0, lc.stream, 1, w, m, v, dbg, g,
             touched, rows, width, hp, bc);
  return 1;
}

}  // namespace ngdb_dev
