// FuseSemantic: frozen PTE vectors fused into the structural embedding by a
// GPU-resident projection (Eq. 12):
//
//   e_fused = sigma(W_p [h | F s] + b_p)        h: entity row (d), s: store row (d_l)
//
// applied to anchors AND candidates. Parameters are fixed within
// a step, so the B200 layout evaluates e_fused ONCE per touched entity row of
// the step (the optimizer CSR rows: ~14k for FB15k-237 instead of 66k
// candidate + ~1k anchor evaluations — the "deduped" 19 GFLOP of SURVEY §8(d))
// as two tcgen05 GEMMs in the step prologue, into the same per-step entity
// table (etab) the BetaE path uses. FuseSemantic nodes then gather from etab
// and the fused score+loss kernel streams candidate rows from it.
//
// With W_p = [W_h | W_s] the pre-activation is Z = h W_h^T + s (W_s F)^T + b_p:
// the product M = W_s F (d x d_l, 0.25 GFLOP at d = 400, d_l = 768) is formed
// once per step and the per-row work is two GEMMs of K = d_l and K = d instead
// of K = d_l (F s) then K = 2d (W_p [h | F s]) — the same linear map, about 30 %
// fewer flops over forward + backward, and the u x d intermediate F s is gone.
//
// Backward (in the optimizer): dL/de_fused per row = anchor gradient rows +
// candidate terms recomputed from (q, coef) as for the plain backbones, times
// sigma' -> dZ; then dh = dZ W_h (the entity rows take Adam on it),
// dW_h += dZ^T h, dM = dZ^T S, dW_s += dM F^T, dF += W_s^T dM, db_p += colsum dZ.
// The store is never written (frozen: its gradient is exactly zero, SPEC.md:416,
// 579).
//
// BetaE (Psi_theta, Eq. 3): h is d wide and the
// fused vector E = sigma(Z) is mapped to the 2d' Beta pre-activations
// Y = E W_psi^T + b_psi by one more GEMM; the step's BetaE entity table (the
// KL linearisation T_e, C_e) is then evaluated from Y by the same prologue
// kernel as the plain backbone (beta_prep), FuseSemantic anchors realise their
// Y rows, and the backward starts from dL/dY (beta_fuse_grad: anchor and
// candidate terms through realize') -> dE = dY W_psi, dW_psi += dY^T E,
// db_psi += colsum dY, dZ = dE * E (1 - E), then the chain above.
#include <algorithm>

#include "common.cuh"
#include "mlp_util.cuh"

namespace ngdb_dev {
namespace {

constexpr int kWarps = 8;

struct FuseBufs {
  int u, uP, d, dl;
  bool beta;
  float* S;  Split Ss;    // [u][dl]   gathered store rows
  float* X;  Split Xs;    // [u][2d]   [h | F s]
  float* dZ; Split dZs;   // [u][d]
  float* dX;              // [u][2d]   dZ W_p
  // BetaE (Psi_theta)
  float* E;  Split Es;    // [u][d]    sigma(Z)
  float* Y;               // [u][2d]   Beta pre-activations (read by the step's kernels)
  float* dY; Split dYs;   // [u][2d]
  float* dE;              // [u][d]
  // per-step products of the weights (d x d_l)
  float* M;  Split Ms;    // M = W_s F
  float* dM; Split dMs;   // dM^T = S^T dZ [d_l][d] (plain + split)
};

FuseBufs carve(float* base, int64_t cap, int u, int d, int dl, bool beta) {
  Scratch sc{base, cap};
  FuseBufs f{};
  f.u = u;
  f.uP = (u + 3) & ~3;
  f.d = d;
  f.dl = dl;
  f.beta = beta;
  const int64_t U = u;
  f.S = sc.take(U * dl);
  f.Ss = take_split(sc, U * dl);
  f.X = sc.take(U * 2 * d);
  f.Xs = take_split(sc, U * 2 * d);
  f.dZ = sc.take(U * d);
  f.dZs = take_split(sc, U * d);
  f.dX = sc.take(U * 2 * d);
  if (beta) {
    f.E = sc.take(U * d);
    f.Es = take_split(sc, U * d);
    f.Y = sc.take(U * 2 * d);
    f.dY = sc.take(U * 2 * d);
    f.dYs = take_split(sc, U * 2 * d);
    f.dE = sc.take(U * d);
  }
  const int64_t DL = int64_t(d) * dl;
  f.M = sc.take(DL);
  f.Ms = take_split(sc, DL);
  f.dM = sc.take(DL);
  f.dMs = take_split(sc, DL);
  return f;
}

// Per touched row r: candidate / anchor -> row maps, the gathered store row
// (plain + split) and X[r][0:d] = h (plain + split).
__global__ void __launch_bounds__(kWarps * 32) fuse_gather_kernel(DevArgs a, SparseTable t, FuseBufs f,
                                                                  int gather_s) {
  pdl_start();
  const int r = blockIdx.x * kWarps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= t.n_rows) return;
  for (int kk = t.seg[r] + lane; kk < t.seg[r + 1]; kk += 32) {
    const int32_t code = t.contrib[kk];
    if (code >= 0) a.cand_local[code] = r;
    else a.anchor_local[-code - 1] = r;
  }
  const int64_t e = t.rows[r];
  const float* s = a.sem + e * f.dl;
  for (int c = lane; gather_s && c < f.dl / 4; c += 32) {
    const float4 v = ldg4(s + 4 * c);
    const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) put(f.S, f.Ss, (int64_t)r * f.dl + 4 * c + q, vv[q]);
  }
  const float* h = a.ent + e * f.d;  // the structural row (d wide)
  for (int c = lane; c < f.d / 4; c += 32) {
    const float4 v = ld4(h + 4 * c);
    const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) put(f.X, f.Xs, (int64_t)r * 2 * f.d + 4 * c + q, vv[q]);
  }
}

// BetaE: dZ = dE * E (1 - E), plain + split
__global__ void fuse_dz_kernel(const float* dE, const float* E, float* dZ, Split dZs, int64_t n) {
  pdl_start();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float e = E[i];
    put(dZ, dZs, i, dE[i] * e * (1.f - e));
  }
}

template <int BB>
__device__ __forceinline__ float cand_term(float v, float qc, float qo, float coef, float alpha) {
  const float delta = v - qc;
  float mag = coef;
  if (BB == NGDB_Q2B) mag = fabsf(delta) > qo ? coef : coef * alpha;
  return delta > 0.f ? mag : (delta < 0.f ? -mag : 0.f);
}

// dZ[r] = (anchor grads + candidate grads of row r) * E (1 - E), plain + split.
// One warp per row, the row's d/4 float4 chunks in registers (NCH per lane);
// contributions outer: each code / coefficient is loaded once by one lane and
// broadcast (32 at a time), and every contribution's query row is read once.
template <int BB, int NCH>
__global__ void __launch_bounds__(kWarps * 32) fuse_grad_kernel(DevArgs a, SparseTable t, FuseBufs f) {
  pdl_start();
  const int r = blockIdx.x * kWarps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= t.n_rows) return;
  const int beg = t.seg[r], end = t.seg[r + 1];
  const int d4 = f.d / 4;
  const float* E = a.etab + (int64_t)r * a.ent_w;
  float4 ev[NCH], g[NCH];
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    const int c = lane + 32 * i;
    ev[i] = c < d4 ? ld4(E + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
    g[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  const float ca_scale = a.alpha_box;
  for (int k0 = beg; k0 < end; k0 += 32) {
    const int nk = min(32, end - k0);
    int32_t my_code = 0;
    float my_coef = 0.f;
    if (lane < nk) {
      my_code = __ldg(t.contrib + k0 + lane);
      if (my_code >= 0) my_coef = __ldg(a.coefbuf + my_code);
    }
    for (int j = 0; j < nk; ++j) {
      const int32_t code = __shfl_sync(0xffffffffu, my_code, j);
      const float coef = __shfl_sync(0xffffffffu, my_coef, j);
      if (code < 0) {
        const float* u = a.agbuf + (int64_t)(-code - 1) * a.ent_w;
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          const int c = lane + 32 * i;
          if (c < d4) {
            const float4 x = ld4(u + 4 * c);
            g[i].x += x.x; g[i].y += x.y; g[i].z += x.z; g[i].w += x.w;
          }
        }
      } else {
        const float* q = a.qbuf + (int64_t)(code / a.ncand) * a.wq;
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          const int c = lane + 32 * i;
          if (c < d4) {
            const float4 qc = ld4(q + 4 * c);
            const float4 qo = BB == NGDB_Q2B ? ld4(q + a.dim + 4 * c) : make_float4(0.f, 0.f, 0.f, 0.f);
            g[i].x += cand_term<BB>(ev[i].x, qc.x, qo.x, coef, ca_scale);
            g[i].y += cand_term<BB>(ev[i].y, qc.y, qo.y, coef, ca_scale);
            g[i].z += cand_term<BB>(ev[i].z, qc.z, qo.z, coef, ca_scale);
            g[i].w += cand_term<BB>(ev[i].w, qc.w, qo.w, coef, ca_scale);
          }
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    const int c = lane + 32 * i;
    if (c < d4) {
      const float e4[4] = {ev[i].x, ev[i].y, ev[i].z, ev[i].w};
      const float gg[4] = {g[i].x, g[i].y, g[i].z, g[i].w};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        put(f.dZ, f.dZs, (int64_t)r * f.d + 4 * c + q, gg[q] * e4[q] * (1.f - e4[q]));
    }
  }
}

// lazy Adam on the touched entity rows with gradient rows G[r][0:width] (stride ldg);
// rows without contributions (the whole-table form) are untouched: skipped
__global__ void __launch_bounds__(kWarps * 32) rows_adam_kernel(SparseTable t, const float* G, int ldg,
                                                                AdamHyper hp, const float* bc) {
  pdl_start();
  const int r = blockIdx.x * kWarps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= t.n_rows || t.seg[r] == t.seg[r + 1]) return;
  const float ibc1 = 1.f / bc[0], ibc2 = 1.f / bc[1];  // bias corrections as reciprocals
  const int64_t row = t.rows[r];
  for (int c = lane; c < t.width / 4; c += 32) {
    const float4 g4 = ld4(G + (int64_t)r * ldg + 4 * c);
    if (t.dbg_g) st4(t.dbg_g + row * t.width + 4 * c, g4);
    const int64_t o = row * t.width + 4 * c;
    float4 w = ld4(t.w + o), m = ld4(t.m + o), v = ld4(t.v + o);
    float* wv = &w.x;
    float* mv = &m.x;
    float* vv = &v.x;
    const float g[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      mv[q] = hp.b1 * mv[q] + (1.f - hp.b1) * g[q];
      vv[q] = hp.b2 * vv[q] + (1.f - hp.b2) * g[q] * g[q];
      wv[q] -= hp.lr * (mv[q] * ibc1) / (sqrtf(vv[q] * ibc2) + hp.eps);
    }
    st4(t.w + o, w);
    st4(t.m + o, m);
    st4(t.v + o, v);
  }
}

inline int row_blocks(int n) { return (n + kWarps - 1) / kWarps; }

// A step that touches every entity (CSR rows ascending and unique, so rows ==
// 0..N-1) reads the frozen store's split made at upload instead of gathering
// and splitting it again (FB15k-237: ~66k candidates cover all 14.5k entities)
inline bool all_rows(const DevArgs& a, const SparseTable& t) {
  return a.sem_hi && t.n_rows == a.n_entities;
}

}  // namespace

// Whole-table form of a step's entity CSR: rows 0..N-1 (row e = entity e) with
// the compact CSR's contribution segments (empty for untouched entities)
__global__ void expand_seg_kernel(const int32_t* rows, const int32_t* seg, int u, int32_t* seg_full,
                                  int n) {
  pdl_start();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e > n) return;
  int lo = 0, hi = u;  // first compact row with entity >= e
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (rows[mid] < e) lo = mid + 1;
    else hi = mid;
  }
  seg_full[e] = seg[lo];
}

int64_t fuse_scratch_floats(int d, int dl, int64_t rows) {
  const int64_t U = rows + 4;
  // S, X, dZ (plain + split), dX; the BetaE (Psi) buffers; M, dM (plain + split)
  return U * (3 * dl + 6 * d + d + 3 * d + 2 * d) + U * (3 * d + 2 * d + 6 * d + d) +
         int64_t(d + 4) * dl * 6 + 4096;
}

int launch_expand_rows(const int32_t* rows, const int32_t* seg, int u, int32_t* seg_full, int n,
                       cudaStream_t s) {
  launch_pdl(expand_seg_kernel, dim3((n + 256) / 256), dim3(256), 0, s, 1, rows, seg, u, seg_full, n);
  return 1;
}

float* fuse_y_table(float* fs, int64_t cap, int u, int d, int dl) {
  return carve(fs, cap, u, d, dl, true).Y;
}

int fuse_prologue(const DevArgs& a, const SparseTable& t, float* fs, int64_t cap, const LaunchCtx& lc) {
  if (t.n_rows <= 0) return 0;
  const bool beta = a.backbone == NGDB_BETAE;
  const int d = a.dim, dl = a.sem_dim, u = t.n_rows;
  FuseBufs f = carve(fs, cap, u, d, dl, beta);
  const float* p = a.dense;
  int launches = 0;
  const bool whole = all_rows(a, t);
  launch_pdl(fuse_gather_kernel, dim3(row_blocks(u)), dim3(kWarps * 32), 0, lc.stream, 1, a, t, f,
             whole ? 0 : 1);
  ++launches;
  // M = W_s F (A = W_p[:, d:2d] row-major, B = F^T), split for the next GEMM
  const SplitOperand wp = wop(a, a.fus_idx + 1, d, 2 * d, false);
  TcGemmArgs gm = gemm_args(d, dl, d, SplitOperand{wp.hi + d, wp.lo + d, 2 * d},
                            wop(a, a.fus_idx, d, dl, true), f.M, dl);
  gm.s_hi = f.Ms.hi;
  gm.s_lo = f.Ms.lo;
  launches += tc_gemm(gm, lc.stream);
  // Z = S M^T + b_p, then Z += h W_h^T
  const Split Ss = whole ? Split{const_cast<float*>(a.sem_hi), const_cast<float*>(a.sem_lo)} : f.Ss;
  float* zE = beta ? f.E : a.etab;  // Z, then sigmoid(Z) in place
  TcGemmArgs g1 = gemm_args(u, d, dl, op(Ss, dl), op(f.Ms, dl), zE, d);
  g1.bias = p + a.dense_off[a.fus_idx + 2];
  launches += tc_gemm(g1, lc.stream);
  // ... + h W_h^T, then E = sigmoid(Z) in the epilogue: the fused rows go
  // straight to the step table (BetaE: to E, plain + split, for Psi_theta)
  TcGemmArgs g2 = gemm_args(u, d, d, op(f.Xs, 2 * d), wp, zE, d);
  g2.accumulate = 1;
  g2.sigmoid = 1;
  if (beta) {
    g2.s_hi = f.Es.hi;
    g2.s_lo = f.Es.lo;
  }
  launches += tc_gemm(g2, lc.stream);
  if (!beta) return launches;
  // Psi_theta: Y = E W_psi^T + b_psi, then the BetaE entity table from Y
  TcGemmArgs gy = gemm_args(u, 2 * d, d, op(f.Es, d), wop(a, a.fus_idx + 3, 2 * d, d, false), f.Y, 2 * d);
  gy.bias = p + a.dense_off[a.fus_idx + 4];
  launches += tc_gemm(gy, lc.stream);
  DevArgs ay = a;
  ay.ytab = f.Y;
  return launches + 1 + launch_beta_prep(ay, t, lc);
}

int fuse_entity_adam(const SparseTable& t, float* fs, int64_t cap, int d, int dl, bool beta,
                     const AdamHyper& hp, const float* bc, const LaunchCtx& lc) {
  if (t.n_rows <= 0) return 0;
  const FuseBufs f = carve(fs, cap, t.n_rows, d, dl, beta);
  launch_pdl(rows_adam_kernel, dim3(row_blocks(t.n_rows)), dim3(kWarps * 32), 0, lc.stream, 1, t,
             (const float*)f.dX, d, hp, bc);
  return 1;
}

int fuse_backward(const DevArgs& a, const SparseTable& t, float* fs, int64_t cap, const AdamHyper& hp,
                  const float* bc, const LaunchCtx& lc, bool adam) {
  if (t.n_rows <= 0) return 0;
  const bool beta = a.backbone == NGDB_BETAE;
  const int d = a.dim, dl = a.sem_dim, u = t.n_rows;
  FuseBufs f = carve(fs, cap, u, d, dl, beta);
  float* g = a.dense_g;
  const int64_t* off = a.dense_off;
  int launches = 0;
  if (beta) {
    // dL/dY through realize' (anchor + candidate terms), then Psi_theta's backward
    DevArgs ay = a;
    ay.ytab = f.Y;
    launches += launch_beta_fuse_grad(ay, t, f.dY, f.dYs, lc);
    TcGemmArgs ge = gemm_args(u, d, 2 * d, op(f.dYs, 2 * d), wop(a, a.fus_idx + 3, 2 * d, d, true),
                              f.dE, d);  // dE = dY W_psi
    launches += tc_gemm(ge, lc.stream);
    // dY and E (prologue epilogue) split row-major, read MN-major
    TcGemmArgs gw = gemm_args(2 * d, d, u, mop(f.dYs, 2 * d), mop(f.Es, d), g + off[a.fus_idx + 3], d);
    gw.accumulate = 1;  // dW_psi += dY^T E
    launches += tc_gemm(gw, lc.stream);
    ColsumJobs pc{};
    pc.job[0] = {f.dY, u, 2 * d, g + off[a.fus_idx + 4]};
    pc.n = 1;
    launches += colsums(pc, 2 * d, lc.stream);
    const int64_t n = (int64_t)u * d;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)lc.num_sms * 8);
    launch_pdl(fuse_dz_kernel, dim3(blocks), dim3(256), 0, lc.stream, 1, (const float*)f.dE,
               (const float*)f.E, f.dZ, f.dZs, n);
    ++launches;
  } else if (a.backbone == NGDB_GQE) {
    if (d <= 512) launch_pdl(fuse_grad_kernel<NGDB_GQE, 4>, dim3(row_blocks(u)), dim3(kWarps * 32), 0, lc.stream, 1, a, t, f);
    else launch_pdl(fuse_grad_kernel<NGDB_GQE, 8>, dim3(row_blocks(u)), dim3(kWarps * 32), 0, lc.stream, 1, a, t, f);
    ++launches;
  } else {
    if (d <= 512) launch_pdl(fuse_grad_kernel<NGDB_Q2B, 4>, dim3(row_blocks(u)), dim3(kWarps * 32), 0, lc.stream, 1, a, t, f);
    else launch_pdl(fuse_grad_kernel<NGDB_Q2B, 8>, dim3(row_blocks(u)), dim3(kWarps * 32), 0, lc.stream, 1, a, t, f);
    ++launches;
  }
  // dh = dZ W_h -> dX[:, 0:d] (the entity rows' gradient)
  const SplitOperand wpt = wop(a, a.fus_idx + 1, d, 2 * d, true);  // W_p^T [2d][d]
  TcGemmArgs g3 = gemm_args(u, d, d, op(f.dZs, d), wpt, f.dX, d);
  launches += tc_gemm(g3, lc.stream);
  const bool whole = all_rows(a, t);
  // the K = rows weight gradients read the row-major splits of dZ, h (= X[:,
  // 0:d], the prologue's split) and the store rows S MN-major: no transposed
  // copies. The two as separate launches: each gets its own tile width and
  // split-K (tc_gemm.cu), which beats one shared launch
  const Split Ss = whole ? Split{const_cast<float*>(a.sem_hi), const_cast<float*>(a.sem_lo)} : f.Ss;
  TcGemmArgs gw = gemm_args(d, d, u, mop(f.dZs, d), mop(f.Xs, 2 * d), g + off[a.fus_idx + 1], 2 * d);
  gw.accumulate = 1;  // dW_h += dZ^T h
  launches += tc_gemm(gw, lc.stream);
  // dM^T = S^T dZ ([d_l][d], plain + split): the d_l-row orientation streams
  // the store operand fewer times than dM = dZ^T S
  TcGemmArgs gt = gemm_args(dl, d, u, mop(Ss, dl), mop(f.dZs, d), f.dM, d);
  gt.s_hi = f.dMs.hi;
  gt.s_lo = f.dMs.lo;
  launches += tc_gemm(gt, lc.stream);
  TcGemmArgs wl[2];
  wl[0] = gemm_args(d, d, dl, mop(f.dMs, d), wop(a, a.fus_idx, d, dl, false),
                    g + off[a.fus_idx + 1] + d, 2 * d);
  wl[0].accumulate = 1;  // dW_s += dM F^T
  wl[1] = gemm_args(d, dl, d, SplitOperand{wpt.hi + int64_t(d) * d, wpt.lo + int64_t(d) * d, d},
                    op(f.dMs, d), g + off[a.fus_idx], dl);
  wl[1].accumulate = 1;  // dF += W_s^T dM
  launches += tc_gemm_batch(wl, 2, lc.stream);
  ColsumJobs cj{};
  cj.job[0] = {f.dZ, u, d, g + off[a.fus_idx + 2]};
  cj.n = 1;
  launches += colsums(cj, d, lc.stream);
  if (!adam) return launches;
  return launches + fuse_entity_adam(t, fs, cap, d, dl, beta, hp, bc, lc);
}

}  // namespace ngdb_dev
