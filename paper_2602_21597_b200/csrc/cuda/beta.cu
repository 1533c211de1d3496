// BetaE backbone (concrete forms DESIGN.md §3.5).
//
// A query / entity is d Beta distributions, stored as [alpha (d) | beta (d)]:
// entities as unconstrained reals realised by clamp(softplus(x), 0.05, 1e9),
// query tensors in the arena as realised parameters.
//
//   Project    out = realize(W2 relu(W1 [q | r] + b1) + b2)   (2d+d -> 2d -> 2d)
//   Intersect  w = softmax_l(A2 relu(A1 q_l + a1) + a2) per dim; alpha, beta = sum_l w_l (.)_l
//   Negate     (alpha, beta) -> clamp(1/alpha, 1/beta)        (rows.cu)
//   Distance   sum_dims KL(Beta(entity) || Beta(query))     (score.cu)
//
// KL linearisation (the B200 layout of the scoring). With (a, b) the entity and
// (A, B) the query parameters of one dimension, s = a + b,
//   KL = lnB(A,B) + [-lnB(a,b) + a psi(a) + b psi(b) - s psi(s)]
//        + A (psi(s) - psi(a)) + B (psi(s) - psi(b)),
// i.e. a per-query constant + a per-entity constant + a dot product. beta_prep
// evaluates the entity side ONCE per touched row per step (digamma/lgamma on
// ~14k rows instead of 66k candidate evaluations); the fused score+loss kernel
// then streams 2d floats per candidate exactly like the L1/box backbones. The
// entity-side gradient is linear in the query too:
//   dKL/da = a psi'(a) - s psi'(s) + A (psi'(s) - psi'(a)) + B psi'(s)
//   dKL/db = b psi'(b) - s psi'(s) + A psi'(s) + B (psi'(s) - psi'(b))
// so the optimizer only needs S = sum coef, GA = sum coef A, GB = sum coef B per
// row (the same CSR walk as the other backbones) and three trigammas per dim.
//
// The MLPs run on the tcgen05 3xTF32 GEMM (tc_gemm.cu) with the same operand
// plumbing as intersect.cu; backward recomputes the forward intermediates from
// the saved inputs.
#include <algorithm>

#include "adam.cuh"
#include "common.cuh"
#include "mlp_util.cuh"
#include "special.cuh"

namespace ngdb_dev {
namespace {

constexpr int kWarps = 8;

// ---- per-step entity table -------------------------------------------------
__global__ void __launch_bounds__(kWarps * 32) beta_prep_kernel(DevArgs a, SparseTable t) {
  pdl_start();
  const int r = blockIdx.x * kWarps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= t.n_rows) return;
  for (int kk = t.seg[r] + lane; kk < t.seg[r + 1]; kk += 32) {
    const int32_t code = t.contrib[kk];
    if (code >= 0) a.cand_local[code] = r;
  }
  const int D = a.dim, d4 = D / 4;
  // the raw Beta pre-activations: the entity row, or (FuseSemantic) Psi_theta's row
  const float* x = a.ytab ? a.ytab + static_cast<int64_t>(r) * a.ent_w
                          : a.ent + static_cast<int64_t>(t.rows[r]) * a.ent_w;
  float* L = a.etab + static_cast<int64_t>(r) * a.ent_w;
  float c = 0.f;
  for (int ch = lane; ch < d4; ch += 32) {
    const float4 xa = ld4(x + 4 * ch), xb = ld4(x + D + 4 * ch);
    float pa[4], pb[4];
    const float va[4] = {xa.x, xa.y, xa.z, xa.w}, vb[4] = {xb.x, xb.y, xb.z, xb.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float al = beta_realize(va[u]), be = beta_realize(vb[u]), s = al + be;
      const float da = dg_digamma_fast(al), db = dg_digamma_fast(be), ds = dg_digamma_fast(s);
      pa[u] = ds - da;
      pb[u] = ds - db;
      c += -dg_lbeta(al, be) + al * da + be * db - s * ds;
    }
    st4(L + 4 * ch, make_float4(pa[0], pa[1], pa[2], pa[3]));
    st4(L + D + 4 * ch, make_float4(pb[0], pb[1], pb[2], pb[3]));
  }
  c = warp_sum(c);
  if (lane == 0) a.etab_c[r] = c;
}

// ---- lazy Adam on touched entity rows (see the header for the gradient) ----
__global__ void __launch_bounds__(kWarps * 32) beta_entity_adam_kernel(DevArgs a, SparseTable t,
                                                                       AdamHyper hp,
                                                                       const float* bc) {
  pdl_start();
  const int row_idx = blockIdx.x * kWarps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row_idx >= t.n_rows) return;
  const AdamK k = adam_consts(hp, bc);
  const int64_t row = t.rows[row_idx];
  const int beg = t.seg[row_idx], end = t.seg[row_idx + 1];
  const int D = a.dim, d4 = D / 4;
  float S = 0.f;  // sum of candidate coefficients (identical in every lane)
  for (int kk = beg; kk < end; ++kk) {
    const int32_t code = __ldg(t.contrib + kk);
    if (code >= 0) S += __ldg(a.coefbuf + code);
  }
  float* wp = t.w + row * t.width;
  float* mp = t.m + row * t.width;
  float* vp = t.v + row * t.width;
  for (int ch = lane; ch < d4; ch += 32) {
    float gA[4] = {0, 0, 0, 0}, gB[4] = {0, 0, 0, 0}, GA[4] = {0, 0, 0, 0}, GB[4] = {0, 0, 0, 0};
    for (int kk = beg; kk < end; ++kk) {
      const int32_t code = __ldg(t.contrib + kk);
      if (code < 0) {
        const float* g = a.agbuf + static_cast<int64_t>(-code - 1) * t.width;
        const float4 u = ld4(g + 4 * ch), v = ld4(g + D + 4 * ch);
        gA[0] += u.x; gA[1] += u.y; gA[2] += u.z; gA[3] += u.w;
        gB[0] += v.x; gB[1] += v.y; gB[2] += v.z; gB[3] += v.w;
      } else {
        const float coef = __ldg(a.coefbuf + code);
        const float* q = a.qbuf + static_cast<int64_t>(code / a.ncand) * a.wq;
        const float4 u = ld4(q + 4 * ch), v = ld4(q + D + 4 * ch);
        GA[0] += coef * u.x; GA[1] += coef * u.y; GA[2] += coef * u.z; GA[3] += coef * u.w;
        GB[0] += coef * v.x; GB[1] += coef * v.y; GB[2] += coef * v.z; GB[3] += coef * v.w;
      }
    }
    const float4 xa = ld4(wp + 4 * ch), xb = ld4(wp + D + 4 * ch);
    const float va[4] = {xa.x, xa.y, xa.z, xa.w}, vb[4] = {xb.x, xb.y, xb.z, xb.w};
    float ga[4], gb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float al, dal, be, dbe;
      beta_realize_pair(va[u], al, dal);
      beta_realize_pair(vb[u], be, dbe);
      const float s = al + be;
      const float ta = dg_trigamma_fast(al), tb = dg_trigamma_fast(be), ts = dg_trigamma_fast(s);
      const float dA = gA[u] + S * (al * ta - s * ts) + GA[u] * (ts - ta) + GB[u] * ts;
      const float dB = gB[u] + S * (be * tb - s * ts) + GA[u] * ts + GB[u] * (ts - tb);
      ga[u] = dA * dal;
      gb[u] = dB * dbe;
    }
    if (t.dbg_g) {
      st4(t.dbg_g + row * t.width + 4 * ch, make_float4(ga[0], ga[1], ga[2], ga[3]));
      st4(t.dbg_g + row * t.width + D + 4 * ch, make_float4(gb[0], gb[1], gb[2], gb[3]));
    }
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int off = half * D + 4 * ch;
      float4 w = ld4(wp + off), m = ld4(mp + off), v = ld4(vp + off);
      const float* g = half ? gb : ga;
      w = adam4(w, m, v, make_float4(g[0], g[1], g[2], g[3]), k);
      st4(wp + off, w);
      st4(mp + off, m);
      st4(vp + off, v);
    }
  }
}

// ---- FuseSemantic (Psi_theta): dL/dY instead of an Adam update ----------------
// The same gradient as beta_entity_adam_kernel with the pre-activations read
// from Y (CSR row order) and the result written out for Psi_theta's backward.
__global__ void __launch_bounds__(kWarps * 32) beta_fuse_grad_kernel(DevArgs a, SparseTable t,
                                                                     float* gY, Split gYs) {
  pdl_start();
  const int r = blockIdx.x * kWarps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= t.n_rows) return;
  const int beg = t.seg[r], end = t.seg[r + 1];
  const int D = a.dim, d4 = D / 4, W = a.ent_w;  // W = 2d
  float S = 0.f;
  for (int kk = beg; kk < end; ++kk) {
    const int32_t code = __ldg(t.contrib + kk);
    if (code >= 0) S += __ldg(a.coefbuf + code);
  }
  const float* yp = a.ytab + static_cast<int64_t>(r) * W;
  for (int ch = lane; ch < d4; ch += 32) {
    float gA[4] = {0, 0, 0, 0}, gB[4] = {0, 0, 0, 0}, GA[4] = {0, 0, 0, 0}, GB[4] = {0, 0, 0, 0};
    for (int kk = beg; kk < end; ++kk) {
      const int32_t code = __ldg(t.contrib + kk);
      if (code < 0) {
        const float* g = a.agbuf + static_cast<int64_t>(-code - 1) * W;
        const float4 u = ld4(g + 4 * ch), v = ld4(g + D + 4 * ch);
        gA[0] += u.x; gA[1] += u.y; gA[2] += u.z; gA[3] += u.w;
        gB[0] += v.x; gB[1] += v.y; gB[2] += v.z; gB[3] += v.w;
      } else {
        const float coef = __ldg(a.coefbuf + code);
        const float* q = a.qbuf + static_cast<int64_t>(code / a.ncand) * a.wq;
        const float4 u = ld4(q + 4 * ch), v = ld4(q + D + 4 * ch);
        GA[0] += coef * u.x; GA[1] += coef * u.y; GA[2] += coef * u.z; GA[3] += coef * u.w;
        GB[0] += coef * v.x; GB[1] += coef * v.y; GB[2] += coef * v.z; GB[3] += coef * v.w;
      }
    }
    const float4 xa = ld4(yp + 4 * ch), xb = ld4(yp + D + 4 * ch);
    const float va[4] = {xa.x, xa.y, xa.z, xa.w}, vb[4] = {xb.x, xb.y, xb.z, xb.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float al, dal, be, dbe;
      beta_realize_pair(va[u], al, dal);
      beta_realize_pair(vb[u], be, dbe);
      const float s = al + be;
      const float ta = dg_trigamma_fast(al), tb = dg_trigamma_fast(be), ts = dg_trigamma_fast(s);
      const float dA = gA[u] + S * (al * ta - s * ts) + GA[u] * (ts - ta) + GB[u] * ts;
      const float dB = gB[u] + S * (be * tb - s * ts) + GA[u] * ts + GB[u] * (ts - tb);
      put(gY, gYs, static_cast<int64_t>(r) * W + 4 * ch + u, dA * dal);
      put(gY, gYs, static_cast<int64_t>(r) * W + D + 4 * ch + u, dB * dbe);
    }
  }
}

// ---- Project -----------------------------------------------------------------
// X[i] = [q_i (2d) | r_i (d)] (plain + split)
__global__ void beta_proj_pack_kernel(DevArgs a, int first, float* X, Split Xs) {
  pdl_start();
  const int i = blockIdx.x;
  const ngdb_node_desc d = a.nodes[first + i];
  const int D = a.dim;
  const bool ok = d.id >= 0 && d.id < a.n_relations;
  if (!ok && threadIdx.x == 0) atomicOr(&a.flags[1], 1);
  const float* q = a.arena + d.in[0];
  const float* r = a.rel + static_cast<int64_t>(ok ? d.id : 0) * a.rel_w;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < 3 * D; e += blockDim.x * gridDim.y)
    put(X, Xs, static_cast<int64_t>(i) * 3 * D + e, e < 2 * D ? q[e] : r[e - 2 * D]);
}
// stash of a Project node (slot = its project slot, node aux): H, Z [2d] each
__device__ __forceinline__ float* proj_stash(const DevArgs& a, int slot) {
  if (slot < 0 || slot >= a.pstash_slots) {
    atomicOr(&a.flags[1], 1);
    slot = 0;
  }
  return a.pstash + static_cast<int64_t>(slot) * 4 * a.dim;
}
// output = realize(Z); H and Z are stashed for the mirror
__global__ void beta_proj_out_kernel(DevArgs a, int first, const float* Z, const float* H) {
  pdl_start();
  const int i = blockIdx.x;
  const ngdb_node_desc d = a.nodes[first + i];
  const int W = 2 * a.dim;
  float* st = proj_stash(a, d.aux);
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < W; e += blockDim.x * gridDim.y) {
    const float z = Z[static_cast<int64_t>(i) * W + e];
    a.arena[d.out + e] = beta_realize(z);
    st[e] = H[static_cast<int64_t>(i) * W + e];
    st[W + e] = z;
  }
}
// Backward gather: X = [q | r] (plain; the weight-gradient operand), the
// stashed H (the ReLU mask) and gZ = dL/dout * realize'(Z) (plain + split)
// (X and relu(H) are written split row-major only: the weight gradients read
// them MN-major; H stays plain as the ReLU mask)
__global__ void beta_proj_bwd_pack_kernel(DevArgs a, int first, Split Xs, float* H, Split RHs,
                                          float* gZ, Split gZs) {
  pdl_start();
  const int i = blockIdx.x;
  const ngdb_node_desc d = a.nodes[first + i];
  const int D = a.dim, W = 2 * D;
  const bool ok = d.id >= 0 && d.id < a.n_relations;
  if (!ok && threadIdx.x == 0) atomicOr(&a.flags[1], 1);
  const float* q = a.arena + d.in[0];
  const float* r = a.rel + static_cast<int64_t>(ok ? d.id : 0) * a.rel_w;
  const float* st = proj_stash(a, d.aux);
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < 3 * D; e += blockDim.x * gridDim.y) {
    put(nullptr, Xs, static_cast<int64_t>(i) * 3 * D + e, e < W ? q[e] : r[e - W]);
    if (e < W) {
      const int64_t o = static_cast<int64_t>(i) * W + e;
      H[o] = st[e];
      put(nullptr, RHs, o, fmaxf(st[e], 0.f));
      put(gZ, gZs, o, a.arena[d.grad + e] * beta_drealize(st[W + e]));
    }
  }
}
__global__ void beta_proj_gz_kernel(DevArgs a, int first, const float* Z, float* gZ, Split gZs) {
  pdl_start();
  const int i = blockIdx.x;
  const ngdb_node_desc d = a.nodes[first + i];
  const int W = 2 * a.dim;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < W; e += blockDim.x * gridDim.y) {
    const int64_t o = static_cast<int64_t>(i) * W + e;
    put(gZ, gZs, o, a.arena[d.grad + e] * beta_drealize(Z[o]));
  }
}
__global__ void beta_proj_scatter_kernel(DevArgs a, int first, const float* gX) {
  pdl_start();
  const int i = blockIdx.x;
  const ngdb_node_desc d = a.nodes[first + i];
  const int D = a.dim;
  const float* g = gX + static_cast<int64_t>(i) * 3 * D;
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < 3 * D; e += blockDim.x * gridDim.y) {
    if (e < 2 * D) a.arena[d.out + e] = g[e];
    else a.rgbuf[static_cast<int64_t>(d.aux) * a.rel_w + (e - 2 * D)] = g[e];
  }
}

int beta_project(const DevArgs& a, int dir, int first, int n, cudaStream_t s) {
  const int D = a.dim, D2 = 2 * D, D3 = 3 * D;
  Scratch sc{a.scratch, a.scratch_cap};
  float* X = sc.take((int64_t)n * D3);
  float* H = sc.take((int64_t)n * D2);
  const float* p = a.dense;
  int launches = 0;
  if (dir == 0) {
    Split Xs = take_split(sc, (int64_t)n * D3);
    Split RHs = take_split(sc, (int64_t)n * D2);
    float* Z = sc.take((int64_t)n * D2);
    launch_pdl(beta_proj_pack_kernel, node_grid(n, a.dim), dim3(128), 0, s, 1, a, first, X, Xs);
    ++launches;
    TcGemmArgs h = gemm_args(n, D2, D3, op(Xs, D3), wop(a, BETA_P1, D2, D3, false), H, D2);
    h.bias = p + a.dense_off[BETA_P1B];
    h.s_hi = RHs.hi; h.s_lo = RHs.lo; h.s_relu = 1;
    launches += tc_gemm(h, s);
    TcGemmArgs z = gemm_args(n, D2, D2, op(RHs, D2), wop(a, BETA_P2, D2, D2, false), Z, D2);
    z.bias = p + a.dense_off[BETA_P2B];
    launches += tc_gemm(z, s);
    launch_pdl(beta_proj_out_kernel, node_grid(n, a.dim), dim3(128), 0, s, 1, a, first,
               (const float*)Z, (const float*)H);
    return launches + 1;
  }
  // Backward: H and Z come from the node's stash (no forward recomputation)
  float* gZ = sc.take((int64_t)n * D2);
  Split gZs = take_split(sc, (int64_t)n * D2);
  float* gH = sc.take((int64_t)n * D2);
  Split gHs = take_split(sc, (int64_t)n * D2);
  Split Xs = take_split(sc, (int64_t)n * D3), RHs = take_split(sc, (int64_t)n * D2);
  float* gX = sc.take((int64_t)n * D3);
  float* g = a.dense_g;
  const int64_t* off = a.dense_off;
  launch_pdl(beta_proj_bwd_pack_kernel, node_grid(n, a.dim), dim3(128), 0, s, 1, a, first, Xs, H,
             RHs, gZ, gZs);
  ++launches;
  // gH = (gZ W2) * (H > 0)
  TcGemmArgs gh = gemm_args(n, D2, D2, op(gZs, D2), wop(a, BETA_P2, D2, D2, true), gH, D2);
  gh.mask = H;
  gh.s_hi = gHs.hi; gh.s_lo = gHs.lo;
  launches += tc_gemm(gh, s);
  // weight gradients: row-major splits read MN-major (no transposed copies)
  TcGemmArgs lvl[3];
  lvl[0] = gemm_args(D2, D2, n, mop(gZs, D2), mop(RHs, D2), g + off[BETA_P2], D2);  // gW2 += gZ^T relu(H)
  lvl[0].accumulate = 1;
  lvl[1] = gemm_args(D2, D3, n, mop(gHs, D2), mop(Xs, D3), g + off[BETA_P1], D3);   // gW1 += gH^T X
  lvl[1].accumulate = 1;
  lvl[2] = gemm_args(n, D3, D2, op(gHs, D2), wop(a, BETA_P1, D2, D3, true), gX, D3);  // gX = gH W1
  launches += tc_gemm_batch(lvl, 3, s);
  ColsumJobs cj{};
  cj.job[0] = {gZ, n, D2, g + off[BETA_P2B]};
  cj.job[1] = {gH, n, D2, g + off[BETA_P1B]};
  cj.n = 2;
  launches += colsums(cj, D2, s);
  launch_pdl(beta_proj_scatter_kernel, node_grid(n, a.dim), dim3(128), 0, s, 1, a, first, (const float*)gX);
  return launches + 1;
}

// ---- Intersect ---------------------------------------------------------------
__global__ void beta_inter_pack_kernel(DevArgs a, KSpan ks, int first, float* Q, Split Qs) {
  pdl_start();
  const int i = blockIdx.x;
  const int k = ks.k(i), r0 = ks.row0(i);
  const ngdb_node_desc d = a.nodes[first + i];
  const int W = 2 * a.dim;
  for (int l = 0; l < k; ++l)
    for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < W; e += blockDim.x * gridDim.y)
      put(Q, Qs, (static_cast<int64_t>(r0) + l) * W + e, a.arena[d.in[l] + e]);
}
__device__ __forceinline__ void softmax3(const float* S, int64_t base, int k, int D, int e, float* w) {
  float mx = S[base + e];
  for (int l = 1; l < k; ++l) mx = fmaxf(mx, S[base + static_cast<int64_t>(l) * D + e]);
  float z = 0.f;
  for (int l = 0; l < k; ++l) {
    w[l] = expf(S[base + static_cast<int64_t>(l) * D + e] - mx);
    z += w[l];
  }
  const float inv = 1.f / z;
  for (int l = 0; l < k; ++l) w[l] *= inv;
}
// stash of an Intersect node (slot = node aux): Z rows [3][2d], then S rows [3][d]
__device__ __forceinline__ float* inter_stash(const DevArgs& a, int slot) {
  if (slot < 0 || slot >= a.istash_slots) {
    atomicOr(&a.flags[1], 1);
    slot = 0;
  }
  return a.istash + static_cast<int64_t>(slot) * kStashPerSlot * a.dim;
}
__global__ void beta_inter_combine_kernel(DevArgs a, KSpan ks, int first, const float* S,
                                          const float* Q, const float* Z) {
  pdl_start();
  const int i = blockIdx.x;
  const int D = a.dim, W = 2 * D;
  const int k = ks.k(i), r0 = ks.row0(i);
  const ngdb_node_desc d = a.nodes[first + i];
  float* st = inter_stash(a, d.aux);
  // stash Z and S rows for the mirror
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < W; e += blockDim.x * gridDim.y)
    for (int l = 0; l < k; ++l) {
      st[l * W + e] = Z[(static_cast<int64_t>(r0) + l) * W + e];
      if (e < D) st[3 * W + l * D + e] = S[(static_cast<int64_t>(r0) + l) * D + e];
    }
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < D; e += blockDim.x * gridDim.y) {
    float w[3];
    softmax3(S, static_cast<int64_t>(r0) * D, k, D, e, w);
    float al = 0.f, be = 0.f;
    for (int l = 0; l < k; ++l) {
      const float* q = Q + (static_cast<int64_t>(r0) + l) * W;
      al += w[l] * q[e];
      be += w[l] * q[D + e];
    }
    a.arena[d.out + e] = al;
    a.arena[d.out + D + e] = be;
  }
}
// Backward combine from the node's stash; also gathers the inputs Q and the
// stashed Z rows into class order (weight-gradient operands, ReLU mask).
__global__ void beta_inter_combine_bwd_kernel(DevArgs a, KSpan ks, int first, Split Qs, float* Z,
                                              Split RZs, float* gS, Split gSs, float* dQ) {
  pdl_start();
  const int i = blockIdx.x;
  const int D = a.dim, W = 2 * D;
  const int k = ks.k(i), r0 = ks.row0(i);
  const ngdb_node_desc d = a.nodes[first + i];
  const float* st = inter_stash(a, d.aux);
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < W; e += blockDim.x * gridDim.y)
    for (int l = 0; l < k; ++l) {
      const int64_t r = (static_cast<int64_t>(r0) + l) * W + e;
      put(nullptr, Qs, r, a.arena[d.in[l] + e]);  // split only: read MN-major
      Z[r] = st[l * W + e];                      // ReLU mask
      put(nullptr, RZs, r, fmaxf(st[l * W + e], 0.f));
    }
  const float* S = st + 3 * W;  // the node's k score rows [k][D]
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < D; e += blockDim.x * gridDim.y) {
    const float gA = a.arena[d.grad + e], gB = a.arena[d.grad + D + e];
    float w[3], gw[3], dot = 0.f;
    softmax3(S, 0, k, D, e, w);
    for (int l = 0; l < k; ++l) {
      const float* q = a.arena + d.in[l];
      gw[l] = gA * q[e] + gB * q[D + e];
      dot += w[l] * gw[l];
    }
    for (int l = 0; l < k; ++l) {
      const int64_t r = static_cast<int64_t>(r0) + l;
      put(gS, gSs, r * D + e, w[l] * (gw[l] - dot));
      dQ[r * W + e] = gA * w[l];
      dQ[r * W + D + e] = gB * w[l];
    }
  }
}
__global__ void beta_inter_scatter_kernel(DevArgs a, KSpan ks, int first, const float* dQ) {
  pdl_start();
  const int i = blockIdx.x;
  const int W = 2 * a.dim;
  const int k = ks.k(i), r0 = ks.row0(i);
  const ngdb_node_desc d = a.nodes[first + i];
  for (int l = 0; l < k; ++l)
    for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < W; e += blockDim.x * gridDim.y)
      a.arena[d.out + l * W + e] = dQ[(static_cast<int64_t>(r0) + l) * W + e];
}

int beta_intersect(const DevArgs& a, int dir, KSpan ks, int first, int n, cudaStream_t s) {
  const int D = a.dim, W = 2 * D;
  const int R = ks.row0(n);
  Scratch sc{a.scratch, a.scratch_cap};
  float* Q = sc.take((int64_t)R * W);
  float* Z = sc.take((int64_t)R * W);
  const float* p = a.dense;
  int launches = 0;
  if (dir == 0) {
    Split Qs = take_split(sc, (int64_t)R * W);
    Split RZs = take_split(sc, (int64_t)R * W);
    float* S = sc.take((int64_t)R * D);
    launch_pdl(beta_inter_pack_kernel, node_grid(n, a.dim), dim3(128), 0, s, 1, a, ks, first, Q, Qs);
    ++launches;
    TcGemmArgs z = gemm_args(R, W, W, op(Qs, W), wop(a, BETA_A1, W, W, false), Z, W);
    z.bias = p + a.dense_off[BETA_A1B];
    z.s_hi = RZs.hi; z.s_lo = RZs.lo; z.s_relu = 1;
    launches += tc_gemm(z, s);
    TcGemmArgs sg = gemm_args(R, D, W, op(RZs, W), wop(a, BETA_A2, D, W, false), S, D);
    sg.bias = p + a.dense_off[BETA_A2B];
    launches += tc_gemm(sg, s);
    launch_pdl(beta_inter_combine_kernel, node_grid(n, a.dim), dim3(128), 0, s, 1, a, ks, first,
               (const float*)S, (const float*)Q, (const float*)Z);
    return launches + 1;
  }
  // Backward: Z and S come from the node's stash (no forward recomputation)
  float* gS = sc.take((int64_t)R * D);
  Split gSs = take_split(sc, (int64_t)R * D);
  float* dQ = sc.take((int64_t)R * W);
  float* gZ = sc.take((int64_t)R * W);
  Split gZs = take_split(sc, (int64_t)R * W);
  Split Qs = take_split(sc, (int64_t)R * W), RZs = take_split(sc, (int64_t)R * W);
  float* g = a.dense_g;
  const int64_t* off = a.dense_off;
  launch_pdl(beta_inter_combine_bwd_kernel, node_grid(n, a.dim), dim3(128), 0, s, 1, a, ks, first,
             Qs, Z, RZs, gS, gSs, dQ);
  ++launches;
  // gZ = (gS A2) * (Z > 0)
  TcGemmArgs gz = gemm_args(R, W, D, op(gSs, D), wop(a, BETA_A2, D, W, true), gZ, W);
  gz.mask = Z;
  gz.s_hi = gZs.hi; gz.s_lo = gZs.lo;
  launches += tc_gemm(gz, s);
  // weight gradients: row-major splits read MN-major (no transposed copies)
  TcGemmArgs lvl[3];
  lvl[0] = gemm_args(D, W, R, mop(gSs, D), mop(RZs, W), g + off[BETA_A2], W);  // gA2 += gS^T relu(Z)
  lvl[0].accumulate = 1;
  lvl[1] = gemm_args(W, W, R, mop(gZs, W), mop(Qs, W), g + off[BETA_A1], W);   // gA1 += gZ^T Q
  lvl[1].accumulate = 1;
  lvl[2] = gemm_args(R, W, W, op(gZs, W), wop(a, BETA_A1, W, W, true), dQ, W);  // dQ += gZ A1
  lvl[2].accumulate = 1;
  launches += tc_gemm_batch(lvl, 3, s);
  ColsumJobs cj{};
  cj.job[0] = {gS, R, D, g + off[BETA_A2B]};
  cj.job[1] = {gZ, R, W, g + off[BETA_A1B]};
  cj.n = 2;
  launches += colsums(cj, W, s);
  launch_pdl(beta_inter_scatter_kernel, node_grid(n, a.dim), dim3(128), 0, s, 1, a, ks, first, (const float*)dQ);
  return launches + 1;
}

}  // namespace

int64_t beta_project_scratch_floats(int dim, int max_nodes) {
  return 50 * (int64_t)(max_nodes + 4) * dim + 64 * (int64_t)dim + 256;
}

int64_t beta_scratch_floats(int dim, int max_nodes) {
  const int64_t nd = (int64_t)(max_nodes + 4) * dim, rd = 3 * nd;
  const int64_t project = 50 * nd;   // X, Xs, H, RHs, Z, gZ(s), gH(s), gX (bound: 30 nd used)
  const int64_t intersect = 38 * rd; // Q(s), Z, RZs, S, gS(s), dQ, gZ(s) (bound)
  return std::max(project, intersect) + 64 * (int64_t)dim + 256;
}

int launch_beta_prep(const DevArgs& a, const SparseTable& t, const LaunchCtx& lc) {
  if (t.n_rows <= 0) return 0;
  launch_pdl(beta_prep_kernel, dim3((t.n_rows + kWarps - 1) / kWarps), dim3(kWarps * 32), 0,
             lc.stream, 1, a, t);
  return 1;
}

int launch_beta_fuse_grad(const DevArgs& a, const SparseTable& t, float* gY, Split gYs,
                          const LaunchCtx& lc) {
  if (t.n_rows <= 0) return 0;
  launch_pdl(beta_fuse_grad_kernel, dim3((t.n_rows + kWarps - 1) / kWarps), dim3(kWarps * 32), 0,
             lc.stream, 1, a, t, gY, gYs);
  return 1;
}

int launch_beta_entity_adam(const DevArgs& a, const SparseTable& t, const AdamHyper& hp,
                            const float* bc, const LaunchCtx& lc) {
  if (t.n_rows <= 0) return 0;
  launch_pdl(beta_entity_adam_kernel, dim3((t.n_rows + kWarps - 1) / kWarps), dim3(kWarps * 32), 0,
             lc.stream, 1, a, t, hp, bc);
  return 1;
}

int launch_beta_project(const DevArgs& a, int dir, int first, int n, const LaunchCtx& lc) {
  if (n <= 0) return 0;
  return beta_project(a, dir, first, n, lc.stream);
}

int launch_beta_intersect(const DevArgs& a, int dir, KSpan ks, int first, int n, const LaunchCtx& lc) {
  if (n <= 0) return 0;
  return beta_intersect(a, dir, ks, first, n, lc.stream);
}

}  // namespace ngdb_dev
