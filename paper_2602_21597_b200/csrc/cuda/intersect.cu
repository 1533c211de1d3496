// Intersection operators per cardinality class (Eq. 8-9).
//
//   GQE:  y = W2 relu(W1 mean_k x)                (no bias)
//   Q2B:  centre = sum_l softmax_l(A2 relu(A1 c_l + a1) + a2) * c_l
//                           offset = min_l o_l * sigmoid(V2 mean_l relu(V1 o_l + v1) + v2)
//
// Every dense contraction runs on the tcgen05 tensor cores as a 3xTF32 GEMM
// (tc_gemm.cu; fp32-grade accuracy — single-pass TF32 cannot hold the 1e-4
// parity bar at K=400). Operands enter pre-split (hi/lo): weights once per
// optimizer step, activations from the packing kernels or from the epilogue of
// the GEMM that produced them; the weight-gradient operands (dY^T, X^T) are
// transposed+split in one batched launch. Independent GEMMs of a dependency
// level share one grouped launch. Backward recomputes the forward
// intermediates from the saved inputs (the only activations the Eq. 7 refcount
// model keeps alive). Rows are node-major: row = i*k + l.
#include <algorithm>

#include "common.cuh"
#include "mlp_util.cuh"

namespace ngdb_dev {

// bias gradients of a class in one launch: db_j += column sums of dy_j
// 32 columns per CTA; the rows are split over a cluster of P CTAs (consecutive
// blockIdx.x), each summing its row range — warp w of 16 takes rows w, w+16,
// ... with four independent accumulators (loads in flight) and the 16 warp
// partials are combined in warp order — then cluster rank 0 adds the P CTA
// partials in rank order through distributed shared memory (deterministic,
// no global scratch). Tall gradients (the fusion backward's 14.5k rows) thus
// spread over 8 x (n / 32) CTAs instead of n / 32.
constexpr int kColsumWarps = 16;
__global__ void __launch_bounds__(kColsumWarps * 32) colsum_kernel(ColsumJobs jobs, int P) {
  pdl_start();
  __shared__ float part[kColsumWarps][32];
  __shared__ float total[32];
  const ColsumJob& j = jobs.job[blockIdx.y];
  const int rank = blockIdx.x % P, cg = blockIdx.x / P;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int c = cg * 32 + lane;
  const int r_beg = static_cast<int>((int64_t)rank * j.rows / P);
  const int r_end = static_cast<int>((int64_t)(rank + 1) * j.rows / P);
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  if (c < j.n) {
    constexpr int W = kColsumWarps;
    int r = r_beg + warp;
    for (; r + 3 * W < r_end; r += 4 * W) {
      s0 += j.dy[(int64_t)r * j.n + c];
      s1 += j.dy[(int64_t)(r + W) * j.n + c];
      s2 += j.dy[(int64_t)(r + 2 * W) * j.n + c];
      s3 += j.dy[(int64_t)(r + 3 * W) * j.n + c];
    }
    for (; r < r_end; r += W) s0 += j.dy[(int64_t)r * j.n + c];
  }
  part[warp][lane] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (warp == 0) {
    float t = 0.f;
    for (int w = 0; w < kColsumWarps; ++w) t += part[w][lane];
    total[lane] = t;
  }
  if (P > 1) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
  else __syncthreads();
  if (rank == 0 && warp == 0 && c < j.n) {
    float t = total[lane];
    const uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(&total[lane]));
    for (int q = 1; q < P; ++q) {  // peers in rank order
      uint32_t remote;
      float v;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(q));
      asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(remote));
      t += v;
    }
    j.db[c] += t;
  }
  // peers' partials stay resident until rank 0 has read them
  if (P > 1) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;");
}
int colsums(const ColsumJobs& jobs, int n, cudaStream_t s) {
  int rows = 0;
  for (int i = 0; i < jobs.n; ++i) rows = std::max(rows, jobs.job[i].rows);
  const int P = std::max(1, std::min(8, rows / 512));  // >= 512 rows per CTA
  launch_pdl(colsum_kernel, dim3(dim3((n + 31) / 32 * P, jobs.n)), dim3(kColsumWarps * 32), 0, s,
             P, jobs, P);
  return 1;
}


namespace {

// ---------------------------------------------------------------------------
// GQE

// M[i] = mean_l x_l (plain + split); optionally G[i] = upstream grad (plain + split)
__global__ void gqe_pack_kernel(DevArgs a, KSpan ks, int first, float* M, Split Ms, float* G,
                                Split Gs) {
  pdl_launch();
  const int i = blockIdx.x;
  const int k = ks.k(i);
  const ngdb_node_desc d = a.nodes[first + i];  // plan data: before the wait
  pdl_wait();
  const float inv_k = 1.f / static_cast<float>(k);
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < a.dim; e += blockDim.x * gridDim.y) {
    float s = 0.f;
    for (int l = 0; l < k; ++l) s += a.arena[d.in[l] + e];
    const int64_t o = (int64_t)i * a.dim + e;
    put(M, Ms, o, s * inv_k);
    if (G) put(G, Gs, o, a.arena[d.grad + e]);
  }
}
// G_X row l of node i = dM[i] / k  (mean adjoint)
__global__ void gqe_scatter_kernel(DevArgs a, KSpan ks, int first, const float* dM) {
  pdl_launch();
  const int i = blockIdx.x;
  const int k = ks.k(i);
  const ngdb_node_desc d = a.nodes[first + i];  // plan data: before the wait
  pdl_wait();
  const float inv_k = 1.f / static_cast<float>(k);
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < a.dim; e += blockDim.x * gridDim.y) {
    const float v = dM[(int64_t)i * a.dim + e] * inv_k;
    for (int l = 0; l < k; ++l) a.arena[d.out + l * a.dim + e] = v;
  }
}

int gqe_intersect(const DevArgs& a, int dir, KSpan ks, int first, int n, cudaStream_t s) {
  const int D = a.dim;
  const int64_t nd = (int64_t)n * D;
  Scratch sc{a.scratch, a.scratch_cap};
  float* M = sc.take(nd);
  Split Ms = take_split(sc, nd);
  float* H = sc.take(nd);
  Split RHs = take_split(sc, nd);  // split(relu(H))
  float* G = dir ? sc.take(nd) : nullptr;
  Split Gs = dir ? take_split(sc, nd) : Split{nullptr, nullptr};
  int launches = 0;

  launch_pdl(gqe_pack_kernel, node_grid(n, a.dim), dim3(128), 0, s, 1, a, ks, first, M, Ms, G, Gs);
  ++launches;
  TcGemmArgs h = gemm_args(n, D, D, op(Ms, D), wop(a, GQE_W1, D, D, false), H, D);
  h.s_hi = RHs.hi; h.s_lo = RHs.lo; h.s_relu = 1;
  launches += tc_gemm(h, s);
  if (dir == 0) {
    // y = relu(H) W2^T, scattered straight into the planned arena slots
    TcGemmArgs y = gemm_args(n, D, D, op(RHs, D), wop(a, GQE_W2, D, D, false), a.arena, D);
    y.c_rowoff = &a.nodes[first].out;
    y.c_stride = sizeof(ngdb_node_desc) / sizeof(int32_t);
    return launches + tc_gemm(y, s);
  }
  float* dH = sc.take(nd);
  Split dHs = take_split(sc, nd);
  float* dM = sc.take(nd);
  float* gW1 = a.dense_g + a.dense_off[GQE_W1];
  float* gW2 = a.dense_g + a.dense_off[GQE_W2];
  // dH = (G W2) * (H > 0), also split for dM = dH W1
  TcGemmArgs da = gemm_args(n, D, D, op(Gs, D), wop(a, GQE_W2, D, D, true), dH, D);
  da.mask = H;
  da.s_hi = dHs.hi; da.s_lo = dHs.lo;
  launches += tc_gemm(da, s);
  // weight gradients read the row-major splits of G, relu(H), dH and M (pack
  // kernel / GEMM epilogues) MN-major: no transposed copies
  TcGemmArgs lvl[3];
  lvl[0] = gemm_args(D, D, n, mop(Gs, D), mop(RHs, D), gW2, D);  // gW2 += G^T relu(H)
  lvl[0].accumulate = 1;
  lvl[1] = gemm_args(D, D, n, mop(dHs, D), mop(Ms, D), gW1, D);  // gW1 += dH^T M
  lvl[1].accumulate = 1;
  lvl[2] = gemm_args(n, D, D, op(dHs, D), wop(a, GQE_W1, D, D, true), dM, D);  // dM = dH W1
  launches += tc_gemm_batch(lvl, 3, s);
  launch_pdl(gqe_scatter_kernel, node_grid(n, a.dim), dim3(128), 0, s, 1, a, ks, first, dM);
  return launches + 1;
}

// ---------------------------------------------------------------------------
// Q2B

__global__ void q2b_pack_kernel(DevArgs a, KSpan ks, int first, float* Cin, Split Cs, float* Oin,
                                Split Os) {
  pdl_launch();
  const int i = blockIdx.x;
  const int k = ks.k(i), r0 = ks.row0(i);
  const ngdb_node_desc d = a.nodes[first + i];  // plan data: before the wait
  pdl_wait();
  for (int l = 0; l < k; ++l)
    for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < a.dim; e += blockDim.x * gridDim.y) {
      const int64_t r = ((int64_t)r0 + l) * a.dim + e;
      put(Cin, Cs, r, a.arena[d.in[l] + e]);
      put(Oin, Os, r, a.arena[d.in[l] + a.dim + e]);
    }
}
// Lm[i] = mean_l relu(P[i*k+l]) (plain + split)
__global__ void q2b_mean_relu_kernel(const float* P, KSpan ks, int D, float* Lm, Split Lms) {
  pdl_start();
  const int i = blockIdx.x;
  const int k = ks.k(i), r0 = ks.row0(i);
  const float inv_k = 1.f / static_cast<float>(k);
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < D; e += blockDim.x * gridDim.y) {
    float s = 0.f;
    for (int l = 0; l < k; ++l) s += fmaxf(P[((int64_t)r0 + l) * D + e], 0.f);
    put(Lm, Lms, (int64_t)i * D + e, s * inv_k);
  }
}
__device__ __forceinline__ void softmax_k(const float* S, int64_t base, int k, int D, int e,
                                          float* w) {
  float mx = S[base + e];
  for (int l = 1; l < k; ++l) mx = fmaxf(mx, S[base + (int64_t)l * D + e]);
  float z = 0.f;
  for (int l = 0; l < k; ++l) {
    w[l] = expf(S[base + (int64_t)l * D + e] - mx);
    z += w[l];
  }
  const float inv = 1.f / z;
  for (int l = 0; l < k; ++l) w[l] *= inv;
}
// stash of a forward node: Z, S, P rows [3][D], then U, Lm [D] (kStashPerSlot)
__device__ __forceinline__ float* q2b_stash(const DevArgs& a, int slot) {
  if (slot < 0 || slot >= a.istash_slots) {
    atomicOr(&a.flags[1], 1);
    slot = 0;
  }
  return a.istash + static_cast<int64_t>(slot) * kStashPerSlot * a.dim;
}

// Forward combine; also stashes the node's MLP intermediates (Z, S, P rows,
// U, Lm) for its mirror, which then skips the forward recomputation.
__global__ void q2b_combine_kernel(DevArgs a, KSpan ks, int first, const float* S, const float* U,
                                   const float* Cin, const float* Oin, const float* Z,
                                   const float* P, const float* Lm) {
  pdl_launch();
  const int i = blockIdx.x;
  const int D = a.dim;
  const int k = ks.k(i);
  const ngdb_node_desc d = a.nodes[first + i];  // plan data: before the wait
  pdl_wait();
  const int64_t base = (int64_t)ks.row0(i) * D;
  float* st = q2b_stash(a, d.aux);
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < D; e += blockDim.x * gridDim.y) {
    float w[3];
    softmax_k(S, base, k, D, e, w);
    float c = 0.f, mn = Oin[base + e];
    for (int l = 0; l < k; ++l) {
      c += w[l] * Cin[base + (int64_t)l * D + e];
      mn = fminf(mn, Oin[base + (int64_t)l * D + e]);
      st[l * D + e] = Z[base + (int64_t)l * D + e];
      st[3 * D + l * D + e] = S[base + (int64_t)l * D + e];
      st[6 * D + l * D + e] = P[base + (int64_t)l * D + e];
    }
    const float u = U[(int64_t)i * D + e];
    st[9 * D + e] = u;
    st[10 * D + e] = Lm[(int64_t)i * D + e];
    a.arena[d.out + e] = c;
    a.arena[d.out + D + e] = mn * sigmoidf(u);
  }
}
// Backward combine. Also gathers the node's inputs (arena) and its stashed Z,
// P rows and Lm into class order: the ReLU masks (Z, P plain) and, split
// row-major, the weight-gradient GEMMs' operands (Cin, Oin, relu(Z), Lm —
// read MN-major by the GEMMs, so no transposed copies).
__global__ void q2b_combine_bwd_kernel(DevArgs a, KSpan ks, int first, Split Cs, Split Os,
                                       float* Z, Split RZs, float* P, Split Lms, float* gS, Split gSs,
                                       float* dCin, float* dOin, float* gU, Split gUs) {
  pdl_launch();
  const int i = blockIdx.x;
  const int D = a.dim;
  const int k = ks.k(i);
  const ngdb_node_desc d = a.nodes[first + i];  // plan data: before the wait
  pdl_wait();
  const int64_t base = (int64_t)ks.row0(i) * D;
  const float* st = q2b_stash(a, d.aux);
  const float* S = st + 3 * D;  // the node's k score rows, stashed by the forward
  for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < D; e += blockDim.x * gridDim.y) {
    const float gC = a.arena[d.grad + e];
    const float gO = a.arena[d.grad + D + e];
    float w[3], cin[3], oin[3];
    softmax_k(S, 0, k, D, e, w);
    float ga[3], dot = 0.f;
    for (int l = 0; l < k; ++l) {
      const int64_t r = base + (int64_t)l * D + e;
      cin[l] = a.arena[d.in[l] + e];
      oin[l] = a.arena[d.in[l] + D + e];
      put(nullptr, Cs, r, cin[l]);
      put(nullptr, Os, r, oin[l]);
      const float z = st[l * D + e];
      Z[r] = z;
      put(nullptr, RZs, r, fmaxf(z, 0.f));
      P[r] = st[6 * D + l * D + e];
      ga[l] = gC * cin[l];
      dot += w[l] * ga[l];
    }
    put(nullptr, Lms, (int64_t)i * D + e, st[10 * D + e]);
    int arg = 0;
    float mn = oin[0];
    for (int l = 1; l < k; ++l)
      if (oin[l] < mn) { mn = oin[l]; arg = l; }  // ties -> lowest index
    const float gate = sigmoidf(st[9 * D + e]);
    for (int l = 0; l < k; ++l) {
      const int64_t r = base + (int64_t)l * D + e;
      put(gS, gSs, r, w[l] * (ga[l] - dot));
      dCin[r] = gC * w[l];
      dOin[r] = (l == arg) ? gO * gate : 0.f;
    }
    put(gU, gUs, (int64_t)i * D + e, gO * mn * gate * (1.f - gate));
  }
}
// The backward tail in ONE launch: blocks [0, n_col) compute the bias
// gradients (the colsum kernel's work), the rest scatter dCin / dOin into the
// planned G slots, one node per block.
__global__ void __launch_bounds__(kColsumWarps * 32) q2b_bwd_tail_kernel(DevArgs a, KSpan ks, int first,
                                                                         const float* dCin,
                                                                         const float* dOin,
                                                                         ColsumJobs jobs, int n_colx) {
  pdl_start();
  const int n_col = n_colx * jobs.n;
  if (static_cast<int>(blockIdx.x) < n_col) {
    __shared__ float part[kColsumWarps][32];
    const ColsumJob& j = jobs.job[blockIdx.x / n_colx];
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int c = (blockIdx.x % n_colx) * 32 + lane;
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    if (c < j.n) {
      constexpr int W = kColsumWarps;
      int r = warp;
      for (; r + 3 * W < j.rows; r += 4 * W) {
        s0 += j.dy[(int64_t)r * j.n + c];
        s1 += j.dy[(int64_t)(r + W) * j.n + c];
        s2 += j.dy[(int64_t)(r + 2 * W) * j.n + c];
        s3 += j.dy[(int64_t)(r + 3 * W) * j.n + c];
      }
      for (; r < j.rows; r += W) s0 += j.dy[(int64_t)r * j.n + c];
    }
    part[warp][lane] = (s0 + s1) + (s2 + s3);
    __syncthreads();
    if (warp == 0 && c < j.n) {
      float t = 0.f;
      for (int w = 0; w < kColsumWarps; ++w) t += part[w][lane];
      j.db[c] += t;
    }
    return;
  }
  const int i = blockIdx.x - n_col;
  const int D = a.dim;
  const int k = ks.k(i), r0 = ks.row0(i);
  const ngdb_node_desc d = a.nodes[first + i];
  for (int l = 0; l < k; ++l)
    for (int e = threadIdx.x; e < D; e += blockDim.x) {
      const int64_t r = ((int64_t)r0 + l) * D + e;
      a.arena[d.out + l * 2 * D + e] = dCin[r];
      a.arena[d.out + l * 2 * D + D + e] = dOin[r];
    }
}

int q2b_intersect(const DevArgs& a, int dir, KSpan ks, int first, int n, cudaStream_t s) {
  const int D = a.dim;
  const int R = ks.row0(n);
  const int64_t rd = (int64_t)R * D, nd = (int64_t)n * D;
  Scratch sc{a.scratch, a.scratch_cap};
  float* Cin = sc.take(rd);
  float* Oin = sc.take(rd);
  float* Z = sc.take(rd);
  float* Lm = sc.take(nd);
  int launches = 0;
  if (dir == 0) {
    Split Cs = take_split(sc, rd);
    Split Os = take_split(sc, rd);
    Split RZs = take_split(sc, rd);  // split(relu(Z))
    float* S = sc.take(rd);
    float* P = sc.take(rd);
    Split Lms = take_split(sc, nd);
    float* U = sc.take(nd);
    const float* p = a.dense;
    const float* a1 = p + a.dense_off[Q2B_A1B];
    const float* a2 = p + a.dense_off[Q2B_A2B];
    const float* v1 = p + a.dense_off[Q2B_V1B];
    const float* v2 = p + a.dense_off[Q2B_V2B];
    launch_pdl(q2b_pack_kernel, node_grid(n, a.dim), dim3(128), 0, s, 1, a, ks, first, Cin, Cs, Oin, Os);
    ++launches;
    {  // level 1: Z = A1 c + a1 (chained split of relu(Z)), P = V1 o + v1
      TcGemmArgs lvl[2];
      lvl[0] = gemm_args(R, D, D, op(Cs, D), wop(a, Q2B_A1, D, D, false), Z, D);
      lvl[0].bias = a1;
      lvl[0].s_hi = RZs.hi; lvl[0].s_lo = RZs.lo; lvl[0].s_relu = 1;
      lvl[1] = gemm_args(R, D, D, op(Os, D), wop(a, Q2B_V1, D, D, false), P, D);
      lvl[1].bias = v1;
      launches += tc_gemm_batch(lvl, 2, s);
    }
    launch_pdl(q2b_mean_relu_kernel, node_grid(n, a.dim), dim3(128), 0, s, 1, P, ks, D, Lm, Lms);
    ++launches;
    {  // level 2: S = A2 relu(Z) + a2, U = V2 Lm + v2
      TcGemmArgs lvl[2];
      lvl[0] = gemm_args(R, D, D, op(RZs, D), wop(a, Q2B_A2, D, D, false), S, D);
      lvl[0].bias = a2;
      lvl[1] = gemm_args(n, D, D, op(Lms, D), wop(a, Q2B_V2, D, D, false), U, D);
      lvl[1].bias = v2;
      launches += tc_gemm_batch(lvl, 2, s);
    }
    launch_pdl(q2b_combine_kernel, node_grid(n, a.dim), dim3(128), 0, s, 1, a, ks, first, (const float*)S,
               (const float*)U, (const float*)Cin, (const float*)Oin, (const float*)Z,
               (const float*)P, (const float*)Lm);
    return launches + 1;
  }
  // Backward: the forward's Z, S, P, U, Lm come from the node's stash slot.
  // The weight gradients dW += dY^T X read dY and X as row-major splits
  // through MN-major UMMA operands (K = rows): no transposed copies.
  float* gS = sc.take(rd);
  Split gSs = take_split(sc, rd);
  float* dCin = sc.take(rd);
  float* dOin = sc.take(rd);
  float* gU = sc.take(nd);
  Split gUs = take_split(sc, nd);
  float* gLm = sc.take(nd);
  float* gP = sc.take(rd);
  Split gPs = take_split(sc, rd);
  float* gZ = sc.take(rd);
  Split gZs = take_split(sc, rd);
  Split Cs = take_split(sc, rd), Os = take_split(sc, rd), RZs = take_split(sc, rd),
        Lms = take_split(sc, nd);
  float* g = a.dense_g;
  const int64_t* off = a.dense_off;

  float* Pc = sc.take(rd);  // stashed P rows in class order (ReLU mask of gP)
  launch_pdl(q2b_combine_bwd_kernel, node_grid(n, a.dim), dim3(128), 0, s, 1, a, ks, first, Cs, Os, Z,
             RZs, Pc, Lms, gS, gSs, dCin, dOin, gU, gUs);
  ++launches;
  {  // level 3: weight grads of V2, A2; gLm = gU V2; gZ = (gS A2) * (Z > 0)
    TcGemmArgs lvl[4];
    lvl[0] = gemm_args(D, D, n, mop(gUs, D), mop(Lms, D), g + off[Q2B_V2], D);
    lvl[0].accumulate = 1;
    lvl[1] = gemm_args(D, D, R, mop(gSs, D), mop(RZs, D), g + off[Q2B_A2], D);
    lvl[1].accumulate = 1;
    lvl[2] = gemm_args(n, D, D, op(gUs, D), wop(a, Q2B_V2, D, D, true), gLm, D);
    lvl[3] = gemm_args(R, D, D, op(gSs, D), wop(a, Q2B_A2, D, D, true), gZ, D);
    lvl[3].mask = Z;
    lvl[3].s_hi = gZs.hi; lvl[3].s_lo = gZs.lo;
    launches += tc_gemm_batch(lvl, 4, s);
  }
  SplitJobs j2{};
  // gP = gLm / k * (P > 0), computed and written plain + split row-major
  j2.job[0] = {gP, R, D, D, 0, nullptr, nullptr, gLm, Pc, ks.n1, ks.k1, ks.k2, gP, gPs.hi, gPs.lo};
  j2.n = 1;
  launches += split_transposed(j2, s);
  {  // level 4: weight grads of V1, A1; input grads dOin += gP V1, dCin += gZ A1
    TcGemmArgs lvl[4];
    lvl[0] = gemm_args(D, D, R, mop(gPs, D), mop(Os, D), g + off[Q2B_V1], D);
    lvl[0].accumulate = 1;
    lvl[1] = gemm_args(D, D, R, mop(gZs, D), mop(Cs, D), g + off[Q2B_A1], D);
    lvl[1].accumulate = 1;
    lvl[2] = gemm_args(R, D, D, op(gPs, D), wop(a, Q2B_V1, D, D, true), dOin, D);
    lvl[2].accumulate = 1;
    lvl[3] = gemm_args(R, D, D, op(gZs, D), wop(a, Q2B_A1, D, D, true), dCin, D);
    lvl[3].accumulate = 1;
    launches += tc_gemm_batch(lvl, 4, s);
  }
  ColsumJobs cj{};
  cj.job[0] = {gU, n, D, g + off[Q2B_V2B]};
  cj.job[1] = {gS, R, D, g + off[Q2B_A2B]};
  cj.job[2] = {gP, R, D, g + off[Q2B_V1B]};
  cj.job[3] = {gZ, R, D, g + off[Q2B_A1B]};
  cj.n = 4;
  const int n_colx = (D + 31) / 32;  // bias gradients and the G-slot scatter: one launch
  launch_pdl(q2b_bwd_tail_kernel, dim3(n_colx * cj.n + n), dim3(kColsumWarps * 32), 0, s, 1, a, ks,
             first, (const float*)dCin, (const float*)dOin, cj, n_colx);
  return launches + 1;
}

}  // namespace

int64_t intersect_scratch_floats(int backbone, int dim, int max_nodes) {
  const int64_t nd = (int64_t)max_nodes * dim, rd = 3 * nd;
  // (upper bounds; the weight gradients read row-major splits MN-major)
  if (backbone == NGDB_GQE) return 24 * nd + 32 * (int64_t)dim + 64;
  if (backbone == NGDB_BETAE) return beta_scratch_floats(dim, max_nodes);
  return 36 * rd + 14 * nd + 64 * (int64_t)dim + 256;
}

int launch_intersect(const DevArgs& a, int dir, KSpan ks, int first, int n, const LaunchCtx& lc) {
  if (n <= 0) return 0;
  if (a.backbone == NGDB_GQE) return gqe_intersect(a, dir, ks, first, n, lc.stream);
  if (a.backbone == NGDB_BETAE) return launch_beta_intersect(a, dir, ks, first, n, lc);
  return q2b_intersect(a, dir, ks, first, n, lc.stream);
}

}  // namespace ngdb_dev
