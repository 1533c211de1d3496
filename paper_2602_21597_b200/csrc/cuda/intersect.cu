// Intersection operators per cardinality class (Eq. 8-9).
//
//   GQE:  y = W2 relu(W1 mean_k x)                (no bias)
//   Q2B:  centre = sum_l softmax_l(A2 relu(A1 c_l + a1) + a2) * c_l
//                           offset = min_l o_l * sigmoid(V2 mean_l relu(V1 o_l + v1) + v2)
//
// The contractions run on the tcgen05 tensor cores as 3xTF32 GEMMs (tc_gemm.cu:
// fp32-level accuracy; single-pass TF32 cannot hold the 1e-4 bar at K=400). Each class is
// packed into contiguous scratch, contracted, and scattered back to the planned
// arena slots; backward recomputes the forward intermediates from the saved
// inputs (the only activations the Eq. 7 refcount model keeps alive).
#include "common.cuh"
#include "tc_gemm.cuh"

namespace ngdb_dev {
namespace {

// ---------------------------------------------------------------------------
// Dense contractions: tcgen05 3xTF32 GEMM (tc_gemm.cu). Weights are stored
// [out][in] (y = x W^T), activations [rows][features].

TcGemmArgs mk(int M, int N, int K, const float* A, int lda, const float* B, int ldb, float* C,
              int ldc, int accumulate = 0, const float* bias = nullptr) {
  TcGemmArgs g{};
  g.M = M; g.N = N; g.K = K;
  g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.C = C; g.ldc = ldc;
  g.accumulate = accumulate; g.bias = bias;
  return g;
}

// y (+)= x W^T (+b): x [rows, in], W [out, in]
void linear(int rows, int out, int in, const float* x, const float* W, const float* b, float* y,
            cudaStream_t s, bool relu_x = false, int accumulate = 0) {
  tc_gemm(mk(rows, out, in, x, in, W, in, y, out, accumulate, b), MAJ_K, MAJ_K,
          relu_x ? AOP_RELU : AOP_NONE, s);
}
// dx (+)= dy W: dy [rows, out], W [out, in]
void linear_dx(int rows, int out, int in, const float* dy, const float* W, float* dx,
               cudaStream_t s, int accumulate = 0) {
  tc_gemm(mk(rows, in, out, dy, out, W, in, dx, in, accumulate), MAJ_K, MAJ_MN, AOP_NONE, s);
}
// dW += dy^T x (or dy^T relu(x)): dy [rows, out], x [rows, in]
void linear_dw(int rows, int out, int in, const float* dy, const float* x, float* dW,
               cudaStream_t s, bool relu_x = false) {
  tc_gemm(mk(out, in, rows, dy, out, x, in, dW, in, 1), MAJ_MN, MAJ_MN,
          relu_x ? BOP_RELU : AOP_NONE, s);
}

// db += column sums of dy [rows, n]
__global__ void colsum_kernel(const float* dy, int rows, int n, float* db) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  float s = 0.f;
  for (int r = 0; r < rows; ++r) s += dy[(int64_t)r * n + c];
  db[c] += s;
}
void colsum(const float* dy, int rows, int n, float* db, cudaStream_t s) {
  colsum_kernel<<<(n + 127) / 128, 128, 0, s>>>(dy, rows, n, db);
}

// ---------------------------------------------------------------------------
// GQE helpers

// M[i] = mean_l x_l ; optionally G[i] = grad row
__global__ void gqe_pack_kernel(DevArgs a, int k, int first, int n, float* M, float* G) {
  const int i = blockIdx.x;
  const ngdb_node_desc d = a.nodes[first + i];
  const float inv_k = 1.f / static_cast<float>(k);
  for (int e = threadIdx.x; e < a.dim; e += blockDim.x) {
    float s = 0.f;
    for (int l = 0; l < k; ++l) s += a.arena[d.in[l] + e];
    M[(int64_t)i * a.dim + e] = s * inv_k;
    if (G) G[(int64_t)i * a.dim + e] = a.arena[d.grad + e];
  }
}
// dH = dA * (H > 0), in place on dA
__global__ void relu_mask_kernel(float* dA, const float* H, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && H[i] <= 0.f) dA[i] = 0.f;
}
void relu_mask(float* dA, const float* H, int64_t n, cudaStream_t s) {
  relu_mask_kernel<<<(int)((n + 255) / 256), 256, 0, s>>>(dA, H, n);
}
// G_X row l of node i = dM[i] / k  (mean adjoint)
__global__ void gqe_scatter_kernel(DevArgs a, int k, int first, const float* dM) {
  const int i = blockIdx.x;
  const ngdb_node_desc d = a.nodes[first + i];
  const float inv_k = 1.f / static_cast<float>(k);
  for (int e = threadIdx.x; e < a.dim; e += blockDim.x) {
    const float v = dM[(int64_t)i * a.dim + e] * inv_k;
    for (int l = 0; l < k; ++l) a.arena[d.out + l * a.dim + e] = v;
  }
}

int gqe_intersect(const DevArgs& a, int dir, int k, int first, int n, cudaStream_t s) {
  const int D = a.dim;
  const int64_t nd = (int64_t)n * D;
  float* M = a.scratch;
  float* H = M + nd;
  float* G = H + nd;
  float* dA = G + nd;
  const float* W1 = a.dense + a.dense_off[GQE_W1];
  const float* W2 = a.dense + a.dense_off[GQE_W2];
  gqe_pack_kernel<<<n, 128, 0, s>>>(a, k, first, n, M, dir ? G : nullptr);
  linear(n, D, D, M, W1, nullptr, H, s);
  if (dir == 0) {
    // out rows live in the arena: map C row i -> desc[first+i].out
    TcGemmArgs g = mk(n, D, D, H, D, W2, D, a.arena, D);
    g.c_rowoff = &a.nodes[first].out;
    g.c_stride = sizeof(ngdb_node_desc) / sizeof(int32_t);
    tc_gemm(g, MAJ_K, MAJ_K, AOP_RELU, s);
    return 3;
  }
  float* gW1 = a.dense_g + a.dense_off[GQE_W1];
  float* gW2 = a.dense_g + a.dense_off[GQE_W2];
  linear_dx(n, D, D, G, W2, dA, s);           // dA = G W2
  linear_dw(n, D, D, G, H, gW2, s, true);     // gW2 += G^T relu(H)
  relu_mask(dA, H, nd, s);                    // dH
  linear_dw(n, D, D, dA, M, gW1, s);          // gW1 += dH^T M
  linear_dx(n, D, D, dA, W1, H, s);           // dM = dH W1 (H reused)
  gqe_scatter_kernel<<<n, 128, 0, s>>>(a, k, first, H);
  return 8;
}

// ---------------------------------------------------------------------------
// Q2B helpers (rows are node-major: row = i*k + l)

__global__ void q2b_pack_kernel(DevArgs a, int k, int first, float* Cin, float* Oin) {
  const int i = blockIdx.x;
  const ngdb_node_desc d = a.nodes[first + i];
  for (int l = 0; l < k; ++l)
    for (int e = threadIdx.x; e < a.dim; e += blockDim.x) {
      Cin[((int64_t)i * k + l) * a.dim + e] = a.arena[d.in[l] + e];
      Oin[((int64_t)i * k + l) * a.dim + e] = a.arena[d.in[l] + a.dim + e];
    }
}
// Lm[i] = mean_l relu(P[i*k+l])
__global__ void q2b_mean_relu_kernel(const float* P, int k, int D, float* Lm) {
  const int i = blockIdx.x;
  const float inv_k = 1.f / static_cast<float>(k);
  for (int e = threadIdx.x; e < D; e += blockDim.x) {
    float s = 0.f;
    for (int l = 0; l < k; ++l) s += fmaxf(P[((int64_t)i * k + l) * D + e], 0.f);
    Lm[(int64_t)i * D + e] = s * inv_k;
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
__global__ void q2b_combine_kernel(DevArgs a, int k, int first, const float* S, const float* U,
                                   const float* Cin, const float* Oin) {
  const int i = blockIdx.x;
  const int D = a.dim;
  const ngdb_node_desc d = a.nodes[first + i];
  const int64_t base = (int64_t)i * k * D;
  for (int e = threadIdx.x; e < D; e += blockDim.x) {
    float w[3];
    softmax_k(S, base, k, D, e, w);
    float c = 0.f, mn = Oin[base + e];
    for (int l = 0; l < k; ++l) {
      c += w[l] * Cin[base + (int64_t)l * D + e];
      mn = fminf(mn, Oin[base + (int64_t)l * D + e]);
    }
    a.arena[d.out + e] = c;
    a.arena[d.out + D + e] = mn * sigmoidf(U[(int64_t)i * D + e]);
  }
}
__global__ void q2b_combine_bwd_kernel(DevArgs a, int k, int first, const float* S, const float* U,
                                       const float* Cin, const float* Oin, float* gS, float* dCin,
                                       float* dOin, float* gU) {
  const int i = blockIdx.x;
  const int D = a.dim;
  const ngdb_node_desc d = a.nodes[first + i];
  const int64_t base = (int64_t)i * k * D;
  for (int e = threadIdx.x; e < D; e += blockDim.x) {
    const float gC = a.arena[d.grad + e];
    const float gO = a.arena[d.grad + D + e];
    float w[3];
    softmax_k(S, base, k, D, e, w);
    float ga[3], dot = 0.f;
    for (int l = 0; l < k; ++l) {
      ga[l] = gC * Cin[base + (int64_t)l * D + e];
      dot += w[l] * ga[l];
    }
    int arg = 0;
    float mn = Oin[base + e];
    for (int l = 1; l < k; ++l) {
      const float o = Oin[base + (int64_t)l * D + e];
      if (o < mn) { mn = o; arg = l; }  // ties -> lowest index
    }
    const float gate = sigmoidf(U[(int64_t)i * D + e]);
    for (int l = 0; l < k; ++l) {
      const int64_t r = base + (int64_t)l * D + e;
      gS[r] = w[l] * (ga[l] - dot);
      dCin[r] = gC * w[l];
      dOin[r] = (l == arg) ? gO * gate : 0.f;
    }
    gU[(int64_t)i * D + e] = gO * mn * gate * (1.f - gate);
  }
}
// gP[i*k+l] = gLm[i] / k * (P > 0)
__global__ void q2b_gp_kernel(const float* gLm, const float* P, int k, int D, float* gP) {
  const int i = blockIdx.x;
  const float inv_k = 1.f / static_cast<float>(k);
  for (int e = threadIdx.x; e < D; e += blockDim.x)
    for (int l = 0; l < k; ++l) {
      const int64_t r = ((int64_t)i * k + l) * D + e;
      gP[r] = P[r] > 0.f ? gLm[(int64_t)i * D + e] * inv_k : 0.f;
    }
}
__global__ void q2b_scatter_kernel(DevArgs a, int k, int first, const float* dCin,
                                   const float* dOin) {
  const int i = blockIdx.x;
  const int D = a.dim;
  const ngdb_node_desc d = a.nodes[first + i];
  for (int l = 0; l < k; ++l)
    for (int e = threadIdx.x; e < D; e += blockDim.x) {
      const int64_t r = ((int64_t)i * k + l) * D + e;
      a.arena[d.out + l * 2 * D + e] = dCin[r];
      a.arena[d.out + l * 2 * D + D + e] = dOin[r];
    }
}

int q2b_intersect(const DevArgs& a, int dir, int k, int first, int n, cudaStream_t s) {
  const int D = a.dim;
  const int R = n * k;
  const int64_t rd = (int64_t)R * D, nd = (int64_t)n * D;
  float* Cin = a.scratch;
  float* Oin = Cin + rd;
  float* Z = Oin + rd;
  float* S = Z + rd;
  float* P = S + rd;
  float* Lm = P + rd;
  float* U = Lm + nd;
  const float* p = a.dense;
  const float *A1 = p + a.dense_off[Q2B_A1], *a1 = p + a.dense_off[Q2B_A1B];
  const float *A2 = p + a.dense_off[Q2B_A2], *a2 = p + a.dense_off[Q2B_A2B];
  const float *V1 = p + a.dense_off[Q2B_V1], *v1 = p + a.dense_off[Q2B_V1B];
  const float *V2 = p + a.dense_off[Q2B_V2], *v2 = p + a.dense_off[Q2B_V2B];

  q2b_pack_kernel<<<n, 128, 0, s>>>(a, k, first, Cin, Oin);
  linear(R, D, D, Cin, A1, a1, Z, s);
  linear(R, D, D, Z, A2, a2, S, s, /*relu_x=*/true);
  linear(R, D, D, Oin, V1, v1, P, s);
  q2b_mean_relu_kernel<<<n, 128, 0, s>>>(P, k, D, Lm);
  linear(n, D, D, Lm, V2, v2, U, s);
  if (dir == 0) {
    q2b_combine_kernel<<<n, 128, 0, s>>>(a, k, first, S, U, Cin, Oin);
    return 7;
  }
  float* gS = U + nd;
  float* dCin = gS + rd;
  float* dOin = dCin + rd;
  float* gU = dOin + rd;
  float* gLm = gU + nd;
  float* gP = gLm + nd;
  float* g = a.dense_g;
  const int64_t* off = a.dense_off;
  q2b_combine_bwd_kernel<<<n, 128, 0, s>>>(a, k, first, S, U, Cin, Oin, gS, dCin, dOin, gU);
  // offset branch: gate = sigmoid(V2 Lm + v2), Lm = mean relu(V1 o + v1)
  linear_dw(n, D, D, gU, Lm, g + off[Q2B_V2], s);
  colsum(gU, n, D, g + off[Q2B_V2B], s);
  linear_dx(n, D, D, gU, V2, gLm, s);
  q2b_gp_kernel<<<n, 128, 0, s>>>(gLm, P, k, D, gP);
  linear_dw(R, D, D, gP, Oin, g + off[Q2B_V1], s);
  colsum(gP, R, D, g + off[Q2B_V1B], s);
  linear_dx(R, D, D, gP, V1, dOin, s, /*accumulate=*/1);
  // centre branch: S = A2 relu(Z) + a2, Z = A1 c + a1
  linear_dw(R, D, D, gS, Z, g + off[Q2B_A2], s, /*relu_x=*/true);
  colsum(gS, R, D, g + off[Q2B_A2B], s);
  linear_dx(R, D, D, gS, A2, gP, s);  // gR (gP buffer reused)
  relu_mask(gP, Z, rd, s);            // gZ
  linear_dw(R, D, D, gP, Cin, g + off[Q2B_A1], s);
  colsum(gP, R, D, g + off[Q2B_A1B], s);
  linear_dx(R, D, D, gP, A1, dCin, s, /*accumulate=*/1);
  q2b_scatter_kernel<<<n, 128, 0, s>>>(a, k, first, dCin, dOin);
  return 22;
}

}  // namespace

int launch_intersect(const DevArgs& a, int dir, int k, int first, int n, const LaunchCtx& lc) {
  if (n <= 0) return 0;
  if (a.backbone == NGDB_GQE) return gqe_intersect(a, dir, k, first, n, lc.stream);
  return q2b_intersect(a, dir, k, first, n, lc.stream);
}

}  // namespace ngdb_dev
