// Helpers shared by the MLP operators (intersect.cu, beta.cu): scratch bump
// allocation, 3xTF32 split operands and GEMM argument builders.
#pragma once

#include "common.cuh"
#include "tc_gemm.cuh"

namespace ngdb_dev {

// bump allocator over the context scratch buffer
struct Scratch {
  float* p;
  int64_t left;
  float* take(int64_t n) {
    n = (n + 3) / 4 * 4;
    float* r = p;
    p += n;
    left -= n;
    return left >= 0 ? r : nullptr;
  }
};

struct Split {
  float* hi;
  float* lo;
};
inline Split take_split(Scratch& s, int64_t n) { return {s.take(n), s.take(n)}; }

// BetaE with FuseSemantic (beta.cu): dL/dY of the touched rows (plain + split)
int launch_beta_fuse_grad(const DevArgs& a, const SparseTable& t, float* gY, Split gYs,
                          const LaunchCtx& lc);

inline SplitOperand op(Split x, int ld) { return {x.hi, x.lo, ld, 0}; }
// a row-major [rows][ld] split read MN-major: the transposed operand of a
// weight gradient (dW += dY^T X, K = rows) without a transposed copy
inline SplitOperand mop(Split x, int ld) { return {x.hi, x.lo, ld, 1}; }

// Grid of the per-node elementwise kernels: blockIdx.x = node, blockIdx.y
// strides the row elements (128 threads each), so every thread handles ~one
// element of a 2d-wide row and all of a node's loads are in flight at once.
inline dim3 node_grid(int n, int dim) { return dim3(n, (2 * dim + 127) / 128); }
// weight W_i [out][in] as B of y = x W^T (K = in), or its transpose as B of dx = dy W (K = out)
inline SplitOperand wop(const DevArgs& a, int i, int rows, int cols, bool transposed) {
  const int64_t n = (int64_t)rows * cols;
  const float* base = a.wsplit + a.wsplit_off[i];
  return transposed ? SplitOperand{base + 2 * n, base + 3 * n, rows, 0}
                    : SplitOperand{base, base + n, cols, 0};
}

inline TcGemmArgs gemm_args(int M, int N, int K, SplitOperand A, SplitOperand B, float* C, int ldc) {
  TcGemmArgs g{};
  g.M = M; g.N = N; g.K = K;
  g.A = A; g.B = B; g.C = C; g.ldc = ldc;
  return g;
}

__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
  lo = x - hi;
}
__device__ __forceinline__ void put(float* plain, Split s, int64_t i, float v) {
  if (plain) plain[i] = v;
  float h, l;
  split_tf32(v, h, l);
  s.hi[i] = h;
  s.lo[i] = l;
}

// bias gradients: db_j += column sums of dy_j [rows][n], up to four per launch
struct ColsumJob {
  const float* dy;
  int rows, n;
  float* db;
};
struct ColsumJobs {
  ColsumJob job[4];
  int n;
};
int colsums(const ColsumJobs& jobs, int n, cudaStream_t s);

}  // namespace ngdb_dev
