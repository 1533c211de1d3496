// tcgen05 GEMM with 3xTF32 split precision for the operator MLPs.
//
//   C[M,N] (+)= A[M,K] * B[N,K]^T (+ bias[n])      fp32 in, fp32 out
//
// Operands arrive PRE-SPLIT: x = hi + lo with hi = tf32_rn(x), lo = x - hi, both
// stored row-major K-contiguous ("K-major"). Weights are split once per
// optimizer step (refresh_weight_splits); activations are split by
// split_matrix (optionally transposed / ReLU'd) or directly by the epilogue of
// the GEMM that produced them. The tensor core accumulates hi*hi + hi*lo + lo*hi
// per BK=32 chunk in a fresh TMEM buffer; chunk partials are summed in fp32
// registers (the accumulator's exponent alignment loses ~5x fp32 precision over
// a full K=400 run; per chunk it does not matter).
//
// Tile: BM = 128 rows (UMMA M=128, cta_group::1), BN = 80 (one UMMA N=80; d=400
// is exactly five tiles), BK = 32 (one 128-byte swizzle atom of fp32). 256
// threads stream hi/lo tiles global -> shared with cp.async straight into the
// 128B-swizzled K-major layout the UMMA descriptors describe (3-stage ring);
// one thread issues 4 k-steps x 3 UMMAs per chunk and commits to the stage's
// mbarrier; two TMEM accumulator buffers alternate between chunks.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ngdb_dev {

struct SplitOperand {
  const float* hi;
  const float* lo;
  int ld;  // row stride (elements); rows are K-contiguous
  // 1: MN-major — stored [K][rows] (element (row, k) at k*ld + row), e.g. dY
  // of a weight gradient dW = dY^T X read in place as [rows][features]; the
  // TMA mainloop loads it in 32-row blocks and the UMMA reads it through an
  // MN-major descriptor (no transposed copy). Needs the TMA path (ld % 4 == 0,
  // 16-byte aligned hi/lo).
  int mn;
};

struct TcGemmArgs {
  int M, N, K;
  SplitOperand A;  // [M][K]
  SplitOperand B;  // [N][K]
  float* C; int ldc;
  const int32_t* c_rowoff; int c_stride;  // optional row scatter: C + c_rowoff[m*stride]
  const float* bias;
  int accumulate;
  // optional ReLU-derivative mask: result *= (mask[m*ldc + n] > 0)
  const float* mask;
  // optional chained output: split(relu?(C)) -> s_hi/s_lo [M][ldc] (no scatter)
  float* s_hi; float* s_lo; int s_relu;
  // optional activation after bias / accumulate: C = sigmoid(C) (FuseSemantic's E)
  int sigmoid;
};

int tc_gemm(const TcGemmArgs& g, cudaStream_t s);
// Process-wide split-K override: 0 = per launch (default), 1..8 = fixed.
void set_gemm_split_override(int s);
// Up to four independent problems in one launch (one dependency level).
int tc_gemm_batch(const TcGemmArgs* probs, int n, cudaStream_t s);

// dst_hi/dst_lo[r][c] = split(op(src[r][c])) (transpose=0, dense [rows][cols]) or
// dst[c][r] = split(op(src[r][c])) (transpose=1, [cols][pad4(rows)], zero padded
// so every row is 16-byte aligned for cp.async); op = relu if relu != 0.
int split_matrix(const float* src, int rows, int cols, int ld_src, int transpose, int relu,
                 float* dst_hi, float* dst_lo, cudaStream_t s);

// Up to four transposed splits in ONE launch (the weight-gradient operands of
// a backward class: dY^T and X^T for each dW += dY^T X).
struct SplitJob {
  const float* src;
  int rows, cols, ld, relu;
  float* hi;
  float* lo;
  // optional computed source (the mean-adjoint of a DeepSets layer):
  // v[r][c] = mask[r][c] > 0 ? node_grad[node(r)][c] / k(node) : 0, with the
  // node layout of a two-class (n1 nodes of k1 rows, then k2) Intersect
  // invocation; v is also written plain (plain) and split row-major (rhi/rlo)
  const float* node_grad;
  const float* mask;
  int n1, k1, k2;
  float* plain;
  float* rhi;
  float* rlo;
  // (hi == nullptr: no transposed output — the computed source is written
  // plain and split row-major only, for MN-major weight-gradient operands)
};
struct SplitJobs {
  SplitJob job[4];
  int n;
};
int split_transposed(const SplitJobs& jobs, cudaStream_t s);

}  // namespace ngdb_dev
