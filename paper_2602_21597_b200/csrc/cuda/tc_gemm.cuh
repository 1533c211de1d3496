// tcgen05 GEMM with 3xTF32 split precision for the operator MLPs.
//
//   C[M,N] (+)= A[M,K] * B[N,K]^T (+ bias[n])      fp32 in, fp32 out
//
// Each fp32 operand x is split into hi = tf32_rn(x) and lo = x - hi; the tensor
// core accumulates hi*hi + hi*lo + lo*hi in fp32 TMEM accumulators, which keeps
// the contraction within ~1e-6 relative of fp32 — the 1e-4 parity bar cannot be
// met by single-pass TF32 at K = 400..1536.
//
// Tile: BM = 128 rows (UMMA M=128, cta_group::1), BN = 80 columns (one UMMA
// N=80; d = 400 is exactly 5 tiles), BK = 32 (one 128-byte swizzle atom of fp32).
// 128 threads: all of them stream A/B K-chunks global -> shared with cp.async
// into a 4-deep raw ring, split them into hi/lo operand tiles laid out K-major
// with the 128B swizzle, and one elected thread issues 4 k-steps x 3 UMMAs per
// chunk; tcgen05.commit on an mbarrier releases the operand stage. The epilogue
// reads the accumulator with tcgen05.ld (thread t owns row t) and applies bias /
// accumulate / row scatter.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ngdb_dev {

enum : int { MAJ_K = 0, MAJ_MN = 1 };  // operand storage: K contiguous or M/N contiguous
enum : int { AOP_NONE = 0, AOP_RELU = 1, BOP_RELU = 2 };  // operand-op bit mask

struct TcGemmArgs {
  int M, N, K;
  const float* A; int lda;   // MAJ_K: A(m,k) = A[m*lda+k]; MAJ_MN: A[k*lda+m]
  const float* B; int ldb;   // MAJ_K: B(n,k) = B[n*ldb+k]; MAJ_MN: B[k*ldb+n]
  float* C; int ldc;
  const int32_t* c_rowoff; int c_stride;  // optional row scatter: C + c_rowoff[m*stride]
  const float* bias;
  int accumulate;
};

// Launch C = A * B^T with the given operand majorness and operand ops (ReLU on
// A and/or B applied while splitting); returns the kernel count (1).
int tc_gemm(const TcGemmArgs& g, int a_major, int b_major, int ops, cudaStream_t s);

}  // namespace ngdb_dev
