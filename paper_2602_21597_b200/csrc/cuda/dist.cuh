// Per-dimension distance terms of the scoring kernels and the loss coefficient
// (score.cu fused score+loss, shard.cu owner scoring).
//   GQE   |v - c|                                     (SURVEY A-7)
//   Q2B   max(0, |v-c| - o) + alpha min(|v-c|, o)
//   BetaE A p + B q over the per-step entity table    (beta.cu)
#pragma once

#include "common.cuh"

namespace ngdb_dev {

template <int BB>
struct Dist;

template <>
struct Dist<NGDB_GQE> {
  static __device__ __forceinline__ float term(float v, float c, float, float) {
    return fabsf(v - c);
  }
  // coef * dd/dq
  static __device__ __forceinline__ void grad(float v, float c, float, float coef, float,
                                              float& gc, float&) {
    gc += coef * sgnf(c - v);
  }
};

// BetaE: v = etab row halves (P | Q); "c", "o" = query alpha, beta
template <>
struct Dist<NGDB_BETAE> {
  static __device__ __forceinline__ float term(float p, float q, float A, float B) {
    return A * p + B * q;
  }
};

template <>
struct Dist<NGDB_Q2B> {
  static __device__ __forceinline__ float term(float v, float c, float o, float alpha) {
    const float a = fabsf(v - c);
    return fmaxf(a - o, 0.f) + alpha * fminf(a, o);
  }
  static __device__ __forceinline__ void grad(float v, float c, float o, float coef, float alpha,
                                              float& gc, float& go) {
    const float delta = v - c;
    const float a = fabsf(delta);
    const float s = sgnf(delta);
    if (a > o) {
      gc -= coef * s;
      go += coef * (alpha - 1.f);
    } else {
      gc -= coef * alpha * s;
    }
  }
};

// psi terms of one candidate: returns coef_j = dL/dd_j and
// adds the candidate's loss term to `loss`
__device__ __forceinline__ float loss_coef(const DevArgs& a, int j, float dj, float& loss) {
  const float inv_k = 1.f / static_cast<float>(a.n_neg);
  if (j == 0) {
    loss += softplusf(dj - a.gamma);
    return sigmoidf(dj - a.gamma);
  }
  loss += inv_k * softplusf(a.gamma - dj);
  return -inv_k * sigmoidf(a.gamma - dj);
}

}  // namespace ngdb_dev
