// Adam element update shared by the optimizer kernels (optim.cu, beta.cu):
// adam_step, SPEC.md:550-558 (bias-corrected, b1 0.9, b2 0.999, eps 1e-8).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace ngdb_dev {

// Adam constants folded once per thread: with s1 = lr / bc1 and s2 = 1/sqrt(bc2),
//   theta -= s1 * m / (s2 * sqrt(v) + eps)  ==  lr * mhat / (sqrt(vhat) + eps)
// The square root and the reciprocal are the SFU approximations (relative error
// ~2^-22, far inside the 1e-4 parity bound) instead of the IEEE sequences, and
// the elementwise math runs as packed f32x2 operations (FFMA2/FMUL2), which
// roughly quarters the per-element instruction count of the update.
struct AdamK {
  float b1, b2, c1, c2, s1, s2, eps;
};

__device__ __forceinline__ AdamK adam_consts(const AdamHyper& h, const float* bc) {
  return AdamK{h.b1, h.b2, 1.f - h.b1, 1.f - h.b2, h.lr / bc[0], rsqrtf(bc[1]), h.eps};
}

__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// two elements at once: w, m, v, g are (x, y) pairs
__device__ __forceinline__ void adam2(float2& w, float2& m, float2& v, float2 g, const AdamK& k) {
  const float2 b1 = make_float2(k.b1, k.b1), b2 = make_float2(k.b2, k.b2);
  m = __ffma2_rn(b1, m, __fmul2_rn(make_float2(k.c1, k.c1), g));
  v = __ffma2_rn(b2, v, __fmul2_rn(make_float2(k.c2, k.c2), __fmul2_rn(g, g)));
  const float2 den = __ffma2_rn(make_float2(k.s2, k.s2), make_float2(sqrt_approx(v.x), sqrt_approx(v.y)),
                                make_float2(k.eps, k.eps));
  const float2 r = make_float2(rcp_approx(den.x), rcp_approx(den.y));
  w = __ffma2_rn(make_float2(-k.s1, -k.s1), __fmul2_rn(m, r), w);
}

__device__ __forceinline__ void adam_update(float& w, float& m, float& v, float g, const AdamK& k) {
  m = k.b1 * m + k.c1 * g;
  v = k.b2 * v + k.c2 * (g * g);
  w -= k.s1 * m * rcp_approx(k.s2 * sqrt_approx(v) + k.eps);
}

__device__ __forceinline__ float4 adam4(float4 w, float4& m, float4& v, float4 g, const AdamK& k) {
  float2 w0 = make_float2(w.x, w.y), w1 = make_float2(w.z, w.w);
  float2 m0 = make_float2(m.x, m.y), m1 = make_float2(m.z, m.w);
  float2 v0 = make_float2(v.x, v.y), v1 = make_float2(v.z, v.w);
  adam2(w0, m0, v0, make_float2(g.x, g.y), k);
  adam2(w1, m1, v1, make_float2(g.z, g.w), k);
  m = make_float4(m0.x, m0.y, m1.x, m1.y);
  v = make_float4(v0.x, v0.y, v1.x, v1.y);
  return make_float4(w0.x, w0.y, w1.x, w1.y);
}

}  // namespace ngdb_dev
