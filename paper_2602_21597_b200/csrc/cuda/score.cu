// Fused negative-sample scoring + loss (SPEC.md:541-549 compute_loss, Eq. 6
// PAPER.md:259-263) and the union-branch Score operator.
//
// One CTA per scoring node. Pass 1 streams the 1+K candidate rows (positive
// first) with 128-bit loads, one warp per candidate pair, warp-
// reduces the distances; the loss and dL/dd_j follow in shared memory; pass 2
// re-reads the (now L2-resident) rows column-wise to form dL/dq. Candidate-row
// gradients are NOT materialised: the optimizer recomputes coef_j * dd_j/dv
// from (q, coef) when it reduces each touched row.
//
//   psi_pos = -log sigma(gamma - d_pos) = softplus(d_pos - gamma)
//   psi_neg = -log sigma(d_neg - gamma) = softplus(gamma - d_neg), mean over K
//   GQE distance: ||v - q||_1                                 (SURVEY A-7)
//   Q2B distance: ||max(0,|v-c|-o)||_1 + alpha ||min(|v-c|,o)||_1
#include "common.cuh"

namespace ngdb_dev {
namespace {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxCand = 1024;

template <int BB>
struct Dist;

template <>
struct Dist<NGDB_GQE> {
  // accumulate distance contribution of one float4 chunk
  static __device__ __forceinline__ float part(float4 v, const float* q, int e, int /*dim*/,
                                               float /*alpha*/) {
    const float4 c = *reinterpret_cast<const float4*>(q + e);
    return fabsf(v.x - c.x) + fabsf(v.y - c.y) + fabsf(v.z - c.z) + fabsf(v.w - c.w);
  }
  // dq contribution for one element: coef * dd/dq
  static __device__ __forceinline__ void grad(float v, float c, float /*o*/, float coef,
                                              float /*alpha*/, float& gc, float& /*go*/) {
    gc += coef * sgnf(c - v);
  }
};

template <>
struct Dist<NGDB_Q2B> {
  static __device__ __forceinline__ float term(float v, float c, float o, float alpha) {
    const float a = fabsf(v - c);
    return fmaxf(a - o, 0.f) + alpha * fminf(a, o);
  }
  static __device__ __forceinline__ float part(float4 v, const float* q, int e, int dim,
                                               float alpha) {
    const float4 c = *reinterpret_cast<const float4*>(q + e);
    const float4 o = *reinterpret_cast<const float4*>(q + dim + e);
    return term(v.x, c.x, o.x, alpha) + term(v.y, c.y, o.y, alpha) + term(v.z, c.z, o.z, alpha) +
           term(v.w, c.w, o.w, alpha);
  }
  static __device__ __forceinline__ void grad(float v, float c, float o, float coef, float alpha,
                                              float& gc, float& go) {
    const float delta = v - c;
    const float a = fabsf(delta);
    if (a > o) {
      gc -= coef * sgnf(delta);
      go += coef * (alpha - 1.f);
    } else {
      gc -= coef * alpha * sgnf(delta);
    }
  }
};

__device__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  if (threadIdx.x < 32) {
    t = threadIdx.x < kWarps ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
  }
  return t;  // valid in warp 0
}

// Pass 1: distances of all candidates of query `qi` against q (smem).
template <int BB>
__device__ void distances(const DevArgs& a, const float* q, int qi, float* dist) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int d4 = a.dim / 4;
  const int32_t* cand = a.cand + static_cast<int64_t>(qi) * a.ncand;
  for (int j0 = warp * 2; j0 < a.ncand; j0 += kWarps * 2) {
    const int j1 = j0 + 1;
    const bool two = j1 < a.ncand;
    const float* v0 = a.ent + static_cast<int64_t>(cand[j0]) * a.ent_w;
    const float* v1 = a.ent + static_cast<int64_t>(cand[two ? j1 : j0]) * a.ent_w;
    float s0 = 0.f, s1 = 0.f;
    for (int c = lane; c < d4; c += 32) {
      const float4 x0 = ldg4(v0 + 4 * c);
      const float4 x1 = ldg4(v1 + 4 * c);
      s0 += Dist<BB>::part(x0, q, 4 * c, a.dim, a.alpha_box);
      s1 += Dist<BB>::part(x1, q, 4 * c, a.dim, a.alpha_box);
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    if (lane == 0) {
      dist[j0] = s0;
      if (two) dist[j1] = s1;
    }
  }
}

// Pass 2: dq = sum_j coef_j * dd_j/dq, written to dst (wq floats).
template <int BB>
__device__ void query_grad(const DevArgs& a, const float* q, int qi, const float* coef, float* dst) {
  const int32_t* cand = a.cand + static_cast<int64_t>(qi) * a.ncand;
  for (int e = threadIdx.x; e < a.dim; e += kThreads) {
    const float c = q[e];
    const float o = BB == NGDB_Q2B ? q[a.dim + e] : 0.f;
    float gc = 0.f, go = 0.f;
#pragma unroll 4
    for (int j = 0; j < a.ncand; ++j) {
      const float v = __ldg(a.ent + static_cast<int64_t>(cand[j]) * a.ent_w + e);
      Dist<BB>::grad(v, c, o, coef[j], a.alpha_box, gc, go);
    }
    dst[e] = gc;
    if (BB == NGDB_Q2B) dst[a.dim + e] = go;
  }
}

// Loss coefficients from distances; returns this thread's loss share.
__device__ __forceinline__ float loss_terms(const DevArgs& a, const float* dist, float* coef) {
  float part = 0.f;
  const float inv_k = 1.f / static_cast<float>(a.n_neg);
  for (int j = threadIdx.x; j < a.ncand; j += kThreads) {
    const float dj = dist[j];
    if (j == 0) {
      part += softplusf(dj - a.gamma);
      coef[j] = sigmoidf(dj - a.gamma);
    } else {
      part += inv_k * softplusf(a.gamma - dj);
      coef[j] = -inv_k * sigmoidf(a.gamma - dj);
    }
  }
  return part;
}

template <int BB>
__global__ void __launch_bounds__(kThreads) loss_fwd_kernel(DevArgs a, int first) {
  __shared__ __align__(16) float q[2 * 1024];
  __shared__ float dist[kMaxCand], coef[kMaxCand];
  __shared__ float red[kWarps];
  const ngdb_node_desc d = a.nodes[first + blockIdx.x];
  const int qi = d.id;
  if (d.aux < 0) {
    // union query: the input already holds min-over-branch distances
    for (int j = threadIdx.x; j < a.ncand; j += kThreads) dist[j] = a.arena[d.in[0] + j];
    __syncthreads();
    float loss = block_sum(loss_terms(a, dist, coef), red);
    __syncthreads();
    for (int j = threadIdx.x; j < a.ncand; j += kThreads)
      a.ddbuf[static_cast<int64_t>(qi) * a.ncand + j] = coef[j];
    if (threadIdx.x == 0) {
      a.loss_out[qi] = loss;
      a.arena[d.out] = loss;
      if (!isfinite(loss)) atomicOr(&a.flags[0], 1);
    }
    return;
  }
  const float* src = a.arena + d.in[0];
  float* qcopy = a.qbuf + static_cast<int64_t>(d.aux) * a.wq;
  for (int e = threadIdx.x * 4; e < a.wq; e += kThreads * 4) {
    const float4 v = ld4(src + e);
    st4(q + e, v);
    st4(qcopy + e, v);
  }
  __syncthreads();
  distances<BB>(a, q, qi, dist);
  __syncthreads();
  float loss = block_sum(loss_terms(a, dist, coef), red);
  __syncthreads();
  for (int j = threadIdx.x; j < a.ncand; j += kThreads)
    a.coefbuf[static_cast<int64_t>(d.aux) * a.ncand + j] = coef[j];
  if (threadIdx.x == 0) {
    a.loss_out[qi] = loss;
    a.arena[d.out] = loss;
    if (!isfinite(loss)) atomicOr(&a.flags[0], 1);
  }
  query_grad<BB>(a, q, qi, coef, a.dqbuf + static_cast<int64_t>(d.aux) * a.wq);
}

// Union branch Score: fwd writes the distance vector; bwd turns the routed
// dL/dd into coef (for the optimizer) and dL/dq (its G slot).
template <int BB>
__global__ void __launch_bounds__(kThreads) score_kernel(DevArgs a, int dir, int first) {
  __shared__ __align__(16) float q[2 * 1024];
  __shared__ float buf[kMaxCand];
  const ngdb_node_desc d = a.nodes[first + blockIdx.x];
  const float* src = a.arena + d.in[0];
  for (int e = threadIdx.x * 4; e < a.wq; e += kThreads * 4) {
    const float4 v = ld4(src + e);
    st4(q + e, v);
    if (dir == 0) st4(a.qbuf + static_cast<int64_t>(d.aux) * a.wq + e, v);
  }
  __syncthreads();
  if (dir == 0) {
    distances<BB>(a, q, d.id, buf);
    __syncthreads();
    for (int j = threadIdx.x; j < a.ncand; j += kThreads) a.arena[d.out + j] = buf[j];
    return;
  }
  for (int j = threadIdx.x; j < a.ncand; j += kThreads) {
    const float g = a.arena[d.grad + j];
    buf[j] = g;
    a.coefbuf[static_cast<int64_t>(d.aux) * a.ncand + j] = g;
  }
  __syncthreads();
  query_grad<BB>(a, q, d.id, buf, a.arena + d.out);
}

}  // namespace

int launch_loss_fwd(const DevArgs& a, int first, int n, const LaunchCtx& lc) {
  if (n <= 0) return 0;
  if (a.backbone == NGDB_GQE) loss_fwd_kernel<NGDB_GQE><<<n, kThreads, 0, lc.stream>>>(a, first);
  else loss_fwd_kernel<NGDB_Q2B><<<n, kThreads, 0, lc.stream>>>(a, first);
  return 1;
}

int launch_score(const DevArgs& a, int dir, int first, int n, const LaunchCtx& lc) {
  if (n <= 0) return 0;
  if (a.backbone == NGDB_GQE) score_kernel<NGDB_GQE><<<n, kThreads, 0, lc.stream>>>(a, dir, first);
  else score_kernel<NGDB_Q2B><<<n, kThreads, 0, lc.stream>>>(a, dir, first);
  return 1;
}

}  // namespace ngdb_dev
