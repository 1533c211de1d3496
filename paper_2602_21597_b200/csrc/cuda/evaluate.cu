// Evaluator hot path: full-entity scoring + filtered rank (SPEC.md:602-646,
// module `evaluator`).
//
//   filtered_rank(scores, target, filter) =
//       1 + |{e not in filter+{target} : score(e) > score(target)}| + floor(ties / 2)
//   (mean-rank tie rule), score = -distance.
//
// Three launches per batch of queries, all on the context stream:
//   1. eval_target_kernel: d_t = dist(target, q) for every query (one thread per
//      query, sequential over the d dimensions);
//   2. eval_count_kernel:  every (entity, query) distance, tiled 64 entities x 32
//      queries per CTA with 32-dimension slices of both staged in shared memory
//      (each entity value is reused by 8 queries per thread, each query slice by
//      64 entities); counts d < d_t and d == d_t over all non-target entities,
//      warp-reduced, one integer atomic per (warp, query);
//   3. eval_filter_kernel: the filtered entities' contributions are removed again
//      (one thread per (query, filter entry)).
// Every distance is accumulated in the same order (dimension 0..d-1, one fp32
// rounding per step, __fadd_rn so nothing is contracted into an FMA), so the
// distance of an entity is bit-identical in all three kernels: comparisons
// against d_t — including exact ties — are consistent, and the counts are
// integers (deterministic regardless of atomic order).
//
// BetaE (KL): KL(entity || query) = lnB(q) + C_e + <q, T_e> with
// the entity side T_e = [psi(s)-psi(a) | psi(s)-psi(b)], C_e evaluated once per
// entity by the training step's own prologue kernel (beta_prep) over the whole
// table: the all-pairs pass is a 2d-long dot product per (entity, query),
// summed in dimension order with __fmul_rn / __fadd_rn, then + C_e. lnB(q) is
// the same for every entity of a query, so it is left out of the compared
// value (ranks are unchanged; the comparison needs one rounding less). The fusion backbone ranks
// against the fused table sigma(W_p [h | F s] + b_p) of every entity (the
// step's FuseSemantic prologue over all rows) with the GQE distance.
#include <cuda_runtime.h>

#include "common.cuh"

namespace ngdb_dev {

namespace {

constexpr int TE = 64;   // entities per CTA
constexpr int TQ = 32;   // queries per CTA
constexpr int KS = 32;   // dimensions per shared-memory slice
constexpr int QPT = 8;   // queries per thread (256 threads = 64 entities x 4 query groups)
constexpr int ES = KS + 4;  // padded entity row: float4-aligned, conflict-free LDS.128

// one dimension of the distance, accumulated in dimension order
template <int BB>
__device__ __forceinline__ void acc_dim(float& out, float& in, float v, float c, float o) {
  if constexpr (BB == NGDB_BETAE) {  // v = T_e[k], c = q[k]
    out = __fadd_rn(out, __fmul_rn(c, v));
    return;
  }
  const float t = fabsf(__fsub_rn(v, c));
  if constexpr (BB == NGDB_GQE) {
    out = __fadd_rn(out, t);
  } else {
    out = __fadd_rn(out, fmaxf(__fsub_rn(t, o), 0.f));
    in = __fadd_rn(in, fminf(t, o));
  }
}
// ce = C_e of the BetaE distance (0 otherwise)
template <int BB>
__device__ __forceinline__ float finish(float out, float in, float alpha, float ce) {
  if constexpr (BB == NGDB_BETAE) return __fadd_rn(out, ce);
  return BB == NGDB_GQE ? out : __fadd_rn(out, __fmul_rn(alpha, in));
}
template <int BB>
__device__ __forceinline__ float ent_const(const EvalArgs& a, int e) {
  if constexpr (BB == NGDB_BETAE) return a.ec[e];
  return 0.f;
}

// one (entity, query) distance by one thread: float4 loads, the additions still
// in dimension order (d is a multiple of 4, rows are 16-byte aligned)
template <int BB>
__device__ float row_distance(const EvalArgs& a, int e, int q) {
  const float* v = a.ent + static_cast<int64_t>(e) * a.ent_w;
  const float* qc = a.q + static_cast<int64_t>(q) * a.wq;
  float out = 0.f, in = 0.f;
#pragma unroll 4
  for (int k = 0; k < a.dim; k += 4) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(v + k));
    const float4 c = __ldg(reinterpret_cast<const float4*>(qc + k));
    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (BB == NGDB_Q2B) o = __ldg(reinterpret_cast<const float4*>(qc + a.dim + k));
    acc_dim<BB>(out, in, x.x, c.x, o.x);
    acc_dim<BB>(out, in, x.y, c.y, o.y);
    acc_dim<BB>(out, in, x.z, c.z, o.z);
    acc_dim<BB>(out, in, x.w, c.w, o.w);
  }
  return finish<BB>(out, in, a.alpha, ent_const<BB>(a, e));
}

// distance of entity e to query qi: the nearest of its branch slots (UnionScore
// takes the max score); one branch for every other pattern
template <int BB>
__device__ float query_distance(const EvalArgs& a, int e, int qi) {
  const int s0 = a.first_slot[qi], nb = a.slot_nb[s0];
  float d = row_distance<BB>(a, e, s0);
  for (int b = 1; b < nb; ++b) d = fminf(d, row_distance<BB>(a, e, s0 + b));
  return d;
}

template <int BB>
__global__ void eval_target_kernel(EvalArgs a) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= a.n_queries) return;
  a.dt[q] = query_distance<BB>(a, a.target[q], q);
  a.better[q] = 0;
  a.ties[q] = 0;
}

template <int BB>
__global__ void __launch_bounds__(256) eval_count_kernel(EvalArgs a) {
  __shared__ __align__(16) float es[TE][ES];
  __shared__ __align__(16) float qcs[TQ][KS];
  __shared__ __align__(16) float qos[BB == NGDB_Q2B ? TQ : 1][KS];
  const int e0 = blockIdx.x * TE, q0 = blockIdx.y * TQ;
  const int tid = threadIdx.x;
  const int el = tid & (TE - 1), qg = tid / TE;  // a warp shares its query group
  float out[QPT], in[QPT];
#pragma unroll
  for (int j = 0; j < QPT; ++j) out[j] = in[j] = 0.f;
  for (int k0 = 0; k0 < a.dim; k0 += KS) {
    // stage the slice: 64 entity rows x 32 dims, 32 queries x 32 dims, as float4
    // pieces (d is a multiple of 4: a piece is wholly inside or zero padding)
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = tid; i < TE * KS / 4; i += 256) {
      const int r = i / (KS / 4), k = 4 * (i % (KS / 4)), e = e0 + r;
      *reinterpret_cast<float4*>(&es[r][k]) =
          (e < a.n_ent && k0 + k < a.dim)
              ? __ldg(reinterpret_cast<const float4*>(a.ent + static_cast<int64_t>(e) * a.ent_w + k0 + k))
              : z4;
    }
    for (int i = tid; i < TQ * KS / 4; i += 256) {
      const int r = i / (KS / 4), k = 4 * (i % (KS / 4)), q = q0 + r;
      const bool ok = q < a.nq && k0 + k < a.dim;
      const float* qr = a.q + static_cast<int64_t>(q) * a.wq + k0 + k;
      *reinterpret_cast<float4*>(&qcs[r][k]) = ok ? __ldg(reinterpret_cast<const float4*>(qr)) : z4;
      if constexpr (BB == NGDB_Q2B)
        *reinterpret_cast<float4*>(&qos[r][k]) =
            ok ? __ldg(reinterpret_cast<const float4*>(qr + a.dim)) : z4;
    }
    __syncthreads();
#pragma unroll 2
    for (int k = 0; k < KS; k += 4) {
      const float4 v = *reinterpret_cast<const float4*>(&es[el][k]);
#pragma unroll
      for (int j = 0; j < QPT; ++j) {
        const int ql = qg * QPT + j;
        const float4 c = *reinterpret_cast<const float4*>(&qcs[ql][k]);
        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
        if constexpr (BB == NGDB_Q2B) o = *reinterpret_cast<const float4*>(&qos[ql][k]);
        acc_dim<BB>(out[j], in[j], v.x, c.x, o.x);
        acc_dim<BB>(out[j], in[j], v.y, c.y, o.y);
        acc_dim<BB>(out[j], in[j], v.z, c.z, o.z);
        acc_dim<BB>(out[j], in[j], v.w, c.w, o.w);
      }
    }
    __syncthreads();
  }
  const int e = e0 + el;
  // the host packs a query's branch slots inside one 8-slot group, so the
  // nearest-branch distance is a min over this thread's own registers
  float d[QPT];
  const float ce = e < a.n_ent ? ent_const<BB>(a, e) : 0.f;
#pragma unroll
  for (int j = 0; j < QPT; ++j) d[j] = finish<BB>(out[j], in[j], a.alpha, ce);
#pragma unroll
  for (int j = 0; j < QPT; ++j) {
    const int slot = q0 + qg * QPT + j;
    const int nbr = slot < a.nq ? a.slot_nb[slot] : 0;  // > 0: first slot of a query
    const int qi = nbr > 0 ? a.slot_query[slot] : -1;
    float dm = d[j];  // min over the query's nbr (1..QPT) consecutive branch slots
#pragma unroll
    for (int b = 1; b < QPT; ++b)
      if (b < nbr && j + b < QPT) dm = fminf(dm, d[j + b < QPT ? j + b : j]);
    bool b = false, t = false;
    if (qi >= 0 && e < a.n_ent && e != a.target[qi]) {
      const float d_t = a.dt[qi];
      b = dm < d_t;
      t = dm == d_t;
    }
    const unsigned nb = __popc(__ballot_sync(0xffffffffu, b));
    const unsigned nt = __popc(__ballot_sync(0xffffffffu, t));
    if ((tid & 31) == 0 && qi >= 0) {
      if (nb) atomicAdd(&a.better[qi], static_cast<int32_t>(nb));
      if (nt) atomicAdd(&a.ties[qi], static_cast<int32_t>(nt));
    }
  }
}

// one thread per (query, filter entry): remove the filtered entities again
template <int BB>
__global__ void eval_filter_kernel(EvalArgs a, int32_t n_filter) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_filter) return;
  int lo = 0, hi = a.n_queries;  // query of entry i: last q with f_off[q] <= i
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (a.f_off[mid] <= i) lo = mid;
    else hi = mid;
  }
  const int q = lo, e = a.f_ids[i];
  if (e == a.target[q]) return;  // excluded by the host (TargetFiltered)
  const float d = query_distance<BB>(a, e, q), d_t = a.dt[q];
  if (d < d_t) atomicSub(&a.better[q], 1);
  else if (d == d_t) atomicSub(&a.ties[q], 1);
}

template <int BB>
void launch_eval(const EvalArgs& a, int32_t n_filter, cudaStream_t s) {
  eval_target_kernel<BB><<<(a.n_queries + 127) / 128, 128, 0, s>>>(a);
  const dim3 grid((a.n_ent + TE - 1) / TE, (a.nq + TQ - 1) / TQ);
  eval_count_kernel<BB><<<grid, 256, 0, s>>>(a);
  if (n_filter > 0) eval_filter_kernel<BB><<<(n_filter + 127) / 128, 128, 0, s>>>(a, n_filter);
}

}  // namespace

// 3 launches; the caller validated shapes and indices
int launch_eval_ranks(const EvalArgs& a, int32_t n_filter, cudaStream_t s) {
  if (a.n_queries <= 0) return 0;
  if (a.backbone == NGDB_GQE) launch_eval<NGDB_GQE>(a, n_filter, s);
  else if (a.backbone == NGDB_Q2B) launch_eval<NGDB_Q2B>(a, n_filter, s);
  else launch_eval<NGDB_BETAE>(a, n_filter, s);
  return n_filter > 0 ? 3 : 2;
}

}  // namespace ngdb_dev
