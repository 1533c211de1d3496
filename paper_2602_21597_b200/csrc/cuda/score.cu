// Fused negative-sample scoring + loss (SPEC.md:541-549 compute_loss, Eq. 6
// PAPER.md:259-263) and the union-branch Score operator (fwd / bwd).
//
// One persistent, streaming kernel serves all three. Work items are (scoring
// node, part): the S parts of a node split its 1+K candidates into contiguous
// ranges, S chosen so that every resident CTA has items. A CTA walks items
// blockIdx.x, +gridDim.x, ...; its producer warp streams each item's query
// row (double-buffered) and candidate rows (a ring of ~32 KB) into shared
// memory with bulk copies (cp.async.bulk + mbarrier complete_tx), running
// ahead across items so HBM never idles through per-item reductions. Eight
// consumer warps take rows round-robin, read them with 128-bit shared loads,
// reduce the distance with shuffles and — because the loss is a sum of
// per-candidate terms, so dL/dd_j depends on d_j alone — fold coef_j *
// dd_j/dq into per-lane registers in the same pass. Every candidate row is read
// exactly once, and candidate-row gradients are never materialised: the
// optimizer recomputes coef_j * dd_j/dv from (q, coef) while it updates each
// touched row. Parts of a node combine their dL/dq partials
// in part order in the last CTA to finish the node (global partials + an
// arrival counter: deterministic).
//
// Rows and queries sit in shared memory with each d-wide half padded to
// 128*NCH floats and the padding zero: every lane processes exactly NCH
// float4 chunks per half with no bounds tests, and padded lanes contribute 0
// to distances and gradients (q = 0, v = 0).
//
//   psi_pos = -log sigma(gamma - d_pos) = softplus(d_pos - gamma)
//   psi_neg = -log sigma(d_neg - gamma) = softplus(gamma - d_neg), mean over K
//   GQE distance: ||v - q||_1                                     (SURVEY A-7)
//   Q2B distance: ||max(0,|v-c|-o)||_1 + alpha ||min(|v-c|,o)||_1
//   BetaE:        sum_dims KL(entity || query) = lnB(q) + etab_c[r] + <q, etab[r]>
//                 over the per-step entity table of beta.cu;
//                 dL/dq = sum_j coef_j etab[r_j] + (sum_j coef_j) [psi(A)-psi(A+B) | psi(B)-psi(A+B)]
#include <algorithm>
#include <map>

#include "common.cuh"
#include "dist.cuh"
#include "special.cuh"

namespace ngdb_dev {
namespace {

constexpr int kCWarps = 8;                        // consumer warps
constexpr int kThreads = 32 * (kCWarps + 1);      // + one producer warp
constexpr int kConsumerThreads = 32 * kCWarps;

enum Mode : int { kLoss = 0, kScoreFwd = 1, kScoreBwd = 2 };

__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumerThreads) : "memory");
}

// Shared-memory layout (dynamic): ring of `depth` padded rows, two padded query
// slots, the consumer warps' dL/dq partial rows, then the mbarriers. A padded row has `halves` halves of HP floats; a
// padded query always has two (GQE uses the first).
template <int NCH>
struct Layout {
  static constexpr int HP = 128 * NCH;  // floats per padded half
  int halves, depth;
  // depth is a multiple of kCWarps: slot s is then always consumed by warp
  // s % kCWarps, in order, so no consumer ever waits on a slot two phases
  // ahead of its last completion (mbarrier parity waits see one phase back)
  __host__ __device__ explicit Layout(int backbone) {
    halves = backbone == NGDB_BETAE ? 2 : 1;
    const int d = 32768 / (halves * HP * 4) / kCWarps * kCWarps;
    depth = d < kCWarps ? kCWarps : (d > 32 ? 32 : d);
  }
  __host__ __device__ int row_floats() const { return halves * HP; }
  // ring rows, two query slots, kCWarps partial rows of dL/dq (two halves)
  __host__ __device__ size_t floats() const {
    return static_cast<size_t>(depth) * row_floats() + 2 * 2 * HP + kCWarps * 2 * HP;
  }
  __host__ __device__ size_t bytes() const {
    return floats() * sizeof(float) + (2 * depth + 4) * sizeof(uint64_t);
  }
};

__device__ __forceinline__ float4 f4(float x) { return make_float4(x, x, x, x); }
__device__ __forceinline__ void acc4(float4& a, float4 b) {
  a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
}

// m * sign(t) with sign(0) = 0 (the subgradient the oracle takes at a kink):
// one sign-bit XOR and a select
__device__ __forceinline__ float mul_sign(float m, float t) {
  const float s = __int_as_float(__float_as_int(m) ^ (__float_as_int(t) & 0x80000000));
  return t != 0.f ? s : 0.f;
}

// -(m * sign(t)) with sign(0) = 0: the sign bit of t, inverted, onto m (one LOP3)
__device__ __forceinline__ float neg_sign(float m, float t) {
  const float s = __int_as_float(__float_as_int(m) ^ (~__float_as_int(t) & 0x80000000));
  return t != 0.f ? s : 0.f;
}

// a += (x, y, z, w) as two packed FADD2
__device__ __forceinline__ void add2(float4& a, float x, float y, float z, float w) {
  const float2 lo = __fadd2_rn(make_float2(a.x, a.y), make_float2(x, y));
  const float2 hi = __fadd2_rn(make_float2(a.z, a.w), make_float2(z, w));
  a = make_float4(lo.x, lo.y, hi.x, hi.y);
}

// Per-backbone distance of one padded row against the lane's query slice and
// its gradient contribution coef * dd/dq.
// The query slice is NOT held in registers: it is re-read from the shared
// query buffer for every row (LDS.128; the mbarrier waits clobber memory), which
// keeps the consumers at <= 72 registers -> 3 CTAs (24 consumer warps) per SM.
template <int BB, int NCH>
struct RowMath {
  const float* qs;          // padded query in shared memory (two halves)
  int lane;
  float4 gc[NCH], go[NCH];  // dL/dq accumulators
  float4 t[NCH], t2[NCH];   // per-row values kept between distance and gradient

  __device__ float4 qc(int i) const { return ld4(qs + 4 * (lane + 32 * i)); }
  __device__ float4 qo(int i) const { return ld4(qs + Layout<NCH>::HP + 4 * (lane + 32 * i)); }

  __device__ void load_q(const float* q, int l) {
    qs = q;
    lane = l;
#pragma unroll
    for (int i = 0; i < NCH; ++i) gc[i] = go[i] = f4(0.f);
  }
  // the lane's part of d_j (warp-summed by the caller)
  __device__ float distance(const float* row, int /*lane*/, float alpha) {
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      const float4 v = ld4(row + 4 * (lane + 32 * i));
      const float4 c = qc(i);
      if constexpr (BB == NGDB_BETAE) {
        const float4 v2 = ld4(row + Layout<NCH>::HP + 4 * (lane + 32 * i));
        const float4 o = qo(i);
        t[i] = v;
        t2[i] = v2;
        s0 += c.x * v.x + o.x * v2.x;
        s1 += c.y * v.y + o.y * v2.y;
        s2 += c.z * v.z + o.z * v2.z;
        s3 += c.w * v.w + o.w * v2.w;
      } else {
        // t = v - c as two packed FFMA2 (v + (-1) c: exact product, one rounding)
        const float2 m1 = make_float2(-1.f, -1.f);
        const float2 t01 = __ffma2_rn(make_float2(c.x, c.y), m1, make_float2(v.x, v.y));
        const float2 t23 = __ffma2_rn(make_float2(c.z, c.w), m1, make_float2(v.z, v.w));
        t[i] = make_float4(t01.x, t01.y, t23.x, t23.y);
        if constexpr (BB == NGDB_GQE) {
          s0 += fabsf(t[i].x); s1 += fabsf(t[i].y); s2 += fabsf(t[i].z); s3 += fabsf(t[i].w);
        } else {  // outside part max(|t|-o, 0) in (s0, s1), inside part min(|t|, o) in (s2, s3)
          const float4 o = qo(i);
          float2 so = make_float2(s0, s1), si = make_float2(s2, s3);
          so = __fadd2_rn(so, make_float2(fmaxf(fabsf(t[i].x) - o.x, 0.f), fmaxf(fabsf(t[i].y) - o.y, 0.f)));
          so = __fadd2_rn(so, make_float2(fmaxf(fabsf(t[i].z) - o.z, 0.f), fmaxf(fabsf(t[i].w) - o.w, 0.f)));
          si = __fadd2_rn(si, make_float2(fminf(fabsf(t[i].x), o.x), fminf(fabsf(t[i].y), o.y)));
          si = __fadd2_rn(si, make_float2(fminf(fabsf(t[i].z), o.z), fminf(fabsf(t[i].w), o.w)));
          s0 = so.x; s1 = so.y; s2 = si.x; s3 = si.y;
        }
      }
    }
    if constexpr (BB == NGDB_Q2B) return (s0 + s1) + alpha * (s2 + s3);
    return (s0 + s1) + (s2 + s3);
  }
  __device__ void grad(float coef, float alpha) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      if constexpr (BB == NGDB_BETAE) {
        gc[i].x += coef * t[i].x; go[i].x += coef * t2[i].x;
        gc[i].y += coef * t[i].y; go[i].y += coef * t2[i].y;
        gc[i].z += coef * t[i].z; go[i].z += coef * t2[i].z;
        gc[i].w += coef * t[i].w; go[i].w += coef * t2[i].w;
      } else if constexpr (BB == NGDB_GQE) {  // d|v-c|/dc = -sign(v-c)
        add2(gc[i], neg_sign(coef, t[i].x), neg_sign(coef, t[i].y), neg_sign(coef, t[i].z),
             neg_sign(coef, t[i].w));
      } else {  // outside the box: dc = -sign, do = alpha - 1; inside: dc = -alpha sign
        const float ca = coef * alpha, co = coef * (alpha - 1.f);
        const float4 o = qo(i);
        const bool ox = fabsf(t[i].x) > o.x, oy = fabsf(t[i].y) > o.y;
        const bool oz = fabsf(t[i].z) > o.z, ow = fabsf(t[i].w) > o.w;
        add2(gc[i], neg_sign(ox ? coef : ca, t[i].x), neg_sign(oy ? coef : ca, t[i].y),
             neg_sign(oz ? coef : ca, t[i].z), neg_sign(ow ? coef : ca, t[i].w));
        add2(go[i], ox ? co : 0.f, oy ? co : 0.f, oz ? co : 0.f, ow ? co : 0.f);
      }
    }
  }
};

// BetaE query-side part of dKL/dq (per unit coefficient): psi(A) - psi(A+B) for
// the alpha half, psi(B) - psi(A+B) for the beta half
__device__ __forceinline__ float beta_qterm(const DevArgs& a, const float* q, int e) {
  const int D = a.dim;
  const int i = e < D ? e : e - D;
  const float A = q[i], B = q[D + i];
  return dg_digamma(e < D ? A : B) - dg_digamma(A + B);
}

// 3 CTAs per SM (<= 72 registers) where that costs no spills; the BetaE
// (linearised KL: query-side digamma terms) and d > 512 variants need more
// registers and run 2 CTAs per SM spill-free
template <int BB, int NCH, int MODE>
__global__ void __launch_bounds__(kThreads, (BB == NGDB_BETAE || NCH > 4) ? 2 : 3)
    stream_kernel(DevArgs a, int first, int n, int S) {
  extern __shared__ __align__(128) float smem[];
  __shared__ float lred[2 * kCWarps];
  __shared__ int last_flag;
  __shared__ float bcast;
  constexpr bool kBeta = BB == NGDB_BETAE;
  constexpr int HP = Layout<NCH>::HP;
  const Layout<NCH> L(BB);
  const int RW = L.row_floats();
  float* rows = smem;
  float* qbuf0 = smem + static_cast<size_t>(L.depth) * RW;
  float* qbuf1 = qbuf0 + 2 * HP;
  float* parts_base = qbuf1 + 2 * HP;  // [kCWarps][2 * HP]
  auto parts = [&](int w) { return parts_base + static_cast<size_t>(w) * 2 * HP; };
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.floats());
  uint64_t* empty = full + L.depth;
  uint64_t* qfull = empty + L.depth;
  uint64_t* qempty = qfull + 2;
  // zero the padding once (bulk copies never write it), then the barriers
  for (size_t e = threadIdx.x * 4; e < L.floats(); e += kThreads * 4) st4(smem + e, f4(0.f));
  if (threadIdx.x == 0) {
    for (int i = 0; i < L.depth; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&qfull[i], 1);
      mbar_init(&qempty[i], 1);
    }
    mbar_fence_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zeros before bulk writes
  __syncthreads();
  pdl_start();

  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int n_items = S * n;
  const bool rows_local = kBeta || a.fused;  // candidate rows from the step table
  const float* rows_base = rows_local ? a.etab : a.ent;
  const int D = a.dim;

  if (warp == kCWarps) {  // ---- producer warp ----
    // the warp stages the candidate indices of 32 rows at a time in shared
    // memory (one coalesced load instead of a serial chain of round trips);
    // lane 0 issues the copies
    __shared__ int32_t idx_s[32];
    const uint32_t half_bytes = static_cast<uint32_t>(D * sizeof(float));
    const int q_halves = a.wq / D;
    int pos = 0, qi = 0;
    for (int t = blockIdx.x; t < n_items; t += gridDim.x) {
      const int node = t / S, part = t % S;
      const ngdb_node_desc d = a.nodes[first + node];
      if (MODE == kLoss && d.aux < 0) continue;  // union query: no candidate rows
      if (lane == 0) {
        const int qs = qi & 1;
        if (qi >= 2) mbar_wait_parity(&qempty[qs], ((qi >> 1) - 1) & 1);
        float* qdst = qs ? qbuf1 : qbuf0;
        mbar_arrive_expect_tx(&qfull[qs], q_halves * half_bytes);
        for (int h = 0; h < q_halves; ++h)
          bulk_g2s(qdst + h * HP, a.arena + d.in[0] + h * D, half_bytes, &qfull[qs]);
      }
      ++qi;
      const int32_t* idx = rows_local ? a.cand_local + static_cast<int64_t>(d.aux) * a.ncand
                                      : a.cand + static_cast<int64_t>(d.id) * a.ncand;
      const int j_beg = part * a.ncand / S, j_end = (part + 1) * a.ncand / S;
      for (int j0 = j_beg; j0 < j_end; j0 += 32) {
        if (j0 + lane < j_end) idx_s[lane] = __ldg(idx + j0 + lane);
        __syncwarp();
        const int cnt = min(32, j_end - j0);
        if (lane == 0)
          for (int r = 0; r < cnt; ++r) {
            const int p = pos + r;
            const int slot = p % L.depth, round = p / L.depth;
            if (round > 0) mbar_wait_parity(&empty[slot], (round - 1) & 1);
            const float* src = rows_base + static_cast<int64_t>(idx_s[r]) * a.ent_w;
            mbar_arrive_expect_tx(&full[slot], L.halves * half_bytes);
            for (int h = 0; h < L.halves; ++h)
              bulk_g2s(rows + slot * RW + h * HP, src + h * D, half_bytes, &full[slot]);
          }
        pos += cnt;
        __syncwarp();  // idx_s is reused by the next chunk
      }
    }
    return;
  }

  // ---- consumers ----
  const int ctid = threadIdx.x;
  int pos = 0, qi = 0;
  for (int t = blockIdx.x; t < n_items; t += gridDim.x) {
    const int node = t / S, part = t % S;
    const ngdb_node_desc d = a.nodes[first + node];
    if (MODE == kLoss && d.aux < 0) {
      // union query: the input already holds min-over-branch distances; part 0
      // computes the whole loss, the other parts have nothing to do
      if (part == 0) {
        float loss = 0.f;
        for (int j = ctid; j < a.ncand; j += kConsumerThreads) {
          const float c = loss_coef(a, j, a.arena[d.in[0] + j], loss);
          a.ddbuf[static_cast<int64_t>(d.id) * a.ncand + j] = c;
        }
        loss = warp_sum(loss);
        if (lane == 0) lred[warp] = loss;
        consumers_sync();
        if (ctid == 0) {
          float total = 0.f;
          for (int w = 0; w < kCWarps; ++w) total += lred[w];
          a.loss_out[d.id] = total;
          a.arena[d.out] = total;
          if (!isfinite(total)) atomicOr(&a.flags[0], 1);
        }
        consumers_sync();
      }
      continue;
    }
    const int qs = qi & 1;
    mbar_wait_parity(&qfull[qs], (qi >> 1) & 1);
    const float* q = qs ? qbuf1 : qbuf0;
    RowMath<BB, NCH> R;
    R.load_q(q, lane);
    if (part == 0 && MODE != kScoreBwd) {  // query copy for the optimizer
      float* qcopy = a.qbuf + static_cast<int64_t>(d.aux) * a.wq;
      for (int e = ctid * 4; e < a.wq; e += kConsumerThreads * 4) {
        const int h = e / D;
        st4(qcopy + e, ld4(q + h * HP + (e - h * D)));
      }
    }
    float qbias = 0.f;
    if constexpr (kBeta) {  // lnB(query) summed over the dims
      float tq = 0.f;
      for (int e = ctid; e < D; e += kConsumerThreads) tq += dg_lbeta(q[e], q[HP + e]);
      tq = warp_sum(tq);
      if (lane == 0) lred[warp] = tq;
      consumers_sync();
      if (ctid == 0) {
        float tt = 0.f;
        for (int w = 0; w < kCWarps; ++w) tt += lred[w];
        bcast = tt;
      }
      consumers_sync();
      qbias = bcast;
    }
    const int32_t* idx = rows_local ? a.cand_local + static_cast<int64_t>(d.aux) * a.ncand
                                    : a.cand + static_cast<int64_t>(d.id) * a.ncand;
    const int j_beg = part * a.ncand / S, j_end = (part + 1) * a.ncand / S;
    const int n_mine = j_end - j_beg;
    float* coefs = a.coefbuf + static_cast<int64_t>(d.aux) * a.ncand;
    const float* g = MODE == kScoreBwd ? a.arena + d.grad : nullptr;
    float* out = MODE == kScoreFwd ? a.arena + d.out : nullptr;
    float loss = 0.f, csum = 0.f;  // identical in every lane of a warp
    for (int u = warp; u < n_mine; u += kCWarps) {
      const int p = pos + u, slot = p % L.depth, j = j_beg + u;
      mbar_wait_parity(&full[slot], (p / L.depth) & 1);
      float dj = R.distance(rows + slot * RW, lane, a.alpha_box);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);  // the row is in registers
      dj = warp_sum(dj);
      if constexpr (kBeta) dj += qbias + __ldg(a.etab_c + __ldg(idx + j));
      if constexpr (MODE == kScoreFwd) {
        if (lane == 0) out[j] = dj;
      } else {
        float coef;
        if constexpr (MODE == kLoss) coef = loss_coef(a, j, dj, loss);
        else coef = g[j];
        csum += coef;
        if (lane == 0) coefs[j] = coef;
        R.grad(coef, a.alpha_box);
      }
    }
    pos += n_mine;
    if constexpr (MODE == kScoreFwd) {
      consumers_sync();
      if (ctid == 0) mbar_arrive(&qempty[qs]);
      ++qi;
    } else {
      // cross-warp partials: one shared row per warp, summed in warp order
      if (lane == 0) {
        lred[2 * warp] = loss;
        lred[2 * warp + 1] = csum;
      }
#pragma unroll
      for (int i = 0; i < NCH; ++i) {
        st4(parts(warp) + 4 * (lane + 32 * i), R.gc[i]);
        if (BB != NGDB_GQE) st4(parts(warp) + HP + 4 * (lane + 32 * i), R.go[i]);
      }
      consumers_sync();
      if (ctid == 0) mbar_arrive(&qempty[qs]);  // every consumer is done with q
      ++qi;
      // this item's dL/dq (compact [wq]) and (loss, coefficient sum)
      float* dq_final = MODE == kLoss ? a.dqbuf + static_cast<int64_t>(d.aux) * a.wq
                                      : a.arena + d.out;
      float* dst = S == 1 ? dq_final : a.lpart + static_cast<int64_t>(t) * a.wq;
      for (int e = ctid * 4; e < a.wq; e += kConsumerThreads * 4) {
        const int h = e / D, ep = h * HP + (e - h * D);
        float4 s4 = ld4(parts(0) + ep);
#pragma unroll
        for (int w = 1; w < kCWarps; ++w) acc4(s4, ld4(parts(w) + ep));
        st4(dst + e, s4);
      }
      float l_item = 0.f, c_item = 0.f;
      if (ctid == 0)
        for (int w = 0; w < kCWarps; ++w) {
          l_item += lred[2 * w];
          c_item += lred[2 * w + 1];
        }
      bool finish = true;
      if (S > 1) {
        if (ctid == 0) {
          a.lpart_scalar[2 * t] = l_item;
          a.lpart_scalar[2 * t + 1] = c_item;
        }
        __threadfence();
        consumers_sync();
        if (ctid == 0) last_flag = atomicAdd(&a.lcount[node], 1) == S - 1;
        consumers_sync();
        finish = last_flag != 0;
        if (finish) {
          __threadfence();  // the other parts' partials are visible
          const float* base = a.lpart + static_cast<int64_t>(node) * S * a.wq;
          for (int e = ctid * 4; e < a.wq; e += kConsumerThreads * 4) {
            float4 s4 = ld4(base + e);
            for (int p2 = 1; p2 < S; ++p2) acc4(s4, ld4(base + static_cast<int64_t>(p2) * a.wq + e));
            st4(dq_final + e, s4);
          }
          if (ctid == 0) {
            l_item = c_item = 0.f;
            for (int p2 = 0; p2 < S; ++p2) {
              l_item += a.lpart_scalar[2 * (node * S + p2)];
              c_item += a.lpart_scalar[2 * (node * S + p2) + 1];
            }
            a.lcount[node] = 0;  // ready for the next launch
          }
        }
      }
      if (finish) {
        if constexpr (kBeta) {
          // dL/dq += (sum_j coef_j) [psi(A)-psi(A+B) | psi(B)-psi(A+B)] (query term)
          consumers_sync();
          if (ctid == 0) bcast = c_item;
          consumers_sync();
          const float sc = bcast;
          const float* qq = a.arena + d.in[0];
          for (int e = ctid; e < a.wq; e += kConsumerThreads) dq_final[e] += sc * beta_qterm(a, qq, e);
        }
        if (MODE == kLoss && ctid == 0) {
          a.loss_out[d.id] = l_item;
          a.arena[d.out] = l_item;
          if (!isfinite(l_item)) atomicOr(&a.flags[0], 1);
        }
      }
      consumers_sync();  // parts[] / lred are reused by the next item
    }
  }
}

// A kernel's max-dynamic-smem attribute must cover every launch: keep it equal
// to the size of the launch at hand (set only when it changes).
template <class K>
void ensure_smem_attr(K kernel, size_t smem) {
  static std::map<const void*, size_t> attr;  // kernel -> value last set
  const void* key = reinterpret_cast<const void*>(kernel);
  auto it = attr.find(key);
  if (it == attr.end() || it->second != smem) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr[key] = smem;
  }
}

template <int BB, int NCH, int MODE>
void launch_stream(const DevArgs& a, int first, int n, cudaStream_t s) {
  auto kernel = stream_kernel<BB, NCH, MODE>;
  const size_t smem = Layout<NCH>(BB).bytes();
  ensure_smem_attr(kernel, smem);
  static int resident = 0;  // per instantiation (fixed smem per instantiation)
  if (!resident) {
    int per_sm = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    resident = std::max(1, per_sm) * sms;
  }
  // parts per node: at most one item per resident CTA (measured: fewer,
  // larger items beat an even spread — the per-item reduction is not free;
  // within the partial
  // buffer's capacity); the persistent grid never exceeds one wave
  int S = std::max(1, std::min(8, resident / n));
  while (S > 1 && S * n > a.lpart_items) --S;
  const int grid = std::min(resident, S * n);
  launch_pdl(kernel, dim3(grid), dim3(kThreads), smem, s, 1, a, first, n, S);
}

template <int NCH, int MODE>
void launch_mode(const DevArgs& a, int first, int n, cudaStream_t s) {
  if (a.backbone == NGDB_GQE) launch_stream<NGDB_GQE, NCH, MODE>(a, first, n, s);
  else if (a.backbone == NGDB_BETAE) launch_stream<NGDB_BETAE, NCH, MODE>(a, first, n, s);
  else launch_stream<NGDB_Q2B, NCH, MODE>(a, first, n, s);
}

template <int MODE>
void launch_any(const DevArgs& a, int first, int n, cudaStream_t s) {
  // each d-wide half is padded to 128 * NCH floats
  if (a.dim <= 512) launch_mode<4, MODE>(a, first, n, s);
  else launch_mode<8, MODE>(a, first, n, s);
}

}  // namespace

int launch_loss_fwd(const DevArgs& a, int first, int n, const LaunchCtx& lc) {
  if (n <= 0) return 0;
  launch_any<kLoss>(a, first, n, lc.stream);
  return 1;
}

int launch_score(const DevArgs& a, int dir, int first, int n, const LaunchCtx& lc) {
  if (n <= 0) return 0;
  if (dir == 0) launch_any<kScoreFwd>(a, first, n, lc.stream);
  else launch_any<kScoreBwd>(a, first, n, lc.stream);
  return 1;
}

}  // namespace ngdb_dev
