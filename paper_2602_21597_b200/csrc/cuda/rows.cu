// Row-parallel operator kernels: EmbedAnchor (gather), Project, Negate,
// UnionScore and the Loss mirror. One warp per operator node, 128-bit loads
// along the row (rows are 1600 B for d=400: 100 float4 per row).
//
// Forms follow SPEC.md:359-367 (gqe_project), 377-378 (q2b_project), 303-311
// (gather / scatter_add), 404-412 (union_score) and DESIGN.md §3.2 (the Q2B
// negation convention, SURVEY A-8).
#include "common.cuh"
#include "special.cuh"

namespace ngdb_dev {
namespace {

constexpr int kWarps = 2;  // 64 threads, one node per warp: a 512-node pop spreads over 256 CTAs

__device__ __forceinline__ bool bad_index(const DevArgs& a, int32_t id, int32_t limit) {
  if (id < 0 || id >= limit) {
    atomicOr(&a.flags[1], 1);
    return true;
  }
  return false;
}

// Lane-chunk loops below load every chunk of the lane's rows first and store
// afterwards: all of a warp's 16-byte loads are in flight at once (one memory
// round trip per node instead of one per chunk). NCH = float4 chunks per lane
// for a row of up to 128 * NCH floats.
#define FOR_CHUNKS(n4) \
  _Pragma("unroll") for (int i = 0; i < NCH; ++i) \
    if (const int c = lane + 32 * i; c < (n4))

template <int NCH>
__global__ void __launch_bounds__(kWarps * 32) embed_kernel(DevArgs a, int dir, int first, int n,
                                                            int n_entities) {
  pdl_launch();
  const int node = blockIdx.x * kWarps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (node >= n) return;
  const ngdb_node_desc d = a.nodes[first + node];  // plan data: before the wait
  pdl_wait();
  if (bad_index(a, d.id, n_entities)) return;
  const int ew4 = a.ent_w / 4;
  float4 u[NCH];
  if (dir == 0) {
    float* out = a.arena + d.out;
    // FuseSemantic: the prologue's fused row of this anchor's entity
    // row-sharded: the row fetched from its owner into this anchor slot
    // (BetaE: Psi_theta's pre-activation row, realised below)
    // (FuseSemantic: the owner sent the fused / Psi_theta row)
    const float* src = a.anc_rows ? a.anc_rows + static_cast<int64_t>(a.anc_pos[d.aux]) * a.ent_w
                       : a.fused  ? (a.ytab ? a.ytab : a.etab) +
                                        static_cast<int64_t>(a.anchor_local[d.aux]) * a.ent_w
                                  : a.ent + static_cast<int64_t>(d.id) * a.ent_w;
    FOR_CHUNKS(ew4) u[i] = ldg4(src + 4 * c);
    if (a.backbone == NGDB_BETAE) {  // realised (alpha | beta); the mirror's
      FOR_CHUNKS(ew4)                // chain rule runs in the optimizer
        st4(out + 4 * c, make_float4(beta_realize(u[i].x), beta_realize(u[i].y),
                                     beta_realize(u[i].z), beta_realize(u[i].w)));
      return;
    }
    FOR_CHUNKS(ew4) st4(out + 4 * c, u[i]);
    // Q2B anchors are point boxes: offset half is zero
    for (int c = ew4 + lane; c < a.wq / 4; c += 32) st4(out + 4 * c, make_float4(0.f, 0.f, 0.f, 0.f));
  } else {
    // adjoint of the gather: keep the entity part of the upstream gradient for
    // the sorted-segment reduce in the optimizer
    const float* g = a.arena + d.grad;
    float* dst = a.agbuf + static_cast<int64_t>(d.aux) * a.ent_w;
    FOR_CHUNKS(ew4) u[i] = ld4(g + 4 * c);
    FOR_CHUNKS(ew4) st4(dst + 4 * c, u[i]);
  }
}

__device__ __forceinline__ float4 add4(float4 u, float4 v) {
  return make_float4(u.x + v.x, u.y + v.y, u.z + v.z, u.w + v.w);
}

template <int NCH>
__global__ void __launch_bounds__(kWarps * 32) project_kernel(DevArgs a, int dir, int first, int n,
                                                              int n_relations) {
  pdl_launch();
  const int node = blockIdx.x * kWarps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (node >= n) return;
  const ngdb_node_desc d = a.nodes[first + node];  // plan data: before the wait
  pdl_wait();
  if (bad_index(a, d.id, n_relations)) return;
  const float* r = a.rel + static_cast<int64_t>(d.id) * a.rel_w;
  const float* x = a.arena + d.in[0];
  float* out = a.arena + d.out;
  const int d4 = a.dim / 4;
  float4 u[NCH], v[NCH];
  if (a.backbone == NGDB_GQE) {
    if (dir == 0) {
      FOR_CHUNKS(d4) {
        u[i] = ld4(x + 4 * c);
        v[i] = ldg4(r + 4 * c);
      }
      FOR_CHUNKS(d4) st4(out + 4 * c, add4(u[i], v[i]));
    } else {
      const float* g = a.arena + d.grad;
      float* rg = a.rgbuf + static_cast<int64_t>(d.aux) * a.rel_w;
      FOR_CHUNKS(d4) u[i] = ld4(g + 4 * c);
      FOR_CHUNKS(d4) {
        st4(out + 4 * c, u[i]);
        st4(rg + 4 * c, u[i]);
      }
    }
    return;
  }
  // Q2B box projection: c' = c + r_c, o' = relu(o + r_o). Chunks 0..d4-1 are
  // the centre half, d4..2*d4-1 the offset half (rows are [c | o]).
  const int w4 = 2 * d4;
  if (dir == 0) {
    FOR_CHUNKS(w4) {
      u[i] = ld4(x + 4 * c);
      v[i] = ldg4(r + 4 * c);
    }
    FOR_CHUNKS(w4) {
      float4 y = add4(u[i], v[i]);
      if (c >= d4) y = make_float4(fmaxf(y.x, 0.f), fmaxf(y.y, 0.f), fmaxf(y.z, 0.f), fmaxf(y.w, 0.f));
      st4(out + 4 * c, y);
    }
  } else {
    const float* g = a.arena + d.grad;
    float* rg = a.rgbuf + static_cast<int64_t>(d.aux) * a.rel_w;
    float4 gg[NCH];
    FOR_CHUNKS(w4) {
      gg[i] = ld4(g + 4 * c);
      if (c >= d4) {
        u[i] = ld4(x + 4 * c);
        v[i] = ldg4(r + 4 * c);
      }
    }
    FOR_CHUNKS(w4) {
      float4 m = gg[i];
      if (c >= d4) {
        const float4 o = add4(u[i], v[i]);
        m = make_float4(o.x > 0.f ? m.x : 0.f, o.y > 0.f ? m.y : 0.f, o.z > 0.f ? m.z : 0.f,
                        o.w > 0.f ? m.w : 0.f);
      }
      st4(out + 4 * c, m);
      st4(rg + 4 * c, m);
    }
  }
}

template <int NCH>
__global__ void __launch_bounds__(kWarps * 32) negate_kernel(DevArgs a, int dir, int first, int n) {
  pdl_launch();
  const int node = blockIdx.x * kWarps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (node >= n) return;
  const ngdb_node_desc d = a.nodes[first + node];  // plan data: before the wait
  pdl_wait();
  const float* src = a.arena + (dir == 0 ? d.in[0] : d.grad);
  float* out = a.arena + d.out;
  const int w4 = a.wq / 4;
  float4 u[NCH];
  if (a.backbone == NGDB_BETAE) {
    // (alpha, beta) -> clamp(1/alpha, 1/beta); bwd: g * -1/x^2 where unclamped
    const float* x = a.arena + d.in[0];
    float4 g[NCH];
    FOR_CHUNKS(w4) {
      u[i] = ld4(x + 4 * c);
      g[i] = ld4(src + 4 * c);
    }
    FOR_CHUNKS(w4) {
      const float xs[4] = {u[i].x, u[i].y, u[i].z, u[i].w}, gs[4] = {g[i].x, g[i].y, g[i].z, g[i].w};
      float o[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float inv = 1.f / xs[t];
        if (dir == 0) o[t] = fminf(fmaxf(inv, kBetaMin), kBetaMax);
        else o[t] = (inv > kBetaMin && inv < kBetaMax) ? -gs[t] * inv * inv : 0.f;
      }
      st4(out + 4 * c, make_float4(o[0], o[1], o[2], o[3]));
    }
    return;
  }
  // GQE: x -> -x. Q2B: (c, o) -> (-c, o). Both are their own adjoints.
  const int neg4 = a.dim / 4;
  FOR_CHUNKS(w4) u[i] = ld4(src + 4 * c);
  FOR_CHUNKS(w4) {
    float4 y = u[i];
    if (c < neg4) y = make_float4(-y.x, -y.y, -y.z, -y.w);
    st4(out + 4 * c, y);
  }
}

// One thread per (node, candidate): the k branch distances of a candidate are
// independent loads.
__global__ void __launch_bounds__(256) union_kernel(DevArgs a, int dir, int k, int first, int n) {
  pdl_start();
  const int nc = a.ncand;
  const int64_t item = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (item >= static_cast<int64_t>(n) * nc) return;
  const int node = static_cast<int>(item / nc), j = static_cast<int>(item % nc);
  const ngdb_node_desc d = a.nodes[first + node];
  float v[3];
  for (int l = 0; l < k; ++l) v[l] = a.arena[d.in[l] + j];
  int arg = 0;
  float best = v[0];
  for (int l = 1; l < k; ++l)
    if (v[l] < best) { best = v[l]; arg = l; }  // ties -> lowest branch index
  if (dir == 0) {
    a.arena[d.out + j] = best;  // min distance == max score
  } else {
    const float g = a.arena[d.grad + j];
    for (int l = 0; l < k; ++l) a.arena[d.out + l * nc + j] = (l == arg) ? g : 0.f;
  }
}

// Loss mirror: the fused Loss forward already produced dL/dq (non-union) or
// dL/dd (union); the mirror materialises it into its planned arena slot.
template <int NCH>
__global__ void __launch_bounds__(kWarps * 32) loss_bwd_kernel(DevArgs a, int first, int n) {
  pdl_launch();
  const int node = blockIdx.x * kWarps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (node >= n) return;
  const ngdb_node_desc d = a.nodes[first + node];  // plan data: before the wait
  pdl_wait();
  float* out = a.arena + d.out;
  if (d.aux >= 0) {
    const float* src = a.dqbuf + static_cast<int64_t>(d.aux) * a.wq;
    const int w4 = a.wq / 4;
    float4 u[NCH];
    FOR_CHUNKS(w4) u[i] = ld4(src + 4 * c);
    FOR_CHUNKS(w4) st4(out + 4 * c, u[i]);
  } else {
    const float* src = a.ddbuf + static_cast<int64_t>(d.id) * a.ncand;
    for (int j = lane; j < a.ncand; j += 32) out[j] = src[j];
  }
}

inline int blocks_for(int n) { return (n + kWarps - 1) / kWarps; }

// chunk-count instantiation for rows of up to `floats` floats
template <template <int> class Sel, class... Args>
void by_width(int floats, Args&&... args) {
  const int w4 = (floats + 3) / 4;
  if (w4 <= 128) Sel<4>::go(args...);
  else if (w4 <= 256) Sel<8>::go(args...);
  else Sel<16>::go(args...);
}
template <int NCH>
struct EmbedL {
  static void go(const DevArgs& a, int dir, int first, int n, cudaStream_t s) {
    launch_pdl(embed_kernel<NCH>, dim3(blocks_for(n)), dim3(kWarps * 32), 0, s, 1, a, dir, first, n, a.n_entities);
  }
};
template <int NCH>
struct ProjectL {
  static void go(const DevArgs& a, int dir, int first, int n, cudaStream_t s) {
    launch_pdl(project_kernel<NCH>, dim3(blocks_for(n)), dim3(kWarps * 32), 0, s, 1, a, dir, first, n, a.n_relations);
  }
};
template <int NCH>
struct NegateL {
  static void go(const DevArgs& a, int dir, int first, int n, cudaStream_t s) {
    launch_pdl(negate_kernel<NCH>, dim3(blocks_for(n)), dim3(kWarps * 32), 0, s, 1, a, dir, first, n);
  }
};
template <int NCH>
struct LossBwdL {
  static void go(const DevArgs& a, int first, int n, cudaStream_t s) {
    launch_pdl(loss_bwd_kernel<NCH>, dim3(blocks_for(n)), dim3(kWarps * 32), 0, s, 1, a, first, n);
  }
};

}  // namespace

int launch_embed(const DevArgs& a, int dir, int first, int n, const LaunchCtx& lc) {
  by_width<EmbedL>(a.ent_w, a, dir, first, n, lc.stream);
  return 1;
}
int launch_project(const DevArgs& a, int dir, int first, int n, const LaunchCtx& lc) {
  if (a.backbone == NGDB_BETAE) return launch_beta_project(a, dir, first, n, lc);
  by_width<ProjectL>(a.wq, a, dir, first, n, lc.stream);
  return 1;
}
int launch_negate(const DevArgs& a, int dir, int first, int n, const LaunchCtx& lc) {
  by_width<NegateL>(a.wq, a, dir, first, n, lc.stream);
  return 1;
}
int launch_union(const DevArgs& a, int dir, int k, int first, int n, const LaunchCtx& lc) {
  const int64_t items = static_cast<int64_t>(n) * a.ncand;
  launch_pdl(union_kernel, dim3(static_cast<int>((items + 255) / 256)), dim3(256), 0, lc.stream, 1,
             a, dir, k, first, n);
  return 1;
}
int launch_loss_bwd(const DevArgs& a, int first, int n, const LaunchCtx& lc) {
  by_width<LossBwdL>(a.wq, a, first, n, lc.stream);
  return 1;
}

}  // namespace ngdb_dev
