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

constexpr int kWarps = 8;  // 256 threads, one node per warp

__device__ __forceinline__ bool bad_index(const DevArgs& a, int32_t id, int32_t limit) {
  if (id < 0 || id >= limit) {
    atomicOr(&a.flags[1], 1);
    return true;
  }
  return false;
}

__global__ void __launch_bounds__(kWarps * 32) embed_kernel(DevArgs a, int dir, int first, int n,
                                                            int n_entities) {
  pdl_start();
  const int node = blockIdx.x * kWarps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (node >= n) return;
  const ngdb_node_desc d = a.nodes[first + node];
  if (bad_index(a, d.id, n_entities)) return;
  const int ew4 = a.ent_w / 4;
  if (dir == 0) {
    float* out = a.arena + d.out;
    // FuseSemantic: the prologue's fused row of this anchor's entity
    // row-sharded: the row fetched from its owner into this anchor slot
    const float* src = a.fused      ? a.etab + static_cast<int64_t>(a.anchor_local[d.aux]) * a.ent_w
                       : a.anc_rows ? a.anc_rows + static_cast<int64_t>(d.aux) * a.ent_w
                                    : a.ent + static_cast<int64_t>(d.id) * a.ent_w;
    if (a.backbone == NGDB_BETAE) {  // realised (alpha | beta); the mirror's
      for (int c = lane; c < ew4; c += 32) {  // chain rule runs in the optimizer
        const float4 x = ldg4(src + 4 * c);
        st4(out + 4 * c, make_float4(beta_realize(x.x), beta_realize(x.y), beta_realize(x.z),
                                     beta_realize(x.w)));
      }
      return;
    }
    for (int c = lane; c < ew4; c += 32) st4(out + 4 * c, ld4(src + 4 * c));
    // Q2B anchors are point boxes: offset half is zero
    for (int c = ew4 + lane; c < a.wq / 4; c += 32) st4(out + 4 * c, make_float4(0.f, 0.f, 0.f, 0.f));
  } else {
    // adjoint of the gather: keep the entity part of the upstream gradient for
    // the sorted-segment reduce in the optimizer
    const float* g = a.arena + d.grad;
    float* dst = a.agbuf + static_cast<int64_t>(d.aux) * a.ent_w;
    for (int c = lane; c < ew4; c += 32) st4(dst + 4 * c, ld4(g + 4 * c));
  }
}

__global__ void __launch_bounds__(kWarps * 32) project_kernel(DevArgs a, int dir, int first, int n,
                                                              int n_relations) {
  pdl_start();
  const int node = blockIdx.x * kWarps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (node >= n) return;
  const ngdb_node_desc d = a.nodes[first + node];
  if (bad_index(a, d.id, n_relations)) return;
  const float* r = a.rel + static_cast<int64_t>(d.id) * a.rel_w;
  const float* x = a.arena + d.in[0];
  const int d4 = a.dim / 4;
  if (a.backbone == NGDB_GQE) {
    if (dir == 0) {
      float* out = a.arena + d.out;
      for (int c = lane; c < d4; c += 32) {
        float4 u = ld4(x + 4 * c), v = ldg4(r + 4 * c);
        st4(out + 4 * c, make_float4(u.x + v.x, u.y + v.y, u.z + v.z, u.w + v.w));
      }
    } else {
      const float* g = a.arena + d.grad;
      float* out = a.arena + d.out;
      float* rg = a.rgbuf + static_cast<int64_t>(d.aux) * a.rel_w;
      for (int c = lane; c < d4; c += 32) {
        float4 u = ld4(g + 4 * c);
        st4(out + 4 * c, u);
        st4(rg + 4 * c, u);
      }
    }
    return;
  }
  // Q2B box projection: c' = c + r_c, o' = relu(o + r_o)
  if (dir == 0) {
    float* out = a.arena + d.out;
    for (int c = lane; c < d4; c += 32) {
      float4 u = ld4(x + 4 * c), v = ldg4(r + 4 * c);
      st4(out + 4 * c, make_float4(u.x + v.x, u.y + v.y, u.z + v.z, u.w + v.w));
      float4 o = ld4(x + a.dim + 4 * c), ro = ldg4(r + a.dim + 4 * c);
      st4(out + a.dim + 4 * c, make_float4(fmaxf(o.x + ro.x, 0.f), fmaxf(o.y + ro.y, 0.f),
                                           fmaxf(o.z + ro.z, 0.f), fmaxf(o.w + ro.w, 0.f)));
    }
  } else {
    const float* g = a.arena + d.grad;
    float* out = a.arena + d.out;
    float* rg = a.rgbuf + static_cast<int64_t>(d.aux) * a.rel_w;
    for (int c = lane; c < d4; c += 32) {
      float4 gc = ld4(g + 4 * c);
      st4(out + 4 * c, gc);
      st4(rg + 4 * c, gc);
      float4 o = ld4(x + a.dim + 4 * c), ro = ldg4(r + a.dim + 4 * c), go = ld4(g + a.dim + 4 * c);
      float4 m = make_float4(o.x + ro.x > 0.f ? go.x : 0.f, o.y + ro.y > 0.f ? go.y : 0.f,
                             o.z + ro.z > 0.f ? go.z : 0.f, o.w + ro.w > 0.f ? go.w : 0.f);
      st4(out + a.dim + 4 * c, m);
      st4(rg + a.dim + 4 * c, m);
    }
  }
}

__global__ void __launch_bounds__(kWarps * 32) negate_kernel(DevArgs a, int dir, int first, int n) {
  pdl_start();
  const int node = blockIdx.x * kWarps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (node >= n) return;
  const ngdb_node_desc d = a.nodes[first + node];
  const float* src = a.arena + (dir == 0 ? d.in[0] : d.grad);
  float* out = a.arena + d.out;
  if (a.backbone == NGDB_BETAE) {
    // (alpha, beta) -> clamp(1/alpha, 1/beta); bwd: g * -1/x^2 where unclamped
    const float* x = a.arena + d.in[0];
    for (int c = lane; c < a.wq / 4; c += 32) {
      const float4 u = ld4(x + 4 * c), g = ld4(src + 4 * c);
      const float xs[4] = {u.x, u.y, u.z, u.w}, gs[4] = {g.x, g.y, g.z, g.w};
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
  for (int c = lane; c < a.wq / 4; c += 32) {
    float4 u = ld4(src + 4 * c);
    if (c < neg4) u = make_float4(-u.x, -u.y, -u.z, -u.w);
    st4(out + 4 * c, u);
  }
}

__global__ void __launch_bounds__(kWarps * 32) union_kernel(DevArgs a, int dir, int k, int first,
                                                            int n) {
  pdl_start();
  const int node = blockIdx.x * kWarps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (node >= n) return;
  const ngdb_node_desc d = a.nodes[first + node];
  const int nc = a.ncand;
  if (dir == 0) {
    float* out = a.arena + d.out;
    for (int j = lane; j < nc; j += 32) {
      float best = a.arena[d.in[0] + j];
      for (int l = 1; l < k; ++l) best = fminf(best, a.arena[d.in[l] + j]);
      out[j] = best;  // min distance == max score
    }
  } else {
    const float* g = a.arena + d.grad;
    float* out = a.arena + d.out;
    for (int j = lane; j < nc; j += 32) {
      int arg = 0;
      float best = a.arena[d.in[0] + j];
      for (int l = 1; l < k; ++l) {
        const float v = a.arena[d.in[l] + j];
        if (v < best) { best = v; arg = l; }  // ties -> lowest branch index
      }
      for (int l = 0; l < k; ++l) out[l * nc + j] = (l == arg) ? g[j] : 0.f;
    }
  }
}

// Loss mirror: the fused Loss forward already produced dL/dq (non-union) or
// dL/dd (union); the mirror materialises it into its planned arena slot.
__global__ void __launch_bounds__(kWarps * 32) loss_bwd_kernel(DevArgs a, int first, int n) {
  pdl_start();
  const int node = blockIdx.x * kWarps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (node >= n) return;
  const ngdb_node_desc d = a.nodes[first + node];
  float* out = a.arena + d.out;
  if (d.aux >= 0) {
    const float* src = a.dqbuf + static_cast<int64_t>(d.aux) * a.wq;
    for (int c = lane; c < a.wq / 4; c += 32) st4(out + 4 * c, ld4(src + 4 * c));
  } else {
    const float* src = a.ddbuf + static_cast<int64_t>(d.id) * a.ncand;
    for (int j = lane; j < a.ncand; j += 32) out[j] = src[j];
  }
}

inline int blocks_for(int n) { return (n + kWarps - 1) / kWarps; }

}  // namespace

int launch_embed(const DevArgs& a, int dir, int first, int n, const LaunchCtx& lc) {
  launch_pdl(embed_kernel, dim3(blocks_for(n)), dim3(kWarps * 32), 0, lc.stream, 1, a, dir, first, n, a.n_entities);
  return 1;
}
int launch_project(const DevArgs& a, int dir, int first, int n, const LaunchCtx& lc) {
  if (a.backbone == NGDB_BETAE) return launch_beta_project(a, dir, first, n, lc);
  launch_pdl(project_kernel, dim3(blocks_for(n)), dim3(kWarps * 32), 0, lc.stream, 1, a, dir, first, n, a.n_relations);
  return 1;
}
int launch_negate(const DevArgs& a, int dir, int first, int n, const LaunchCtx& lc) {
  launch_pdl(negate_kernel, dim3(blocks_for(n)), dim3(kWarps * 32), 0, lc.stream, 1, a, dir, first, n);
  return 1;
}
int launch_union(const DevArgs& a, int dir, int k, int first, int n, const LaunchCtx& lc) {
  launch_pdl(union_kernel, dim3(blocks_for(n)), dim3(kWarps * 32), 0, lc.stream, 1, a, dir, k, first, n);
  return 1;
}
int launch_loss_bwd(const DevArgs& a, int first, int n, const LaunchCtx& lc) {
  launch_pdl(loss_bwd_kernel, dim3(blocks_for(n)), dim3(kWarps * 32), 0, lc.stream, 1, a, first, n);
  return 1;
}

}  // namespace ngdb_dev
