// Shared device-side definitions for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "ngdb/ngdb_cuda.h"

namespace ngdb_dev {

constexpr int kMaxDenseTensors = 16;
// Intersect stash slot size in units of d floats: Q2B Z, S, P [3][d] + U, Lm [d]
constexpr int kStashPerSlot = 11;

// Named dense tensors (offsets into the flat dense parameter buffer).
enum DenseName : int {
  // GQE intersection MLP: out = W2 relu(W1 mean_k x)
  GQE_W1 = 0, GQE_W2 = 1,
  // Q2B attention (centre) and DeepSets (offset) MLPs
  Q2B_A1 = 0, Q2B_A1B = 1, Q2B_A2 = 2, Q2B_A2B = 3,
  Q2B_V1 = 4, Q2B_V1B = 5, Q2B_V2 = 6, Q2B_V2B = 7,
  // BetaE projection MLP [q | r] -> 2d -> 2d and attention MLP 2d -> 2d -> d
  //
  BETA_P1 = 0, BETA_P1B = 1, BETA_P2 = 2, BETA_P2B = 3,
  BETA_A1 = 4, BETA_A1B = 5, BETA_A2 = 6, BETA_A2B = 7,
};

// Everything a kernel needs, passed by value.
struct DevArgs {
  int32_t backbone;
  int32_t dim;        // d
  int32_t wq;         // query width (GQE d, Q2B 2d)
  int32_t ent_w;      // entity row width
  int32_t rel_w;      // relation row width
  int32_t ncand;      // 1 + K
  int32_t n_neg;
  int32_t n_entities;
  int32_t n_relations;
  float gamma;
  float alpha_box;
  float* arena;
  const ngdb_node_desc* nodes;
  const int32_t* cand;
  float* ent;         // entity table
  float* rel;         // relation table
  float* dense;       // flat dense params
  float* dense_g;     // flat dense grads
  int64_t dense_off[kMaxDenseTensors];
  // 3xTF32 operand splits of every dense weight matrix W [out][in], refreshed
  // after each optimizer step: W_hi, W_lo, (W^T)_hi, (W^T)_lo at wsplit_off[i]
  float* wsplit;
  int64_t wsplit_off[kMaxDenseTensors];
  float* qbuf;        // [S][wq]   query copy per score slot
  float* dqbuf;       // [S][wq]   dL/dq per score slot (fused Loss)
  float* coefbuf;     // [S][ncand] dL/dd per score slot and candidate
  float* ddbuf;       // [B][ncand] dL/dd per union query
  float* agbuf;       // [A][ent_w] anchor gradient rows
  float* rgbuf;       // [P][rel_w] relation gradient rows
  float* loss_out;    // [B]
  int32_t* flags;     // [0] non-finite loss, [1] index out of range
  float* scratch;     // GEMM scratch
  int64_t scratch_cap;
  // BetaE per-step entity table: for every touched entity row
  // r (the optimizer CSR order) etab[r] = [psi(s)-psi(a) | psi(s)-psi(b)] and
  // etab_c[r] = sum_e (-lnB(a,b) + a psi(a) + b psi(b) - s psi(s)), so that
  // KL(entity || query) = lnB(query) + etab_c[r] + <query, etab[r]>.
  // cand_local[slot*ncand + j] = CSR row of candidate j of score slot `slot`.
  float* etab;
  float* etab_c;
  int32_t* cand_local;
  // FuseSemantic (fuse.cu): etab holds e_fused of every touched row; anchors
  // map to rows through anchor_local[anchor slot]
  int32_t fused;
  int32_t sem_dim;
  const float* sem;      // frozen store [n_entities][sem_dim]
  // its 3xTF32 split, made once at upload: [n][sem_dim] hi / lo (used when a
  // step touches every entity; read MN-major by the weight gradients)
  const float* sem_hi;
  const float* sem_lo;
  int32_t* anchor_local;
  int32_t fus_idx;       // dense index of fus_f (fus_wp = +1, fus_bp = +2)
  // row-sharded step (shard.cu): anchor rows fetched from their owners, in
  // receive order [n_recv][ent_w]; anc_pos[anchor slot] = its receive position
  const float* anc_rows;
  const int32_t* anc_pos;
  // BetaE with FuseSemantic: Psi_theta output rows Y [touched row][2d] (the
  // pre-activation Beta parameters, CSR row order); nullptr otherwise
  const float* ytab;
  // Intersect stash: per forward node (slot = node aux) the MLP intermediates
  // its mirror reads instead of recomputing them; istash_slots slots of
  // kStashPerSlot * dim floats
  float* istash;
  int32_t istash_slots;
  // BetaE Project stash: per project slot (node aux) H, Z [2d] each
  float* pstash;
  int32_t pstash_slots;
  // fused score+loss: per-(node, part) partials of dL/dq [items][wq] and of
  // (loss, coefficient sum) [items][2], and per-node arrival counters (zero
  // between launches)
  float* lpart;
  float* lpart_scalar;
  int32_t* lcount;
  int32_t lpart_items;
};

// Device view of the sharded step's owner work (ngdb_shard_plan + buffers).
struct ShardDev {
  int32_t world, rank, batch, max_slots;
  int32_t n_send, n_recv;
  int64_t dq_block;         // floats per rank block of dq_part: max_slots*wq + batch
  const int32_t* send_rows; // [n_send] local entity rows of the lookup send, requester-major
  const int32_t* recv_slot; // [n_recv] this rank's anchor slots, owner-major
  const int32_t* unit_k;
  const int32_t* unit_slots;
  const int32_t* cand;
  const int32_t* unit_off;
  const int32_t* owned;
  const float* query_all;  // [world*max_slots][wq]
  float* dq_part;          // [world][max_slots*wq + batch]: partial dL/dq, then partial losses
  float* coef_all;         // [world*max_slots][ncand]
};

// Programmatic dependent launch: let the next kernel in the stream start its
// launch/prologue now, then wait until the previous kernel's results are
// visible. Every kernel of the step calls this before touching step data.
__device__ __forceinline__ void pdl_start() {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// The two halves of pdl_start(), for kernels that read step-invariant plan
// data (node descriptors, CSR) before waiting: the descriptor loads then
// overlap the previous kernel's tail. Nothing written by an earlier kernel may
// be read before pdl_wait().
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float4 ldg4(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
// streaming load: do not allocate in L1 (each row is touched once per kernel)
__device__ __forceinline__ float4 ld_stream4(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// --- mbarrier + bulk async copy (TMA 1-D) helpers ---------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
// global -> shared bulk copy (16-byte aligned, size a multiple of 16) that
// completes `bytes` of transaction count on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ float sgnf(float x) { return (x > 0.f) - (x < 0.f); }
// numerically stable softplus and logistic
__device__ __forceinline__ float softplusf(float x) {
  return x > 0.f ? x + log1pf(expf(-x)) : log1pf(expf(x));
}
__device__ __forceinline__ float sigmoidf(float x) {
  return x >= 0.f ? 1.f / (1.f + expf(-x)) : expf(x) / (1.f + expf(x));
}

}  // namespace ngdb_dev

// ---- launchers (defined in the k_*.cu files) --------------------------------
namespace ngdb_dev {

// Launch with programmatic stream serialization (PDL) and an optional 1-D
// cluster; kernels pair this with pdl_start().
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int n = 0;
  attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[n].val.programmaticStreamSerializationAllowed = 1;
  ++n;
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

struct LaunchCtx {
  cudaStream_t stream;
  int num_sms;
};
// Cardinality layout of an Intersect invocation: one class (k2 == k1), or the
// two classes of one PopBatch run as one set of launches — nodes [0, n1) take
// k1 inputs, the rest k2. Per-input rows are node-major: node i owns rows
// [row0(i), row0(i) + k(i)).
struct KSpan {
  int n1, k1, k2;
  __host__ __device__ int k(int i) const { return i < n1 ? k1 : k2; }
  __host__ __device__ int row0(int i) const { return i < n1 ? i * k1 : n1 * k1 + (i - n1) * k2; }
  static KSpan single(int n, int k) { return KSpan{n, k, k}; }
};
// rows.cu
// evaluator (evaluate.cu): full-entity scoring + filtered rank counts
struct EvalArgs {
  // entity table [n_ent][ent_w]: GQE/Q2B rows are d-wide points; BetaE: the
  // entity side T_e [2d] of the linearised KL (dim = 2d then); fusion: fused rows
  const float* ent;
  int64_t ent_w;
  int32_t n_ent, dim, backbone;
  float alpha;       // Q2B inside weight
  const float* q;    // [nq][wq] query slots: GQE q; Q2B centre | offset
  int32_t wq, nq;    // nq = slots (a union query has one slot per DNF branch)
  int32_t n_queries;
  const int32_t* slot_query;  // [nq] query of the slot, -1 = padding
  const int32_t* slot_nb;     // [nq] branches starting at this slot (its query's first), else 0
  const int32_t* first_slot;  // [n_queries]
  const int32_t* target;      // per query
  const int32_t* f_off;  // [n_queries + 1] CSR of filter entities
  const int32_t* f_ids;
  const float* ec;       // BetaE: [n_ent] C_e
  float* dt;             // [n_queries] target distances (nearest branch)
  int32_t* better;       // [n_queries]
  int32_t* ties;         // [n_queries]
};
int launch_eval_ranks(const EvalArgs& a, int32_t n_filter, cudaStream_t s);

int launch_embed(const DevArgs& a, int dir, int first, int n, const LaunchCtx& lc);
int launch_project(const DevArgs& a, int dir, int first, int n, const LaunchCtx& lc);
int launch_negate(const DevArgs& a, int dir, int first, int n, const LaunchCtx& lc);
int launch_union(const DevArgs& a, int dir, int k, int first, int n, const LaunchCtx& lc);
int launch_loss_bwd(const DevArgs& a, int first, int n, const LaunchCtx& lc);
// score.cu
int launch_loss_fwd(const DevArgs& a, int first, int n, const LaunchCtx& lc);
int launch_score(const DevArgs& a, int dir, int first, int n, const LaunchCtx& lc);
// beta.cu (BetaE backbone)
int launch_beta_project(const DevArgs& a, int dir, int first, int n, const LaunchCtx& lc);
int launch_beta_intersect(const DevArgs& a, int dir, KSpan ks, int first, int n, const LaunchCtx& lc);
int64_t beta_scratch_floats(int dim, int max_nodes);
// the Project MLP's share alone (ctx scratch2, sized for merged drains)
int64_t beta_project_scratch_floats(int dim, int max_nodes);
// intersect.cu
int launch_intersect(const DevArgs& a, int dir, KSpan ks, int first, int n, const LaunchCtx& lc);
// scratch floats the intersect operators need for classes of up to max_nodes
int64_t intersect_scratch_floats(int backbone, int dim, int max_nodes);
// tc_gemm.cu: refresh the hi/lo (and transposed) splits of dense weight i
int split_weight(const float* w, int rows, int cols, float* dst, cudaStream_t s);
void tc_gemm_init();
// optim.cu
struct SparseTable {
  float* w; float* m; float* v; float* dbg_g;
  int32_t width;
  int32_t n_rows;
  const int32_t* rows; const int32_t* seg; const int32_t* contrib;
};
struct AdamHyper {
  float lr, b1, b2, eps;
};
// bc: device pointer to {1 - b1^t, 1 - b2^t} for the current step t
int launch_sparse_adam_entity(const DevArgs& a, const SparseTable& t, const AdamHyper& hp,
                              const float* bc, const LaunchCtx& lc);
int launch_sparse_adam_relation(const DevArgs& a, const SparseTable& t, const AdamHyper& hp,
                                const float* bc, const LaunchCtx& lc);
// BetaE: per-step entity table + candidate -> CSR-row map (before any pool)
int launch_beta_prep(const DevArgs& a, const SparseTable& t, const LaunchCtx& lc);
// fuse.cu: step prologue (etab = e_fused of the touched rows) and the fused
// backward + entity Adam
int64_t fuse_scratch_floats(int d, int dl, int64_t rows);
// whole-table CSR segments (row e = entity e) from a step's compact entity CSR
int launch_expand_rows(const int32_t* rows, const int32_t* seg, int u, int32_t* seg_full, int n,
                       cudaStream_t s);
// BetaE with FuseSemantic: the Psi_theta output rows Y [u][2d] inside the scratch
float* fuse_y_table(float* fs, int64_t cap, int u, int d, int dl);

int fuse_prologue(const DevArgs& a, const SparseTable& t, float* fs, int64_t cap, const LaunchCtx& lc);
// adam = false (row-sharded step): the dense gradients and dh only; the
// entity rows' Adam then runs as fuse_entity_adam after the all-reduce
int fuse_backward(const DevArgs& a, const SparseTable& t, float* fs, int64_t cap, const AdamHyper& hp,
                  const float* bc, const LaunchCtx& lc, bool adam = true);
int fuse_entity_adam(const SparseTable& t, float* fs, int64_t cap, int d, int dl, bool beta,
                     const AdamHyper& hp, const float* bc, const LaunchCtx& lc);
int launch_beta_entity_adam(const DevArgs& a, const SparseTable& t, const AdamHyper& hp,
                            const float* bc, const LaunchCtx& lc);
// shard.cu (row-sharded step)
int launch_shard_anchor_pack(const DevArgs& a, const ShardDev& sd, float* send, const LaunchCtx& lc);
int launch_shard_query_pack(const DevArgs& a, int first, int n, float* dst, const LaunchCtx& lc);
int launch_shard_score(const DevArgs& a, const ShardDev& sd, const LaunchCtx& lc);
int launch_shard_score_done(const DevArgs& a, const float* dq_mine, int64_t n_dq,
                            const float* loss_mine, int nq, const LaunchCtx& lc);
int launch_shard_grad_pack(const DevArgs& a, const ShardDev& sd, float* send, const LaunchCtx& lc);
int launch_shard_rel_pack(const DevArgs& a, const SparseTable& t, float* rel_g, float* touched,
                          const LaunchCtx& lc);
int launch_masked_rows_adam(float* w, float* m, float* v, float* dbg, const float* g,
                            const float* touched, int rows, int width, const AdamHyper& hp,
                            const float* bc, const LaunchCtx& lc);
int launch_dense_adam(float* w, float* m, float* v, float* g, int64_t n, const AdamHyper& hp,
                      const float* bc, const LaunchCtx& lc);
// dense tensors of the flat buffer: Adam + (weights) the 3xTF32 split refresh
struct DenseJob {
  int64_t off;        // element offset in the flat dense buffers
  int rows, cols;
  int64_t split_off;  // W_hi offset in the split buffer (W_lo, W^T_hi, W^T_lo follow); -1: none
  int tile_begin;     // first 32x32 tile of this tensor in the launch grid
};
struct DenseJobs {
  DenseJob job[kMaxDenseTensors];
  int n, tiles;
};
int launch_dense_adam_split(float* w, float* m, float* v, const float* g, float* wsplit,
                            const DenseJobs& jobs, const AdamHyper& hp, const float* bc,
                            const LaunchCtx& lc);
}  // namespace ngdb_dev
