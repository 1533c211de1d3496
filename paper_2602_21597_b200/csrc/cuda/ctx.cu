#include <cstdlib>
#include <cstdio>
// Device context and the C ABI of include/ngdb/ngdb_cuda.h.
//
// The context owns all device memory for one training run on one GPU:
// parameters + Adam moments, the activation arena
// whose slots the host planner assigned (SPEC.md:257-330 as static offsets),
// the per-step gradient staging buffers, and the packed step plans. All launches
// go to one non-blocking stream; a step issues no host synchronisation until
// ngdb_step_end.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "nccl_loader.hpp"
#include "tc_gemm.cuh"

using namespace ngdb_dev;

namespace {

thread_local std::string g_last_error;

struct Fail {
  int code;
  std::string msg;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Fail{NGDB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}
#define CK(x) ck((x), #x)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return NGDB_OK;
  } catch (const Fail& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return NGDB_ERR_CUDA;
  }
}

enum Family : int {
  F_EMBED = 0, F_PROJECT, F_NEGATE, F_INTERSECT, F_SCORE, F_UNION, F_LOSS_FWD, F_LOSS_BWD,
  F_OPT_ENTITY, F_OPT_RELATION, F_OPT_DENSE, F_ENTITY_PREP, F_COUNT
};
const char* kFamilyNames[F_COUNT] = {"embed",     "project",   "negate",      "intersect",
                                     "score",     "union",     "loss_fwd",    "loss_bwd",
                                     "opt_entity", "opt_relation", "opt_dense", "entity_prep"};

struct Param {
  std::string name;
  int64_t rows = 0, cols = 0;
  bool sparse = false;
  int dense_idx = -1;
  float *w = nullptr, *m = nullptr, *v = nullptr, *g = nullptr;
  int64_t n() const { return rows * cols; }
};

template <class T>
T* dmalloc(int64_t count) {
  void* p = nullptr;
  if (count <= 0) count = 1;
  CK(cudaMalloc(&p, static_cast<size_t>(count) * sizeof(T)));
  return static_cast<T*>(p);
}

// Packed plan blob: [nodes][cand][erows][eseg][econ][rrows][rseg][rcon] (int32)
struct PlanLayout {
  int64_t nodes, cand, erows, eseg, econ, rrows, rseg, rcon, total;
  static int64_t up4(int64_t x) { return (x + 3) / 4 * 4; }
  explicit PlanLayout(const ngdb_step_plan& p) {
    int64_t o = 0;
    nodes = o; o += up4(int64_t(p.n_nodes) * 8);
    cand = o; o += up4(int64_t(p.n_queries) * p.n_candidates);
    erows = o; o += up4(p.n_entity_rows);
    eseg = o; o += up4(p.n_entity_rows + 1);
    econ = o; o += up4(p.n_entity_rows ? p.entity_seg[p.n_entity_rows] : 0);
    rrows = o; o += up4(p.n_relation_rows);
    rseg = o; o += up4(p.n_relation_rows + 1);
    rcon = o; o += up4(p.n_relation_rows ? p.relation_seg[p.n_relation_rows] : 0);
    total = o;
  }
};

void pack_plan(const ngdb_step_plan& p, const PlanLayout& L, int32_t* dst) {
  std::memcpy(dst + L.nodes, p.nodes, sizeof(ngdb_node_desc) * p.n_nodes);
  std::memcpy(dst + L.cand, p.candidates, sizeof(int32_t) * int64_t(p.n_queries) * p.n_candidates);
  if (p.n_entity_rows) {
    std::memcpy(dst + L.erows, p.entity_rows, sizeof(int32_t) * p.n_entity_rows);
    std::memcpy(dst + L.eseg, p.entity_seg, sizeof(int32_t) * (p.n_entity_rows + 1));
    std::memcpy(dst + L.econ, p.entity_contrib, sizeof(int32_t) * p.entity_seg[p.n_entity_rows]);
  }
  if (p.n_relation_rows) {
    std::memcpy(dst + L.rrows, p.relation_rows, sizeof(int32_t) * p.n_relation_rows);
    std::memcpy(dst + L.rseg, p.relation_seg, sizeof(int32_t) * (p.n_relation_rows + 1));
    std::memcpy(dst + L.rcon, p.relation_contrib,
                sizeof(int32_t) * p.relation_seg[p.n_relation_rows]);
  }
}

// Host-side summary of a plan the device copy needs for dispatch.
struct PlanMeta {
  std::vector<ngdb_pool_desc> pools;
  int32_t n_queries = 0, n_candidates = 0, n_nodes = 0;
  int32_t n_score = 0, n_anchor = 0, n_project = 0;
  int32_t n_erows = 0, n_rrows = 0, n_econ = 0, n_rcon = 0;
  int64_t arena_elems = 0;
  std::vector<int32_t> node_counts_by_kind;  // for algorithmic-byte accounting
  std::vector<int32_t> dep_off, deps;        // pool dependencies (empty: serial)
};

PlanMeta meta_of(const ngdb_step_plan& p) {
  PlanMeta m;
  m.pools.assign(p.pools, p.pools + p.n_pools);
  m.n_queries = p.n_queries;
  m.n_candidates = p.n_candidates;
  m.n_nodes = p.n_nodes;
  m.n_score = p.n_score_slots;
  m.n_anchor = p.n_anchor_slots;
  m.n_project = p.n_project_slots;
  m.n_erows = p.n_entity_rows;
  m.n_rrows = p.n_relation_rows;
  m.n_econ = p.n_entity_rows ? p.entity_seg[p.n_entity_rows] : 0;
  m.n_rcon = p.n_relation_rows ? p.relation_seg[p.n_relation_rows] : 0;
  m.arena_elems = p.arena_elems;
  if (p.pool_dep_off && p.pool_deps) {
    m.dep_off.assign(p.pool_dep_off, p.pool_dep_off + p.n_pools + 1);
    m.deps.assign(p.pool_deps, p.pool_deps + m.dep_off.back());
  }
  return m;
}

void validate_plan(const ngdb_step_plan& p) {
  if (p.n_queries < 0 || p.n_nodes < 0 || p.n_pools < 0 || p.n_candidates < 2)
    throw Fail{NGDB_ERR_SHAPE_MISMATCH, "invalid plan sizes"};
  for (int i = 0; i < p.n_pools; ++i) {
    const ngdb_pool_desc& d = p.pools[i];
    if (d.first < 0 || d.count < 0 || d.first + d.count > p.n_nodes)
      throw Fail{NGDB_ERR_INDEX_OUT_OF_RANGE, "pool descriptor out of range"};
  }
  if (p.pool_dep_off && p.pool_deps) {
    if (p.pool_dep_off[0] != 0) throw Fail{NGDB_ERR_SHAPE_MISMATCH, "pool_dep_off[0] != 0"};
    for (int i = 0; i < p.n_pools; ++i) {
      if (p.pool_dep_off[i + 1] < p.pool_dep_off[i])
        throw Fail{NGDB_ERR_SHAPE_MISMATCH, "pool_dep_off not ascending"};
      for (int k = p.pool_dep_off[i]; k < p.pool_dep_off[i + 1]; ++k)
        if (p.pool_deps[k] < 0 || p.pool_deps[k] >= i)
          throw Fail{NGDB_ERR_INDEX_OUT_OF_RANGE, "pool dependency must name an earlier pool"};
    }
  }
}

}  // namespace

struct ngdb_plan {
  int32_t* blob = nullptr;
  PlanLayout layout{ngdb_step_plan{}};
  PlanMeta meta;
  // CUDA graph of the whole step (resident plans), valid while the context's
  // buffer generation is unchanged
  cudaGraphExec_t graph = nullptr;
  int64_t graph_gen = -1;
  int64_t graph_launches = 0;
};

struct ngdb_ctx {
  ngdb_model_desc desc{};
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  std::vector<Param> params;
  int ent_idx = -1, rel_idx = -1;
  float *dense_w = nullptr, *dense_m = nullptr, *dense_v = nullptr, *dense_g = nullptr;
  int64_t dense_n = 0;
  int64_t dense_off[kMaxDenseTensors] = {};
  float* sem = nullptr;
  int64_t sem_n = 0;
  float* wsplit = nullptr;
  int64_t wsplit_off[kMaxDenseTensors] = {};
  // per-step staging
  float *qbuf = nullptr, *dqbuf = nullptr, *coefbuf = nullptr, *ddbuf = nullptr, *agbuf = nullptr,
        *rgbuf = nullptr, *loss_out = nullptr;
  int32_t* flags = nullptr;
  int64_t cap_score = 0, cap_anchor = 0, cap_project = 0, cap_queries = 0, cap_cand = 0;
  float* scratch = nullptr;
  int64_t scratch_cap = 0;
  float* scratch2 = nullptr;  // BetaE Project GEMM scratch (independent of the intersect's)
  float* sem_split = nullptr;  // frozen store splits: hi, lo [N][dl]
  // whole-table fusion form (a step touching >= 90 % of the entities fuses every
  // entity: no per-step gather / split of the store, rows = identity)
  int32_t* iota_rows = nullptr;  // [N] 0..N-1
  int32_t* seg_full = nullptr;   // [N+1]
  int64_t scratch2_cap = 0;
  float* arena = nullptr;
  int64_t arena_cap = 0;
  // BetaE per-step entity table (beta.cu) and candidate -> CSR-row map
  float *etab = nullptr, *etab_c = nullptr;
  int32_t* cand_local = nullptr;
  int64_t cap_erows = 0;
  // FuseSemantic: anchor slot -> etab row, fusion scratch (fuse.cu)
  int32_t* anchor_local = nullptr;
  float* fscratch = nullptr;
  int64_t fscratch_cap = 0;
  int fus_idx = -1;
  // row-sharded step (shard.cu)
  int world = 1, rank = 0;
  cudaStream_t own_stream = nullptr;
  // concurrent pools (exec_pools_concurrent): side streams, one event per
  // invocation of the widest plan seen, fork / join events
  static constexpr int kSide = 3;
  cudaStream_t side[kSide] = {nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> inv_ev;
  cudaEvent_t fork_ev = nullptr, join_ev[kSide] = {nullptr, nullptr, nullptr};
  bool concurrent = true;  // NGDB_SERIAL_POOLS=1 turns it off
  // streaming plans are uploaded on a copy stream one step ahead, overlapping
  // the previous step's kernels: blob_free[i] marks the end of the last step
  // that read stream_plan[i], blob_ready[i] the end of its upload
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t blob_free[2] = {nullptr, nullptr}, blob_ready[2] = {nullptr, nullptr};
  const float* anc_rows = nullptr;  // set while a sharded step runs
  const int32_t* anc_pos = nullptr;
  // NCCL communicators owned by the context (ngdb_comm_init): `comm` carries
  // the step's collectives on the context stream, `meta_comm` the host
  // metadata all-gather of upcoming steps on its own stream (another thread)
  ncclComm_t comm = nullptr, meta_comm = nullptr;
  cudaStream_t meta_stream = nullptr;
  std::mutex meta_mu;
  int32_t* meta_dev = nullptr;
  int64_t meta_cap = 0;
  float* istash = nullptr;           // Intersect stash (DevArgs::istash)
  int32_t istash_slots = 0;
  float* pstash = nullptr;           // BetaE Project stash (DevArgs::pstash)
  int32_t pstash_slots = 0;
  int32_t proj_merge_cap = 0;        // BetaE Project nodes one merged launch may cover
  float* lpart = nullptr;            // fused score+loss partials (DevArgs::lpart)
  float* lpart_scalar = nullptr;
  int32_t* lcount = nullptr;
  int32_t lpart_items = 0;
  struct ShardState {
    int32_t* blobs[2] = {nullptr, nullptr};  // owner lists of streaming steps (double-buffered)
    int64_t blobs_cap[2] = {0, 0};
    int32_t* staging[2] = {nullptr, nullptr};  // pinned, alternating with the plan staging
    int64_t staging_cap[2] = {0, 0};
    cudaEvent_t staged[2] = {nullptr, nullptr};
    float* buf = nullptr;
    int64_t buf_cap = 0;
    ShardDev dev{};
    ngdb_shard_buffers bufs{};
    std::vector<int32_t> send_cnt, recv_cnt;  // host copies: NCCL send/recv counts (rows)
    float* coef_all = nullptr;
    // BetaE: the step entity table of the rows this rank owns (beta_prep over
    // the shard CSR) and global score code -> table row
    float *etab = nullptr, *etab_c = nullptr;
    int32_t* cand_local = nullptr;
    // FuseSemantic: the fusion scratch over the owned rows, lookup-send position -> CSR row
    float* fscratch = nullptr;
    int64_t fscratch_cap = 0;
    int32_t* anchor_local = nullptr;
    int32_t n_rows = 0;
    const int32_t *rows = nullptr, *seg = nullptr, *contrib = nullptr;
    bool active = false;
  } sh;
  // streaming plans: double-buffered pinned staging + device blobs
  int32_t* staging[2] = {nullptr, nullptr};
  int64_t staging_cap[2] = {0, 0};
  cudaEvent_t staged[2] = {nullptr, nullptr};
  ngdb_plan stream_plan[2];
  int64_t stream_cap[2] = {0, 0};
  int cur = 0;
  ngdb_plan* active = nullptr;
  // streaming ABI: an Intersect class held back one call so the next class of
  // the same PopBatch can share its launches (exec_pools / mergeable)
  ngdb_pool_desc held{};
  bool has_held = false;
  // ngdb_step_begin_ex(NGDB_BEGIN_DEFER_PROLOGUE): the step prologue (flag and
  // dense-gradient resets, step table) runs inside ngdb_step_launch's graph
  bool prologue_pending = false;
  // asynchronous step ends: a ring of pinned result slots (losses + flags)
  static constexpr int kResultSlots = 4;
  struct ResultSlot {
    float* host = nullptr;  // [cap] losses, then 4 int32 flags
    int64_t cap = 0;
    int32_t n_queries = 0;
    int64_t ticket = -1;    // outstanding ticket, -1 when free
    cudaEvent_t done = nullptr;
  } results[kResultSlots];
  int64_t next_ticket = 0;
  // streaming steps launched as CUDA graphs (ngdb_step_launch): two
  // alternating executable graphs, updated in place when the topology allows
  // small cache of executable step graphs keyed by the step's invocation
  // structure: a step whose structure was seen before is launched through
  // cudaGraphExecUpdate (new parameters, same topology) instead of a fresh
  // instantiation; an entry is only touched once its last launch completed
  struct ExecEntry {
    uint64_t sig = 0;
    cudaGraphExec_t exec = nullptr;
    cudaEvent_t done = nullptr;
    int64_t used = 0;
  };
  static constexpr int kExecCache = 16;
  ExecEntry exec_cache[kExecCache];
  int64_t exec_clock = 0;
  int64_t exec_updates = 0, exec_instantiations = 0;
  uint64_t launch_sig = 0;  // FNV-1a over the merged invocation structure (exec_pools)
  bool debug = false;
  // timing / accounting
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  bool profiling = false;
  struct Rec { int fam; cudaEvent_t a, b; double bytes; int launches; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> event_pool;
  double fam_ms[F_COUNT] = {}, fam_bytes[F_COUNT] = {}, fam_flops[F_COUNT] = {};
  int64_t fam_launches[F_COUNT] = {};
  int64_t launches = 0;
  int64_t h2d_bytes = 0, d2h_bytes = 0;  // step data copied by the streaming ABI
  float* d_bc = nullptr;        // Adam bias corrections of the current step
  int64_t buffer_gen = 0;       // bumped whenever a buffer captured by a graph moves
  bool use_graphs = true;
  float* l2_flush = nullptr;
  int64_t l2_flush_bytes = 0;
  // step timeline (NGDB_STEP_TIMELINE=1): timing events around each graph-launched step
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timeline;
  // pinned ring of pre-packed plans (ngdb_ctx_pinned_ring; the trainer loop)
  int32_t* pinned_ring = nullptr;
  int64_t pinned_ring_ints = 0;
  // evaluator staging (ngdb_eval_ranks)
  char* eval_buf = nullptr;
  // evaluator entity table of the BetaE / fusion backbones over ALL entities
  // (T_e | C_e, or the fused rows), its row list and the fusion scratch
  float* evtab = nullptr;
  int32_t* ev_rows = nullptr;
  float* ev_scratch = nullptr;
  int64_t ev_scratch_cap = 0;
  int64_t eval_cap = 0;

  Param* find(const std::string& name) {
    for (auto& p : params)
      if (p.name == name) return &p;
    return nullptr;
  }
  int32_t query_width() const {
    return desc.backbone == NGDB_GQE ? desc.dim : 2 * desc.dim;
  }
  bool beta() const { return desc.backbone == NGDB_BETAE; }
  bool fused() const { return desc.semantic_dim > 0; }
  bool step_table() const { return beta() || fused(); }  // per-step entity table
  // width of the entity rows the operators see (anchors, candidates, anchor
  // gradients, the step table): BetaE 2d (with FuseSemantic: Psi_theta's rows)
  int64_t op_ent_w() const { return beta() ? 2 * int64_t(desc.dim) : params[ent_idx].cols; }
  cudaEvent_t take_event() {
    if (!event_pool.empty()) {
      cudaEvent_t e = event_pool.back();
      event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
  }
  void drain_profile() {
    if (recs.empty()) return;
    CK(cudaStreamSynchronize(stream));
    for (auto& r : recs) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, r.a, r.b));
      fam_ms[r.fam] += ms;
      fam_bytes[r.fam] += r.bytes;
      fam_launches[r.fam] += r.launches;
      event_pool.push_back(r.a);
      event_pool.push_back(r.b);
    }
    recs.clear();
  }
};

namespace {

void add_param(ngdb_ctx* c, const char* name, int64_t rows, int64_t cols, bool sparse) {
  Param p;
  p.name = name;
  p.rows = rows;
  p.cols = cols;
  p.sparse = sparse;
  c->params.push_back(p);
}

void ensure_f(float*& p, int64_t& cap, int64_t need) {
  if (need <= cap) return;
  if (p) CK(cudaFree(p));
  cap = std::max<int64_t>(need + need / 2, cap + cap / 2);
  p = dmalloc<float>(cap);
}

// Rows the fusion prologue / backward work on: every entity (whole-table form)
// when the step touches >= 90 % of them and the store's split exists, else the
// step's touched rows.
bool fusion_whole(const ngdb_ctx* c, const PlanMeta& m) {
  return c->fused() && c->iota_rows && int64_t(m.n_erows) * 10 >= int64_t(c->desc.n_entities) * 9;
}

void ensure_step_buffers(ngdb_ctx* c, const PlanMeta& m) {
  const int64_t wq = c->query_width();
  const int64_t ew = c->op_ent_w(), rw = c->params[c->rel_idx].cols;
  bool grow = m.n_score > c->cap_score || m.n_anchor > c->cap_anchor ||
              m.n_project > c->cap_project || m.n_queries > c->cap_queries ||
              m.n_candidates != c->cap_cand;
  if (grow) {
    CK(cudaStreamSynchronize(c->stream));
    auto realloc_f = [&](float*& p, int64_t n) {
      if (p) CK(cudaFree(p));
      p = dmalloc<float>(n);
    };
    // grow with headroom: every growth is a device sync + reallocation, and
    // streaming plans vary from step to step. First sizing covers any batch of
    // max_queries queries (<= 2 score slots, 3 anchors, 4 projects per query
    // after DNF, query.hpp:14-29)
    auto grow_to = [](int64_t need, int64_t cap, int64_t floor) {
      return need <= cap ? cap : std::max<int64_t>({need + need / 4, cap + cap / 4, floor});
    };
    const int64_t B = std::max<int64_t>(c->desc.max_queries, 1);
    c->cap_score = grow_to(m.n_score, c->cap_score, 2 * B);
    c->cap_anchor = grow_to(m.n_anchor, c->cap_anchor, 3 * B);
    c->cap_project = grow_to(m.n_project, c->cap_project, 4 * B);
    c->cap_queries = grow_to(m.n_queries, c->cap_queries, B);
    c->cap_cand = m.n_candidates;
    realloc_f(c->qbuf, c->cap_score * wq);
    realloc_f(c->dqbuf, c->cap_score * wq);
    realloc_f(c->coefbuf, c->cap_score * c->cap_cand);
    realloc_f(c->ddbuf, c->cap_queries * c->cap_cand);
    realloc_f(c->agbuf, c->cap_anchor * ew);
    realloc_f(c->rgbuf, c->cap_project * rw);
    realloc_f(c->loss_out, c->cap_queries);
    if (c->step_table()) {
      if (c->cand_local) CK(cudaFree(c->cand_local));
      c->cand_local = dmalloc<int32_t>(c->cap_score * c->cap_cand);
    }
    if (c->fused()) {
      if (c->anchor_local) CK(cudaFree(c->anchor_local));
      c->anchor_local = dmalloc<int32_t>(c->cap_anchor);
    }
    ++c->buffer_gen;
  }
  const int64_t erows = fusion_whole(c, m) ? int64_t(c->desc.n_entities) : m.n_erows;
  // (row-sharded: the step table lives in the shard buffers, sized per step)
  if (c->step_table() && c->world == 1 && erows > c->cap_erows) {
    CK(cudaStreamSynchronize(c->stream));
    c->cap_erows = std::max<int64_t>(erows, c->cap_erows + c->cap_erows / 4);
    if (c->etab) CK(cudaFree(c->etab));
    if (c->etab_c) CK(cudaFree(c->etab_c));
    c->etab = dmalloc<float>(c->cap_erows * ew);
    c->etab_c = dmalloc<float>(c->cap_erows);
    if (c->fused()) {
      if (c->fscratch) CK(cudaFree(c->fscratch));
      c->fscratch_cap = fuse_scratch_floats(c->desc.dim, c->desc.semantic_dim, c->cap_erows);
      c->fscratch = dmalloc<float>(c->fscratch_cap);
    }
    ++c->buffer_gen;
  }
  if (m.arena_elems > c->arena_cap) {
    CK(cudaStreamSynchronize(c->stream));
    ensure_f(c->arena, c->arena_cap, m.arena_elems + 64);
    ++c->buffer_gen;
  }
}

DevArgs make_args(ngdb_ctx* c, const ngdb_plan* p) {
  DevArgs a{};
  a.backbone = c->desc.backbone;
  a.dim = c->desc.dim;
  a.wq = c->query_width();
  a.ent_w = static_cast<int32_t>(c->op_ent_w());
  a.rel_w = static_cast<int32_t>(c->params[c->rel_idx].cols);
  a.ncand = p ? p->meta.n_candidates : 0;
  a.n_neg = c->desc.n_neg;
  a.n_entities = c->desc.n_entities;
  a.n_relations = c->desc.n_relations;
  a.gamma = c->desc.gamma;
  a.alpha_box = c->desc.alpha_box;
  a.arena = c->arena;
  a.nodes = p ? reinterpret_cast<const ngdb_node_desc*>(p->blob + p->layout.nodes) : nullptr;
  a.cand = p ? p->blob + p->layout.cand : nullptr;
  a.ent = c->params[c->ent_idx].w;
  a.rel = c->params[c->rel_idx].w;
  a.dense = c->dense_w;
  a.dense_g = c->dense_g;
  for (int i = 0; i < kMaxDenseTensors; ++i) {
    a.dense_off[i] = c->dense_off[i];
    a.wsplit_off[i] = c->wsplit_off[i];
  }
  a.wsplit = c->wsplit;
  a.qbuf = c->qbuf;
  a.dqbuf = c->dqbuf;
  a.coefbuf = c->coefbuf;
  a.ddbuf = c->ddbuf;
  a.agbuf = c->agbuf;
  a.rgbuf = c->rgbuf;
  a.loss_out = c->loss_out;
  a.flags = c->flags;
  a.scratch = c->scratch;
  a.scratch_cap = c->scratch_cap;
  a.etab = c->etab;
  a.etab_c = c->etab_c;
  a.cand_local = c->cand_local;
  if (c->sh.active) {  // a row-sharded step (any world size): its own step table
    a.etab = c->sh.etab;
    a.etab_c = c->sh.etab_c;
    a.cand_local = c->sh.cand_local;
    a.anchor_local = c->sh.anchor_local;
  }
  a.fused = c->fused() ? 1 : 0;
  a.sem_dim = c->desc.semantic_dim;
  a.sem = c->sem;
  if (c->sem_split) {
    const int64_t N = c->desc.n_entities, L = c->desc.semantic_dim;
    a.sem_hi = c->sem_split;
    a.sem_lo = a.sem_hi + N * L;
  }
  a.anchor_local = c->anchor_local;
  a.fus_idx = c->fus_idx;
  a.anc_rows = c->anc_rows;
  a.anc_pos = c->anc_pos;
  a.ytab = (c->beta() && c->fused() && p && c->fscratch)
               ? fuse_y_table(c->fscratch, c->fscratch_cap,
                              fusion_whole(c, p->meta) ? c->desc.n_entities : p->meta.n_erows,
                              c->desc.dim, c->desc.semantic_dim)
               : nullptr;
  if (c->sh.active)  // row-sharded: the fusion runs over the owned rows of the shard CSR
    a.ytab = (c->beta() && c->fused() && c->sh.fscratch)
                 ? fuse_y_table(c->sh.fscratch, c->sh.fscratch_cap, c->sh.n_rows, c->desc.dim,
                                c->desc.semantic_dim)
                 : nullptr;
  a.istash = c->istash;
  a.istash_slots = c->istash_slots;
  a.pstash = c->pstash;
  a.pstash_slots = c->pstash_slots;
  a.lpart = c->lpart;
  a.lpart_scalar = c->lpart_scalar;
  a.lcount = c->lcount;
  a.lpart_items = c->lpart_items;
  return a;
}

// Algorithmic bytes of one invocation (unique bytes a kernel must
// move; L2 re-reads inside a kernel are not counted).
double pool_bytes(const ngdb_ctx* c, const ngdb_pool_desc& d, int ncand) {
  const double wq = c->query_width() * 4.0, ew = c->params[c->ent_idx].cols * 4.0,
               rw = c->params[c->rel_idx].cols * 4.0, n = d.count, k = d.k;
  switch (d.kind) {
    case NGDB_OP_EMBED_ANCHOR: return n * (d.dir == 0 ? ew + wq : 2 * ew) + n * 32;
    case NGDB_OP_PROJECT: return n * (d.dir == 0 ? (wq + rw + wq) : (2 * wq + 2 * rw)) + n * 32;
    case NGDB_OP_NEGATE: return n * 2 * wq + n * 32;
    case NGDB_OP_INTERSECT: {
      // node rows in and out (+ the G slots backward), plus the MLP contractions'
      // operand traffic: every GEMM row reads its hi/lo split A row (8 B per
      // element), writes its fp32 output and a chained hi/lo split (12 B), and
      // every GEMM reads its hi/lo weight (8 B per weight element) — the
      // intermediates of the class, not only its inputs
      const double D = c->desc.dim, R = n * k;
      double rows, gemms, w = D;  // GEMM rows of width w, and GEMMs per launch set
      if (c->desc.backbone == NGDB_GQE) {
        rows = d.dir == 0 ? 2 * n : 4 * n;
        gemms = d.dir == 0 ? 2 : 4;
      } else if (c->beta()) {
        rows = d.dir == 0 ? 3 * R : 6 * R;
        gemms = d.dir == 0 ? 2 : 5;
        w = 2 * D;
      } else {
        rows = d.dir == 0 ? 3 * R + n : 6 * R + 2 * n;
        gemms = d.dir == 0 ? 4 : 8;
      }
      return n * (k + 1) * wq * (d.dir == 0 ? 1 : 2) + n * 32 + rows * w * 20.0 +
             gemms * w * w * 8.0;
    }
    case NGDB_OP_UNION_SCORE: return n * (k + 1) * ncand * 4.0 * (d.dir == 0 ? 1 : 2) + n * 32;
    case NGDB_OP_SCORE:
      return n * (ncand * (ew + 4) + wq * (d.dir == 0 ? 2 : 2) + ncand * 4.0) + n * 32;
    case NGDB_OP_LOSS:
      if (d.dir == 1) return n * 2 * wq + n * 32;
      return n * (ncand * (ew + 4) + 3 * wq + ncand * 4.0 + 8) + n * 32;
  }
  return 0.0;
}

int family_of(int kind, int dir) {
  switch (kind) {
    case NGDB_OP_EMBED_ANCHOR: return F_EMBED;
    case NGDB_OP_PROJECT: return F_PROJECT;
    case NGDB_OP_NEGATE: return F_NEGATE;
    case NGDB_OP_INTERSECT: return F_INTERSECT;
    case NGDB_OP_SCORE: return F_SCORE;
    case NGDB_OP_UNION_SCORE: return F_UNION;
    case NGDB_OP_LOSS: return dir == 0 ? F_LOSS_FWD : F_LOSS_BWD;
  }
  return F_EMBED;
}

template <class Launch>
void timed(ngdb_ctx* c, int fam, double bytes, Launch&& launch) {
  if (!c->profiling) {
    c->launches += launch();
    return;
  }
  cudaEvent_t a = c->take_event(), b = c->take_event();
  CK(cudaEventRecord(a, c->stream));
  const int n = launch();
  CK(cudaEventRecord(b, c->stream));
  c->launches += n;
  c->recs.push_back({fam, a, b, bytes, n});
}

// `merged` (optional): the next Intersect class of the same PopBatch, run in
// the same set of launches (see mergeable()).
void exec_pool(ngdb_ctx* c, const ngdb_plan* p, const ngdb_pool_desc& d,
               const ngdb_pool_desc* merged = nullptr) {
  if (d.count <= 0) return;
  const DevArgs a = make_args(c, p);
  const LaunchCtx lc{c->stream, c->num_sms};
  const int fam = family_of(d.kind, d.dir);
  const double bytes = c->profiling ? pool_bytes(c, d, p->meta.n_candidates) : 0.0;
  switch (d.kind) {
    case NGDB_OP_EMBED_ANCHOR:
      if (c->fused()) throw Fail{NGDB_ERR_CONFIG, "EmbedAnchor pool on a FuseSemantic context"};
      timed(c, fam, bytes, [&] { return launch_embed(a, d.dir, d.first, d.count, lc); });
      break;
    case NGDB_OP_FUSE_SEMANTIC:  // gather of the prologue's fused rows / its adjoint
      if (!c->fused()) throw Fail{NGDB_ERR_MISSING_KERNEL, "FuseSemantic pool without a semantic store"};
      timed(c, fam, bytes, [&] { return launch_embed(a, d.dir, d.first, d.count, lc); });
      break;
    case NGDB_OP_PROJECT: {
      if (c->profiling && c->beta())  // [q|r] 3d -> 2d -> 2d MLP, in units of 2 d^2 flops
        c->fam_flops[fam] += (d.dir == 0 ? 10.0 : 20.0) * d.count * 2.0 * c->desc.dim * c->desc.dim;
      DevArgs ap = a;
      if (c->scratch2) {
        ap.scratch = c->scratch2;
        ap.scratch_cap = c->scratch2_cap;
      }
      timed(c, fam, bytes, [&] { return launch_project(ap, d.dir, d.first, d.count, lc); });
      break;
    }
    case NGDB_OP_NEGATE:
      timed(c, fam, bytes, [&] { return launch_negate(a, d.dir, d.first, d.count, lc); });
      break;
    case NGDB_OP_INTERSECT: {
      if (d.k < 2 || d.k > 3) throw Fail{NGDB_ERR_SHAPE_MISMATCH, "intersect cardinality"};
      const KSpan ks = merged ? KSpan{d.count, d.k, merged->k} : KSpan::single(d.count, d.k);
      const int n_all = d.count + (merged ? merged->count : 0);
      if (c->profiling) {
        // algorithmic fp32 GEMM flops of the classes (2*M*N*K per contraction;
        // neither the 3xTF32 split nor any forward recomputation in backward
        // counts): DESIGN.md §4
        const double n = n_all, R = ks.row0(n_all), D2 = 2.0 * c->desc.dim * c->desc.dim;
        double gemm_rows;
        if (c->desc.backbone == NGDB_GQE) gemm_rows = d.dir == 0 ? 2 * n : 4 * n;
        else if (c->beta()) gemm_rows = d.dir == 0 ? 6 * R : 12 * R;  // 2d->2d->d attention
        else gemm_rows = d.dir == 0 ? 3 * R + n : 6 * R + 2 * n;
        c->fam_flops[fam] += gemm_rows * D2;
      }
      const double all_bytes =
          merged && c->profiling ? bytes + pool_bytes(c, *merged, p->meta.n_candidates) : bytes;
      timed(c, fam, all_bytes, [&] { return launch_intersect(a, d.dir, ks, d.first, n_all, lc); });
      break;
    }
    case NGDB_OP_SCORE:
      timed(c, fam, bytes, [&] { return launch_score(a, d.dir, d.first, d.count, lc); });
      break;
    case NGDB_OP_UNION_SCORE:
      if (d.k < 2 || d.k > 3) throw Fail{NGDB_ERR_SHAPE_MISMATCH, "union cardinality"};
      timed(c, fam, bytes, [&] { return launch_union(a, d.dir, d.k, d.first, d.count, lc); });
      break;
    case NGDB_OP_LOSS:
      if (d.dir == 0)
        timed(c, fam, bytes, [&] { return launch_loss_fwd(a, d.first, d.count, lc); });
      else
        timed(c, fam, bytes, [&] { return launch_loss_bwd(a, d.first, d.count, lc); });
      break;
    default:
      throw Fail{NGDB_ERR_MISSING_KERNEL,
                 "no kernel registered for operator kind " + std::to_string(d.kind)};
  }
  CK(cudaGetLastError());
}

// The cardinality classes of one Intersect PopBatch (consecutive invocations of
// the same direction over contiguous node ranges, ascending k) are independent
// of each other, so they share one set of launches: half the intersect
// launches and larger GEMMs. The invocation list (the trace) is unchanged.
bool mergeable(const ngdb_ctx* c, const ngdb_pool_desc& a, const ngdb_pool_desc& b) {
  return a.kind == NGDB_OP_INTERSECT && b.kind == NGDB_OP_INTERSECT && a.dir == b.dir &&
         a.cycle == b.cycle && a.count > 0 && b.count > 0 && b.first == a.first + a.count &&
         a.k < b.k && b.k <= 3 && a.k >= 2 && a.count + b.count <= c->desc.max_batch;
}

// The ⌈n/B_max⌉ pops that drain one pool snapshot (same cycle) are
// independent; for operators whose kernels have no per-invocation scratch they
// run as one launch over the concatenated node range.
bool drain_mergeable(const ngdb_ctx* c, const ngdb_pool_desc& a, const ngdb_pool_desc& b) {
  if (a.kind != b.kind || a.dir != b.dir || a.cycle != b.cycle || a.k != b.k) return false;
  if (a.count <= 0 || b.count <= 0 || b.first != a.first + a.count) return false;
  switch (a.kind) {
    case NGDB_OP_EMBED_ANCHOR:
    case NGDB_OP_FUSE_SEMANTIC:
    case NGDB_OP_NEGATE:
    case NGDB_OP_UNION_SCORE:
    case NGDB_OP_SCORE:
    case NGDB_OP_LOSS:
      return true;
    case NGDB_OP_PROJECT:  // the BetaE projection MLP: up to its scratch's node capacity
      return !c->beta() || a.count + b.count <= c->proj_merge_cap;
    default:
      return false;
  }
}

void flush_held(ngdb_ctx* c) {
  if (!c->has_held) return;
  c->has_held = false;
  exec_pool(c, c->active, c->held);
}

// Runs invocations in order, merging Intersect classes (mergeable()) and the
// pops of one drain (drain_mergeable()).
void sig_mix(ngdb_ctx* c, uint64_t x) {
  c->launch_sig = (c->launch_sig ^ x) * 1099511628211ull;
}

void exec_pools(ngdb_ctx* c, const ngdb_plan* p, const std::vector<ngdb_pool_desc>& v) {
  for (size_t i = 0; i < v.size(); ++i) {
    if (i + 1 < v.size() && mergeable(c, v[i], v[i + 1])) {
      sig_mix(c, 0x100u | (v[i].dir << 4) | v[i].kind);
      exec_pool(c, p, v[i], &v[i + 1]);
      ++i;
      continue;
    }
    ngdb_pool_desc d = v[i];
    while (i + 1 < v.size() && drain_mergeable(c, d, v[i + 1])) d.count += v[++i].count;
    sig_mix(c, (static_cast<uint64_t>(d.k) << 8) | (d.dir << 4) | d.kind);
    exec_pool(c, p, d);
  }
}

// Events for the invocations of a plan (created outside any stream capture).
void ensure_inv_events(ngdb_ctx* c, size_t n) {
  while (c->inv_ev.size() < n) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->inv_ev.push_back(e);
  }
}

// The plan's pools as a DAG over the context stream and its side streams
// (DESIGN.md §3.2 "concurrent pools"): invocation i waits only for the pools
// the planner named (data, slab-reuse and side-buffer hazards), so independent
// pools of the latency-bound small launches overlap. The MLP chain
// (intersect classes, BetaE projections: one GEMM scratch, dense-gradient
// accumulation) runs on side stream 0, the scoring chain (shared partials) on
// side stream 1; every other invocation follows its latest dependency's stream
// (none: the context stream). Kernels and their inputs are those of the serial
// order, so results are bit-identical.
void exec_pools_concurrent(ngdb_ctx* c, const ngdb_plan* p) {
  const auto& v = p->meta.pools;
  const auto& off = p->meta.dep_off;
  const auto& deps = p->meta.deps;
  struct Inv {
    ngdb_pool_desc d, m;
    bool merged;
    int p0, p1;  // pool index range [p0, p1]
  };
  std::vector<Inv> invs;
  std::vector<int> inv_of_pool(v.size());
  for (size_t i = 0; i < v.size(); ++i) {
    Inv in{v[i], ngdb_pool_desc{}, false, static_cast<int>(i), static_cast<int>(i)};
    if (i + 1 < v.size() && mergeable(c, v[i], v[i + 1])) {
      in.merged = true;
      in.m = v[i + 1];
      in.p1 = static_cast<int>(++i);
    } else {
      while (i + 1 < v.size() && drain_mergeable(c, in.d, v[i + 1])) {
        in.d.count += v[++i].count;
        in.p1 = static_cast<int>(i);
      }
    }
    for (int q = in.p0; q <= in.p1; ++q) inv_of_pool[q] = static_cast<int>(invs.size());
    invs.push_back(in);
  }
  const int n = static_cast<int>(invs.size());
  if (static_cast<int>(c->inv_ev.size()) < n)
    throw Fail{NGDB_ERR_CONFIG, "concurrent pools: invocation events not allocated"};
  std::vector<std::vector<int>> dep_inv(n);
  std::vector<char> waited_on(n, 0);
  for (int i = 0; i < n; ++i) {
    for (int q = invs[i].p0; q <= invs[i].p1; ++q)
      for (int k = off[q]; k < off[q + 1]; ++k) {
        const int d = inv_of_pool[deps[k]];
        if (d != i) dep_inv[i].push_back(d);
      }
    std::sort(dep_inv[i].begin(), dep_inv[i].end());
    dep_inv[i].erase(std::unique(dep_inv[i].begin(), dep_inv[i].end()), dep_inv[i].end());
  }
  cudaStream_t main = c->stream;
  cudaStream_t streams[1 + ngdb_ctx::kSide] = {main, c->side[0], c->side[1], c->side[2]};
  constexpr int S = 1 + ngdb_ctx::kSide;
  std::vector<int> stream_of(n, 0);
  auto chain_stream = [&](const ngdb_pool_desc& d) {
    if (d.kind == NGDB_OP_INTERSECT) return 1;
    if (d.kind == NGDB_OP_SCORE || d.kind == NGDB_OP_UNION_SCORE || d.kind == NGDB_OP_LOSS) return 2;
    if (d.kind == NGDB_OP_PROJECT && c->beta()) return 3;
    return -1;
  };
  for (int i = 0; i < n; ++i) {
    const int cs = chain_stream(invs[i].d);
    stream_of[i] = cs >= 0 ? cs : (dep_inv[i].empty() ? 0 : stream_of[dep_inv[i].back()]);
    for (int d : dep_inv[i])
      if (stream_of[d] != stream_of[i]) waited_on[d] = 1;
  }
  bool used[S] = {true, false, false, false};
  for (int i = 0; i < n; ++i) used[stream_of[i]] = true;
  CK(cudaEventRecord(c->fork_ev, main));
  for (int s = 1; s < S; ++s)
    if (used[s]) CK(cudaStreamWaitEvent(streams[s], c->fork_ev, 0));
  int waited[S][S];
  for (auto& row : waited)
    for (int& x : row) x = -1;
  try {
    for (int i = 0; i < n; ++i) {
      const int s = stream_of[i];
      uint64_t sig = static_cast<uint64_t>(s) << 12;
      for (int d : dep_inv[i]) {
        const int t = stream_of[d];
        if (t == s || d <= waited[s][t]) continue;  // FIFO: a later event implies earlier ones
        CK(cudaStreamWaitEvent(streams[s], c->inv_ev[d], 0));
        waited[s][t] = d;
        sig = sig * 31 + static_cast<uint64_t>(d) + 1;
      }
      const Inv& in = invs[i];
      c->stream = streams[s];
      if (in.merged) {
        sig_mix(c, sig ^ (0x100u | (in.d.dir << 4) | in.d.kind));
        exec_pool(c, p, in.d, &in.m);
      } else {
        sig_mix(c, sig ^ ((static_cast<uint64_t>(in.d.k) << 8) | (in.d.dir << 4) | in.d.kind));
        exec_pool(c, p, in.d);
      }
      c->stream = main;
      if (waited_on[i]) CK(cudaEventRecord(c->inv_ev[i], streams[s]));
    }
  } catch (...) {
    c->stream = main;
    throw;
  }
  for (int s = 1; s < S; ++s)
    if (used[s]) {
      CK(cudaEventRecord(c->join_ev[s - 1], streams[s]));
      CK(cudaStreamWaitEvent(main, c->join_ev[s - 1], 0));
    }
}

bool use_concurrent(const ngdb_ctx* c, const ngdb_plan* p) {
  return c->concurrent && !c->profiling && !p->meta.dep_off.empty() && c->world == 1;
}

void begin_step_device(ngdb_ctx* c) {
  CK(cudaMemsetAsync(c->flags, 0, 4 * sizeof(int32_t), c->stream));
  if (c->dense_n) CK(cudaMemsetAsync(c->dense_g, 0, c->dense_n * sizeof(float), c->stream));
  if (c->debug)
    for (auto& p : c->params)
      if (p.sparse && p.g) CK(cudaMemsetAsync(p.g, 0, p.n() * sizeof(float), c->stream));
}

// 3xTF32 operand splits of the dense weight matrices (W and W^T, hi and lo),
// consumed by every MLP GEMM of the next step.
int refresh_weight_splits(ngdb_ctx* c) {
  int launches = 0;
  for (const auto& p : c->params)
    if (!p.sparse && p.rows > 1)
      launches += split_weight(p.w, static_cast<int>(p.rows), static_cast<int>(p.cols),
                               c->wsplit + c->wsplit_off[p.dense_idx], c->stream);
  return launches;
}

// Every dense tensor as one job of the fused dense Adam + split refresh.
DenseJobs dense_jobs(const ngdb_ctx* c) {
  DenseJobs j{};
  for (const auto& p : c->params) {
    if (p.sparse || j.n >= kMaxDenseTensors) continue;
    DenseJob& d = j.job[j.n++];
    d.off = c->dense_off[p.dense_idx];
    d.rows = static_cast<int>(p.rows);
    d.cols = static_cast<int>(p.cols);
    d.split_off = p.rows > 1 ? c->wsplit_off[p.dense_idx] : -1;
    d.tile_begin = j.tiles;
    j.tiles += static_cast<int>(((p.rows + 31) / 32) * ((p.cols + 31) / 32));
  }
  return j;
}

// Adam bias corrections of step t -> device scalars (read by the optimizer
// kernels, so a captured graph of the step replays with the current t).
__global__ void set_bc_kernel(float* bc, float bc1, float bc2) {
  bc[0] = bc1;
  bc[1] = bc2;
}
// A one-thread kernel with the values as arguments: no host-to-device copy in
// the kernel stream (a pageable memcpy would put a copy-engine op between
// kernels), and capturable.
void set_step_scalars(ngdb_ctx* c, int64_t step) {
  if (step < 1) throw Fail{NGDB_ERR_CONFIG, "optimizer step must be >= 1"};
  const ngdb_model_desc& d = c->desc;
  const float bc1 = static_cast<float>(1.0 - std::pow(static_cast<double>(d.beta1), double(step)));
  const float bc2 = static_cast<float>(1.0 - std::pow(static_cast<double>(d.beta2), double(step)));
  set_bc_kernel<<<1, 1, 0, c->stream>>>(c->d_bc, bc1, bc2);
  CK(cudaGetLastError());
}

SparseTable entity_table(ngdb_ctx* c, const ngdb_plan* p);

// The fusion's entity table: the whole-table form (rows 0..N-1, the step's
// segments expanded by `expand` on the stream) or the step's CSR.
SparseTable fusion_table(ngdb_ctx* c, const ngdb_plan* p, bool expand) {
  SparseTable t = entity_table(c, p);
  if (!fusion_whole(c, p->meta)) return t;
  if (expand)
    c->launches += launch_expand_rows(t.rows, t.seg, t.n_rows, c->seg_full,
                                      static_cast<int>(c->desc.n_entities), c->stream);
  t.n_rows = static_cast<int32_t>(c->desc.n_entities);
  t.rows = c->iota_rows;
  t.seg = c->seg_full;
  return t;
}

SparseTable entity_table(ngdb_ctx* c, const ngdb_plan* p) {
  Param& ent = c->params[c->ent_idx];
  return SparseTable{ent.w, ent.m, ent.v, c->debug ? ent.g : nullptr, static_cast<int32_t>(ent.cols),
                     p->meta.n_erows, p->blob + p->layout.erows, p->blob + p->layout.eseg,
                     p->blob + p->layout.econ};
}

void optimizer(ngdb_ctx* c, const ngdb_plan* p) {
  const ngdb_model_desc& d = c->desc;
  const AdamHyper hp{d.lr, d.beta1, d.beta2, d.eps_adam};
  const float* bc = c->d_bc;
  const DevArgs a = make_args(c, p);
  const LaunchCtx lc{c->stream, c->num_sms};
  Param& ent = c->params[c->ent_idx];
  Param& rel = c->params[c->rel_idx];
  const SparseTable te = entity_table(c, p);
  if (c->fused()) {
    const SparseTable tf = fusion_table(c, p, false);  // expanded by prep_step
    const double u = tf.n_rows, D = c->desc.dim, L = c->desc.semantic_dim;
    // dh, dW_h, dM (+ Psi_theta's dE, dW_psi) and the d x d_l products dW_s, dF
    if (c->profiling)
      c->fam_flops[F_OPT_ENTITY] += 2.0 * u * D * (2 * D + L + (c->beta() ? 4 * D : 0)) + 4.0 * D * D * L;
    timed(c, F_OPT_ENTITY, 6.0 * u * D * 4 + 8.0 * p->meta.n_econ + u * L * 4, [&] {
      return fuse_backward(a, tf, c->fscratch, c->fscratch_cap, hp, bc, lc);
    });
  }
  SparseTable tr{rel.w, rel.m, rel.v, c->debug ? rel.g : nullptr, static_cast<int32_t>(rel.cols),
                 p->meta.n_rrows, p->blob + p->layout.rrows, p->blob + p->layout.rseg,
                 p->blob + p->layout.rcon};
  const double eb = 6.0 * p->meta.n_erows * ent.cols * 4 + 8.0 * p->meta.n_econ +
                    p->meta.n_score * double(c->query_width()) * 4;
  if (!c->fused())
    timed(c, F_OPT_ENTITY, eb, [&] { return launch_sparse_adam_entity(a, te, hp, bc, lc); });
  const double rb = 6.0 * p->meta.n_rrows * rel.cols * 4 + p->meta.n_rcon * (4.0 + rel.cols * 4);
  timed(c, F_OPT_RELATION, rb, [&] { return launch_sparse_adam_relation(a, tr, hp, bc, lc); });
  timed(c, F_OPT_DENSE, 28.0 * c->dense_n, [&] {
    return launch_dense_adam_split(c->dense_w, c->dense_m, c->dense_v, c->dense_g, c->wsplit,
                                   dense_jobs(c), hp, bc, lc);
  });
  CK(cudaGetLastError());
}

// Step prologue of the BetaE backbone: the entity table of the step's touched
// rows (beta.cu). Parameters are fixed within a step, so evaluating the entity
// side of every KL once up front is exact.
void prep_step(ngdb_ctx* c, const ngdb_plan* p) {
  if (!c->step_table()) return;
  const DevArgs a = make_args(c, p);
  const LaunchCtx lc{c->stream, c->num_sms};
  const SparseTable te = entity_table(c, p);
  if (c->fused()) {
    if (!c->sem) throw Fail{NGDB_ERR_CONFIG, "semantic store not uploaded (ngdb_semantic_upload)"};
    const SparseTable tf = fusion_table(c, p, true);
    const double u = tf.n_rows, D = c->desc.dim, L = c->desc.semantic_dim;
    // M = W_s F, Z = S M^T + h W_h^T (+ Psi_theta's Y = E W_psi^T)
    if (c->profiling)
      c->fam_flops[F_ENTITY_PREP] += 2.0 * D * D * L + 2.0 * u * D * (L + D + (c->beta() ? 2 * D : 0));
    timed(c, F_ENTITY_PREP, u * (L * 4 + D * 4 * 2) + 4.0 * p->meta.n_econ,
          [&] { return fuse_prologue(a, tf, c->fscratch, c->fscratch_cap, lc); });
    CK(cudaGetLastError());
    return;
  }
  timed(c, F_ENTITY_PREP, p->meta.n_erows * (2.0 * te.width * 4 + 4) + 4.0 * p->meta.n_econ,
        [&] { return launch_beta_prep(a, te, lc); });
  CK(cudaGetLastError());
}

// Every launch of one planned step, in order (capturable: no host syncs,
// no host-side allocation).
void launch_step(ngdb_ctx* c, const ngdb_plan* p) {
  begin_step_device(c);
  prep_step(c, p);
  if (use_concurrent(c, p)) exec_pools_concurrent(c, p);
  else exec_pools(c, p, p->meta.pools);
  optimizer(c, p);
}

void upload_plan(ngdb_ctx* c, const ngdb_step_plan& plan, ngdb_plan* dst, int64_t& dst_cap,
                 int32_t* staging, cudaStream_t s, const int32_t* prepacked = nullptr) {
  PlanLayout L(plan);
  if (L.total > dst_cap) {
    if (dst->blob) {
      CK(cudaStreamSynchronize(c->stream));
      if (c->copy_stream) CK(cudaStreamSynchronize(c->copy_stream));
      CK(cudaFree(dst->blob));
    }
    dst_cap = std::max<int64_t>(L.total + L.total / 2, dst_cap + dst_cap / 2);
    dst->blob = dmalloc<int32_t>(dst_cap);
  }
  if (!prepacked) pack_plan(plan, L, staging);
  CK(cudaMemcpyAsync(dst->blob, prepacked ? prepacked : staging, L.total * sizeof(int32_t),
                     cudaMemcpyHostToDevice, s));
  c->h2d_bytes += L.total * sizeof(int32_t);
  dst->layout = L;
  dst->meta = meta_of(plan);
  ensure_inv_events(c, dst->meta.pools.size());
}

}  // namespace

namespace ngdb_internal {
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace ngdb_internal

extern "C" {

const char* ngdb_last_error(void) { return g_last_error.c_str(); }

int ngdb_ctx_desc(const ngdb_ctx* c, ngdb_model_desc* out) {
  if (!c || !out) return NGDB_ERR_CONFIG;
  *out = c->desc;
  return NGDB_OK;
}

int ngdb_ctx_create(const ngdb_model_desc* desc, int device, ngdb_ctx** out) {
  ngdb_ctx* c = nullptr;
  int rc = guarded([&] {
    if (!desc || !out) throw Fail{NGDB_ERR_CONFIG, "null argument"};
    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0)
      throw Fail{NGDB_ERR_NO_DEVICE, "no CUDA device visible (the sm_100a kernels have no CPU fallback)"};
    if (device < 0 || device >= n_dev) throw Fail{NGDB_ERR_NO_DEVICE, "device index out of range"};
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      throw Fail{NGDB_ERR_NO_DEVICE, std::string("device is sm_") + std::to_string(prop.major) +
                                         std::to_string(prop.minor) + ", kernels are built for sm_100a"};
    const ngdb_model_desc& d = *desc;
    if (d.backbone != NGDB_GQE && d.backbone != NGDB_Q2B && d.backbone != NGDB_BETAE)
      throw Fail{NGDB_ERR_MISSING_KERNEL, "backbone not built into this library"};
    if (d.dim <= 0 || d.dim % 4 != 0 || d.dim > 1024)
      throw Fail{NGDB_ERR_CONFIG, "dim must be a positive multiple of 4, <= 1024"};
    if (d.n_neg < 1 || d.n_neg + 1 > 1024) throw Fail{NGDB_ERR_CONFIG, "n_neg out of range"};
    if (d.n_entities < 1 || d.n_relations < 1) throw Fail{NGDB_ERR_CONFIG, "empty tables"};
    if (d.semantic_dim < 0 || d.semantic_dim % 4 != 0 || d.semantic_dim > 4096)
      throw Fail{NGDB_ERR_CONFIG, "semantic_dim must be a multiple of 4, <= 4096"};
    const int world = d.world > 1 ? d.world : 1;
    if (world > 1 && (d.rank < 0 || d.rank >= world)) throw Fail{NGDB_ERR_CONFIG, "rank out of range"};
    c = new ngdb_ctx();
    c->desc = d;
    c->world = world;
    c->rank = world > 1 ? d.rank : 0;
    if (c->desc.max_batch <= 0) c->desc.max_batch = 512;
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    for (auto& st : c->side) CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
    for (auto& ev : c->join_ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    if (const char* e = std::getenv("NGDB_SERIAL_POOLS")) c->concurrent = e[0] == '0';
    c->stream = c->own_stream;
    for (int k = 0; k < 2; ++k) CK(cudaEventCreateWithFlags(&c->sh.staged[k], cudaEventDisableTiming));
    const int64_t D = d.dim;
    // this rank's entity rows e = rank (mod world), local row e div world
    const int64_t n_ent_local = (d.n_entities - c->rank + world - 1) / world;
    if (d.backbone == NGDB_GQE) {
      add_param(c, "entity", n_ent_local, D, true);
      add_param(c, "relation", d.n_relations, D, true);
      add_param(c, "int_w1", D, D, false);
      add_param(c, "int_w2", D, D, false);
    } else if (d.backbone == NGDB_BETAE) {  // DESIGN.md §3.5; order = trainer.hpp param_specs
      // with FuseSemantic the structural row h is d wide; Psi_theta makes the 2d
      add_param(c, "entity", n_ent_local, d.semantic_dim > 0 ? D : 2 * D, true);
      add_param(c, "relation", d.n_relations, D, true);
      add_param(c, "prj_w1", 2 * D, 3 * D, false);
      add_param(c, "prj_b1", 1, 2 * D, false);
      add_param(c, "prj_w2", 2 * D, 2 * D, false);
      add_param(c, "prj_b2", 1, 2 * D, false);
      add_param(c, "att_w1", 2 * D, 2 * D, false);
      add_param(c, "att_b1", 1, 2 * D, false);
      add_param(c, "att_w2", D, 2 * D, false);
      add_param(c, "att_b2", 1, D, false);
    } else {
      add_param(c, "entity", n_ent_local, D, true);
      add_param(c, "relation", d.n_relations, 2 * D, true);
      add_param(c, "att_w1", D, D, false);
      add_param(c, "att_b1", 1, D, false);
      add_param(c, "att_w2", D, D, false);
      add_param(c, "att_b2", 1, D, false);
      add_param(c, "off_w1", D, D, false);
      add_param(c, "off_b1", 1, D, false);
      add_param(c, "off_w2", D, D, false);
      add_param(c, "off_b2", 1, D, false);
    }
    if (d.semantic_dim > 0) {  // FusionParams, after the backbone's
      int n_dense = 0;
      for (const auto& p : c->params) n_dense += p.sparse ? 0 : 1;
      c->fus_idx = n_dense;
      add_param(c, "fus_f", D, d.semantic_dim, false);
      add_param(c, "fus_wp", D, 2 * D, false);
      add_param(c, "fus_bp", 1, D, false);
      if (d.backbone == NGDB_BETAE) {  // Psi_theta (Eq. 3)
        add_param(c, "fus_psi", 2 * D, D, false);
        add_param(c, "fus_psi_b", 1, 2 * D, false);
      }
    }
    // dense tensors share one flat buffer (one Adam launch, one memset)
    int64_t off = 0;
    int dense_i = 0;
    for (auto& p : c->params) {
      if (p.sparse) continue;
      c->dense_off[dense_i++] = off;
      off += (p.n() + 3) / 4 * 4;
    }
    c->dense_n = off;
    if (off) {
      c->dense_w = dmalloc<float>(off);
      c->dense_m = dmalloc<float>(off);
      c->dense_v = dmalloc<float>(off);
      c->dense_g = dmalloc<float>(off);
      CK(cudaMemset(c->dense_w, 0, off * 4));
      CK(cudaMemset(c->dense_m, 0, off * 4));
      CK(cudaMemset(c->dense_v, 0, off * 4));
      CK(cudaMemset(c->dense_g, 0, off * 4));
    }
    dense_i = 0;
    for (size_t i = 0; i < c->params.size(); ++i) {
      Param& p = c->params[i];
      if (p.sparse) {
        p.w = dmalloc<float>(p.n());
        p.m = dmalloc<float>(p.n());
        p.v = dmalloc<float>(p.n());
        CK(cudaMemset(p.w, 0, p.n() * 4));
        CK(cudaMemset(p.m, 0, p.n() * 4));
        CK(cudaMemset(p.v, 0, p.n() * 4));
        if (p.name == "entity") c->ent_idx = static_cast<int>(i);
        if (p.name == "relation") c->rel_idx = static_cast<int>(i);
      } else {
        p.dense_idx = dense_i;
        const int64_t o = c->dense_off[dense_i++];
        p.w = c->dense_w + o;
        p.m = c->dense_m + o;
        p.v = c->dense_v + o;
        p.g = c->dense_g + o;
      }
    }
    int64_t woff = 0;
    for (const auto& p : c->params)
      if (!p.sparse) {
        c->wsplit_off[p.dense_idx] = woff;
        if (p.rows > 1) woff += 4 * p.n();
      }
    c->wsplit = dmalloc<float>(woff);
    CK(cudaMemset(c->wsplit, 0, woff * 4));
    c->flags = reinterpret_cast<int32_t*>(dmalloc<float>(4));
    CK(cudaMemset(c->flags, 0, 16));
    c->scratch_cap = intersect_scratch_floats(d.backbone, d.dim, c->desc.max_batch);
    c->istash_slots = std::max(c->desc.max_queries, 1);
    c->istash = dmalloc<float>(int64_t(c->istash_slots) * kStashPerSlot * d.dim);
    if (d.backbone == NGDB_BETAE) {  // <= 4 Project nodes per query after DNF
      c->pstash_slots = 4 * std::max(c->desc.max_queries, 1);
      c->pstash = dmalloc<float>(int64_t(c->pstash_slots) * 4 * d.dim);
    }
    // (node, part) items of one loss launch: at most 8 parts of max_batch nodes
    c->lpart_items = 8 * c->desc.max_batch;
    c->lpart = dmalloc<float>(int64_t(c->lpart_items) * c->query_width());
    c->lpart_scalar = dmalloc<float>(2 * int64_t(c->lpart_items));
    c->lcount = reinterpret_cast<int32_t*>(dmalloc<float>(c->desc.max_batch));
    CK(cudaMemset(c->lcount, 0, sizeof(int32_t) * c->desc.max_batch));
    c->scratch = dmalloc<float>(c->scratch_cap);
    if (d.backbone == NGDB_BETAE) {  // BetaE Project MLPs: their own scratch, so a Project
      // pool can run beside an Intersect pool (§3.2), sized for up to 4 drains
      // of a pool merged into one launch (bigger, fewer GEMMs)
      const char* pm = std::getenv("NGDB_PROJ_MERGE");  // drains per launch (A/B)
      c->proj_merge_cap = (pm ? std::max(1, std::atoi(pm)) : 4) * std::max(c->desc.max_batch, 1);
      c->scratch2_cap = beta_project_scratch_floats(d.dim, c->proj_merge_cap);
      c->scratch2 = dmalloc<float>(c->scratch2_cap);
    }
    c->d_bc = dmalloc<float>(4);
    tc_gemm_init();
    CK(cudaEventCreate(&c->t0));
    CK(cudaEventCreate(&c->t1));
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&c->staged[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->blob_free[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->blob_ready[i], cudaEventDisableTiming));
    }
    CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    *out = c;
  });
  if (rc != NGDB_OK && c) ngdb_ctx_destroy(c);
  return rc;
}

int ngdb_ctx_destroy(ngdb_ctx* c) {
  if (!c) return NGDB_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->own_stream) cudaStreamSynchronize(c->own_stream);
  for (auto& st : c->side)
    if (st) cudaStreamDestroy(st);
  for (auto ev : c->inv_ev) cudaEventDestroy(ev);
  if (c->fork_ev) cudaEventDestroy(c->fork_ev);
  for (auto ev : c->join_ev)
    if (ev) cudaEventDestroy(ev);
  if (c->comm) nccl_api().CommDestroy(c->comm);
  if (c->meta_comm) nccl_api().CommDestroy(c->meta_comm);
  if (c->meta_stream) cudaStreamDestroy(c->meta_stream);
  if (c->meta_dev) cudaFree(c->meta_dev);
  for (auto& p : c->params)
    if (p.sparse) {
      cudaFree(p.w);
      cudaFree(p.m);
      cudaFree(p.v);
      if (p.g) cudaFree(p.g);
    }
  if (c->eval_buf) cudaFree(c->eval_buf);
  if (c->pinned_ring) cudaFreeHost(c->pinned_ring);
  if (c->evtab) cudaFree(c->evtab);
  if (c->ev_rows) cudaFree(c->ev_rows);
  if (c->ev_scratch) cudaFree(c->ev_scratch);
  if (c->cand_local) cudaFree(c->cand_local);
  if (c->anchor_local) cudaFree(c->anchor_local);
  if (c->fscratch) cudaFree(c->fscratch);
  if (c->istash) cudaFree(c->istash);
  if (c->pstash) cudaFree(c->pstash);
  if (c->lpart) cudaFree(c->lpart);
  if (c->lpart_scalar) cudaFree(c->lpart_scalar);
  if (c->lcount) cudaFree(c->lcount);
  for (float* p : {c->etab, c->etab_c, c->dense_w, c->dense_m, c->dense_v, c->dense_g, c->wsplit, c->sem, c->qbuf, c->dqbuf,
                   c->coefbuf, c->ddbuf, c->agbuf, c->rgbuf, c->loss_out, c->scratch, c->arena,
                   c->l2_flush, c->d_bc, c->scratch2, c->sem_split})
    if (p) cudaFree(p);
  for (int32_t* p : {c->iota_rows, c->seg_full})
    if (p) cudaFree(p);
  if (c->flags) cudaFree(c->flags);
  for (int i = 0; i < 2; ++i) {
    if (c->staging[i]) cudaFreeHost(c->staging[i]);
    if (c->stream_plan[i].blob) cudaFree(c->stream_plan[i].blob);
    if (c->staged[i]) cudaEventDestroy(c->staged[i]);
    if (c->blob_free[i]) cudaEventDestroy(c->blob_free[i]);
    if (c->blob_ready[i]) cudaEventDestroy(c->blob_ready[i]);
  }
  for (auto& e : c->exec_cache) {
    if (e.exec) cudaGraphExecDestroy(e.exec);
    if (e.done) cudaEventDestroy(e.done);
  }
  for (auto& r : c->results) {
    if (r.host) cudaFreeHost(r.host);
    if (r.done) cudaEventDestroy(r.done);
  }
  for (auto& r : c->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : c->event_pool) cudaEventDestroy(e);
  if (c->t0) cudaEventDestroy(c->t0);
  if (c->t1) cudaEventDestroy(c->t1);
  for (int32_t* b : c->sh.blobs)
    if (b) cudaFree(b);
  if (c->sh.buf) cudaFree(c->sh.buf);
  for (int k = 0; k < 2; ++k) {
    if (c->sh.staging[k]) cudaFreeHost(c->sh.staging[k]);
    if (c->sh.staged[k]) cudaEventDestroy(c->sh.staged[k]);
  }
  if (c->copy_stream) {
    cudaStreamSynchronize(c->copy_stream);
    cudaStreamDestroy(c->copy_stream);
  }
  if (c->own_stream) cudaStreamDestroy(c->own_stream);
  delete c;
  return NGDB_OK;
}

int ngdb_param_count(ngdb_ctx* c, int32_t* n) {
  return guarded([&] { *n = static_cast<int32_t>(c->params.size()); });
}

int ngdb_param_info(ngdb_ctx* c, int32_t i, const char** name, int64_t* rows, int64_t* cols,
                    int32_t* sparse) {
  return guarded([&] {
    if (i < 0 || i >= static_cast<int32_t>(c->params.size()))
      throw Fail{NGDB_ERR_INDEX_OUT_OF_RANGE, "param index"};
    const Param& p = c->params[i];
    if (name) *name = p.name.c_str();
    if (rows) *rows = p.rows;
    if (cols) *cols = p.cols;
    if (sparse) *sparse = p.sparse ? 1 : 0;
  });
}

namespace {
float* resolve(ngdb_ctx* c, const char* name, int64_t n) {
  std::string s(name);
  char kind = 'w';
  if (s.size() > 2 && s[1] == ':') {
    kind = s[0];
    s = s.substr(2);
  }
  Param* p = c->find(s);
  if (!p) throw Fail{NGDB_ERR_CONFIG, "unknown parameter " + s};
  if (n != p->n()) throw Fail{NGDB_ERR_SHAPE_MISMATCH, "size mismatch for " + s};
  switch (kind) {
    case 'w': return p->w;
    case 'm': return p->m;
    case 'v': return p->v;
    case 'g':
      if (!p->g) throw Fail{NGDB_ERR_CONFIG, "gradient of " + s + " not kept (ngdb_set_debug)"};
      return p->g;
  }
  throw Fail{NGDB_ERR_CONFIG, "unknown parameter prefix"};
}
}  // namespace

int ngdb_param_upload(ngdb_ctx* c, const char* name, const float* host, int64_t n) {
  return guarded([&] {
    float* dst = resolve(c, name, n);
    CK(cudaMemcpyAsync(dst, host, n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    refresh_weight_splits(c);  // dense weights feed the GEMMs through their splits
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ngdb_param_download(ngdb_ctx* c, const char* name, float* host, int64_t n) {
  return guarded([&] {
    const float* src = resolve(c, name, n);
    CK(cudaMemcpyAsync(host, src, n * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ngdb_semantic_upload(ngdb_ctx* c, const float* host, int64_t n) {
  return guarded([&] {
    if (c->desc.semantic_dim <= 0) throw Fail{NGDB_ERR_CONFIG, "context has no semantic store"};
    // row-sharded: this rank's rows (entity e = rank + world * local row)
    const int64_t rows = c->world > 1 ? c->params[c->ent_idx].rows : int64_t(c->desc.n_entities);
    if (n != rows * c->desc.semantic_dim)
      throw Fail{NGDB_ERR_SHAPE_MISMATCH, "semantic store size"};
    if (!c->sem) c->sem = dmalloc<float>(n);
    CK(cudaMemcpy(c->sem, host, n * 4, cudaMemcpyHostToDevice));
    if (c->world > 1) return;  // the whole-table form is single-GPU only
    // the frozen store's operand splits, once (the fusion GEMMs read them
    // directly when a step touches every entity: no per-step gather / split;
    // the weight gradients read them MN-major, so no transposed copy)
    const int64_t N = c->desc.n_entities, L = c->desc.semantic_dim;
    if (!c->sem_split) c->sem_split = dmalloc<float>(2 * N * L);
    float* hi = c->sem_split;
    float* lo = hi + N * L;
    split_matrix(c->sem, static_cast<int>(N), static_cast<int>(L), static_cast<int>(L), 0, 0, hi, lo,
                 c->stream);
    if (!c->iota_rows) {
      std::vector<int32_t> iota(N);
      for (int64_t e = 0; e < N; ++e) iota[e] = static_cast<int32_t>(e);
      c->iota_rows = dmalloc<int32_t>(N);
      c->seg_full = dmalloc<int32_t>(N + 1);
      CK(cudaMemcpy(c->iota_rows, iota.data(), N * 4, cudaMemcpyHostToDevice));
    }
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ngdb_set_debug(ngdb_ctx* c, int32_t keep) {
  return guarded([&] {
    c->debug = keep != 0;
    if (c->debug)
      for (auto& p : c->params)
        if (p.sparse && !p.g) {
          p.g = dmalloc<float>(p.n());
          CK(cudaMemset(p.g, 0, p.n() * 4));
        }
  });
}

int ngdb_step_begin(ngdb_ctx* c, const ngdb_step_plan* plan) {
  return ngdb_step_begin_ex(c, plan, 0);
}

int ngdb_step_begin_ex(ngdb_ctx* c, const ngdb_step_plan* plan, int32_t flags) {
  return guarded([&] {
    c->has_held = false;
    if (c->world > 1) throw Fail{NGDB_ERR_CONFIG, "context is row-sharded: use ngdb_shard_begin"};
    validate_plan(*plan);
    const int i = c->cur;
    c->cur ^= 1;
    const PlanLayout L(*plan);
    // the pinned buffer may still be feeding the H2D copy issued two steps ago
    CK(cudaEventSynchronize(c->staged[i]));
    if (L.total > c->staging_cap[i]) {
      if (c->staging[i]) CK(cudaFreeHost(c->staging[i]));
      c->staging_cap[i] = L.total + L.total / 2;
      void* p = nullptr;
      CK(cudaMallocHost(&p, c->staging_cap[i] * sizeof(int32_t)));
      c->staging[i] = static_cast<int32_t*>(p);
    }
    // everything enqueued so far on the context stream belongs to the steps
    // before this one: the last reader of stream_plan[1-i] is among them
    CK(cudaEventRecord(c->blob_free[i ^ 1], c->stream));
    // upload on the copy stream once the step two back (the last reader of
    // stream_plan[i]) is done; the kernels of this step wait for the upload
    CK(cudaStreamWaitEvent(c->copy_stream, c->blob_free[i], 0));
    upload_plan(c, *plan, &c->stream_plan[i], c->stream_cap[i], c->staging[i], c->copy_stream);
    CK(cudaEventRecord(c->staged[i], c->copy_stream));
    CK(cudaEventRecord(c->blob_ready[i], c->copy_stream));
    CK(cudaStreamWaitEvent(c->stream, c->blob_ready[i], 0));
    ensure_step_buffers(c, c->stream_plan[i].meta);
    c->active = &c->stream_plan[i];
    c->prologue_pending = (flags & NGDB_BEGIN_DEFER_PROLOGUE) != 0;
    if (!c->prologue_pending) {
      begin_step_device(c);
      prep_step(c, &c->stream_plan[i]);
    }
  });
}

int64_t ngdb_plan_packed_size(const ngdb_step_plan* plan) { return PlanLayout(*plan).total; }

int ngdb_plan_pack(const ngdb_step_plan* plan, int32_t* out, int64_t cap) {
  return guarded([&] {
    validate_plan(*plan);
    const PlanLayout L(*plan);
    if (cap < L.total) throw Fail{NGDB_ERR_SHAPE_MISMATCH, "plan_pack: buffer too small"};
    pack_plan(*plan, L, out);
  });
}

int ngdb_ctx_pinned_ring(ngdb_ctx* c, int64_t ints, int32_t** base) {
  return guarded([&] {
    if (ints > c->pinned_ring_ints) {
      CK(cudaDeviceSynchronize());  // no copy may still read the old ring
      if (c->pinned_ring) CK(cudaFreeHost(c->pinned_ring));
      c->pinned_ring = nullptr;
      void* p = nullptr;
      CK(cudaMallocHost(&p, static_cast<size_t>(ints) * sizeof(int32_t)));
      c->pinned_ring = static_cast<int32_t*>(p);
      c->pinned_ring_ints = ints;
    }
    *base = c->pinned_ring;
  });
}

int ngdb_host_alloc(int64_t bytes, void** out) {
  return guarded([&] { CK(cudaMallocHost(out, static_cast<size_t>(bytes))); });
}

int ngdb_host_free(void* p) {
  return guarded([&] {
    if (p) CK(cudaFreeHost(p));
  });
}

int ngdb_step_begin_packed(ngdb_ctx* c, const ngdb_step_plan* plan, const int32_t* packed,
                           int64_t n, int32_t flags) {
  return guarded([&] {
    c->has_held = false;
    if (c->world > 1) throw Fail{NGDB_ERR_CONFIG, "context is row-sharded: use ngdb_shard_begin"};
    const PlanLayout L(*plan);
    if (n != L.total) throw Fail{NGDB_ERR_SHAPE_MISMATCH, "step_begin_packed: packed size"};
    const int i = c->cur;
    c->cur ^= 1;
    CK(cudaEventRecord(c->blob_free[i ^ 1], c->stream));
    CK(cudaStreamWaitEvent(c->copy_stream, c->blob_free[i], 0));
    upload_plan(c, *plan, &c->stream_plan[i], c->stream_cap[i], nullptr, c->copy_stream, packed);
    CK(cudaEventRecord(c->blob_ready[i], c->copy_stream));
    CK(cudaStreamWaitEvent(c->stream, c->blob_ready[i], 0));
    ensure_step_buffers(c, c->stream_plan[i].meta);
    c->active = &c->stream_plan[i];
    c->prologue_pending = (flags & NGDB_BEGIN_DEFER_PROLOGUE) != 0;
    if (!c->prologue_pending) {
      begin_step_device(c);
      prep_step(c, &c->stream_plan[i]);
    }
  });
}

int ngdb_exec_pool(ngdb_ctx* c, const ngdb_pool_desc* pool) {
  return guarded([&] {
    if (!c->active) throw Fail{NGDB_ERR_CONFIG, "exec_pool outside a step"};
    if (c->prologue_pending) {
      begin_step_device(c);
      prep_step(c, c->active);
      c->prologue_pending = false;
    }
    if (c->has_held) {
      c->has_held = false;
      if (mergeable(c, c->held, *pool)) {
        exec_pool(c, c->active, c->held, pool);
        return;
      }
      exec_pool(c, c->active, c->held);
    }
    if (pool->kind == NGDB_OP_INTERSECT && pool->count > 0) {
      c->held = *pool;
      c->has_held = true;
      return;
    }
    exec_pool(c, c->active, *pool);
  });
}

int ngdb_exec_flush(ngdb_ctx* c) {
  return guarded([&] {
    if (!c->active) throw Fail{NGDB_ERR_CONFIG, "exec_flush outside a step"};
    if (c->has_held) {
      c->has_held = false;
      exec_pool(c, c->active, c->held);
    }
  });
}

int ngdb_read_arena(ngdb_ctx* c, int64_t offset, int64_t n, float* out) {
  return guarded([&] {
    if (!c->arena || offset < 0 || n < 0 || offset + n > c->arena_cap)
      throw Fail{NGDB_ERR_INDEX_OUT_OF_RANGE, "read_arena: range outside the arena"};
    CK(cudaMemcpyAsync(out, c->arena + offset, n * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ngdb_set_gemm_split(int32_t split) {
  return guarded([&] {
    if (split < 0 || split > 8) throw Fail{NGDB_ERR_CONFIG, "gemm split-K must be 0 (auto) or 1..8"};
    ngdb_dev::set_gemm_split_override(split);
  });
}

int ngdb_optimizer_step(ngdb_ctx* c, int64_t step) {
  return guarded([&] {
    if (!c->active) throw Fail{NGDB_ERR_CONFIG, "optimizer_step outside a step"};
    if (c->prologue_pending) {
      begin_step_device(c);
      prep_step(c, c->active);
      c->prologue_pending = false;
    }
    flush_held(c);
    set_step_scalars(c, step);
    optimizer(c, c->active);
  });
}

int ngdb_step_launch(ngdb_ctx* c, int64_t step, int32_t use_graph) {
  return guarded([&] {
    if (!c->active) throw Fail{NGDB_ERR_CONFIG, "step_launch outside a step"};
    flush_held(c);
    ngdb_plan* p = c->active;
    auto body = [&] {
      if (c->prologue_pending) {
        begin_step_device(c);
        prep_step(c, p);
      }
      set_step_scalars(c, step);
      // streaming steps keep the serial chain: re-capturing and updating the
      // DAG-shaped graph every step costs the consumer thread more host time
      // (C2: 0.18 -> 0.25 ms/step) than the concurrency saves on the device
      // (steady-state e2e measured 1.21 M serial vs 1.14-1.19 M concurrent)
      exec_pools(c, p, p->meta.pools);
      optimizer(c, p);
    };
    if (!use_graph || c->profiling) {
      body();
      c->prologue_pending = false;
      return;
    }
    // the whole step (prologue, step scalars, every pool, the optimizer) as one
    // graph: the device runs it with graph-launch overheads instead of ~60
    // stream operations
    cudaGraph_t g = nullptr;
    c->launch_sig = 1469598103934665603ull;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    try {
      body();
    } catch (...) {
      cudaStreamEndCapture(c->stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    CK(cudaStreamEndCapture(c->stream, &g));
    c->prologue_pending = false;
    const uint64_t sig = c->launch_sig;
    ngdb_ctx::ExecEntry* hit = nullptr;
    ngdb_ctx::ExecEntry* victim = nullptr;
    for (auto& en : c->exec_cache) {
      const bool idle = !en.exec || cudaEventQuery(en.done) == cudaSuccess;
      cudaGetLastError();  // cudaErrorNotReady is not an error here
      if (!idle) continue;
      if (en.exec && en.sig == sig && !hit) hit = &en;
      if (!victim || !en.exec || (victim->exec && en.used < victim->used)) victim = &en;
    }
    cudaGraphExec_t e = nullptr;
    if (hit) {
      cudaGraphExecUpdateResultInfo info{};
      if (cudaGraphExecUpdate(hit->exec, g, &info) == cudaSuccess) {
        e = hit->exec;
        ++c->exec_updates;
      } else {
        cudaGetLastError();
        victim = hit;  // same structure, incompatible parameters: replace it
      }
    }
    if (!e) {
      if (!victim) throw Fail{NGDB_ERR_CONFIG, "no idle step-graph slot"};
      if (victim->exec) CK(cudaGraphExecDestroy(victim->exec));
      victim->exec = nullptr;
      const cudaError_t err = cudaGraphInstantiate(&victim->exec, g, 0);
      if (err != cudaSuccess) {
        cudaGraphDestroy(g);
        CK(err);
      }
      if (!victim->done) CK(cudaEventCreateWithFlags(&victim->done, cudaEventDisableTiming));
      victim->sig = sig;
      e = victim->exec;
      hit = victim;
      ++c->exec_instantiations;
    }
    hit->used = ++c->exec_clock;
    CK(cudaGraphDestroy(g));
    // upload the (re)instantiated / updated exec on the copy stream now, so
    // the launch below does not pay it between the previous step's last
    // kernel and this step's first (steady-state gap 0.09 -> 0.05 ms/step on
    // C2, NGDB_STEP_TIMELINE); NGDB_GRAPH_UPLOAD=0 leaves it to the launch
    static const bool pre_upload = [] {
      const char* u = std::getenv("NGDB_GRAPH_UPLOAD");
      return !(u && u[0] == '0');
    }();
    if (pre_upload) CK(cudaGraphUpload(e, c->copy_stream));
    static const bool timeline = std::getenv("NGDB_STEP_TIMELINE") != nullptr;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (timeline) {
      CK(cudaEventCreate(&t0));
      CK(cudaEventCreate(&t1));
      CK(cudaEventRecord(t0, c->stream));
    }
    CK(cudaGraphLaunch(e, c->stream));
    if (timeline) {
      CK(cudaEventRecord(t1, c->stream));
      c->timeline.emplace_back(t0, t1);
    }
    CK(cudaEventRecord(hit->done, c->stream));
  });
}

int ngdb_step_end(ngdb_ctx* c, float* per_query_loss, int32_t n_queries, double* loss_sum,
                  int32_t* nonfinite) {
  return guarded([&] {
    if (!c->active) throw Fail{NGDB_ERR_CONFIG, "step_end outside a step"};
    flush_held(c);
    const int32_t nq = c->active->meta.n_queries;
    std::vector<float> tmp;
    float* dst = per_query_loss;
    if (!dst || n_queries < nq) {
      tmp.resize(nq);
      dst = tmp.data();
    }
    int32_t flags[4] = {0, 0, 0, 0};
    CK(cudaMemcpyAsync(dst, c->loss_out, nq * sizeof(float), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(flags, c->flags, sizeof(flags), cudaMemcpyDeviceToHost, c->stream));
    c->d2h_bytes += nq * sizeof(float) + sizeof(flags);
    CK(cudaStreamSynchronize(c->stream));
    c->drain_profile();
    if (loss_sum) {
      double s = 0.0;
      for (int32_t i = 0; i < nq; ++i) s += dst[i];
      *loss_sum = s;
    }
    if (nonfinite) *nonfinite = flags[0];
    c->active = nullptr;
    if (flags[1]) throw Fail{NGDB_ERR_INDEX_OUT_OF_RANGE, "embedding index out of range in plan"};
  });
}

namespace {
// host: pinned (UVA-mapped) [nq] losses then 4 int32 flags
__global__ void results_to_host_kernel(float* host, const float* loss, const int32_t* flags,
                                       int32_t nq) {
  for (int i = threadIdx.x; i < nq; i += blockDim.x) host[i] = loss[i];
  if (threadIdx.x < 4) reinterpret_cast<int32_t*>(host + nq)[threadIdx.x] = flags[threadIdx.x];
}
}  // namespace

int ngdb_step_end_async(ngdb_ctx* c, int64_t* ticket) {
  return guarded([&] {
    if (!c->active) throw Fail{NGDB_ERR_CONFIG, "step_end outside a step"};
    flush_held(c);
    if (c->profiling) throw Fail{NGDB_ERR_CONFIG, "step_end_async while profiling"};
    const int64_t t = c->next_ticket;
    auto& r = c->results[t % ngdb_ctx::kResultSlots];
    if (r.ticket >= 0) throw Fail{NGDB_ERR_CONFIG, "too many outstanding steps (ngdb_step_wait)"};
    const int32_t nq = c->active->meta.n_queries;
    if (nq + 4 > r.cap) {
      if (r.host) CK(cudaFreeHost(r.host));
      void* p = nullptr;
      r.cap = std::max<int64_t>(nq + 4, 1024);
      CK(cudaMallocHost(&p, r.cap * sizeof(float)));
      r.host = static_cast<float*>(p);
    }
    if (!r.done) CK(cudaEventCreateWithFlags(&r.done, cudaEventDisableTiming));
    // the step's losses + flags written straight into the pinned slot by one
    // small kernel (zero-copy over PCIe): unlike two copy-engine D2H operations
    // it does not hold the stream between this step's graph and the next one's
    // (measured: ~40 us of idle device time per step)
    results_to_host_kernel<<<1, 256, 0, c->stream>>>(r.host, c->loss_out, c->flags, nq);
    CK(cudaGetLastError());
    ++c->launches;
    c->d2h_bytes += nq * sizeof(float) + 4 * sizeof(int32_t);
    CK(cudaEventRecord(r.done, c->stream));
    r.n_queries = nq;
    r.ticket = t;
    ++c->next_ticket;
    c->active = nullptr;
    *ticket = t;
  });
}

int ngdb_step_wait(ngdb_ctx* c, int64_t ticket, float* per_query_loss, int32_t n_queries,
                   double* loss_sum, int32_t* nonfinite) {
  return guarded([&] {
    if (ticket < 0) throw Fail{NGDB_ERR_CONFIG, "invalid ticket"};
    auto& r = c->results[ticket % ngdb_ctx::kResultSlots];
    if (r.ticket != ticket) throw Fail{NGDB_ERR_CONFIG, "unknown or already collected ticket"};
    CK(cudaEventSynchronize(r.done));
    r.ticket = -1;
    const int32_t nq = r.n_queries;
    if (per_query_loss && n_queries >= nq) std::memcpy(per_query_loss, r.host, nq * sizeof(float));
    if (loss_sum) {
      double s = 0.0;
      for (int32_t i = 0; i < nq; ++i) s += r.host[i];
      *loss_sum = s;
    }
    int32_t flags[4];
    std::memcpy(flags, r.host + nq, sizeof(flags));
    if (nonfinite) *nonfinite = flags[0];
    if (flags[1]) throw Fail{NGDB_ERR_INDEX_OUT_OF_RANGE, "embedding index out of range in plan"};
  });
}

int ngdb_plan_create(ngdb_ctx* c, const ngdb_step_plan* plan, ngdb_plan** out) {
  ngdb_plan* p = nullptr;
  int rc = guarded([&] {
    if (c->world > 1) throw Fail{NGDB_ERR_CONFIG, "context is row-sharded: use ngdb_shard_begin"};
    validate_plan(*plan);
    p = new ngdb_plan();
    const PlanLayout L(*plan);
    std::vector<int32_t> host(L.total);
    pack_plan(*plan, L, host.data());
    p->blob = dmalloc<int32_t>(L.total);
    CK(cudaMemcpy(p->blob, host.data(), L.total * sizeof(int32_t), cudaMemcpyHostToDevice));
    p->layout = L;
    p->meta = meta_of(*plan);
    ensure_step_buffers(c, p->meta);
    ensure_inv_events(c, p->meta.pools.size());
    *out = p;
  });
  if (rc != NGDB_OK && p) ngdb_plan_destroy(p);
  return rc;
}

namespace {
// capture the step's ~100+ launches once; replays cost one launch
void capture_plan(ngdb_ctx* c, ngdb_plan* p) {
  if (p->graph) CK(cudaGraphExecDestroy(p->graph));
  p->graph = nullptr;
  cudaGraph_t g = nullptr;
  ngdb_plan* prev = c->active;
  c->active = p;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  const int64_t l0 = c->launches;
  try {
    launch_step(c, p);
  } catch (...) {
    cudaStreamEndCapture(c->stream, &g);
    if (g) cudaGraphDestroy(g);
    c->launches = l0;
    c->active = prev;
    throw;
  }
  p->graph_launches = c->launches - l0;
  c->launches = l0;
  c->active = prev;
  CK(cudaStreamEndCapture(c->stream, &g));
  const cudaError_t e = cudaGraphInstantiate(&p->graph, g, 0);
  cudaGraphDestroy(g);
  CK(e);
  p->graph_gen = c->buffer_gen;
}
}  // namespace

int ngdb_plan_prepare(ngdb_ctx* c, ngdb_plan* p) {
  return guarded([&] {
    ensure_step_buffers(c, p->meta);
    if (!c->use_graphs) return;
    if (!p->graph || p->graph_gen != c->buffer_gen) capture_plan(c, p);
  });
}

int ngdb_plan_run(ngdb_ctx* c, ngdb_plan* p, int64_t step) {
  return guarded([&] {
    ensure_step_buffers(c, p->meta);
    set_step_scalars(c, step);
    c->active = p;
    if (c->profiling || !c->use_graphs) {
      launch_step(c, p);
      return;
    }
    if (!p->graph || p->graph_gen != c->buffer_gen) capture_plan(c, p);
    static const bool timeline = std::getenv("NGDB_STEP_TIMELINE") != nullptr;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (timeline) {
      CK(cudaEventCreate(&t0));
      CK(cudaEventCreate(&t1));
      CK(cudaEventRecord(t0, c->stream));
    }
    CK(cudaGraphLaunch(p->graph, c->stream));
    if (timeline) {
      CK(cudaEventRecord(t1, c->stream));
      c->timeline.emplace_back(t0, t1);
    }
    c->launches += p->graph_launches;
  });
}

int ngdb_plan_destroy(ngdb_plan* p) {
  if (!p) return NGDB_OK;
  if (p->graph) cudaGraphExecDestroy(p->graph);
  if (p->blob) cudaFree(p->blob);
  delete p;
  return NGDB_OK;
}

int ngdb_sync(ngdb_ctx* c) {
  return guarded([&] { CK(cudaStreamSynchronize(c->stream)); });
}

int ngdb_timer_start(ngdb_ctx* c) {
  return guarded([&] { CK(cudaEventRecord(c->t0, c->stream)); });
}

int ngdb_timer_stop(ngdb_ctx* c, float* ms) {
  return guarded([&] {
    CK(cudaEventRecord(c->t1, c->stream));
    CK(cudaEventSynchronize(c->t1));
    CK(cudaEventElapsedTime(ms, c->t0, c->t1));
  });
}

int ngdb_profile_enable(ngdb_ctx* c, int32_t on) {
  return guarded([&] {
    c->drain_profile();
    c->profiling = on != 0;
    for (int i = 0; i < F_COUNT; ++i) {
      c->fam_ms[i] = 0;
      c->fam_bytes[i] = 0;
      c->fam_flops[i] = 0;
      c->fam_launches[i] = 0;
    }
  });
}

int ngdb_profile_flops(ngdb_ctx* c, int32_t family, double* flops) {
  return guarded([&] {
    if (family < 0 || family >= F_COUNT) throw Fail{NGDB_ERR_INDEX_OUT_OF_RANGE, "family"};
    *flops = c->fam_flops[family];
  });
}

int ngdb_profile_read(ngdb_ctx* c, int32_t family, double* ms, int64_t* launches, double* bytes) {
  return guarded([&] {
    if (family < 0 || family >= F_COUNT) throw Fail{NGDB_ERR_INDEX_OUT_OF_RANGE, "family"};
    c->drain_profile();
    if (ms) *ms = c->fam_ms[family];
    if (launches) *launches = c->fam_launches[family];
    if (bytes) *bytes = c->fam_bytes[family];
  });
}

int32_t ngdb_profile_families(void) { return F_COUNT; }

const char* ngdb_profile_family_name(int32_t f) {
  return (f >= 0 && f < F_COUNT) ? kFamilyNames[f] : "?";
}

int64_t ngdb_launch_count(ngdb_ctx* c) { return c ? c->launches : 0; }

int ngdb_graph_stats(ngdb_ctx* c, int64_t* updates, int64_t* instantiations) {
  return guarded([&] {
    if (updates) *updates = c->exec_updates;
    if (instantiations) *instantiations = c->exec_instantiations;
  });
}

// ---- checkpoint ("versioned binary blob of named parameter
// tensors + config hash"; cadence SPEC.md:587) --------------------------------
// Layout, little-endian: "NGCK", u32 version = 2, u64 config hash, i64 step,
// i32 backbone, i32 dim, i32 world, i32 rank, u32 tensor count; per tensor (registry order): u32 name
// length, name, i64 rows, i64 cols, then theta, Adam m, Adam v as rows*cols f32
// each; trailer: u64 FNV-1a of every preceding byte. The Adam moments and the
// step make a resumed run bit-identical to an uninterrupted one. A row-sharded
// context (world > 1) writes its own rows only; world and rank are recorded and a
// blob loads only into the same (world, rank) slot. Version-1 blobs (no world /
// rank fields) load into unsharded contexts.
namespace {
constexpr uint32_t kCkptVersion = 2;
struct Fnv {
  uint64_t h = 1469598103934665603ull;
  void add(const void* p, size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  }
};
}  // namespace

int ngdb_checkpoint_save(ngdb_ctx* c, const char* path, uint64_t config_hash, int64_t step) {
  return guarded([&] {
    if (!path) throw Fail{NGDB_ERR_CONFIG, "checkpoint: null path"};
    std::vector<char> blob;
    auto put = [&](const void* p, size_t n) {
      const char* b = static_cast<const char*>(p);
      blob.insert(blob.end(), b, b + n);
    };
    const uint32_t ver = kCkptVersion, nt = static_cast<uint32_t>(c->params.size());
    const int32_t bb = c->desc.backbone, dim = c->desc.dim, world = c->world, rank = c->rank;
    put("NGCK", 4);
    put(&ver, 4);
    put(&config_hash, 8);
    put(&step, 8);
    put(&bb, 4);
    put(&dim, 4);
    put(&world, 4);
    put(&rank, 4);
    put(&nt, 4);
    CK(cudaStreamSynchronize(c->stream));
    std::vector<float> host;
    for (const auto& p : c->params) {
      const uint32_t len = static_cast<uint32_t>(p.name.size());
      put(&len, 4);
      put(p.name.data(), len);
      put(&p.rows, 8);
      put(&p.cols, 8);
      host.resize(p.n());
      for (const float* src : {p.w, p.m, p.v}) {
        CK(cudaMemcpy(host.data(), src, p.n() * sizeof(float), cudaMemcpyDeviceToHost));
        put(host.data(), p.n() * sizeof(float));
      }
    }
    Fnv f;
    f.add(blob.data(), blob.size());
    put(&f.h, 8);
    FILE* fp = std::fopen(path, "wb");
    if (!fp) throw Fail{NGDB_ERR_CONFIG, std::string("checkpoint: cannot write ") + path};
    const size_t wrote = std::fwrite(blob.data(), 1, blob.size(), fp);
    const bool ok = std::fclose(fp) == 0 && wrote == blob.size();
    if (!ok) throw Fail{NGDB_ERR_CONFIG, std::string("checkpoint: short write to ") + path};
  });
}

int ngdb_checkpoint_load(ngdb_ctx* c, const char* path, uint64_t config_hash, int64_t* step) {
  return guarded([&] {
    if (!path) throw Fail{NGDB_ERR_CONFIG, "checkpoint: null path"};
    FILE* fp = std::fopen(path, "rb");
    if (!fp) throw Fail{NGDB_ERR_CONFIG, std::string("checkpoint: cannot read ") + path};
    std::vector<char> blob;
    char buf[1 << 16];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof(buf), fp)) > 0) blob.insert(blob.end(), buf, buf + got);
    std::fclose(fp);
    if (blob.size() < 44 || std::memcmp(blob.data(), "NGCK", 4) != 0)
      throw Fail{NGDB_ERR_DOMAIN, "checkpoint: not an NGCK blob"};
    uint64_t stored;
    std::memcpy(&stored, blob.data() + blob.size() - 8, 8);
    Fnv f;
    f.add(blob.data(), blob.size() - 8);
    if (f.h != stored) throw Fail{NGDB_ERR_DOMAIN, "checkpoint: checksum mismatch (corrupt file)"};
    size_t at = 4;
    auto get = [&](void* p, size_t n) {
      if (at + n > blob.size() - 8) throw Fail{NGDB_ERR_DOMAIN, "checkpoint: truncated"};
      std::memcpy(p, blob.data() + at, n);
      at += n;
    };
    uint32_t ver, nt;
    uint64_t hash;
    int64_t st;
    int32_t bb, dim, world = 1, rank = 0;
    get(&ver, 4);
    if (ver != 1 && ver != kCkptVersion) throw Fail{NGDB_ERR_CONFIG, "checkpoint: unsupported version"};
    get(&hash, 8);
    get(&st, 8);
    get(&bb, 4);
    get(&dim, 4);
    if (ver >= 2) {
      get(&world, 4);
      get(&rank, 4);
    }
    get(&nt, 4);
    if (world != c->world || rank != c->rank)
      throw Fail{NGDB_ERR_CONFIG, "checkpoint: written by rank " + std::to_string(rank) + " of " +
                                      std::to_string(world) + ", context is rank " +
                                      std::to_string(c->rank) + " of " + std::to_string(c->world)};
    if (bb != c->desc.backbone || dim != c->desc.dim)
      throw Fail{NGDB_ERR_CONFIG, "checkpoint: BackboneMismatch (backbone / dim differ from the context)"};
    if (config_hash && hash != config_hash) throw Fail{NGDB_ERR_CONFIG, "checkpoint: config hash mismatch"};
    if (nt != c->params.size()) throw Fail{NGDB_ERR_SHAPE_MISMATCH, "checkpoint: tensor count"};
    std::vector<std::pair<const char*, Param*>> plan;
    for (auto& p : c->params) {
      uint32_t len;
      get(&len, 4);
      std::string name(len, '\0');
      get(name.data(), len);
      int64_t rows, cols;
      get(&rows, 8);
      get(&cols, 8);
      if (name != p.name || rows != p.rows || cols != p.cols)
        throw Fail{NGDB_ERR_SHAPE_MISMATCH, "checkpoint: tensor " + name + " does not match " + p.name};
      if (at + 3 * p.n() * sizeof(float) > blob.size() - 8) throw Fail{NGDB_ERR_DOMAIN, "checkpoint: truncated"};
      plan.emplace_back(blob.data() + at, &p);
      at += 3 * p.n() * sizeof(float);
    }
    if (at != blob.size() - 8) throw Fail{NGDB_ERR_DOMAIN, "checkpoint: trailing bytes"};
    CK(cudaStreamSynchronize(c->stream));
    for (auto& [src, p] : plan) {
      const size_t nb = p->n() * sizeof(float);
      CK(cudaMemcpy(p->w, src, nb, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(p->m, src + nb, nb, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(p->v, src + 2 * nb, nb, cudaMemcpyHostToDevice));
    }
    refresh_weight_splits(c);
    CK(cudaStreamSynchronize(c->stream));
    if (step) *step = st;
  });
}

}  // extern "C"

namespace {

// Width of the evaluator's entity rows: BetaE T_e [2d], fusion / GQE / Q2B d.
int64_t eval_row_width(const ngdb_ctx* c) {
  return c->beta() ? 2 * int64_t(c->desc.dim) : int64_t(c->desc.dim);
}

// The evaluator's entity table for the current parameters (BetaE: T_e and C_e
// of every entity by the step prologue kernel beta_prep; fusion: every fused
// row by the FuseSemantic prologue's GEMMs). Returns (table, C_e or nullptr).
std::pair<const float*, const float*> eval_entity_table(ngdb_ctx* c) {
  const Param& ent = c->params[c->ent_idx];
  if (!c->beta() && !c->fused()) return {ent.w, nullptr};
  const int64_t N = c->desc.n_entities, w = eval_row_width(c);
  if (!c->evtab) {
    c->evtab = dmalloc<float>(N * w + N);
    std::vector<int32_t> idx(2 * N + 1, 0);
    for (int64_t i = 0; i < N; ++i) idx[i] = static_cast<int32_t>(i);  // rows; seg = 0
    c->ev_rows = dmalloc<int32_t>(2 * N + 1);
    CK(cudaMemcpy(c->ev_rows, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice));
  }
  DevArgs a = make_args(c, nullptr);
  a.etab = c->evtab;
  a.etab_c = c->evtab + N * w;
  const SparseTable t{ent.w, ent.m, ent.v, nullptr, static_cast<int32_t>(ent.cols),
                      static_cast<int32_t>(N), c->ev_rows, c->ev_rows + N, nullptr};
  const LaunchCtx lc{c->stream, c->num_sms};
  if (c->beta() && !c->fused()) {
    c->launches += launch_beta_prep(a, t, lc);
  } else {  // fusion (BetaE: Psi_theta rows, then the same prologue kernel)
    if (!c->sem) throw Fail{NGDB_ERR_CONFIG, "semantic store not uploaded (ngdb_semantic_upload)"};
    const int64_t need = fuse_scratch_floats(c->desc.dim, c->desc.semantic_dim, N);
    if (need > c->ev_scratch_cap) {
      CK(cudaStreamSynchronize(c->stream));
      if (c->ev_scratch) CK(cudaFree(c->ev_scratch));
      c->ev_scratch = dmalloc<float>(need);
      c->ev_scratch_cap = need;
    }
    c->launches += fuse_prologue(a, t, c->ev_scratch, c->ev_scratch_cap, lc);
  }
  CK(cudaGetLastError());
  return {c->evtab, c->beta() ? c->evtab + N * w : nullptr};
}

}  // namespace

extern "C" {

int ngdb_eval_entity_table(ngdb_ctx* c, float* rows, int64_t n_rows_floats, float* consts,
                           int64_t n_consts) {
  return guarded([&] {
    if (c->world > 1) throw Fail{NGDB_ERR_CONFIG, "eval_entity_table: row-sharded context"};
    const int64_t N = c->desc.n_entities, w = eval_row_width(c);
    if (n_rows_floats != N * w) throw Fail{NGDB_ERR_SHAPE_MISMATCH, "eval_entity_table: rows size"};
    const auto tab = eval_entity_table(c);
    CK(cudaMemcpyAsync(rows, tab.first, N * w * 4, cudaMemcpyDeviceToHost, c->stream));
    if (consts) {
      if (!tab.second || n_consts != N)
        throw Fail{NGDB_ERR_SHAPE_MISMATCH, "eval_entity_table: consts exist for BetaE only"};
      CK(cudaMemcpyAsync(consts, tab.second, N * 4, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ngdb_read_score_queries(ngdb_ctx* c, float* host, int64_t n_slots) {
  return guarded([&] {
    if (c->world > 1) throw Fail{NGDB_ERR_CONFIG, "read_score_queries: row-sharded context"};
    if (n_slots <= 0) return;
    if (!c->qbuf || n_slots > c->cap_score)
      throw Fail{NGDB_ERR_SHAPE_MISMATCH, "read_score_queries: more slots than the last step had"};
    CK(cudaMemcpyAsync(host, c->qbuf, n_slots * c->query_width() * sizeof(float),
                       cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ngdb_eval_ranks_multi(ngdb_ctx* c, const float* units, int32_t n_queries,
                          const int32_t* unit_offsets, const int32_t* targets,
                          const int32_t* filter_offsets, const int32_t* filter_ids, int32_t* ranks) {
  return guarded([&] {
    if (n_queries < 0 || (n_queries > 0 && (!units || !unit_offsets || !targets ||
                                            !filter_offsets || !ranks)))
      throw Fail{NGDB_ERR_CONFIG, "eval_ranks: null argument"};
    if (c->world > 1) throw Fail{NGDB_ERR_CONFIG, "eval_ranks: row-sharded context"};
    if (n_queries == 0) return;
    const Param& ent = c->params[c->ent_idx];
    const int32_t n_ent = c->desc.n_entities, wq = c->query_width();
    if (filter_offsets[0] != 0 || unit_offsets[0] != 0)
      throw Fail{NGDB_ERR_SHAPE_MISMATCH, "eval_ranks: offsets[0] != 0"};
    // slots: a query's branch units packed inside one aligned group of 8 (the
    // count kernel takes the nearest branch over a thread's 8 slots)
    constexpr int kGroup = 8;
    std::vector<int32_t> slot_query, slot_nb, first(n_queries);
    std::vector<int32_t> slot_unit;
    for (int32_t q = 0; q < n_queries; ++q) {
      const int32_t nb = unit_offsets[q + 1] - unit_offsets[q];
      if (nb < 1 || nb > kGroup) throw Fail{NGDB_ERR_SHAPE_MISMATCH, "eval_ranks: 1..8 branches per query"};
      if (static_cast<int>(slot_query.size() % kGroup) + nb > kGroup)
        while (slot_query.size() % kGroup) {
          slot_query.push_back(-1);
          slot_nb.push_back(0);
          slot_unit.push_back(-1);
        }
      first[q] = static_cast<int32_t>(slot_query.size());
      for (int32_t b = 0; b < nb; ++b) {
        slot_query.push_back(q);
        slot_nb.push_back(b == 0 ? nb : 0);
        slot_unit.push_back(unit_offsets[q] + b);
      }
    }
    const int64_t ns = static_cast<int64_t>(slot_query.size());
    std::vector<float> packed(ns * wq, 0.f);
    for (int64_t i = 0; i < ns; ++i)
      if (slot_unit[i] >= 0)
        std::memcpy(&packed[i * wq], units + static_cast<int64_t>(slot_unit[i]) * wq, wq * 4);
    // filter sets: validated, sorted and de-duplicated per query (they are sets)
    std::vector<int32_t> off(n_queries + 1, 0), ids;
    ids.reserve(filter_offsets[n_queries] > 0 ? filter_offsets[n_queries] : 0);
    for (int32_t q = 0; q < n_queries; ++q) {
      const int32_t t = targets[q];
      if (t < 0 || t >= n_ent) throw Fail{NGDB_ERR_INDEX_OUT_OF_RANGE, "eval_ranks: target out of range"};
      const int32_t b = filter_offsets[q], e = filter_offsets[q + 1];
      if (e < b) throw Fail{NGDB_ERR_SHAPE_MISMATCH, "eval_ranks: filter_offsets not ascending"};
      const size_t first_id = ids.size();
      for (int32_t i = b; i < e; ++i) {
        const int32_t f = filter_ids[i];
        if (f < 0 || f >= n_ent) throw Fail{NGDB_ERR_INDEX_OUT_OF_RANGE, "eval_ranks: filter id out of range"};
        if (f == t) throw Fail{NGDB_ERR_DOMAIN, "eval_ranks: TargetFiltered (target in its filter set)"};
        ids.push_back(f);
      }
      if (!std::is_sorted(ids.begin() + first_id, ids.end())) std::sort(ids.begin() + first_id, ids.end());
      ids.erase(std::unique(ids.begin() + first_id, ids.end()), ids.end());
      off[q + 1] = static_cast<int32_t>(ids.size());
    }
    const int64_t nq = n_queries, nf = static_cast<int64_t>(ids.size());
    auto al = [](int64_t b) { return (b + 255) & ~int64_t(255); };
    const int64_t b_q = al(ns * wq * 4), b_s = al(ns * 4), b_t = al(nq * 4), b_off = al((nq + 1) * 4),
                  b_ids = al(std::max<int64_t>(nf, 1) * 4);
    const int64_t need = b_q + 2 * b_s + b_off + b_ids + 5 * b_t;
    if (need > c->eval_cap) {
      CK(cudaStreamSynchronize(c->stream));
      if (c->eval_buf) CK(cudaFree(c->eval_buf));
      c->eval_cap = need + need / 2;
      CK(cudaMalloc(&c->eval_buf, c->eval_cap));
    }
    char* p = c->eval_buf;
    EvalArgs a{};
    const auto tab = eval_entity_table(c);  // BetaE: T_e | C_e; fusion: fused rows
    a.ent = tab.first;
    a.ent_w = c->beta() ? eval_row_width(c) : (c->fused() ? c->desc.dim : ent.cols);
    a.n_ent = n_ent;
    a.dim = c->beta() ? 2 * c->desc.dim : c->desc.dim;  // BetaE: the 2d-long dot product
    a.backbone = c->beta() ? NGDB_BETAE : (c->fused() ? NGDB_GQE : c->desc.backbone);
    a.ec = tab.second;
    a.alpha = c->desc.alpha_box;
    a.wq = wq;
    a.nq = static_cast<int32_t>(ns);
    a.n_queries = n_queries;
    float* dq = reinterpret_cast<float*>(p);        p += b_q;
    int32_t* dsq = reinterpret_cast<int32_t*>(p);   p += b_s;
    int32_t* dsn = reinterpret_cast<int32_t*>(p);   p += b_s;
    int32_t* dfs = reinterpret_cast<int32_t*>(p);   p += b_t;
    int32_t* dtg = reinterpret_cast<int32_t*>(p);   p += b_t;
    int32_t* doff = reinterpret_cast<int32_t*>(p);  p += b_off;
    int32_t* dids = reinterpret_cast<int32_t*>(p);  p += b_ids;
    a.dt = reinterpret_cast<float*>(p);             p += b_t;
    a.better = reinterpret_cast<int32_t*>(p);       p += b_t;
    a.ties = reinterpret_cast<int32_t*>(p);
    a.q = dq;
    a.slot_query = dsq;
    a.slot_nb = dsn;
    a.first_slot = dfs;
    a.target = dtg;
    a.f_off = doff;
    a.f_ids = dids;
    CK(cudaMemcpyAsync(dq, packed.data(), ns * wq * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dsq, slot_query.data(), ns * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dsn, slot_nb.data(), ns * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dfs, first.data(), nq * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(dtg, targets, nq * 4, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(doff, off.data(), (nq + 1) * 4, cudaMemcpyHostToDevice, c->stream));
    if (nf) CK(cudaMemcpyAsync(dids, ids.data(), nf * 4, cudaMemcpyHostToDevice, c->stream));
    c->h2d_bytes += ns * wq * 4 + 2 * ns * 4 + 2 * nq * 4 + (nq + 1) * 4 + nf * 4;
    c->launches += launch_eval_ranks(a, static_cast<int32_t>(nf), c->stream);
    CK(cudaGetLastError());
    std::vector<int32_t> cnt(2 * nq);
    CK(cudaMemcpyAsync(cnt.data(), a.better, nq * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(cnt.data() + nq, a.ties, nq * 4, cudaMemcpyDeviceToHost, c->stream));
    c->d2h_bytes += 2 * nq * 4;
    CK(cudaStreamSynchronize(c->stream));
    for (int64_t q = 0; q < nq; ++q) ranks[q] = 1 + cnt[q] + cnt[nq + q] / 2;
  });
}

int ngdb_eval_ranks(ngdb_ctx* c, const float* queries, int32_t n_queries, const int32_t* targets,
                    const int32_t* filter_offsets, const int32_t* filter_ids, int32_t* ranks) {
  if (n_queries < 0) return ngdb_eval_ranks_multi(c, queries, n_queries, nullptr, targets,
                                                  filter_offsets, filter_ids, ranks);
  std::vector<int32_t> uo(static_cast<size_t>(n_queries) + 1);
  for (int32_t i = 0; i <= n_queries; ++i) uo[i] = i;
  return ngdb_eval_ranks_multi(c, queries, n_queries, uo.data(), targets, filter_offsets,
                               filter_ids, ranks);
}

// Diagnostics of graph-launched steps recorded under NGDB_STEP_TIMELINE=1:
// busy = sum over steps of (graph end - graph start) on the device, gap = sum of
// idle time between a step's end and the next step's start (the stream waiting
// for the host). Synchronizes and clears the record.
int ngdb_step_timeline(ngdb_ctx* c, double* busy_ms, double* gap_ms, int64_t* n_steps) {
  return guarded([&] {
    CK(cudaStreamSynchronize(c->stream));
    double busy = 0.0, gap = 0.0;
    for (size_t i = 0; i < c->timeline.size(); ++i) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c->timeline[i].first, c->timeline[i].second));
      busy += ms;
      if (i > 0) {
        CK(cudaEventElapsedTime(&ms, c->timeline[i - 1].second, c->timeline[i].first));
        gap += ms;
      }
    }
    if (n_steps) *n_steps = static_cast<int64_t>(c->timeline.size());
    for (auto& [a, b] : c->timeline) {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
    c->timeline.clear();
    if (busy_ms) *busy_ms = busy;
    if (gap_ms) *gap_ms = gap;
  });
}

int ngdb_transfer_bytes(ngdb_ctx* c, int64_t* h2d, int64_t* d2h) {
  return guarded([&] {
    if (h2d) *h2d = c->h2d_bytes;
    if (d2h) *d2h = c->d2h_bytes;
  });
}

int ngdb_flush_l2(ngdb_ctx* c) {
  return guarded([&] {
    if (!c->l2_flush) {
      c->l2_flush_bytes = 512ll << 20;  // > 126 MB L2
      c->l2_flush = dmalloc<float>(c->l2_flush_bytes / 4);
    }
    CK(cudaMemsetAsync(c->l2_flush, c->launches & 0xff, c->l2_flush_bytes, c->stream));
  });
}

// ---- row-sharded step -----------------------------------------

int ngdb_ctx_set_stream(ngdb_ctx* c, void* stream) {
  return guarded([&] {
    CK(cudaStreamSynchronize(c->stream));
    c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
  });
}

namespace {
int64_t up64(int64_t x) { return (x + 63) / 64 * 64; }
}  // namespace

}  // extern "C"

namespace {

// Device blob layout of a rank's owner work lists (ngdb_shard_plan).
struct ShardLayout {
  int64_t o_k = 0, o_slots = 0, o_cand = 0, o_off = 0, o_owned = 0, o_rows = 0, o_seg = 0,
          o_con = 0, o_send = 0, o_recv = 0, o_pos = 0, total = 0, n_owned = 0, n_con = 0;
  ShardLayout() = default;
  explicit ShardLayout(const ngdb_shard_plan& sp) {
    const int64_t G = sp.world, B = sp.batch, nc = sp.n_candidates, U = G * B;
    n_owned = sp.unit_off[U];
    n_con = sp.n_rows ? sp.seg[sp.n_rows] : 0;
    o_slots = o_k + up64(U);
    o_cand = o_slots + up64(U * 3);
    o_off = o_cand + up64(U * nc);
    o_owned = o_off + up64(U + 1);
    o_rows = o_owned + up64(n_owned);
    o_seg = o_rows + up64(sp.n_rows);
    o_con = o_seg + up64(sp.n_rows + 1);
    o_send = o_con + up64(n_con);
    o_recv = o_send + up64(sp.n_send);
    o_pos = o_recv + up64(sp.n_recv);
    total = o_pos + up64(sp.n_anchor_pos);
  }
  void pack(const ngdb_shard_plan& sp, int32_t* h) const {
    const int64_t G = sp.world, B = sp.batch, nc = sp.n_candidates, U = G * B;
    std::memcpy(h + o_k, sp.unit_k, U * 4);
    std::memcpy(h + o_slots, sp.unit_slots, U * 3 * 4);
    std::memcpy(h + o_cand, sp.cand, U * nc * 4);
    std::memcpy(h + o_off, sp.unit_off, (U + 1) * 4);
    if (n_owned) std::memcpy(h + o_owned, sp.owned, n_owned * 4);
    if (sp.n_rows) {
      std::memcpy(h + o_rows, sp.rows, sp.n_rows * 4);
      std::memcpy(h + o_seg, sp.seg, (sp.n_rows + 1) * 4);
      std::memcpy(h + o_con, sp.contrib, n_con * 4);
    }
    if (sp.n_send) std::memcpy(h + o_send, sp.send_rows, int64_t(sp.n_send) * 4);
    if (sp.n_recv) std::memcpy(h + o_recv, sp.recv_slot, int64_t(sp.n_recv) * 4);
    if (sp.n_anchor_pos) std::memcpy(h + o_pos, sp.anchor_pos, int64_t(sp.n_anchor_pos) * 4);
  }
};

// the scalars of a shard plan a device step needs (+ the exchange counts)
struct ShardShape {
  int32_t world = 1, rank = 0, batch = 0, max_anchors = 0, max_slots = 0, n_candidates = 0,
          n_rows = 0, n_send = 0, n_recv = 0;
  std::vector<int32_t> send_cnt, recv_cnt;
  ShardShape() = default;
  explicit ShardShape(const ngdb_shard_plan& sp)
      : world(sp.world), rank(sp.rank), batch(sp.batch), max_anchors(sp.max_anchors),
        max_slots(sp.max_slots), n_candidates(sp.n_candidates), n_rows(sp.n_rows),
        n_send(sp.n_send), n_recv(sp.n_recv), send_cnt(sp.send_cnt, sp.send_cnt + sp.world),
        recv_cnt(sp.recv_cnt, sp.recv_cnt + sp.world) {}
};

void validate_shard(ngdb_ctx* c, const ngdb_step_plan& plan, const ngdb_shard_plan& sp) {
  if (sp.world != c->world || sp.rank != c->rank)
    throw Fail{NGDB_ERR_CONFIG, "shard plan world/rank do not match the context"};
  if (c->beta() && c->desc.dim > 512) throw Fail{NGDB_ERR_MISSING_KERNEL, "sharded BetaE: dim > 512"};
  validate_plan(plan);
  if (plan.n_score_slots > sp.max_slots || plan.n_anchor_slots > sp.max_anchors ||
      plan.n_queries > sp.batch || plan.n_candidates != sp.n_candidates)
    throw Fail{NGDB_ERR_SHAPE_MISMATCH, "step plan exceeds the shard plan's padding"};
  if (!sp.send_cnt || !sp.recv_cnt || sp.n_anchor_pos < plan.n_anchor_slots)
    throw Fail{NGDB_ERR_SHAPE_MISMATCH, "shard plan without lookup exchange lists"};
  int64_t ns = 0, nr = 0;
  for (int q = 0; q < sp.world; ++q) {
    ns += sp.send_cnt[q];
    nr += sp.recv_cnt[q];
  }
  if (ns != sp.n_send || nr != sp.n_recv)
    throw Fail{NGDB_ERR_SHAPE_MISMATCH, "shard plan exchange counts do not add up"};
}

// Exchange buffer sizes of a shard shape (ngdb_shard_buffers order + coef_all,
// then the step table etab, etab_c, cand_local of BetaE / FuseSemantic, and
// FuseSemantic's scratch and anchor_local).
constexpr int kShardBufs = 15;
void shard_buffer_sizes(const ngdb_ctx* c, const ShardShape& sp, int64_t sizes[kShardBufs]) {
  const int64_t G = sp.world, B = sp.batch, S = sp.max_slots, nc = sp.n_candidates;
  const int64_t ew = c->op_ent_w(), wq = c->query_width();
  const Param& rel = c->params[c->rel_idx];
  const int64_t n_red = c->dense_n + rel.n() + rel.rows;
  const int64_t blk = S * wq + B;
  const int64_t z[kShardBufs] = {sp.n_send * ew, sp.n_recv * ew, S * wq,     G * S * wq, G * blk,
                                 blk,            sp.n_recv * ew, sp.n_send * ew, n_red, G * S * nc,
                                 c->step_table() ? sp.n_rows * c->op_ent_w() : 0,
                                 c->step_table() ? sp.n_rows : 0,
                                 c->step_table() ? G * S * nc : 0,
                                 c->fused() ? fuse_scratch_floats(c->desc.dim, c->desc.semantic_dim, sp.n_rows) : 0,
                                 c->fused() ? int64_t(sp.n_send) : 0};
  for (int k = 0; k < kShardBufs; ++k) sizes[k] = z[k];
}
bool shard_buffers_fit(const ngdb_ctx* c, const ShardShape& sp) {
  int64_t sizes[kShardBufs], need = 0;
  shard_buffer_sizes(c, sp, sizes);
  for (int64_t z : sizes) need += up64(std::max<int64_t>(z, 1));
  return need <= c->sh.buf_cap;
}
// (Re)size the exchange buffers (may synchronize) and point sh.bufs at them.
void shard_exchange_buffers(ngdb_ctx* c, const ShardShape& sp) {
  auto& sh = c->sh;
  int64_t sizes[kShardBufs], need = 0;
  shard_buffer_sizes(c, sp, sizes);
  for (int64_t z : sizes) need += up64(std::max<int64_t>(z, 1));
  if (need > sh.buf_cap) {
    CK(cudaStreamSynchronize(c->stream));
    if (sh.buf) CK(cudaFree(sh.buf));
    sh.buf_cap = need + need / 2;
    sh.buf = dmalloc<float>(sh.buf_cap);
    ++c->buffer_gen;
  }
  float* ptr[kShardBufs];
  float* cur = sh.buf;
  for (int k = 0; k < kShardBufs; ++k) {
    ptr[k] = cur;
    cur += up64(std::max<int64_t>(sizes[k], 1));
  }
  ngdb_shard_buffers& b = sh.bufs;
  b.anchor_send = ptr[0]; b.n_anchor_send = sizes[0];
  b.anchor_rows = ptr[1]; b.n_anchor_rows = sizes[1];
  b.query_mine = ptr[2]; b.n_query_mine = sizes[2];
  b.query_all = ptr[3]; b.n_query_all = sizes[3];
  b.dq_part = ptr[4]; b.n_dq_part = sizes[4];
  b.dq_mine = ptr[5]; b.n_dq_mine = sizes[5];
  b.grad_send = ptr[6]; b.n_grad_send = sizes[6];
  b.grad_all = ptr[7]; b.n_grad_all = sizes[7];
  b.reduce = ptr[8]; b.n_reduce = sizes[8];
  sh.coef_all = ptr[9];
  sh.etab = ptr[10];
  sh.etab_c = ptr[11];
  sh.cand_local = reinterpret_cast<int32_t*>(ptr[12]);
  sh.fscratch = ptr[13];
  sh.fscratch_cap = sizes[13];
  sh.anchor_local = reinterpret_cast<int32_t*>(ptr[14]);
}
// Make (plan, owner lists in `blob`) the active sharded step: the step
// prologue on the stream (capturable) and the device views.
void shard_activate(ngdb_ctx* c, ngdb_plan* plan, const ShardShape& sp, const int32_t* blob,
                    const ShardLayout& L) {
  auto& sh = c->sh;
  c->active = plan;
  begin_step_device(c);
  const ngdb_shard_buffers& b = sh.bufs;
  // unset query slots stay defined (their rows are gathered but never read)
  CK(cudaMemsetAsync(b.query_mine, 0, b.n_query_mine * 4, c->stream));
  ShardDev& d = sh.dev;
  d.world = sp.world;
  d.rank = sp.rank;
  d.batch = sp.batch;
  d.max_slots = sp.max_slots;
  d.n_send = sp.n_send;
  d.n_recv = sp.n_recv;
  d.dq_block = int64_t(sp.max_slots) * c->query_width() + sp.batch;
  d.send_rows = blob + L.o_send;
  d.recv_slot = blob + L.o_recv;
  d.unit_k = blob + L.o_k;
  d.unit_slots = blob + L.o_slots;
  d.cand = blob + L.o_cand;
  d.unit_off = blob + L.o_off;
  d.owned = blob + L.o_owned;
  d.query_all = b.query_all;
  d.dq_part = b.dq_part;
  d.coef_all = sh.coef_all;
  sh.n_rows = sp.n_rows;
  sh.rows = blob + L.o_rows;
  sh.seg = blob + L.o_seg;
  sh.contrib = blob + L.o_con;
  sh.send_cnt = sp.send_cnt;
  sh.recv_cnt = sp.recv_cnt;
  sh.active = true;
  c->anc_pos = blob + L.o_pos;
  c->anc_rows = b.anchor_rows;
  const Param& ent = c->params[c->ent_idx];
  const SparseTable te{ent.w, ent.m, ent.v, nullptr, static_cast<int32_t>(ent.cols),
                       sh.n_rows, sh.rows, sh.seg, sh.contrib};
  if (c->fused()) {  // fused rows of every owned row (+ BetaE: Psi_theta, the KL table)
    if (!c->sem) throw Fail{NGDB_ERR_CONFIG, "semantic store not uploaded (ngdb_semantic_upload)"};
    const DevArgs a = make_args(c, plan);
    const double u = sp.n_rows, D = c->desc.dim, L = c->desc.semantic_dim;
    if (c->profiling)
      c->fam_flops[F_ENTITY_PREP] += 2.0 * D * D * L + 2.0 * u * D * (L + D + (c->beta() ? 2 * D : 0));
    timed(c, F_ENTITY_PREP, u * (L * 4 + D * 4 * 2), [&] {
      return fuse_prologue(a, te, sh.fscratch, sh.fscratch_cap, LaunchCtx{c->stream, c->num_sms});
    });
  } else if (c->beta()) {  // the entity side of every owned KL, once per owned row (beta.cu)
    const DevArgs a = make_args(c, plan);
    timed(c, F_ENTITY_PREP, sp.n_rows * (2.0 * ent.cols * 4 + 4),
          [&] { return launch_beta_prep(a, te, LaunchCtx{c->stream, c->num_sms}); });
  }
}

}  // namespace

// Resident sharded step: both blobs in device memory owned by the handle.
struct ngdb_shard_step {
  ngdb_plan plan;
  int32_t* blob = nullptr;
  ShardLayout layout;
  ShardShape shape;
  cudaGraphExec_t exec = nullptr;  // ngdb_shard_step_capture
};

namespace {
// ngdb_shard_begin[_packed]: plan_pk / shard_pk are the caller's pre-packed
// pinned blobs (or null: packed here into the context's staging)
void shard_begin_impl(ngdb_ctx* c, const ngdb_step_plan* plan, const ngdb_shard_plan* sp,
                      const int32_t* plan_pk, int64_t plan_n, const int32_t* shard_pk,
                      int64_t shard_n, ngdb_shard_buffers* out) {
    validate_shard(c, *plan, *sp);
    // Both blobs of this step (its step plan and its owner work lists) go up on
    // the copy stream into double-buffered device slots, as ngdb_step_begin
    // does for the plan: slot i is rewritten once the step two back (its last
    // reader) is done, and this step's kernels wait for the upload — the H2D
    // overlaps the previous step's kernels instead of sitting between them.
    const int i = c->cur;
    c->cur ^= 1;
    auto& sh = c->sh;
    const PlanLayout L(*plan);
    const ShardLayout SL(*sp);
    if ((plan_pk && plan_n != L.total) || (shard_pk && shard_n != SL.total))
      throw Fail{NGDB_ERR_SHAPE_MISMATCH, "shard_begin_packed: packed sizes"};
    // host staging of slot i: its previous H2D (two steps back) must be done
    CK(cudaEventSynchronize(c->staged[i]));
    CK(cudaEventSynchronize(sh.staged[i]));
    if (!plan_pk && L.total > c->staging_cap[i]) {
      if (c->staging[i]) CK(cudaFreeHost(c->staging[i]));
      c->staging_cap[i] = L.total + L.total / 2;
      void* hp = nullptr;
      CK(cudaMallocHost(&hp, c->staging_cap[i] * sizeof(int32_t)));
      c->staging[i] = static_cast<int32_t*>(hp);
    }
    if (!shard_pk && SL.total > sh.staging_cap[i]) {
      if (sh.staging[i]) CK(cudaFreeHost(sh.staging[i]));
      sh.staging_cap[i] = SL.total + SL.total / 2;
      void* hp = nullptr;
      CK(cudaMallocHost(&hp, sh.staging_cap[i] * sizeof(int32_t)));
      sh.staging[i] = static_cast<int32_t*>(hp);
    }
    if (SL.total > sh.blobs_cap[i]) {  // growth: nothing may still read the slot
      CK(cudaStreamSynchronize(c->stream));
      CK(cudaStreamSynchronize(c->copy_stream));
      if (sh.blobs[i]) CK(cudaFree(sh.blobs[i]));
      sh.blobs_cap[i] = SL.total + SL.total / 2;
      sh.blobs[i] = dmalloc<int32_t>(sh.blobs_cap[i]);
    }
    CK(cudaEventRecord(c->blob_free[i ^ 1], c->stream));
    CK(cudaStreamWaitEvent(c->copy_stream, c->blob_free[i], 0));
    upload_plan(c, *plan, &c->stream_plan[i], c->stream_cap[i], c->staging[i], c->copy_stream,
                plan_pk);
    CK(cudaEventRecord(c->staged[i], c->copy_stream));
    if (!shard_pk) SL.pack(*sp, sh.staging[i]);
    CK(cudaMemcpyAsync(sh.blobs[i], shard_pk ? shard_pk : sh.staging[i], SL.total * 4,
                       cudaMemcpyHostToDevice, c->copy_stream));
    c->h2d_bytes += SL.total * 4;
    CK(cudaEventRecord(sh.staged[i], c->copy_stream));
    CK(cudaEventRecord(c->blob_ready[i], c->copy_stream));
    CK(cudaStreamWaitEvent(c->stream, c->blob_ready[i], 0));
    ensure_step_buffers(c, c->stream_plan[i].meta);

    // exchange buffers, then the step prologue and device views
    const ShardShape shape(*sp);
    shard_exchange_buffers(c, shape);
    shard_activate(c, &c->stream_plan[i], shape, sh.blobs[i], SL);
    if (out) *out = sh.bufs;
}
}  // namespace

extern "C" {

int ngdb_shard_begin(ngdb_ctx* c, const ngdb_step_plan* plan, const ngdb_shard_plan* sp,
                     ngdb_shard_buffers* out) {
  return guarded([&] { shard_begin_impl(c, plan, sp, nullptr, 0, nullptr, 0, out); });
}

int64_t ngdb_shard_packed_size(const ngdb_shard_plan* sp) { return ShardLayout(*sp).total; }

int ngdb_shard_pack(const ngdb_shard_plan* sp, int32_t* out, int64_t cap) {
  return guarded([&] {
    const ShardLayout SL(*sp);
    if (cap < SL.total) throw Fail{NGDB_ERR_SHAPE_MISMATCH, "shard_pack: buffer too small"};
    SL.pack(*sp, out);
  });
}

int ngdb_shard_begin_packed(ngdb_ctx* c, const ngdb_step_plan* plan, const int32_t* plan_packed,
                            int64_t plan_n, const ngdb_shard_plan* sp, const int32_t* shard_packed,
                            int64_t shard_n, ngdb_shard_buffers* out) {
  return guarded([&] {
    shard_begin_impl(c, plan, sp, plan_packed, plan_n, shard_packed, shard_n, out);
  });
}

int ngdb_shard_step_create(ngdb_ctx* c, const ngdb_step_plan* plan, const ngdb_shard_plan* sp,
                           ngdb_shard_step** out) {
  ngdb_shard_step* r = nullptr;
  const int rc = guarded([&] {
    validate_shard(c, *plan, *sp);
    r = new ngdb_shard_step();
    const PlanLayout L(*plan);
    std::vector<int32_t> host(L.total);
    pack_plan(*plan, L, host.data());
    r->plan.blob = dmalloc<int32_t>(L.total);
    CK(cudaMemcpy(r->plan.blob, host.data(), L.total * 4, cudaMemcpyHostToDevice));
    r->plan.layout = L;
    r->plan.meta = meta_of(*plan);
    r->layout = ShardLayout(*sp);
    r->shape = ShardShape(*sp);
    host.assign(r->layout.total, 0);
    r->layout.pack(*sp, host.data());
    r->blob = dmalloc<int32_t>(r->layout.total);
    CK(cudaMemcpy(r->blob, host.data(), r->layout.total * 4, cudaMemcpyHostToDevice));
    // size every buffer now: a later begin inside a stream capture must not grow
    ensure_step_buffers(c, r->plan.meta);
    shard_exchange_buffers(c, r->shape);
    *out = r;
  });
  if (rc != NGDB_OK && r) ngdb_shard_step_destroy(r);
  return rc;
}

int ngdb_shard_step_begin(ngdb_ctx* c, ngdb_shard_step* r, ngdb_shard_buffers* out) {
  return guarded([&] {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(c->stream, &cs));
    const bool fits = shard_buffers_fit(c, r->shape);
    if (cs != cudaStreamCaptureStatusNone && !fits)
      throw Fail{NGDB_ERR_CONFIG, "sharded step buffers must be sized before capture"};
    ensure_step_buffers(c, r->plan.meta);
    shard_exchange_buffers(c, r->shape);
    shard_activate(c, &r->plan, r->shape, r->blob, r->layout);
    if (out) *out = c->sh.bufs;
  });
}

int ngdb_shard_step_destroy(ngdb_shard_step* r) {
  if (!r) return NGDB_OK;
  if (r->exec) cudaGraphExecDestroy(r->exec);
  if (r->plan.blob) cudaFree(r->plan.blob);
  if (r->blob) cudaFree(r->blob);
  delete r;
  return NGDB_OK;
}

int ngdb_set_step(ngdb_ctx* c, int64_t step) {
  return guarded([&] { set_step_scalars(c, step); });
}

int ngdb_shard_run(ngdb_ctx* c, int32_t stage) {
  return guarded([&] {
    auto& sh = c->sh;
    if (!sh.active || !c->active) throw Fail{NGDB_ERR_CONFIG, "ngdb_shard_run outside a sharded step"};
    const ngdb_plan* p = c->active;
    const DevArgs a = make_args(c, p);
    const LaunchCtx lc{c->stream, c->num_sms};
    const ngdb_shard_buffers& b = sh.bufs;
    switch (stage) {
      case NGDB_SHARD_ANCHOR_PACK:
        timed(c, F_EMBED, double(b.n_anchor_send) * 4,
              [&] { return launch_shard_anchor_pack(a, sh.dev, b.anchor_send, lc); });
        break;
      case NGDB_SHARD_FORWARD: {
        std::vector<ngdb_pool_desc> v;
        for (const auto& d : p->meta.pools)
          if (d.dir == 0 && d.kind != NGDB_OP_SCORE && d.kind != NGDB_OP_UNION_SCORE &&
              d.kind != NGDB_OP_LOSS)
            v.push_back(d);
        exec_pools(c, p, v);
        break;
      }
      case NGDB_SHARD_QUERY_PACK:
        for (const auto& d : p->meta.pools)
          if (d.dir == 0 && (d.kind == NGDB_OP_SCORE || d.kind == NGDB_OP_LOSS))
            timed(c, F_SCORE, 2.0 * d.count * c->query_width() * 4 + 32.0 * d.count,
                  [&] { return launch_shard_query_pack(a, d.first, d.count, b.query_mine, lc); });
        break;
      case NGDB_SHARD_SCORE: {
        const double nc = p->meta.n_candidates, ew = c->params[c->ent_idx].cols * 4.0;
        const double owned = double(sh.dev.world) * sh.dev.batch * nc / sh.dev.world;
        timed(c, F_LOSS_FWD, owned * (ew + 8) + 2.0 * b.n_dq_part * 4, [&] {
          CK(cudaMemsetAsync(b.dq_part, 0, b.n_dq_part * 4, c->stream));
          return launch_shard_score(a, sh.dev, lc);
        });
        break;
      }
      case NGDB_SHARD_SCORE_DONE:
        timed(c, F_LOSS_FWD, 0.0, [&] {
          return launch_shard_score_done(a, b.dq_mine, int64_t(p->meta.n_score) * c->query_width(),
                                         b.dq_mine + int64_t(sh.dev.max_slots) * c->query_width(),
                                         p->meta.n_queries, lc);
        });
        break;
      case NGDB_SHARD_BACKWARD: {
        const auto& pools = p->meta.pools;
        for (size_t i = 0; i < pools.size(); ++i) {
          const auto& d = pools[i];
          if (d.dir != 1 || d.kind == NGDB_OP_UNION_SCORE) continue;  // routing done by the owners
          if (d.kind == NGDB_OP_SCORE) {  // dL/dq of a union branch arrived in dqbuf
            timed(c, F_SCORE, pool_bytes(c, d, p->meta.n_candidates), [&] { return launch_loss_bwd(a, d.first, d.count, lc); });
          } else if (i + 1 < pools.size() && mergeable(c, d, pools[i + 1])) {
            exec_pool(c, p, d, &pools[i + 1]);
            ++i;
          } else {
            exec_pool(c, p, d);
          }
        }
        break;
      }
      case NGDB_SHARD_GRAD_PACK: {
        const Param& rel = c->params[c->rel_idx];
        SparseTable tr{rel.w, rel.m, rel.v, nullptr, static_cast<int32_t>(rel.cols),
                       p->meta.n_rrows, p->blob + p->layout.rrows, p->blob + p->layout.rseg,
                       p->blob + p->layout.rcon};
        timed(c, F_OPT_RELATION, double(b.n_reduce) * 4 + double(b.n_grad_send) * 4, [&] {
          CK(cudaMemsetAsync(b.reduce, 0, b.n_reduce * 4, c->stream));
          if (c->dense_n)
            CK(cudaMemcpyAsync(b.reduce, c->dense_g, c->dense_n * 4, cudaMemcpyDeviceToDevice, c->stream));
          return launch_shard_grad_pack(a, sh.dev, b.grad_send, lc) +
                 launch_shard_rel_pack(a, tr, b.reduce + c->dense_n, b.reduce + c->dense_n + rel.n(), lc);
        });
        break;
      }
      case NGDB_SHARD_FUSE_BWD: {
        if (!c->fused()) break;
        // dL/d(fused row) of the owned rows: returned anchor rows (grad_all,
        // send order) + owned candidates (every rank's queries and coefs)
        DevArgs af = a;
        af.agbuf = b.grad_all;
        af.qbuf = b.query_all;
        af.coefbuf = sh.coef_all;
        const Param& ent = c->params[c->ent_idx];
        const SparseTable te{ent.w, ent.m, ent.v, c->debug ? ent.g : nullptr,
                             static_cast<int32_t>(ent.cols), sh.n_rows, sh.rows, sh.seg, sh.contrib};
        const ngdb_model_desc& md = c->desc;
        const AdamHyper hp{md.lr, md.beta1, md.beta2, md.eps_adam};
        const double u = sh.n_rows, D = md.dim, L = md.semantic_dim;
        if (c->profiling)
          c->fam_flops[F_OPT_ENTITY] += 2.0 * u * D * (2 * D + L + (c->beta() ? 4 * D : 0)) + 4.0 * D * D * L;
        timed(c, F_OPT_ENTITY, 4.0 * u * D * 4 + u * L * 4, [&] {
          return fuse_backward(af, te, sh.fscratch, sh.fscratch_cap, hp, c->d_bc, lc, false);
        });
        // the fusion's dense gradients join the all-reduce
        if (c->dense_n)
          CK(cudaMemcpyAsync(b.reduce, c->dense_g, c->dense_n * 4, cudaMemcpyDeviceToDevice, c->stream));
        break;
      }
      default: throw Fail{NGDB_ERR_CONFIG, "unknown shard stage"};
    }
    CK(cudaGetLastError());
  });
}

int ngdb_shard_optimizer(ngdb_ctx* c, int64_t step) {
  return guarded([&] {
    auto& sh = c->sh;
    if (!sh.active || !c->active) throw Fail{NGDB_ERR_CONFIG, "ngdb_shard_optimizer outside a sharded step"};
    const ngdb_plan* p = c->active;
    if (step > 0) set_step_scalars(c, step);  // else: ngdb_set_step (capturable)
    const ngdb_model_desc& d = c->desc;
    const AdamHyper hp{d.lr, d.beta1, d.beta2, d.eps_adam};
    const LaunchCtx lc{c->stream, c->num_sms};
    const ngdb_shard_buffers& b = sh.bufs;
    if (c->dense_n)
      CK(cudaMemcpyAsync(c->dense_g, b.reduce, c->dense_n * 4, cudaMemcpyDeviceToDevice, c->stream));
    // entity rows this rank owns: anchors of every rank + owned candidates of every rank's slots
    DevArgs a = make_args(c, p);
    a.agbuf = b.grad_all;
    a.qbuf = b.query_all;
    a.coefbuf = sh.coef_all;
    Param& ent = c->params[c->ent_idx];
    Param& rel = c->params[c->rel_idx];
    SparseTable te{ent.w, ent.m, ent.v, c->debug ? ent.g : nullptr, static_cast<int32_t>(ent.cols),
                   sh.n_rows, sh.rows, sh.seg, sh.contrib};
    if (c->fused())  // Adam on dh (fuse_backward ran in NGDB_SHARD_FUSE_BWD)
      timed(c, F_OPT_ENTITY, 6.0 * sh.n_rows * ent.cols * 4, [&] {
        return fuse_entity_adam(te, sh.fscratch, sh.fscratch_cap, c->desc.dim, c->desc.semantic_dim,
                                c->beta(), hp, c->d_bc, lc);
      });
    else
      timed(c, F_OPT_ENTITY, 6.0 * sh.n_rows * ent.cols * 4,
            [&] { return launch_sparse_adam_entity(a, te, hp, c->d_bc, lc); });
    timed(c, F_OPT_RELATION, 6.0 * rel.n() * 4, [&] {
      return launch_masked_rows_adam(rel.w, rel.m, rel.v, c->debug ? rel.g : nullptr,
                                     b.reduce + c->dense_n, b.reduce + c->dense_n + rel.n(),
                                     static_cast<int>(rel.rows), static_cast<int>(rel.cols), hp,
                                     c->d_bc, lc);
    });
    timed(c, F_OPT_DENSE, 28.0 * c->dense_n, [&] {
      return launch_dense_adam_split(c->dense_w, c->dense_m, c->dense_v, c->dense_g, c->wsplit,
                                     dense_jobs(c), hp, c->d_bc, lc);
    });
    CK(cudaGetLastError());
    sh.active = false;
    c->anc_rows = nullptr;
    c->anc_pos = nullptr;
  });
}

// ---- NCCL owned by the context -------------------------------

}  // extern "C"

namespace {

const NcclApi& nccl_or_fail() {
  const NcclApi& n = nccl_api();
  if (!n.error.empty()) throw Fail{NGDB_ERR_CONFIG, n.error};
  return n;
}
void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Fail{NGDB_ERR_CUDA, std::string(what) + ": " + nccl_api().GetErrorString(r)};
}
void rc_throw(int rc) {
  if (rc != NGDB_OK) throw Fail{rc, g_last_error};
}

// Uneven all-to-all of rows (`width` floats each): scnt[q] rows to rank q from
// `send` (rank-major), rcnt[q] rows from rank q into `recv` (rank-major). One
// NCCL group of point-to-point calls: only rows that are needed travel.
void all_to_all_rows(ngdb_ctx* c, const float* send, const std::vector<int32_t>& scnt, float* recv,
                     const std::vector<int32_t>& rcnt, int64_t width) {
  const NcclApi& n = nccl_api();
  nck(n.GroupStart(), "ncclGroupStart");
  int64_t so = 0, ro = 0;
  for (int q = 0; q < c->world; ++q) {
    if (scnt[q])
      nck(n.Send(send + so * width, size_t(scnt[q]) * width, ncclFloat32, q, c->comm, c->stream),
          "ncclSend");
    if (rcnt[q])
      nck(n.Recv(recv + ro * width, size_t(rcnt[q]) * width, ncclFloat32, q, c->comm, c->stream),
          "ncclRecv");
    so += scnt[q];
    ro += rcnt[q];
  }
  nck(n.GroupEnd(), "ncclGroupEnd");
}

// Stages + collectives + optimizer of the active sharded step, all enqueued on
// the context stream (capturable: no host synchronisation).
void shard_exec(ngdb_ctx* c, int64_t step) {
  if (!c->comm) throw Fail{NGDB_ERR_CONFIG, "ngdb_shard_step_exec: call ngdb_comm_init first"};
  auto& sh = c->sh;
  if (!sh.active) throw Fail{NGDB_ERR_CONFIG, "ngdb_shard_step_exec outside a sharded step"};
  const NcclApi& n = nccl_api();
  const ngdb_shard_buffers b = sh.bufs;
  const int64_t ew = c->op_ent_w();  // rows exchanged at the operators' width
  const int64_t blk = sh.dev.dq_block;
  rc_throw(ngdb_shard_run(c, NGDB_SHARD_ANCHOR_PACK));
  all_to_all_rows(c, b.anchor_send, sh.send_cnt, b.anchor_rows, sh.recv_cnt, ew);
  rc_throw(ngdb_shard_run(c, NGDB_SHARD_FORWARD));
  rc_throw(ngdb_shard_run(c, NGDB_SHARD_QUERY_PACK));
  nck(n.AllGather(b.query_mine, b.query_all, size_t(b.n_query_mine), ncclFloat32, c->comm,
                  c->stream), "ncclAllGather");
  rc_throw(ngdb_shard_run(c, NGDB_SHARD_SCORE));
  nck(n.ReduceScatter(b.dq_part, b.dq_mine, size_t(blk), ncclFloat32, ncclSum, c->comm, c->stream),
      "ncclReduceScatter");
  rc_throw(ngdb_shard_run(c, NGDB_SHARD_SCORE_DONE));
  rc_throw(ngdb_shard_run(c, NGDB_SHARD_BACKWARD));
  rc_throw(ngdb_shard_run(c, NGDB_SHARD_GRAD_PACK));
  all_to_all_rows(c, b.grad_send, sh.recv_cnt, b.grad_all, sh.send_cnt, ew);
  if (c->fused()) rc_throw(ngdb_shard_run(c, NGDB_SHARD_FUSE_BWD));
  nck(n.AllReduce(b.reduce, b.reduce, size_t(b.n_reduce), ncclFloat32, ncclSum, c->comm, c->stream),
      "ncclAllReduce");
  rc_throw(ngdb_shard_optimizer(c, step));
}

}  // namespace

extern "C" {

int ngdb_comm_unique_id(uint8_t* id) {
  return guarded([&] {
    static_assert(sizeof(ncclUniqueId) == NGDB_COMM_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId u;
    nck(nccl_or_fail().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

int ngdb_comm_init(ngdb_ctx* c, const uint8_t* id) {
  return guarded([&] {
    const NcclApi& n = nccl_or_fail();
    if (c->comm) throw Fail{NGDB_ERR_CONFIG, "ngdb_comm_init: communicator already set"};
    CK(cudaSetDevice(c->device));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    nck(n.CommInitRank(&c->comm, c->world, u, c->rank), "ncclCommInitRank");
    // the metadata channel: same ranks, its own communicator and stream, so an
    // exchange thread can all-gather upcoming steps' records while this
    // thread's step collectives are in flight
    nck(n.CommSplit(c->comm, 0, c->rank, &c->meta_comm, nullptr), "ncclCommSplit");
    CK(cudaStreamCreateWithFlags(&c->meta_stream, cudaStreamNonBlocking));
  });
}

int ngdb_comm_allgather_i32(ngdb_ctx* c, const int32_t* send, int64_t count, int32_t* recv) {
  return guarded([&] {
    if (!c->meta_comm) throw Fail{NGDB_ERR_CONFIG, "ngdb_comm_allgather_i32: call ngdb_comm_init first"};
    std::lock_guard<std::mutex> lock(c->meta_mu);
    CK(cudaSetDevice(c->device));
    const int64_t need = count * (c->world + 1);
    if (need > c->meta_cap) {
      CK(cudaStreamSynchronize(c->meta_stream));
      if (c->meta_dev) CK(cudaFree(c->meta_dev));
      c->meta_dev = nullptr;
      CK(cudaMalloc(&c->meta_dev, need * sizeof(int32_t)));
      c->meta_cap = need;
    }
    int32_t* dsend = c->meta_dev + count * c->world;
    CK(cudaMemcpyAsync(dsend, send, count * 4, cudaMemcpyHostToDevice, c->meta_stream));
    nck(nccl_api().AllGather(dsend, c->meta_dev, size_t(count), ncclInt32, c->meta_comm,
                             c->meta_stream), "ncclAllGather");
    CK(cudaMemcpyAsync(recv, c->meta_dev, count * c->world * 4, cudaMemcpyDeviceToHost,
                       c->meta_stream));
    CK(cudaStreamSynchronize(c->meta_stream));
  });
}

int ngdb_shard_step_exec(ngdb_ctx* c, int64_t step) {
  return guarded([&] { shard_exec(c, step); });
}

int ngdb_shard_step_capture(ngdb_ctx* c, ngdb_shard_step* r) {
  return guarded([&] {
    if (!c->comm) throw Fail{NGDB_ERR_CONFIG, "ngdb_shard_step_capture: call ngdb_comm_init first"};
    if (r->exec) CK(cudaGraphExecDestroy(r->exec));
    r->exec = nullptr;
    ensure_step_buffers(c, r->plan.meta);
    shard_exchange_buffers(c, r->shape);  // sized before capture
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    cudaGraph_t g = nullptr;
    try {
      rc_throw(ngdb_shard_step_begin(c, r, nullptr));
      shard_exec(c, 0);
    } catch (...) {
      cudaStreamEndCapture(c->stream, &g);
      if (g) cudaGraphDestroy(g);
      c->sh.active = false;
      throw;
    }
    CK(cudaStreamEndCapture(c->stream, &g));
    const cudaError_t e = cudaGraphInstantiate(&r->exec, g, 0);
    cudaGraphDestroy(g);
    CK(e);
  });
}

int ngdb_shard_step_replay(ngdb_ctx* c, ngdb_shard_step* r, int64_t step) {
  return guarded([&] {
    if (!r->exec) throw Fail{NGDB_ERR_CONFIG, "ngdb_shard_step_replay: capture the step first"};
    set_step_scalars(c, step);
    CK(cudaGraphLaunch(r->exec, c->stream));
  });
}

}  // extern "C"
