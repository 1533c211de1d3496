/* ngdb_cuda.h — C ABI between the host scheduler and the sm_100a kernels.
 *
 * This is the drop-in boundary of the operator-level training step. In the
 * reference it is the KernelRegistry: (OperatorType x backbone) -> batched
 * forward/backward kernels, called by scheduler::run once per popped pool or
 * cardinality class, plus the trainer's
 * adam_step / compute_loss and the arena's gather /
 * scatter_add. The reference ships no header for these (only
 * proj/include/ngdb/{common,kg,query}.hpp exist), so each entry point below cites
 * the SPEC operation it replaces.
 *
 * Conventions: plain C types only; every call returns an ngdb_status (0 = OK) and
 * never throws; ngdb_last_error() returns a thread-local message. Calls after
 * ngdb_ctx_create are asynchronous on the context's CUDA stream unless stated.
 * All device memory (parameters, Adam moments, activation arena, gradient
 * staging, frozen PTE store) is owned by the context.
 */
#ifndef NGDB_CUDA_H_
#define NGDB_CUDA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror the ngdb::Error taxonomy (common.hpp:23-56). */
typedef enum ngdb_status {
  NGDB_OK = 0,
  NGDB_ERR_SHAPE_MISMATCH = 1,     /* ShapeMismatch      (kernels)   */
  NGDB_ERR_INDEX_OUT_OF_RANGE = 2, /* IndexOutOfRange    (arena)     */
  NGDB_ERR_PARAM_OUT_OF_RANGE = 3, /* ParamOutOfRange    (kernels)   */
  NGDB_ERR_DOMAIN = 4,             /* DomainError        (kernels)   */
  NGDB_ERR_MISSING_KERNEL = 5,     /* MissingKernel      (scheduler) */
  NGDB_ERR_NON_FINITE = 6,         /* NonFinite          (trainer)   */
  NGDB_ERR_CONFIG = 7,             /* ConfigError        (cli)       */
  NGDB_ERR_CUDA = 8,               /* CUDA runtime failure           */
  NGDB_ERR_NO_DEVICE = 9           /* no sm_100 device: no CPU fallback exists */
} ngdb_status;

typedef enum ngdb_backbone { NGDB_GQE = 0, NGDB_Q2B = 1, NGDB_BETAE = 2 } ngdb_backbone;

/* Operator kinds in scheduler tie-break order (dag.hpp OpKind). */
typedef enum ngdb_op_kind {
  NGDB_OP_EMBED_ANCHOR = 0,
  NGDB_OP_FUSE_SEMANTIC = 1,
  NGDB_OP_PROJECT = 2,
  NGDB_OP_NEGATE = 3,
  NGDB_OP_INTERSECT = 4,
  NGDB_OP_SCORE = 5,
  NGDB_OP_UNION_SCORE = 6,
  NGDB_OP_LOSS = 7
} ngdb_op_kind;

typedef struct ngdb_model_desc {
  int32_t backbone;     /* ngdb_backbone */
  int32_t n_entities;
  int32_t n_relations;
  int32_t dim;          /* d (GQE, Q2B) or d' (BetaE: rows are 2d' wide) */
  int32_t n_neg;        /* K negatives per query */
  int32_t semantic_dim; /* d_l of the frozen PTE store; 0 = no fusion */
  float gamma;          /* margin, 12.0 */
  float alpha_box;      /* Q2B inside weight, 0.02 */
  float lr;             /* Adam, 1e-4 */
  float beta1, beta2, eps_adam; /* 0.9, 0.999, 1e-8 */
  int32_t max_batch;    /* B_max: widest kernel invocation */
  int32_t max_queries;  /* queries per step the plan buffers are sized for */
  int32_t world;        /* > 1: entity table row-sharded over `world` ranks; this */
  int32_t rank;         /*   context holds rows e = rank (mod world) */
} ngdb_model_desc;

/* One operator node of a kernel invocation. Offsets are float-element offsets
 * into the context's activation arena (the statically planned Eq. 7 slots);
 * -1 = absent. For Bwd nodes `in`/`self` describe the forward mirror. */
typedef struct ngdb_node_desc {
  int32_t out;   /* output tensor (fwd: T_X; bwd: G_X, one row per mirror input) */
  int32_t in[3]; /* forward inputs' tensors */
  int32_t grad;  /* bwd: upstream gradient row; -1 for the Loss mirror */
  int32_t self;  /* bwd: the mirror's forward output */
  int32_t id;    /* entity (EmbedAnchor/FuseSemantic), relation (Project), query (Score/Loss) */
  int32_t aux;   /* anchor slot / project slot / score slot s / intersect stash slot;
                    -1 = union Loss */
} ngdb_node_desc;

/* One kernel invocation = one PopBatch or one cardinality class of it. */
typedef struct ngdb_pool_desc {
  int32_t kind;   /* ngdb_op_kind */
  int32_t dir;    /* 0 = Fwd, 1 = Bwd */
  int32_t k;      /* cardinality class for Intersect/UnionScore, else 0 */
  int32_t first;  /* index of the first node descriptor */
  int32_t count;  /* number of nodes */
  int32_t cycle;  /* Alg. 1 selection index: the invocations of one cycle drain one
                     pool snapshot, so their nodes are independent of each other */
} ngdb_pool_desc;

/* A fully planned training step (host memory; copied by plan_create/step_begin).
 * Sparse-gradient CSR: rows ascending; entity contribution code c >= 0 is the
 * candidate slot s*(1+K)+j of score slot s, c < 0 is anchor slot (-c-1);
 * relation contribution codes are project slots. */
typedef struct ngdb_step_plan {
  int32_t n_queries;
  int32_t n_candidates;          /* 1 + K */
  const int32_t* candidates;     /* [n_queries][n_candidates]: positive, then negatives */
  int32_t n_pools;
  const ngdb_pool_desc* pools;
  int32_t n_nodes;
  const ngdb_node_desc* nodes;
  int64_t arena_elems;           /* activation arena high-water mark (floats) */
  int32_t n_score_slots;         /* Loss (non-union) + Score nodes */
  int32_t n_anchor_slots;        /* EmbedAnchor / FuseSemantic nodes */
  int32_t n_project_slots;       /* Project nodes */
  int32_t n_entity_rows;
  const int32_t* entity_rows;    /* [n_entity_rows] ascending */
  const int32_t* entity_seg;     /* [n_entity_rows + 1] */
  const int32_t* entity_contrib; /* [entity_seg[n]] */
  int32_t n_relation_rows;
  const int32_t* relation_rows;
  const int32_t* relation_seg;
  const int32_t* relation_contrib;
  /* Optional (NULL: the pools run one after another): invocation i may start
   * once pools pool_deps[pool_dep_off[i] .. pool_dep_off[i+1]) are done
   * (earlier indices; data, arena-slab reuse and side-buffer hazards, from the
   * planner). Graph-launched steps then run independent pools concurrently
   * on the context's side streams; results are unchanged. */
  const int32_t* pool_dep_off; /* [n_pools + 1] */
  const int32_t* pool_deps;
} ngdb_step_plan;

/* Owner-side work of one rank in the row-sharded step (ngdb/shard.hpp). */
typedef struct ngdb_shard_plan {
  int32_t world, rank, batch, max_anchors, max_slots, n_candidates;
  const int32_t* anchor_ids; /* [world][max_anchors] entity of every rank's anchor slot */
  const int32_t* unit_k;     /* [world][batch] score slots of each query (1, or 2-3 union branches) */
  const int32_t* unit_slots; /* [world][batch][3] */
  const int32_t* cand;       /* [world][batch][n_candidates] global entity ids */
  const int32_t* unit_off;   /* [world*batch + 1] owned candidate positions per unit */
  const int32_t* owned;
  int32_t n_rows;            /* owner CSR over local entity rows */
  const int32_t* rows;
  const int32_t* seg;
  const int32_t* contrib;    /* code < 0: anchor row at lookup send position -code-1 */
  /* uneven lookup all-to-all (the anchor-gradient return is its reverse) */
  const int32_t* send_cnt;   /* [world] rows sent to each rank (its anchors this rank owns) */
  const int32_t* recv_cnt;   /* [world] rows received from each owner */
  int32_t n_send, n_recv;    /* sums of send_cnt / recv_cnt */
  const int32_t* send_rows;  /* [n_send] local entity rows, requester-major */
  const int32_t* recv_slot;  /* [n_recv] this rank's anchor slots, owner-major */
  int32_t n_anchor_pos;
  const int32_t* anchor_pos; /* [n_anchor_pos] anchor slot -> receive position */
} ngdb_shard_plan;

/* Exchange buffers of the sharded step, owned by the context (device memory,
 * float32, sizes in elements; ew = entity row width, wq = query width,
 * S = max_slots, B = batch). The collectives between the stages:
 *   all-to-all(v)       anchor_send [n_send][ew]    -> anchor_rows [n_recv][ew]
 *                       (rows send_cnt[r] to rank r, recv_cnt[q] from rank q)
 *   all-gather          query_mine [S][wq]          -> query_all [world][S][wq]
 *   reduce-scatter(sum) dq_part [world][S*wq + B]   -> dq_mine [S*wq + B]
 *                       (per rank block: dL/dq of its score slots, then its losses)
 *   all-to-all(v)       grad_send [n_recv][ew]      -> grad_all [n_send][ew]
 *                       (the lookup exchange reversed)
 *   all-reduce(sum)     reduce [dense grads | relation grads | relation touched] */
typedef struct ngdb_shard_buffers {
  float *anchor_send, *anchor_rows, *query_mine, *query_all, *dq_part, *dq_mine, *grad_send,
      *grad_all, *reduce;
  int64_t n_anchor_send, n_anchor_rows, n_query_mine, n_query_all, n_dq_part, n_dq_mine,
      n_grad_send, n_grad_all, n_reduce;
} ngdb_shard_buffers;

typedef enum ngdb_shard_stage {
  NGDB_SHARD_ANCHOR_PACK = 0, /* owned rows of every rank's anchors -> anchor_send */
  NGDB_SHARD_FORWARD = 1,     /* forward pools except Score / UnionScore / Loss (trace order) */
  NGDB_SHARD_QUERY_PACK = 2,  /* score-slot queries -> query_mine */
  NGDB_SHARD_SCORE = 3,       /* owner scoring of all ranks' units over owned candidates */
  NGDB_SHARD_SCORE_DONE = 4,  /* dq_mine / loss_mine -> this rank's Loss results */
  NGDB_SHARD_BACKWARD = 5,    /* backward pools (trace order) */
  NGDB_SHARD_GRAD_PACK = 6,   /* anchor grads -> grad_send; dense + relation grads -> reduce */
  NGDB_SHARD_FUSE_BWD = 7     /* FuseSemantic only, after the gradient all-to-all: the fusion
                                 backward over the owned rows (returned anchor rows + owned
                                 candidates) into the dense grads, which are re-copied into
                                 reduce (the all-reduce follows) */
} ngdb_shard_stage;

typedef struct ngdb_ctx ngdb_ctx;
typedef struct ngdb_plan ngdb_plan;

const char* ngdb_last_error(void);

/* Context: device memory for params + Adam state + arena; one CUDA stream. */
int ngdb_ctx_create(const ngdb_model_desc* desc, int device, ngdb_ctx** out);
int ngdb_ctx_destroy(ngdb_ctx* ctx);
int ngdb_ctx_desc(const ngdb_ctx* ctx, ngdb_model_desc* out);

/* Parameter registry (SPEC.md:337-352 GqeParams/Q2bParams/BetaParams/FusionParams).
 * Names: see DESIGN.md §3.1. Prefix "m:" / "v:" selects Adam moments, "g:" the
 * gradient of the last step (dense: accumulated; sparse: reduced touched rows,
 * only when ngdb_set_debug(ctx, 1)). Synchronous. */
int ngdb_param_count(ngdb_ctx* ctx, int32_t* n);
int ngdb_param_info(ngdb_ctx* ctx, int32_t index, const char** name, int64_t* rows,
                    int64_t* cols, int32_t* sparse);
int ngdb_param_upload(ngdb_ctx* ctx, const char* name, const float* host, int64_t n);
int ngdb_param_download(ngdb_ctx* ctx, const char* name, float* host, int64_t n);
int ngdb_semantic_upload(ngdb_ctx* ctx, const float* host, int64_t n); /* frozen PTE store */
int ngdb_set_debug(ngdb_ctx* ctx, int32_t keep_sparse_grads);

/* Streaming step: packs the plan into pinned staging and issues one H2D copy
 * (on a copy stream, overlapping the previous step's kernels). */
int ngdb_step_begin(ngdb_ctx* ctx, const ngdb_step_plan* plan);
/* flags: NGDB_BEGIN_DEFER_PROLOGUE leaves the step prologue (flag and
 * dense-gradient resets) to the first ngdb_exec_pool / ngdb_step_launch, so a
 * graph-launched step carries it inside its graph. */
#define NGDB_BEGIN_DEFER_PROLOGUE 1
int ngdb_step_begin_ex(ngdb_ctx* ctx, const ngdb_step_plan* plan, int32_t flags);
/* Launch one kernel invocation of the current step (KernelRegistry fwd/bwd).
 * An Intersect class is held until the next call, so that the next class of
 * the same PopBatch shares its launches; errors of a held class surface at the
 * next exec_pool / optimizer_step / step_end call. */
/* Pre-packed plans (the trainer loop's producers pack off the consumer
 * thread): the packed blob of a plan, pinned host memory for it, and a
 * step_begin that only issues its H2D. The packed buffer must stay unchanged
 * until the step's results have been collected (its copy is then long done). */
int64_t ngdb_plan_packed_size(const ngdb_step_plan* plan);
int ngdb_plan_pack(const ngdb_step_plan* plan, int32_t* out, int64_t cap);
int ngdb_host_alloc(int64_t bytes, void** out); /* pinned (cudaMallocHost) */
/* A context-owned pinned ring of at least `ints` int32 (kept across calls, so
 * only the first trainer-loop call pays for the allocation). */
int ngdb_ctx_pinned_ring(ngdb_ctx* ctx, int64_t ints, int32_t** base);
int ngdb_host_free(void* p);
int ngdb_step_begin_packed(ngdb_ctx* ctx, const ngdb_step_plan* plan, const int32_t* packed,
                           int64_t n, int32_t flags);
int ngdb_exec_pool(ngdb_ctx* ctx, const ngdb_pool_desc* pool);
/* Sparse sorted-segment gradient reduce + touched-row Adam, then dense Adam
 * (SPEC.md:550-558 adam_step; Alg. 1 l.21 OptimizerStep). `step` is 1-based. */
int ngdb_optimizer_step(ngdb_ctx* ctx, int64_t step);
/* Every pool of the active streaming step + the optimizer in one call: with
 * use_graph, captured into a CUDA graph (an executable graph is updated in
 * place when the step's topology allows, else instantiated) and launched —
 * ~60 stream launches become one graph launch. Same kernels, same results as
 * ngdb_exec_pool for each pool + ngdb_optimizer_step. */
int ngdb_step_launch(ngdb_ctx* ctx, int64_t step, int32_t use_graph);
/* Waits for the step; copies per-query losses (may be NULL) and the non-finite
 * flag. */
int ngdb_step_end(ngdb_ctx* ctx, float* per_query_loss, int32_t n_queries, double* loss_sum,
                  int32_t* nonfinite);
/* Asynchronous step end: enqueues the D2H of the per-query losses and device
 * flags into a pinned result slot and returns a ticket at once, so the host can
 * plan and launch step i+1 while step i runs. At most 4 tickets outstanding;
 * ngdb_step_wait blocks on one and reports it like ngdb_step_end. */
int ngdb_step_end_async(ngdb_ctx* ctx, int64_t* ticket);
int ngdb_step_wait(ngdb_ctx* ctx, int64_t ticket, float* per_query_loss, int32_t n_queries,
                   double* loss_sum, int32_t* nonfinite);

/* Resident plans: upload once, replay many times (benchmark / graph replay). */
int ngdb_plan_create(ngdb_ctx* ctx, const ngdb_step_plan* plan, ngdb_plan** out);
int ngdb_plan_run(ngdb_ctx* ctx, ngdb_plan* plan, int64_t step); /* all pools + optimizer */
/* Capture (without running) the CUDA graph plan_run replays, so a resident
 * plan's first run costs one graph launch. Call after the last plan_create of
 * a context (a later buffer growth invalidates the capture). */
int ngdb_plan_prepare(ngdb_ctx* ctx, ngdb_plan* plan);

/* Row-sharded step: begin, then stages with the collectives of
 * ngdb_shard_buffers between them, then ngdb_shard_optimizer and ngdb_step_end. */
int ngdb_shard_begin(ngdb_ctx* ctx, const ngdb_step_plan* plan, const ngdb_shard_plan* shard,
                     ngdb_shard_buffers* bufs);
/* The same with the plan and the owner lists pre-packed by the caller (e.g. on
 * producer threads) into pinned memory that stays unchanged until the step's
 * results are collected: only the H2D copies are issued here. */
int64_t ngdb_shard_packed_size(const ngdb_shard_plan* shard);
int ngdb_shard_pack(const ngdb_shard_plan* shard, int32_t* out, int64_t cap);
int ngdb_shard_begin_packed(ngdb_ctx* ctx, const ngdb_step_plan* plan, const int32_t* plan_packed,
                            int64_t plan_n, const ngdb_shard_plan* shard,
                            const int32_t* shard_packed, int64_t shard_n,
                            ngdb_shard_buffers* bufs);
int ngdb_shard_run(ngdb_ctx* ctx, int32_t stage);
/* step <= 0: keep the Adam step scalars of the last ngdb_set_step (graph capture) */
int ngdb_shard_optimizer(ngdb_ctx* ctx, int64_t step);
/* Resident sharded step: the step plan and owner lists uploaded once into
 * device memory owned by the handle, every context buffer sized at create.
 * ngdb_shard_step_begin then only enqueues the step prologue and sets the
 * device views, so begin + stages + collectives + ngdb_shard_optimizer(ctx, 0)
 * can be captured into a CUDA graph and replayed (after ngdb_set_step). */
typedef struct ngdb_shard_step ngdb_shard_step;
int ngdb_shard_step_create(ngdb_ctx* ctx, const ngdb_step_plan* plan,
                           const ngdb_shard_plan* shard, ngdb_shard_step** out);
int ngdb_shard_step_begin(ngdb_ctx* ctx, ngdb_shard_step* step, ngdb_shard_buffers* bufs);
int ngdb_shard_step_destroy(ngdb_shard_step* step);
/* --- NCCL owned by the context (no framework needed) -------
 * Rank 0 creates an id, the caller ships its NGDB_COMM_ID_BYTES to every rank
 * by any channel (MPI, a file, a TCP store), and every rank's context calls
 * ngdb_comm_init (world / rank from ngdb_model_desc). libnccl.so.2 is loaded at
 * run time (the framework's copy when one is already loaded). */
#define NGDB_COMM_ID_BYTES 128
int ngdb_comm_unique_id(uint8_t* id);
int ngdb_comm_init(ngdb_ctx* ctx, const uint8_t* id);
/* Host all-gather of `count` int32 per rank (the packed step metadata of
 * ngdb_step_shard_pack) over the context's metadata communicator (split from
 * the step communicator, own stream): synchronous, and safe to call from ONE
 * exchange thread while another thread launches steps (call order must be the
 * same on every rank). */
int ngdb_comm_allgather_i32(ngdb_ctx* ctx, const int32_t* send, int64_t count, int32_t* recv);
/* The whole active sharded step (after ngdb_shard_begin / ngdb_shard_step_begin):
 * stages, NCCL collectives (uneven all-to-alls of owned rows, all-gather,
 * reduce-scatter, all-reduce) and the optimizer, enqueued on the context
 * stream. step <= 0: Adam scalars of the last ngdb_set_step. */
int ngdb_shard_step_exec(ngdb_ctx* ctx, int64_t step);
/* Capture begin + exec of a resident sharded step into one CUDA graph (NCCL
 * collectives inside); replay sets the Adam scalars of `step` and launches it. */
int ngdb_shard_step_capture(ngdb_ctx* ctx, ngdb_shard_step* step);
int ngdb_shard_step_replay(ngdb_ctx* ctx, ngdb_shard_step* step, int64_t step_no);
/* Streaming ABI helpers of the operator microbench: run an
 * Intersect invocation held back for class merging now; read arena floats
 * [offset, offset + n) (synchronous); fix the tcgen05 GEMMs' split-K for the
 * process (0 = per launch; 1 makes a row's result independent of the rows
 * sharing its launch, so batched and per-op executions agree bit for bit). */
int ngdb_exec_flush(ngdb_ctx* ctx);
int ngdb_read_arena(ngdb_ctx* ctx, int64_t offset, int64_t n, float* out);
int ngdb_set_gemm_split(int32_t split);
/* Adam bias-correction scalars of 1-based step t (host -> device, not capturable). */
int ngdb_set_step(ngdb_ctx* ctx, int64_t step);
/* Run the context's launches on an external stream (e.g. the framework stream
 * that also carries the collectives); NULL restores the private stream. */
int ngdb_ctx_set_stream(ngdb_ctx* ctx, void* cuda_stream);
int ngdb_plan_destroy(ngdb_plan* plan);

/* Device timing on the context stream (CUDA events). */
int ngdb_sync(ngdb_ctx* ctx);
int ngdb_timer_start(ngdb_ctx* ctx);
int ngdb_timer_stop(ngdb_ctx* ctx, float* ms);
/* Per-kernel-family timing: when enabled, exec/optimizer calls record CUDA
 * events around every launch; read accumulated ms and launch counts by family. */
int ngdb_profile_enable(ngdb_ctx* ctx, int32_t on);
int ngdb_profile_read(ngdb_ctx* ctx, int32_t family, double* ms, int64_t* launches,
                      double* bytes);
/* algorithmic fp32 GEMM flops accumulated by a family while profiling */
int ngdb_profile_flops(ngdb_ctx* ctx, int32_t family, double* flops);
int32_t ngdb_profile_families(void);
const char* ngdb_profile_family_name(int32_t family);
/* Kernel launches issued so far by this context (all families). */
int64_t ngdb_launch_count(ngdb_ctx* ctx);
/* Cumulative bytes of step data the streaming ABI copied: plan uploads (H2D)
 * and loss/flag read-backs (D2H). */
/* Checkpoint (versioned binary blob of named parameter tensors +
 * config hash; cadence SPEC.md:587). Writes every registry tensor's theta and
 * Adam m, v plus `step` (so a resumed run continues bit-identically) with an
 * FNV-1a trailer. Load checks magic/version/checksum (NGDB_ERR_DOMAIN when
 * corrupt), backbone + dim (NGDB_ERR_CONFIG: BackboneMismatch), config_hash
 * unless 0 (NGDB_ERR_CONFIG), tensor names/shapes (NGDB_ERR_SHAPE_MISMATCH). */
int ngdb_checkpoint_save(ngdb_ctx* ctx, const char* path, uint64_t config_hash, int64_t step);
int ngdb_checkpoint_load(ngdb_ctx* ctx, const char* path, uint64_t config_hash, int64_t* step);

/* Query embeddings of the last executed step's score slots (each query's Loss
 * slot, or its union branches' Score slots; ngdb_node_desc.aux), [n_slots][wq],
 * copied back synchronously. With the forward pools of a plan executed alone
 * (no backward, no optimizer) this is the evaluator's query encoder. */
int ngdb_read_score_queries(ngdb_ctx* ctx, float* host, int64_t n_slots);

/* Evaluator hot path (SPEC.md:602-646 `evaluator`: filtered_rank over all
 * entities, mean-rank ties; replaces the per-query full-entity scoring loop of
 * evaluate()). queries [n_queries][wq] (GQE: q; Q2B: centre |
 * offset) scored against the context's current entity table; targets [n];
 * filter CSR filter_offsets [n+1] (offsets[0] = 0), filter_ids (sets; duplicates
 * ignored). ranks[q] = 1 + #{e not in filter+target: d(e) < d(target)}
 * + floor(#ties / 2). Synchronous. Backbones: GQE (L1), Q2B (box), BetaE
 * (queries alpha | beta, distance KL(entity || query)), GQE + FuseSemantic (L1
 * against the fused rows), BetaE + FuseSemantic (KL against Psi_theta's Beta
 * parameters). A target inside its own filter is NGDB_ERR_DOMAIN (SPEC
 * TargetFiltered). */
/* The evaluator's entity table for the current parameters (tests / callers):
 * BetaE rows T_e = [psi(s)-psi(a) | psi(s)-psi(b)] [n_entities][2d] and consts
 * C_e [n_entities] of KL(entity || query) = lnB(q) + C_e + <q, T_e>; fusion
 * rows sigma(W_p [h | F s] + b_p) [n_entities][d] (consts NULL; BetaE +
 * fusion: T_e, C_e of Psi_theta's rows); GQE / Q2B the entity table itself. */
int ngdb_eval_entity_table(ngdb_ctx* ctx, float* rows, int64_t n_rows_floats, float* consts,
                           int64_t n_consts);
int ngdb_eval_ranks(ngdb_ctx* ctx, const float* queries, int32_t n_queries, const int32_t* targets,
                    const int32_t* filter_offsets, const int32_t* filter_ids, int32_t* ranks);
/* The same for queries with several embeddings (union patterns: one per DNF
 * branch): query q's branches are units[unit_offsets[q] ..
 * unit_offsets[q+1]) (1..8), an entity's distance is the nearest branch's
 * (UnionScore = max score). */
int ngdb_eval_ranks_multi(ngdb_ctx* ctx, const float* units, int32_t n_queries,
                          const int32_t* unit_offsets, const int32_t* targets,
                          const int32_t* filter_offsets, const int32_t* filter_ids, int32_t* ranks);
/* Diagnostics: with NGDB_STEP_TIMELINE=1 in the environment, graph-launched
 * steps record device timestamps; returns the summed device time of the steps
 * and the summed idle gaps between them, then clears the record. */
int ngdb_step_timeline(ngdb_ctx* ctx, double* busy_ms, double* gap_ms, int64_t* n_steps);
int ngdb_transfer_bytes(ngdb_ctx* ctx, int64_t* h2d, int64_t* d2h);
/* ngdb_step_launch graphs: launches served by updating a cached executable
 * graph of the same invocation structure vs fresh instantiations. */
int ngdb_graph_stats(ngdb_ctx* ctx, int64_t* updates, int64_t* instantiations);
/* Flush L2 by writing a buffer larger than it (timing hygiene). */
int ngdb_flush_l2(ngdb_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* NGDB_CUDA_H_ */
