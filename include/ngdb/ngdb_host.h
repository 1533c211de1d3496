/* ngdb_host.h — C ABI over the host C++ engine (graph, sampler, planner, trainer).
 *
 * The reference exposes these as C++ (kg.hpp, query.hpp, and the SPEC's sampler /
 * scheduler / trainer modules); this flat C surface is what a foreign binding
 * (ctypes here, see INTEGRATION.md for cgo/JNI stubs) links against. Every call
 * returns an ngdb_status from ngdb_cuda.h; messages via ngdb_last_error().
 */
#ifndef NGDB_HOST_H_
#define NGDB_HOST_H_

#include <stdint.h>

#include "ngdb/ngdb_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ngdb_graph ngdb_graph; /* GraphSplit (kg.hpp:72-77) */
typedef struct ngdb_batch ngdb_batch; /* sampled training batch + negatives */
typedef struct ngdb_step ngdb_step;   /* a planned step (trace + device plan) */

/* --- knowledge graph (kg.hpp:25-89) ------------------------ */
int ngdb_graph_synthetic(const char* shape, uint64_t seed, ngdb_graph** out);
int ngdb_graph_from_triples(int32_t n_entities, int32_t n_relations, const int32_t* train,
                            int64_t n_train, const int32_t* valid, int64_t n_valid,
                            const int32_t* test, int64_t n_test, ngdb_graph** out);
int ngdb_graph_load(const char* dir, ngdb_graph** out); /* load_graph (kg.hpp:79-81) */
int ngdb_graph_info(const ngdb_graph* g, int32_t* n_entities, int32_t* n_relations,
                    int64_t* n_train, int64_t* n_valid, int64_t* n_test);
/* split: 0 train, 1 valid, 2 test; writes 3*n int32 (h, r, t) */
int ngdb_graph_triples(const ngdb_graph* g, int32_t split, int32_t* out, int64_t n);
/* answer_query on train (full=0) or full (full=1) graph; returns count via *n,
 * writes up to cap ids (kg.hpp:83-85) */
int ngdb_graph_answer(const ngdb_graph* g, int32_t full, int32_t pattern, const int32_t* anchors,
                      const int32_t* relations, int32_t* out, int64_t cap, int64_t* n);
/* predictive_answers (kg.hpp:87-89): obs = answers on the train
 * graph, miss = full-graph answers not in obs (obs ⊎ miss = full answers);
 * counts via *n_obs / *n_miss, up to the caps written */
int ngdb_graph_predictive_answers(const ngdb_graph* g, int32_t pattern, const int32_t* anchors,
                                  const int32_t* relations, int32_t* obs, int64_t obs_cap,
                                  int64_t* n_obs, int32_t* miss, int64_t miss_cap, int64_t* n_miss);
int ngdb_graph_destroy(ngdb_graph* g);

/* --- sampler ----------------------------------- */
/* Samples b queries with patterns ~ weights (14, enum order) from
 * Rng(seed).fork(tag), then negatives against full-graph answers. */
int ngdb_batch_sample(const ngdb_graph* g, const double* pattern_weights, int32_t b,
                      int32_t n_neg, uint64_t seed, uint64_t tag, ngdb_batch** out);
/* Builds a batch from arrays: anchors [b][3], relations [b][4] (-1 padded). */
int ngdb_batch_from_arrays(int32_t b, const int32_t* patterns, const int32_t* anchors,
                           const int32_t* relations, const int32_t* positives, int32_t n_neg,
                           const int32_t* negatives, ngdb_batch** out);
int ngdb_batch_info(const ngdb_batch* bt, int32_t* b, int32_t* n_neg);
int ngdb_batch_arrays(const ngdb_batch* bt, int32_t* patterns, int32_t* anchors,
                      int32_t* relations, int32_t* positives, int32_t* negatives);
int ngdb_batch_destroy(ngdb_batch* bt);

/* --- planner (Alg. 1) ------------------------------------- */
int ngdb_step_build(const ngdb_batch* bt, int32_t backbone, int32_t dim, int32_t b_max,
                    int32_t semantic, ngdb_step** out);
/* flags: bit0 semantic (FuseSemantic anchors), bit1 sharded (phase-ordered
 * execution of the row-sharded step: every tensor gets a private device slot;
 * the trace is unchanged), bit2 query-level baseline executor (SPEC.md:664-672:
 * queries grouped by pattern, groups run sequentially, no operator batching
 * across patterns; same kernels, same sinks and gradients), bit3 device slab
 * reuse along the Eq. 7 free list (default: a private slab per tensor, so
 * independent pools can run concurrently; the trace is the same) */
int ngdb_step_build_ex(const ngdb_batch* bt, int32_t backbone, int32_t dim, int32_t b_max,
                       int32_t flags, ngdb_step** out);
int ngdb_step_view(const ngdb_step* s, ngdb_step_plan* view);
/* ExecutionTrace as JSON; with_nodes=1 includes popped node ids per record. */
int ngdb_step_trace_json(const ngdb_step* s, int32_t with_nodes, char* buf, int64_t cap,
                         int64_t* len);
int ngdb_step_destroy(ngdb_step* s);

/* --- row-sharded step (ngdb/shard.hpp) ---------------------- */
typedef struct ngdb_shard ngdb_shard;
/* this rank's metadata for the host all-gather */
int ngdb_step_shard_info(const ngdb_step* s, int32_t* n_anchor_slots, int32_t* n_score_slots,
                         int32_t* batch, int32_t* n_candidates);
int ngdb_step_shard_meta(const ngdb_step* s, int32_t* anchor_ids, int32_t* unit_k,
                         int32_t* unit_slots, int32_t* cand);
int ngdb_shard_build(int32_t world, int32_t rank, int32_t batch, int32_t max_anchors,
                     int32_t max_slots, int32_t n_candidates, const int32_t* anchor_ids_all,
                     const int32_t* unit_k_all, const int32_t* unit_slots_all,
                     const int32_t* cand_all, ngdb_shard** out);
/* Packed metadata: ONE int32 record per rank (fixed stride for a batch
 * capacity; layout in ngdb/shard.hpp). Each rank packs its planned step, the
 * records are all-gathered (ngdb_comm_allgather_i32, or any host channel) and
 * ngdb_shard_build_packed turns the rank-major records into this rank's plan. */
int64_t ngdb_shard_meta_stride(int32_t batch_cap, int32_t n_candidates);
int ngdb_step_shard_pack(const ngdb_step* s, int32_t batch_cap, int32_t* out, int64_t stride);
int ngdb_shard_build_packed(int32_t world, int32_t rank, const int32_t* gathered, int64_t stride,
                            int32_t batch_cap, ngdb_shard** out);
int ngdb_shard_view(const ngdb_shard* s, ngdb_shard_plan* view);
int ngdb_shard_destroy(ngdb_shard* s);
/* rows e = rank (mod world) of a parameter's deterministic init (entity table) */
int ngdb_param_init_shard(int32_t backbone, int32_t n_entities, int32_t n_relations, int32_t dim,
                          const char* name, uint64_t seed, int32_t world, int32_t rank,
                          float* out, int64_t n);

/* --- reference-interface helpers (common.hpp:60-127) ----- */
/* Rng(seed) (forked with fork_tag when >= 0), `skip` draws discarded, next draw */
uint64_t ngdb_rng_next(uint64_t seed, int64_t fork_tag, int32_t skip);
/* out[i*reps + j] = j-th Rng(seed).below(ns[i]) in draw order */
int ngdb_rng_below(uint64_t seed, const uint64_t* ns, int32_t count, int32_t reps, uint64_t* out);
/* Eq. 4 selection over the 16 pools (Fwd kinds then Bwd kinds) */
int ngdb_select_pool(const int64_t* counts, const int64_t* head_timestamps, int32_t* pool);
/* JSON-lines round trip of one query record (query.hpp:57-69) */
int ngdb_jsonl_roundtrip(const char* line, char* out, int64_t cap);

/* --- parameters ------------------------------------------- */
int ngdb_param_init(int32_t backbone, int32_t n_entities, int32_t n_relations, int32_t dim,
                    const char* name, uint64_t seed, float* out, int64_t n);
/* same, for a model with semantic fusion of a d_l-wide store (fus_f, fus_wp,
 * fus_bp follow the backbone's tensors in the registry) */
int ngdb_param_init_ex(int32_t backbone, int32_t n_entities, int32_t n_relations, int32_t dim,
                       int32_t semantic_dim, const char* name, uint64_t seed, float* out,
                       int64_t n);

/* --- semantic store (NGSE format SPEC.md:593) ---- */
/* Synthetic frozen PTE rows: N(0,1)/sqrt(d_l) from Rng(seed), row-major. */
int ngdb_semantic_synth(int32_t n_entities, int32_t dim, uint64_t seed, float* out);
/* NGSE file: "NGSE", u32 version 1, u64 count, u32 dim, count*dim f32 (all LE). */
int ngdb_ngse_write(const char* path, const float* data, int64_t count, int32_t dim);
/* *count, *dim from the header; rows copied when out != NULL and cap >= count*dim. */
int ngdb_ngse_read(const char* path, float* out, int64_t cap, int64_t* count, int32_t* dim);

/* --- the public training call: plan + run one step on a context ----------- */
int ngdb_train_step(ngdb_ctx* ctx, const ngdb_batch* bt, int32_t b_max, int64_t step,
                    float* per_query_loss, double* loss_sum);
/* The trainer loop (SPEC.md:568-576 train; producers SPEC.md:591): n_steps
 * steps of freshly sampled batches, batch i from Rng(seed).fork(first_tag + i)
 * with patterns ~ pattern_weights. n_producers host threads sample and plan
 * (0 = hardware threads - 1); the calling thread uploads each plan, launches
 * it and reads step i's losses back while step i+1 runs. Same batches, plans
 * and update order as sampling + ngdb_train_step in a loop. Adam steps are
 * first_step+1 .. first_step+n_steps. loss_per_step [n_steps] (may be NULL),
 * per_query_loss [n_steps][batch] (may be NULL). timings: see below. */
typedef struct ngdb_train_opts {
  const double* pattern_weights; /* 14, enum order (query.hpp:14-29) */
  int32_t batch;                 /* queries per step (512) */
  int32_t n_neg;                 /* must equal the context's n_neg */
  int32_t b_max;                 /* Max-Fillness B_max (512) */
  int32_t n_producers;           /* 0: hardware threads - 1 */
  int32_t queue_depth;           /* planned batches ahead; 0: 2 * n_producers */
  uint64_t seed;                 /* sampler seed (3) */
  uint64_t first_tag;
  int32_t in_flight;             /* steps submitted ahead of the oldest uncollected one; 0: 3 */
  int32_t flags;                 /* NGDB_TRAIN_NO_GRAPHS: stream launches instead of step graphs */
  int32_t steady_from;           /* > 0: timings[6] = host seconds from the consumer reaching step
                                    steady_from (its plan wait included) to the last step's losses
                                    read back — the steady-state window after warm-up steps
                                    of the same call (timings then needs 7 entries) */
} ngdb_train_opts;
#define NGDB_TRAIN_NO_GRAPHS 1
int ngdb_train_run(ngdb_ctx* ctx, const ngdb_graph* g, const ngdb_train_opts* opts,
                   int64_t first_step, int32_t n_steps, double* loss_per_step,
                   float* per_query_loss, double* timings);
/* The trainer loop with the trainer's feedback paths (SPEC.md:218-235, 571,
 * 587, 594-595): difficulty tracking (always: after every step, the mean
 * per-query loss of each pattern in the batch goes into the EMA tracker),
 * adaptive π (refreshed every refresh_every steps over the support of
 * opts->pattern_weights; batch i is sampled with refresh floor(i / R), so runs
 * do not depend on the producer count), a JSON-lines metrics log and a
 * checkpoint cadence. fb may be NULL (= ngdb_train_run). */
typedef struct ngdb_train_feedback {
  int32_t adaptive;          /* 1: adaptive π */
  int32_t refresh_every;     /* 0: 100 */
  double decay, eta, floor;  /* EMA decay, temperature η, floor ε; 0: 0.9, 1.0, 0.01 */
  double* ema_loss;          /* [14] tracker state in/out (NULL: fresh tracker) */
  int64_t* observations;     /* [14] in/out (with ema_loss) */
  double* pi_per_step;       /* [n_steps][14] π each batch was sampled with (may be NULL) */
  const char* metrics_path;  /* JSON-lines {step, loss, ema[14], queries_per_s, peak_bytes}; NULL: off */
  const char* checkpoint_path;
  int32_t checkpoint_every;  /* 0: off (SPEC default 1,000) */
  uint64_t config_hash;
} ngdb_train_feedback;
int ngdb_train_run_ex(ngdb_ctx* ctx, const ngdb_graph* g, const ngdb_train_opts* opts,
                      const ngdb_train_feedback* fb, int64_t first_step, int32_t n_steps,
                      double* loss_per_step, float* per_query_loss, double* timings);
/* The row-sharded trainer loop (needs ngdb_comm_init): batch i of
 * rank r from Rng(seed).fork((first_tag + i) * world + r); producer threads
 * sample, plan and pack, an exchange thread all-gathers the packed metadata in
 * step order (ngdb_comm_allgather_i32) and builds the owner lists, the calling
 * thread launches ngdb_shard_step_exec per step and reads losses back one step
 * behind. timings (may be NULL): 6 doubles — consumer seconds waiting for
 * plans, submitting, waiting for results; exchange-thread seconds in the
 * all-gather; consumer seconds in ngdb_shard_begin; producer count (with
 * opts->steady_from > 0: 8 doubles, + the steady-state window and the
 * consumer seconds in ngdb_shard_step_exec). */
int ngdb_shard_train_run(ngdb_ctx* ctx, const ngdb_graph* g, const ngdb_train_opts* opts,
                         int64_t first_step, int32_t n_steps, double* loss_per_step,
                         double* timings);
/* The sampler's adaptive rule, exposed for tests and callers:
 * record_difficulty on one (pattern, loss); update_distribution over the
 * support of `base` (NULL: all 14 patterns). */
int ngdb_record_difficulty(double* ema_loss, int64_t* observations, double decay, int32_t pattern,
                           double loss);
int ngdb_update_distribution(const double* ema_loss, const int64_t* observations, double eta,
                             double floor, const double* base, double* weights_out);
/* timings (may be NULL) receives 6 doubles: seconds the calling thread spent
 * waiting for planned batches, submitting (upload + launches), waiting for
 * step results, and of the submit time: step_begin, exec_pool calls,
 * optimizer_step. */

/* Streaming run of an already built step (H2D of its plan inside the call). */
int ngdb_run_step(ngdb_ctx* ctx, const ngdb_step* s, int64_t step, float* per_query_loss,
                  double* loss_sum);

#ifdef __cplusplus
}
#endif

#endif /* NGDB_HOST_H_ */
