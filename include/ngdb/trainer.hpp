// ngdb/trainer.hpp — training-step planning and the consumer loop
// (SPEC.md:513-600 trainer module; Alg. 1).
//
// plan_training_step is the host half of the hot path: build + fuse + augment
// the batch DAG, run the Max-Fillness planner, and emit the packed device plan
// (node descriptors per kernel invocation, candidate ids, sparse-gradient CSR).
// Trainer drives one ngdb_ctx (one GPU) through the C ABI in ngdb_cuda.h.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ngdb/dag.hpp"
#include "ngdb/ngdb_cuda.h"
#include "ngdb/sampler.hpp"
#include "ngdb/scheduler.hpp"

namespace ngdb {

// Defaults from Appendix C and SPEC.md:518-521, 586.
struct TrainConfig {
  Backbone backbone = Backbone::GQE;
  int32_t dim = 400;
  int32_t batch = 512;
  double lr = 1e-4;
  double gamma = 12.0;
  double alpha_box = 0.02;
  int32_t n_neg = 128;
  int32_t b_max = 512;
  bool semantic = false;
  int32_t semantic_dim = 0;
  bool sharded = false;  // entity table row-sharded across ranks
  bool query_level = false;  // query-level baseline executor (SchedulerConfig::query_level)
  // Device arena slabs reused along the Eq. 7 free list (true), or a private
  // slab per tensor (false, default): the trace and its byte statistics are
  // the same; private slabs drop the write-after-read hazards between pools so
  // independent pools can run concurrently (+7-10 MB per step).
  bool device_reuse = false;
  uint64_t seed_params = 2;
  uint64_t seed_sampler = 3;
};

int32_t query_width(Backbone b, int32_t dim);
int32_t entity_width(Backbone b, int32_t dim);
int32_t relation_width(Backbone b, int32_t dim);

// Parameter registry + deterministic host init (SURVEY A-12):
// tensor i is filled row-major from Rng(seed).fork(i).
struct ParamSpec {
  std::string name;
  int64_t rows = 0, cols = 0;
  bool sparse = false;
};
// semantic_dim > 0 appends the fusion tensors fus_f [d][d_l], fus_wp [d][2d],
// fus_bp [1][d] (no bias on F, SURVEY A-7).
std::vector<ParamSpec> param_specs(Backbone b, int32_t n_entities, int32_t n_relations,
                                   int32_t dim, int32_t semantic_dim = 0);
std::vector<float> init_param(Backbone b, int32_t n_entities, int32_t n_relations, int32_t dim,
                              const std::string& name, uint64_t seed, double gamma = 12.0,
                              int32_t semantic_dim = 0);

// Frozen semantic store helpers.
std::vector<float> synth_semantic_store(int32_t n_entities, int32_t dim, uint64_t seed);
void write_ngse(const std::string& path, const float* data, int64_t count, int32_t dim);
std::vector<float> read_ngse(const std::string& path, int64_t* count, int32_t* dim);

struct StepPlanHost {
  std::vector<ngdb_pool_desc> pools;
  std::vector<ngdb_node_desc> nodes;
  std::vector<int32_t> candidates;
  std::vector<int32_t> entity_rows, entity_seg, entity_contrib;
  std::vector<int32_t> relation_rows, relation_seg, relation_contrib;
  int32_t n_queries = 0, n_candidates = 0;
  int32_t n_score_slots = 0, n_anchor_slots = 0, n_project_slots = 0;
  int64_t arena_elems = 0;
  // scoring units (sharded step): per query, its score slots — the Loss slot,
  // or the branch Score slots of a union in UnionScore input order — and the
  // entity of every anchor slot
  std::vector<int32_t> unit_k, unit_slots;  // [B], [B][3] (-1 padded)
  std::vector<int32_t> anchor_ids;          // [n_anchor_slots]
  // invocation dependencies (Planner::inv_deps), CSR over pools
  std::vector<int32_t> pool_dep_off, pool_deps;
  ExecutionTrace trace;
  ngdb_step_plan view() const;
};

StepPlanHost plan_training_step(const TrainingBatch& batch, const TrainConfig& cfg);

// One GPU's trainer: owns the device context, uploads the initial parameters.
class Trainer {
 public:
  Trainer(const TrainConfig& cfg, int32_t n_entities, int32_t n_relations, int device = 0);
  ~Trainer();
  Trainer(const Trainer&) = delete;
  Trainer& operator=(const Trainer&) = delete;

  // Plans and runs one step (all pools + OptimizerStep); returns Σ_i loss_i.
  double step(const TrainingBatch& batch, std::vector<float>* per_query_loss = nullptr);
  // Runs an already planned step through the streaming ABI.
  double run_planned(const StepPlanHost& plan, std::vector<float>* per_query_loss = nullptr);

  ngdb_ctx* ctx() const { return ctx_; }
  int64_t steps_done() const { return step_; }

 private:
  TrainConfig cfg_;
  ngdb_ctx* ctx_ = nullptr;
  int64_t step_ = 0;
};

void check_status(int rc);  // throws the ngdb::Error matching an ngdb_status

}  // namespace ngdb
