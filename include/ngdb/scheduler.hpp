// ngdb/scheduler.hpp — Max-Fillness operator scheduler with eager reference
// counting (SPEC.md:444-511 scheduler, SPEC.md:257-330 tensor-arena; Alg. 1,
// PAPER.md:663-698; Eq. 4; Eq. 7).
//
// B200 design: the schedule depends only on DAG structure, never on values, so
// the whole step is planned on the host before any launch. The planner runs
// Alg. 1 symbolically — pools, Max-Fillness selection, ⌈n/B_max⌉ drains,
// cardinality classes, refcount release, successor unlock — and assigns every
// tensor a static slot in one device arena by replaying the size-class free list
// (Eq. 7 reclamation becomes slot reuse). Each kernel invocation is reported to a
// callback that emits device node descriptors; the trace is the parity artefact
// compared bit-for-bit with the oracle's literal executor.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <string>
#include <utility>
#include <vector>

#include "ngdb/dag.hpp"

namespace ngdb {

enum class ReleasePolicy : uint8_t { Eager = 0, EndOfDag = 1 };

struct SchedulerConfig {
  Backbone backbone = Backbone::GQE;
  int32_t b_max = 512;
  int32_t query_width = 400;  // elements of a query embedding (GQE d, Q2B 2d, BetaE 2d')
  int32_t n_candidates = 129; // 1 + K
  int32_t elem_bytes = 4;     // trace byte accounting (f32 throughput mode)
  ReleasePolicy policy = ReleasePolicy::Eager;
  // Device slots: reuse freed slots (the Eq. 7 replay) or give every tensor its
  // own slot. The sharded step runs forward / scoring / backward as phases
  // (DESIGN.md §6), an order the reuse plan does not cover; the trace itself is
  // always the Eq. 7 replay of `policy`.
  bool device_reuse = true;
  // Query-level baseline executor (SPEC.md:664-672 run_query_level): queries
  // are grouped by pattern and the groups run one after another (enum order),
  // each group's DAG stage by stage with its own kernel invocations (Alg. 1
  // restricted to the group) — no operator batching across patterns.
  bool query_level = false;
};

// One PopBatch: a drain of the selected pool.
struct TraceRecord {
  int32_t step = 0;    // pop index (the Eq. 7 scheduling step)
  int32_t cycle = 0;   // selection index (Alg. 1 loop iteration)
  OperatorType type;
  int32_t batch = 0;
  std::vector<std::pair<int32_t, int32_t>> classes;  // (k, n_k) for set operators
  int64_t bytes_reclaimed = 0;
  int64_t live_bytes = 0;  // after the pop's releases
  std::vector<int32_t> nodes;  // popped node ids in pop order
};

struct ExecutionTrace {
  std::vector<TraceRecord> records;
  int64_t invocations = 0;  // kernel calls (one per cardinality class for set ops)
  int64_t peak_bytes = 0;
  int64_t free_list_hits = 0;
  int64_t total_nodes = 0;
  std::string to_json() const;
};

// Eq. 4 with the SPEC tie rules: max count, then oldest head timestamp, then
// pool order. Throws AllPoolsEmpty.
int select_pool(const std::array<int64_t, kPoolCount>& counts,
                const std::array<int64_t, kPoolCount>& head_timestamp);

// Tensor model (SURVEY A-2): forward node X owns
// T_X, consumed by its forward consumer and — when the consumer's backward
// kernel re-reads its inputs (bwd_reads_inputs) — by Bwd(consumer); a Loss
// sink's T_X is consumed by Bwd(Loss). Bwd(X) owns G_X with one row per
// forward input of X, consumed by Bwd(input_i).
bool bwd_reads_inputs(OpKind kind, Backbone backbone);

struct TensorModel {
  int32_t query_width;
  int32_t n_candidates;
  int64_t fwd_elems(const FusedDag& f, const OperatorNode& x) const;
  int64_t bwd_rows(const FusedDag& f, const OperatorNode& bwd) const;      // n_in of mirror
  int64_t bwd_row_elems(const FusedDag& f, const OperatorNode& bwd) const; // width of a row
};

struct Invocation {
  OperatorType type;
  int32_t k = 0;          // cardinality class (set ops), else 0
  const int32_t* nodes = nullptr;
  int32_t n = 0;
  int32_t step = 0;
  int32_t cycle = 0;  // selection index: the pops of one cycle are one drain
};

class Planner {
 public:
  explicit Planner(SchedulerConfig cfg) : cfg_(cfg) {}

  using InvokeFn = std::function<void(const Invocation&)>;
  // Runs Alg. 1 over f (forward + gradient nodes). `invoke` is called once per
  // kernel invocation, in execution order, after that invocation's output slots
  // are assigned and before its inputs are released.
  ExecutionTrace run(const FusedDag& f, const InvokeFn& invoke);

  // Device arena slot (byte offset, 16-byte aligned) of T_X / G_X; -1 if none.
  int64_t fwd_slot(int32_t node) const { return fwd_slot_[node]; }
  int64_t bwd_slot(int32_t node) const { return bwd_slot_[node]; }
  int64_t arena_bytes() const { return arena_top_; }
  const SchedulerConfig& config() const { return cfg_; }
  // Invocation i (emission order) must follow inv_deps[inv_dep_off[i] ..
  // inv_dep_off[i+1]) (earlier invocations: data, slab-reuse and side-buffer
  // hazards); any order consistent with these runs the step identically.
  const std::vector<int32_t>& inv_dep_off() const { return inv_dep_off_; }
  const std::vector<int32_t>& inv_deps() const { return inv_deps_; }

 private:
  SchedulerConfig cfg_;
  std::vector<int32_t> inv_dep_off_, inv_deps_;
  std::vector<int64_t> fwd_slot_, bwd_slot_;
  int64_t arena_top_ = 0;
};

}  // namespace ngdb
