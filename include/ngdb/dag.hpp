// ngdb/dag.hpp — operator DAGs (SPEC.md query-model module).
//
// No reference header exists for this module (only common/kg/query.hpp ship);
// the types and functions follow the SPEC operations:
//   OperatorType / OperatorNode / QueryDag / FusedDag
//   build_dag
//   dnf_rewrite
//   fuse                                                SPEC.md:142-150  (Alg. 1 l.1)
//   add_gradient_nodes                                  SPEC.md:151-159  (Alg. 1 l.2)
// Node-id order, edge order and the training-sink convention are pinned in
// DESIGN.md §2.4 and are part of the bit-exact contract.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "ngdb/query.hpp"

namespace ngdb {

// Kind order is the fixed tie-break order of the scheduler (A-4).
enum class OpKind : uint8_t {
  EmbedAnchor = 0,
  FuseSemantic = 1,
  Project = 2,
  Negate = 3,
  Intersect = 4,
  Score = 5,
  UnionScore = 6,
  Loss = 7,
};
constexpr int kOpKinds = 8;
enum class Direction : uint8_t { Fwd = 0, Bwd = 1 };
enum class Backbone : uint8_t { GQE = 0, Q2B = 1, BETAE = 2 };

const char* op_kind_name(OpKind k);
const char* backbone_name(Backbone b);
Backbone parse_backbone(const std::string& s);  // throws ConfigError

struct OperatorType {
  OpKind kind = OpKind::EmbedAnchor;
  Direction dir = Direction::Fwd;
  // pool index: Fwd before Bwd, then kind order — 16 pools
  int pool() const { return static_cast<int>(dir) * kOpKinds + static_cast<int>(kind); }
  static OperatorType from_pool(int pool) {
    return {static_cast<OpKind>(pool % kOpKinds), static_cast<Direction>(pool / kOpKinds)};
  }
  bool is_set_op() const { return kind == OpKind::Intersect || kind == OpKind::UnionScore; }
};
constexpr int kPoolCount = 2 * kOpKinds;

struct OperatorNode {
  int32_t id = -1;
  OperatorType op;
  // forward data inputs (fwd nodes) or scheduling predecessor (bwd nodes)
  int32_t inputs[3] = {-1, -1, -1};
  int32_t n_inputs = 0;
  int32_t cardinality = 0;   // |inputs| for Intersect/UnionScore (k in {2,3})
  int32_t payload = -1;      // EmbedAnchor/FuseSemantic: entity; Project: relation
  int32_t query = 0;         // origin query index (FusedDag) / 0 in a QueryDag
  int32_t mirror = -1;       // Fwd<->Bwd partner (after add_gradient_nodes)
  int32_t consumer = -1;     // forward consumer (fwd nodes), -1 for the sink
  int32_t consumer_slot = 0; // position of this node in consumer's inputs
};

// Per-query DAG. Sinks are Loss nodes (training) or Score/UnionScore (eval).
struct QueryDag {
  Pattern pattern = Pattern::P1;
  std::vector<OperatorNode> nodes;
  std::vector<std::pair<int32_t, int32_t>> edges;  // (from, to) in creation order
  std::vector<int32_t> sinks;
};

struct FusedDag {
  std::vector<OperatorNode> nodes;                 // fwd nodes first; bwd appended
  std::vector<std::pair<int32_t, int32_t>> edges;  // creation order
  std::vector<int32_t> sinks;                      // forward sinks, batch order
  std::vector<int32_t> origin;                     // query index per node
  std::vector<Pattern> patterns;                   // per query
  int32_t n_fwd = 0;
  bool has_gradients = false;
};

enum class DagMode : uint8_t { Train = 0, Eval = 1 };

// Forward DAG of one query. `semantic` replaces EmbedAnchor by FuseSemantic
// (SPEC.md:589). Union patterns are DNF-rewritten first.
QueryDag build_dag(const QueryInstance& q, DagMode mode = DagMode::Train, bool semantic = false);

// 2u -> [1p, 1p]; up -> [2p, 2p] (projection distributed over the union).
std::vector<QueryInstance> dnf_rewrite(const QueryInstance& q);  // throws NotAUnionPattern

FusedDag fuse(const std::vector<QueryDag>& batch);
FusedDag add_gradient_nodes(FusedDag f);

// Convenience: build + fuse + augment for a whole batch.
FusedDag build_training_dag(const std::vector<QueryInstance>& batch, bool semantic = false);

// Successor lists (CSR) in edge-creation order; indegrees per node.
struct DagAdjacency {
  std::vector<int32_t> succ_begin;  // n+1
  std::vector<int32_t> succ;        // targets
  std::vector<int32_t> indegree;
};
DagAdjacency adjacency(const FusedDag& f);

// Topological sort check (acyclicity invariant).
bool is_acyclic(const FusedDag& f);

}  // namespace ngdb
