// Operator DAG construction (Alg. 1 lines 1-2).
//
// Node-id order: depth-first over the pattern's branches in
// definition order, trailing projection after the intersection/union, sink last.
// Union patterns are DNF-rewritten: each branch ends in its own Score node, the
// branches meet in UnionScore. Training DAGs end in Loss:
// non-union patterns use Loss as the fused scoring+loss sink (no Score node);
// union patterns append Loss after UnionScore.
#include "ngdb/dag.hpp"

#include <queue>

namespace ngdb {
namespace {

class Builder {
 public:
  explicit Builder(QueryDag& d, bool semantic) : d_(d), semantic_(semantic) {}

  int32_t add(OpKind kind, std::initializer_list<int32_t> inputs, int32_t payload = -1) {
    OperatorNode n;
    n.id = static_cast<int32_t>(d_.nodes.size());
    n.op = {kind, Direction::Fwd};
    int slot = 0;
    for (int32_t in : inputs) {
      n.inputs[slot] = in;
      d_.nodes[in].consumer = n.id;
      d_.nodes[in].consumer_slot = slot;
      d_.edges.emplace_back(in, n.id);
      ++slot;
    }
    n.n_inputs = slot;
    if (kind == OpKind::Intersect || kind == OpKind::UnionScore) n.cardinality = slot;
    n.payload = payload;
    d_.nodes.push_back(n);
    return n.id;
  }
  int32_t anchor(int32_t entity) {
    return add(semantic_ ? OpKind::FuseSemantic : OpKind::EmbedAnchor, {}, entity);
  }
  int32_t proj(int32_t in, int32_t rel) { return add(OpKind::Project, {in}, rel); }
  // anchor followed by a chain of projections
  int32_t path(int32_t entity, std::initializer_list<int32_t> rels) {
    int32_t cur = anchor(entity);
    for (int32_t r : rels) cur = proj(cur, r);
    return cur;
  }

 private:
  QueryDag& d_;
  bool semantic_;
};

}  // namespace

const char* op_kind_name(OpKind k) {
  static const char* kNames[kOpKinds] = {"EmbedAnchor", "FuseSemantic", "Project", "Negate",
                                         "Intersect",   "Score",        "UnionScore", "Loss"};
  return kNames[static_cast<int>(k)];
}

const char* backbone_name(Backbone b) {
  switch (b) {
    case Backbone::GQE: return "gqe";
    case Backbone::Q2B: return "q2b";
    case Backbone::BETAE: return "betae";
  }
  return "?";
}

Backbone parse_backbone(const std::string& s) {
  if (s == "gqe") return Backbone::GQE;
  if (s == "q2b") return Backbone::Q2B;
  if (s == "betae") return Backbone::BETAE;
  throw ConfigError("backbone: " + s);
}

std::vector<QueryInstance> dnf_rewrite(const QueryInstance& q) {
  q.validate();
  const auto& a = q.anchors;
  const auto& r = q.relations;
  if (q.pattern == Pattern::U2)
    return {QueryInstance{Pattern::P1, {a[0]}, {r[0]}}, QueryInstance{Pattern::P1, {a[1]}, {r[1]}}};
  if (q.pattern == Pattern::UP)
    return {QueryInstance{Pattern::P2, {a[0]}, {r[0], r[2]}},
            QueryInstance{Pattern::P2, {a[1]}, {r[1], r[2]}}};
  throw NotAUnionPattern(std::string("not a union pattern: ") + pattern_info(q.pattern).name);
}

QueryDag build_dag(const QueryInstance& q, DagMode mode, bool semantic) {
  q.validate();
  QueryDag d;
  d.pattern = q.pattern;
  d.nodes.reserve(12);
  Builder b(d, semantic);
  const auto& a = q.anchors;
  const auto& r = q.relations;
  const bool train = mode == DagMode::Train;
  const OpKind sink_kind = train ? OpKind::Loss : OpKind::Score;
  int32_t top = -1;
  switch (q.pattern) {
    case Pattern::P1: top = b.path(a[0], {r[0]}); break;
    case Pattern::P2: top = b.path(a[0], {r[0], r[1]}); break;
    case Pattern::P3: top = b.path(a[0], {r[0], r[1], r[2]}); break;
    case Pattern::I2: {
      int32_t x = b.path(a[0], {r[0]});
      int32_t y = b.path(a[1], {r[1]});
      top = b.add(OpKind::Intersect, {x, y});
      break;
    }
    case Pattern::I3: {
      int32_t x = b.path(a[0], {r[0]});
      int32_t y = b.path(a[1], {r[1]});
      int32_t z = b.path(a[2], {r[2]});
      top = b.add(OpKind::Intersect, {x, y, z});
      break;
    }
    case Pattern::PI: {
      int32_t x = b.path(a[0], {r[0], r[1]});
      int32_t y = b.path(a[1], {r[2]});
      top = b.add(OpKind::Intersect, {x, y});
      break;
    }
    case Pattern::IP: {
      int32_t x = b.path(a[0], {r[0]});
      int32_t y = b.path(a[1], {r[1]});
      top = b.proj(b.add(OpKind::Intersect, {x, y}), r[2]);
      break;
    }
    case Pattern::U2:
    case Pattern::UP: {
      int32_t branch_scores[2];
      auto branches = dnf_rewrite(q);
      for (int i = 0; i < 2; ++i) {
        const auto& br = branches[i];
        int32_t cur = b.anchor(br.anchors[0]);
        for (int32_t rel : br.relations) cur = b.proj(cur, rel);
        branch_scores[i] = b.add(OpKind::Score, {cur});
      }
      int32_t u = b.add(OpKind::UnionScore, {branch_scores[0], branch_scores[1]});
      if (train) d.sinks.push_back(b.add(OpKind::Loss, {u}));
      else d.sinks.push_back(u);
      return d;
    }
    case Pattern::IN2: {
      int32_t x = b.path(a[0], {r[0]});
      int32_t y = b.add(OpKind::Negate, {b.path(a[1], {r[1]})});
      top = b.add(OpKind::Intersect, {x, y});
      break;
    }
    case Pattern::IN3: {
      int32_t x = b.path(a[0], {r[0]});
      int32_t y = b.path(a[1], {r[1]});
      int32_t z = b.add(OpKind::Negate, {b.path(a[2], {r[2]})});
      top = b.add(OpKind::Intersect, {x, y, z});
      break;
    }
    case Pattern::PIN: {
      int32_t x = b.path(a[0], {r[0], r[1]});
      int32_t y = b.add(OpKind::Negate, {b.path(a[1], {r[2]})});
      top = b.add(OpKind::Intersect, {x, y});
      break;
    }
    case Pattern::PNI: {
      int32_t x = b.add(OpKind::Negate, {b.path(a[0], {r[0], r[1]})});
      int32_t y = b.path(a[1], {r[2]});
      top = b.add(OpKind::Intersect, {x, y});
      break;
    }
    case Pattern::INP: {
      int32_t x = b.path(a[0], {r[0]});
      int32_t y = b.add(OpKind::Negate, {b.path(a[1], {r[1]})});
      top = b.proj(b.add(OpKind::Intersect, {x, y}), r[2]);
      break;
    }
  }
  d.sinks.push_back(b.add(sink_kind, {top}));
  return d;
}

FusedDag fuse(const std::vector<QueryDag>& batch) {
  FusedDag f;
  size_t total = 0, edges = 0;
  for (const auto& d : batch) {
    total += d.nodes.size();
    edges += d.edges.size();
  }
  f.nodes.reserve(total * 2);
  f.edges.reserve(edges * 2 + total);
  f.origin.reserve(total * 2);
  f.patterns.reserve(batch.size());
  for (size_t qi = 0; qi < batch.size(); ++qi) {
    const QueryDag& d = batch[qi];
    const int32_t base = static_cast<int32_t>(f.nodes.size());
    for (OperatorNode n : d.nodes) {
      n.id += base;
      for (int k = 0; k < n.n_inputs; ++k) n.inputs[k] += base;
      if (n.consumer >= 0) n.consumer += base;
      n.query = static_cast<int32_t>(qi);
      f.nodes.push_back(n);
      f.origin.push_back(static_cast<int32_t>(qi));
    }
    for (auto [u, v] : d.edges) f.edges.emplace_back(u + base, v + base);
    for (int32_t s : d.sinks) f.sinks.push_back(s + base);
    f.patterns.push_back(d.pattern);
  }
  f.n_fwd = static_cast<int32_t>(f.nodes.size());
  return f;
}

FusedDag add_gradient_nodes(FusedDag f) {
  const int32_t n = f.n_fwd;
  f.nodes.reserve(2 * static_cast<size_t>(n));
  f.origin.reserve(2 * static_cast<size_t>(n));
  for (int32_t i = 0; i < n; ++i) {
    const OperatorNode x = f.nodes[i];
    OperatorNode b;
    b.id = n + i;
    b.op = {x.op.kind, Direction::Bwd};
    b.cardinality = x.cardinality;
    b.payload = x.payload;
    b.query = x.query;
    b.mirror = i;
    // Scheduling predecessor: the mirror of the forward consumer (it produces
    // this node's upstream gradient), or the forward Loss for the new source.
    b.inputs[0] = x.consumer >= 0 ? n + x.consumer : i;
    b.n_inputs = 1;
    f.nodes[i].mirror = b.id;
    f.nodes.push_back(b);
    f.origin.push_back(x.query);
    f.edges.emplace_back(b.inputs[0], b.id);
  }
  f.has_gradients = true;
  return f;
}

FusedDag build_training_dag(const std::vector<QueryInstance>& batch, bool semantic) {
  std::vector<QueryDag> dags;
  dags.reserve(batch.size());
  for (const auto& q : batch) dags.push_back(build_dag(q, DagMode::Train, semantic));
  return add_gradient_nodes(fuse(dags));
}

DagAdjacency adjacency(const FusedDag& f) {
  const size_t n = f.nodes.size();
  DagAdjacency a;
  a.succ_begin.assign(n + 1, 0);
  a.indegree.assign(n, 0);
  for (auto [u, v] : f.edges) {
    ++a.succ_begin[u + 1];
    ++a.indegree[v];
  }
  for (size_t i = 0; i < n; ++i) a.succ_begin[i + 1] += a.succ_begin[i];
  a.succ.resize(f.edges.size());
  std::vector<int32_t> fill(a.succ_begin.begin(), a.succ_begin.end() - 1);
  for (auto [u, v] : f.edges) a.succ[fill[u]++] = v;
  return a;
}

bool is_acyclic(const FusedDag& f) {
  DagAdjacency a = adjacency(f);
  std::queue<int32_t> q;
  for (size_t i = 0; i < f.nodes.size(); ++i)
    if (a.indegree[i] == 0) q.push(static_cast<int32_t>(i));
  size_t seen = 0;
  while (!q.empty()) {
    int32_t u = q.front();
    q.pop();
    ++seen;
    for (int32_t k = a.succ_begin[u]; k < a.succ_begin[u + 1]; ++k)
      if (--a.indegree[a.succ[k]] == 0) q.push(a.succ[k]);
  }
  return seen == f.nodes.size();
}

}  // namespace ngdb
