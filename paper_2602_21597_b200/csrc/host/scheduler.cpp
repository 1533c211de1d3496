// Max-Fillness planner: Alg. 1 run symbolically on the host,
// with Eq. 7 eager reclamation replayed as static device-arena slot reuse.
// Scheduler rules follow SPEC.md:463-510 and DESIGN.md §2.6 (SURVEY A-4).
#include "ngdb/scheduler.hpp"

#include <algorithm>
#include <unordered_map>

namespace ngdb {

int select_pool(const std::array<int64_t, kPoolCount>& counts,
                const std::array<int64_t, kPoolCount>& head_timestamp) {
  int best = -1;
  for (int p = 0; p < kPoolCount; ++p) {
    if (counts[p] <= 0) continue;
    if (best < 0 || counts[p] > counts[best] ||
        (counts[p] == counts[best] && head_timestamp[p] < head_timestamp[best]))
      best = p;  // equal count + equal timestamp keeps the earlier pool (type order)
  }
  if (best < 0) throw AllPoolsEmpty("select_pool: every pool is empty");
  return best;
}

// Which backward kernels re-read their forward inputs (the activations the
// refcount must keep alive): set operators and scoring recompute from inputs;
// Q2B / BetaE projections need the pre-activation offset; BetaE negation needs
// alpha, beta. GQE/Q2B Project/Negate backward use only the upstream gradient.
bool bwd_reads_inputs(OpKind kind, Backbone backbone) {
  switch (kind) {
    case OpKind::Intersect:
    case OpKind::Score:
    case OpKind::UnionScore:
    case OpKind::Loss: return true;
    case OpKind::Project: return backbone != Backbone::GQE;
    case OpKind::Negate: return backbone == Backbone::BETAE;
    default: return false;
  }
}

int64_t TensorModel::fwd_elems(const FusedDag& f, const OperatorNode& x) const {
  (void)f;
  switch (x.op.kind) {
    case OpKind::Score:
    case OpKind::UnionScore: return n_candidates;
    case OpKind::Loss: return 1;
    default: return query_width;
  }
}

int64_t TensorModel::bwd_rows(const FusedDag& f, const OperatorNode& bwd) const {
  return f.nodes[bwd.mirror].n_inputs;
}

int64_t TensorModel::bwd_row_elems(const FusedDag& f, const OperatorNode& bwd) const {
  const OperatorNode& x = f.nodes[bwd.mirror];
  if (x.n_inputs == 0) return 0;
  return fwd_elems(f, f.nodes[x.inputs[0]]);
}

namespace {

struct Slot {
  int64_t bytes = 0;
  int64_t offset = -1;
  int32_t rc = 0;
};

class SlotArena {
 public:
  SlotArena(ReleasePolicy policy, bool reuse) : policy_(policy), reuse_(reuse) {}

  int32_t alloc(int64_t bytes, int32_t rc) {
    if (rc < 1) throw ZeroRefcount("alloc with refcount < 1");
    Slot s;
    s.bytes = bytes;
    s.rc = rc;
    int32_t prev = -1;  // previous tenant of the reused slab
    auto& fl = free_[bytes];
    if (!fl.empty()) {
      prev = fl.back();
      s.offset = slots_[prev].offset;
      fl.pop_back();
      ++hits_;
    } else {
      s.offset = top_;
      top_ += (bytes + 15) / 16 * 16;
    }
    if (!reuse_) {  // private device slot; the trace statistics are unchanged
      s.offset = dev_top_;
      dev_top_ += (bytes + 15) / 16 * 16;
      prev = -1;
    }
    live_ += bytes;
    peak_ = std::max(peak_, live_);
    slots_.push_back(s);
    prev_.push_back(prev);
    return static_cast<int32_t>(slots_.size() - 1);
  }
  // tensor that occupied this tensor's device slab before it (-1: fresh slab)
  int32_t prev_tenant(int32_t id) const { return prev_[id]; }
  int32_t size() const { return static_cast<int32_t>(slots_.size()); }
  // returns bytes reclaimed (0 if still referenced)
  int64_t release(int32_t id) {
    Slot& s = slots_[id];
    if (s.rc <= 0) throw DoubleRelease("tensor released with refcount 0");
    if (--s.rc > 0) return 0;
    if (policy_ == ReleasePolicy::EndOfDag) return 0;
    free_[s.bytes].push_back(id);
    live_ -= s.bytes;
    return s.bytes;
  }
  void check_live(int32_t id) const {
    if (slots_[id].rc <= 0) throw ZeroRefcount("use after reclamation");
  }
  int64_t offset(int32_t id) const { return slots_[id].offset; }
  int64_t live() const { return live_; }
  int64_t peak() const { return peak_; }
  int64_t hits() const { return hits_; }
  int64_t top() const { return reuse_ ? top_ : dev_top_; }

 private:
  ReleasePolicy policy_;
  bool reuse_;
  int64_t dev_top_ = 0;
  std::vector<Slot> slots_;
  std::vector<int32_t> prev_;
  std::unordered_map<int64_t, std::vector<int32_t>> free_;  // size class -> released slot ids
  int64_t live_ = 0, peak_ = 0, hits_ = 0, top_ = 0;
};

struct Pool {
  std::vector<std::pair<int32_t, int32_t>> q;  // (node, enqueue cycle)
  size_t head = 0;
  int64_t size() const { return static_cast<int64_t>(q.size() - head); }
};

}  // namespace

ExecutionTrace Planner::run(const FusedDag& f, const InvokeFn& invoke) {
  if (!f.has_gradients) throw MissingKernel("planner requires a training DAG with gradient nodes");
  const int32_t n = static_cast<int32_t>(f.nodes.size());
  const int32_t nf = f.n_fwd;
  const TensorModel tm{cfg_.query_width, cfg_.n_candidates};
  const int64_t eb = cfg_.elem_bytes;

  DagAdjacency adj = adjacency(f);
  std::vector<int32_t> indeg = adj.indegree;

  SlotArena arena(cfg_.policy, cfg_.device_reuse);
  std::vector<int32_t> t_fwd(nf, -1), t_bwd(n, -1);
  fwd_slot_.assign(nf, -1);
  bwd_slot_.assign(n, -1);

  ExecutionTrace tr;
  tr.total_nodes = n;
  std::array<Pool, kPoolCount> pools;
  std::vector<int32_t> ready;
  ready.reserve(n);
  for (int32_t i = 0; i < n; ++i)
    if (indeg[i] == 0) ready.push_back(i);

  std::vector<int32_t> batch, cls;
  int64_t executed = 0;
  int32_t cycle = 0, step = 0;


  // query-level mode: nodes of later pattern groups wait in `deferred` until
  // every node of the current group has executed
  const bool ql = cfg_.query_level;
  std::vector<int32_t> deferred;
  int32_t group = -1;
  auto group_of = [&](int32_t v) { return static_cast<int32_t>(f.patterns[f.origin[v]]); };
  if (ql) {
    for (int32_t v : ready) deferred.push_back(v);
    ready.clear();
  }

  // Output allocation for node o (its T or G tensor).
  auto allocate = [&](int32_t o) {
    const OperatorNode& x = f.nodes[o];
    if (x.op.dir == Direction::Fwd) {
      int32_t rc = 1;  // the forward consumer, or Bwd(Loss) for the sink
      if (x.consumer >= 0 && bwd_reads_inputs(f.nodes[x.consumer].op.kind, cfg_.backbone)) ++rc;
      t_fwd[o] = arena.alloc(tm.fwd_elems(f, x) * eb, rc);
      fwd_slot_[o] = arena.offset(t_fwd[o]);
    } else {
      const int64_t rows = tm.bwd_rows(f, x);
      if (rows == 0) return;
      t_bwd[o] = arena.alloc(rows * tm.bwd_row_elems(f, x) * eb, static_cast<int32_t>(rows));
      bwd_slot_[o] = arena.offset(t_bwd[o]);
    }
  };
  // Tensors consumed by node o, in release order.
  auto for_each_input = [&](int32_t o, auto&& fn) {
    const OperatorNode& x = f.nodes[o];
    if (x.op.dir == Direction::Fwd) {
      for (int k = 0; k < x.n_inputs; ++k) fn(t_fwd[x.inputs[k]]);
    } else {
      const OperatorNode& m = f.nodes[x.mirror];
      if (m.consumer >= 0) fn(t_bwd[nf + m.consumer]);
      if (bwd_reads_inputs(m.op.kind, cfg_.backbone))
        for (int k = 0; k < m.n_inputs; ++k) fn(t_fwd[m.inputs[k]]);
      if (m.consumer < 0) fn(t_fwd[x.mirror]);
    }
  };

  // Invocation dependencies (DESIGN.md §3.2 "concurrent pools"): an invocation
  // waits for the writers of the tensors it reads (RAW), and — when its
  // output reuses a slab — for the writer and every reader of the slab's
  // previous tenant (WAW / WAR); invocations sharing a side buffer (the MLP
  // scratch and dense-gradient accumulators of the intersect MLPs, of the BetaE
  // projection MLPs; the scoring partials) form chains.
  std::vector<int32_t> writer, rhead, dep_scratch;  // per tensor: writer, first reader entry
  std::vector<std::pair<int32_t, int32_t>> rlist;   // reader entries (invocation, next)
  rlist.reserve(4 * static_cast<size_t>(n));
  int32_t chain_last[3] = {-1, -1, -1};
  inv_dep_off_.assign(1, 0);
  inv_deps_.clear();
  auto chain_of = [&](OpKind k) {
    if (k == OpKind::Intersect) return 0;
    if (k == OpKind::Score || k == OpKind::UnionScore || k == OpKind::Loss) return 1;
    // BetaE projections: their own GEMM scratch and dense gradients (prj_*)
    if (k == OpKind::Project && cfg_.backbone == Backbone::BETAE) return 2;
    return -1;
  };
  auto track = [&](const int32_t* nodes, int32_t count, OpKind kind) {
    const int32_t inv = static_cast<int32_t>(inv_dep_off_.size()) - 1;
    if (static_cast<int32_t>(writer.size()) < arena.size()) {
      writer.resize(arena.size() + 1024, -1);
      rhead.resize(arena.size() + 1024, -1);
    }
    dep_scratch.clear();
    auto add = [&](int32_t d) {
      if (d >= 0 && d != inv) dep_scratch.push_back(d);
    };
    for (int32_t i = 0; i < count; ++i) {
      const int32_t o = nodes[i];
      for_each_input(o, [&](int32_t t) {
        if (t < 0) return;
        add(writer[t]);
        rlist.emplace_back(inv, rhead[t]);
        rhead[t] = static_cast<int32_t>(rlist.size()) - 1;
      });
      const int32_t t_out = f.nodes[o].op.dir == Direction::Fwd ? t_fwd[o] : t_bwd[o];
      if (t_out >= 0) {
        writer[t_out] = inv;
        const int32_t p = arena.prev_tenant(t_out);
        if (p >= 0) {
          add(writer[p]);
          for (int32_t r = rhead[p]; r >= 0; r = rlist[r].second) add(rlist[r].first);
        }
      }
    }
    const int c = chain_of(kind);
    if (c >= 0) {
      add(chain_last[c]);
      chain_last[c] = inv;
    }
    std::sort(dep_scratch.begin(), dep_scratch.end());
    dep_scratch.erase(std::unique(dep_scratch.begin(), dep_scratch.end()), dep_scratch.end());
    inv_deps_.insert(inv_deps_.end(), dep_scratch.begin(), dep_scratch.end());
    inv_dep_off_.push_back(static_cast<int32_t>(inv_deps_.size()));
  };

  while (!ready.empty() || executed < n) {
    for (int32_t v : ready) {
      if (ql && group_of(v) != group) deferred.push_back(v);
      else pools[f.nodes[v].op.pool()].q.emplace_back(v, cycle);
    }
    ready.clear();
    std::array<int64_t, kPoolCount> counts{}, heads{};
    int64_t queued = 0;
    for (int p = 0; p < kPoolCount; ++p) {
      counts[p] = pools[p].size();
      heads[p] = counts[p] > 0 ? pools[p].q[pools[p].head].second : 0;
      queued += counts[p];
    }
    if (ql && queued == 0) {
      // the current group is done: the next pattern present, its ready nodes in id order
      if (deferred.empty()) throw MissingKernel("query-level planner: no ready node");
      group = kPatternCount;
      for (int32_t v : deferred) group = std::min(group, group_of(v));
      std::vector<int32_t> keep;
      for (int32_t v : deferred) (group_of(v) == group ? ready : keep).push_back(v);
      deferred.swap(keep);
      std::sort(ready.begin(), ready.end());
      continue;
    }
    const int tau = select_pool(counts, heads);
    const OperatorType type = OperatorType::from_pool(tau);
    Pool& pool = pools[tau];
    const int64_t total = pool.size();
    const int64_t n_pops = (total + cfg_.b_max - 1) / cfg_.b_max;
    int64_t remaining = total;
    for (int64_t p = 0; p < n_pops; ++p) {
      const int64_t take = std::min<int64_t>(remaining, cfg_.b_max);
      remaining -= take;
      batch.clear();
      for (int64_t i = 0; i < take; ++i) batch.push_back(pool.q[pool.head++].first);

      TraceRecord rec;
      rec.step = step;
      rec.cycle = cycle;
      rec.type = type;
      rec.batch = static_cast<int32_t>(take);
      rec.nodes = batch;

      // use-after-free guard: every consumed tensor must still be referenced
      for (int32_t o : batch) for_each_input(o, [&](int32_t t) { arena.check_live(t); });
      for (int32_t o : batch) allocate(o);

      if (type.is_set_op()) {
        for (int k = 2; k <= 3; ++k) {
          cls.clear();
          for (int32_t o : batch)
            if (f.nodes[o].cardinality == k) cls.push_back(o);
          if (cls.empty()) continue;
          rec.classes.emplace_back(k, static_cast<int32_t>(cls.size()));
          track(cls.data(), static_cast<int32_t>(cls.size()), type.kind);
          invoke(Invocation{type, k, cls.data(), static_cast<int32_t>(cls.size()), step, cycle});
          ++tr.invocations;
        }
      } else {
        track(batch.data(), static_cast<int32_t>(batch.size()), type.kind);
        invoke(Invocation{type, 0, batch.data(), static_cast<int32_t>(batch.size()), step, cycle});
        ++tr.invocations;
      }

      for (int32_t o : batch) {
        for_each_input(o, [&](int32_t t) { rec.bytes_reclaimed += arena.release(t); });
        for (int32_t k = adj.succ_begin[o]; k < adj.succ_begin[o + 1]; ++k) {
          const int32_t s = adj.succ[k];
          if (--indeg[s] == 0) ready.push_back(s);
        }
      }
      executed += take;
      rec.live_bytes = arena.live();
      tr.records.push_back(std::move(rec));
      ++step;
    }
    ++cycle;
  }
  tr.peak_bytes = arena.peak();
  tr.free_list_hits = arena.hits();
  arena_top_ = arena.top();
  return tr;
}

std::string ExecutionTrace::to_json() const {
  std::string s = "{\"invocations\":" + std::to_string(invocations) +
                  ",\"peak_bytes\":" + std::to_string(peak_bytes) +
                  ",\"free_list_hits\":" + std::to_string(free_list_hits) +
                  ",\"total_nodes\":" + std::to_string(total_nodes) + ",\"records\":[";
  for (size_t i = 0; i < records.size(); ++i) {
    const TraceRecord& r = records[i];
    if (i) s += ',';
    s += "{\"step\":" + std::to_string(r.step) + ",\"cycle\":" + std::to_string(r.cycle) +
         ",\"kind\":\"" + op_kind_name(r.type.kind) + "\",\"dir\":\"" +
         (r.type.dir == Direction::Fwd ? "fwd" : "bwd") + "\",\"batch\":" +
         std::to_string(r.batch) + ",\"classes\":[";
    for (size_t c = 0; c < r.classes.size(); ++c) {
      if (c) s += ',';
      s += "[" + std::to_string(r.classes[c].first) + "," + std::to_string(r.classes[c].second) + "]";
    }
    s += "],\"bytes_reclaimed\":" + std::to_string(r.bytes_reclaimed) +
         ",\"live_bytes\":" + std::to_string(r.live_bytes) + "}";
  }
  s += "]}";
  return s;
}

}  // namespace ngdb
