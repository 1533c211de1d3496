// ORACLE (test infrastructure only). A literal, deliberately simple CPU
// restatement of the reference's training-step path, written independently of
// the product code in paper_2602_21597_b200/. Only tests/, __graft_entry__.smoke()
// and bench.py's CPU-baseline leg may load it.
//
// Parity status: the reference ships no implementation and no tests,
// so this restatement is pinned by (a) golden vectors from the reference's own
// executable header (tests/golden/rng_golden.json, oracle/ref/), and (b) every
// [TRIVIAL]/[DERIVED] known-answer example of /root/reference/SPEC.md on this path
// (tests/test_spec_examples.py, tests/test_golden_rng.py). Beyond those it is "parity unpinned" against a
// running reference — none exists.
#pragma once

#include <cstdint>
#include <map>
#include <set>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "rng.hpp"

namespace oracle {

// ---------------- graph (kg.hpp:25-89) ----------------------
struct OTriple {
  int h, r, t;
  bool operator<(const OTriple& o) const {
    if (h != o.h) return h < o.h;
    if (r != o.r) return r < o.r;
    return t < o.t;
  }
  bool operator==(const OTriple& o) const { return h == o.h && r == o.r && t == o.t; }
};

struct OGraph {
  int ne = 0, nr = 0;
  std::vector<OTriple> triples;                      // sorted, unique
  std::map<std::pair<int, int>, std::set<int>> fwd;  // (h, r) -> tails
  std::vector<std::vector<std::pair<int, int>>> out_edges, in_edges;  // sorted (r, other)
  std::vector<int> has_in;
  static OGraph build(int ne, int nr, std::vector<OTriple> t);
  std::set<int> nbr(int e, int r) const;
  bool has(int h, int r, int t) const;
};

// ---------------- query model (query.hpp:14-69) ------------
enum OPat { P1, P2, P3, I2, I3, PI, IP, U2, UP, IN2, IN3, PIN, PNI, INP, NPAT };
struct OQuery {
  int pattern = 0;
  std::vector<int> a, r;
};
int o_n_anchors(int p);
int o_n_relations(int p);
std::set<int> o_answer(const OGraph& g, const OQuery& q);

// ---------------- sampler -----------------------
struct OBatch {
  std::vector<OQuery> q;
  std::vector<int> pos;
  std::vector<int> neg;  // [B][k]
  int k = 0;
};
OBatch o_sample_batch(const OGraph& train, const OGraph& full, const double* w, int b, int k,
                      OrRng& rng);

// ---------------- DAG ------------------------------------
enum OKind { K_EMB = 0, K_FUSE, K_PROJ, K_NEG, K_INTER, K_SCORE, K_UNION, K_LOSS };
struct ONode {
  int kind = 0;
  bool bwd = false;
  std::vector<int> in;  // fwd: data inputs; bwd: scheduling predecessor
  int payload = -1;     // entity / relation
  int query = 0;
  int mirror = -1;
  int consumer = -1;
  int slot = 0;  // position among the consumer's inputs
};
struct ODag {
  std::vector<ONode> nodes;
  std::vector<std::pair<int, int>> edges;
  int nf = 0;
};
ODag o_build_training_dag(const std::vector<OQuery>& batch);

// ---------------- execution trace -----------------------
struct ORecord {
  int step = 0, cycle = 0, kind = 0;
  bool bwd = false;
  int batch = 0;
  std::vector<std::pair<int, int>> classes;
  int64_t reclaimed = 0, live = 0;
  std::vector<int> nodes;
};
struct OTrace {
  std::vector<ORecord> recs;
  int64_t invocations = 0, peak = 0, hits = 0, total_nodes = 0;
  std::vector<int> release_step;  // per tensor handle: step at which rc hit 0 (-1 never)
  std::vector<int> last_consumer_step;
  std::string json(bool with_nodes) const;
};

// ---------------- synthetic KGs — oracle/src/synth.cpp ----------
struct OShape {
  int ne, nr;
  int64_t ntr, nva, nte;
};
OShape o_shape(const std::string& name);
std::vector<OTriple> o_synth_triples(const OShape& sh, uint64_t seed);  // train|valid|test
std::vector<float> o_semantic_store(int ne, int dl, uint64_t seed);

}  // namespace oracle
