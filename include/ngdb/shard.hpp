// ngdb/shard.hpp — host planning of the row-sharded training step (SURVEY §8(e),
// DESIGN.md §6; BASELINE.json configs[4]).
//
// Entity e lives on rank e mod G at local row e div G; relations and MLPs are
// replicated. Every rank plans its own 512-query batch exactly as on one GPU
// (bit-exact per-rank trace). Scoring is query-shipping: the score-slot query
// vectors are all-gathered, each rank scores the candidates it OWNS for every
// rank's queries and the partial dL/dq are reduce-scattered back. This module
// turns the all-gathered per-rank metadata into the owner's work lists.
#pragma once

#include <cstdint>
#include <vector>

namespace ngdb {

struct ShardSpec {
  int32_t world = 1, rank = 0;
  int32_t batch = 0;        // queries per rank (B)
  int32_t max_anchors = 0;  // A_max over ranks (anchor slot padding)
  int32_t max_slots = 0;    // S_max over ranks (score slot padding)
  int32_t n_candidates = 0; // 1 + K
};

struct ShardPlanHost {
  ShardSpec spec;
  // all ranks' metadata, rank-major: anchor entity ids [G][A_max] (-1 pad);
  // scoring units [G][B] with their score slots [G][B][3] and candidates [G][B][nc]
  std::vector<int32_t> anchor_ids, unit_k, unit_slots, cand;
  // candidate positions j of unit u this rank owns: owned[unit_off[u] .. unit_off[u+1])
  std::vector<int32_t> unit_off, owned;
  // owner CSR over LOCAL entity rows (e div G), rows ascending, codes ascending:
  //   anchor of rank q, slot a:        code = -(q*A_max + a) - 1
  //   candidate j of global slot g:    code = g*nc + j,  g = q*S_max + slot
  std::vector<int32_t> rows, seg, contrib;
};

inline int32_t shard_owner(int32_t e, int32_t world) { return e % world; }
inline int32_t shard_local_row(int32_t e, int32_t world) { return e / world; }
inline int32_t shard_local_rows(int32_t n_entities, int32_t world, int32_t rank) {
  return (n_entities - rank + world - 1) / world;
}

ShardPlanHost build_shard_plan(const ShardSpec& spec, const int32_t* anchor_ids_all,
                               const int32_t* unit_k_all, const int32_t* unit_slots_all,
                               const int32_t* cand_all);

}  // namespace ngdb
