// ngdb/shard.hpp — host planning of the row-sharded training step (SURVEY §8(e),
// DESIGN.md §6; BASELINE.json configs[4]).
//
// Entity e lives on rank e mod G at local row e div G; relations and MLPs are
// replicated. Every rank plans its own 512-query batch exactly as on one GPU
// (bit-exact per-rank trace). Each rank publishes its scoring metadata as ONE
// packed int32 record (shard_meta_pack); the records are all-gathered and
// turned into this rank's work lists:
//   * embedding lookups: an uneven all-to-all — owner q sends rank r exactly the
//     rows of r's anchors it owns (send_rows), r places them by recv_slot /
//     anchor_pos; the anchor-gradient return is the same exchange reversed;
//   * scoring is query-shipping: the score-slot query vectors are all-gathered,
//     each rank scores the candidates it OWNS for every rank's queries and the
//     partial dL/dq (+ partial losses) are reduce-scattered back.
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
  // lookup all-to-all (the gradient return runs it in reverse):
  //   send_cnt[r]  rows this rank sends rank r = rows of r's anchors it owns
  //   recv_cnt[q]  rows this rank receives from owner q
  //   send_rows    [sum send_cnt] local entity rows, requester-major, slot-ascending
  //   recv_slot    [sum recv_cnt] this rank's anchor slots, owner-major, slot-ascending
  //   anchor_pos   [A_mine] anchor slot -> its position in the receive order
  std::vector<int32_t> send_cnt, recv_cnt, send_rows, recv_slot, anchor_pos;
  // owner CSR over LOCAL entity rows (e div G), rows ascending, codes ascending:
  //   anchor sent at lookup position p: code = -p - 1 (its gradient row comes
  //                                     back at position p of the reverse exchange)
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

// Packed per-rank metadata record (int32, fixed stride for a batch capacity):
//   [0] n_anchor_slots  [1] n_score_slots  [2] n_queries  [3] n_candidates
//   [4 ..)              anchor ids   [3*B_cap]  (a query has at most 3 anchors)
//                       unit_k       [B_cap]
//                       unit_slots   [3*B_cap]
//                       candidates   [B_cap * nc]
int64_t shard_meta_stride(int32_t batch_cap, int32_t n_candidates);
// This rank's record of a planned (sharded) step.
struct StepPlanHost;
void pack_shard_meta(const StepPlanHost& plan, int32_t batch_cap, int32_t* out, int64_t stride);
// All-gathered records (rank-major, `stride` apart) -> this rank's plan.
ShardPlanHost build_shard_plan_packed(int32_t world, int32_t rank, const int32_t* gathered,
                                      int64_t stride, int32_t batch_cap);

}  // namespace ngdb
