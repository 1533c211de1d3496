// Owner-side work lists of the row-sharded step (include/ngdb/shard.hpp).
#include "ngdb/shard.hpp"

#include <algorithm>

#include "ngdb/common.hpp"
#include "ngdb/radix.hpp"
#include "ngdb/trainer.hpp"

namespace ngdb {

ShardPlanHost build_shard_plan(const ShardSpec& spec, const int32_t* anchor_ids_all,
                               const int32_t* unit_k_all, const int32_t* unit_slots_all,
                               const int32_t* cand_all) {
  const int32_t G = spec.world, r = spec.rank, B = spec.batch, A = spec.max_anchors,
                S = spec.max_slots, nc = spec.n_candidates;
  if (G < 1 || r < 0 || r >= G || B < 1 || nc < 2 || A < 0 || S < 0)
    throw ConfigError("invalid shard spec");
  ShardPlanHost p;
  p.spec = spec;
  const int64_t U = int64_t(G) * B;
  p.anchor_ids.assign(anchor_ids_all, anchor_ids_all + int64_t(G) * A);
  p.unit_k.assign(unit_k_all, unit_k_all + U);
  p.unit_slots.assign(unit_slots_all, unit_slots_all + U * 3);
  p.cand.assign(cand_all, cand_all + U * nc);

  // lookup exchange: requester-major send list, owner-major receive list
  p.send_cnt.assign(G, 0);
  p.recv_cnt.assign(G, 0);
  int32_t a_mine = 0;
  for (int32_t a = 0; a < A; ++a)
    if (p.anchor_ids[int64_t(r) * A + a] >= 0) a_mine = a + 1;
  p.anchor_pos.assign(a_mine, -1);
  std::vector<int32_t> send_pos(int64_t(G) * A, -1);  // (q, a) -> lookup send position
  for (int32_t q = 0; q < G; ++q)
    for (int32_t a = 0; a < A; ++a) {
      const int32_t e = p.anchor_ids[int64_t(q) * A + a];
      if (e < 0 || shard_owner(e, G) != r) continue;
      send_pos[int64_t(q) * A + a] = static_cast<int32_t>(p.send_rows.size());
      p.send_rows.push_back(shard_local_row(e, G));
      ++p.send_cnt[q];
    }
  for (int32_t q = 0; q < G; ++q)
    for (int32_t a = 0; a < a_mine; ++a) {
      const int32_t e = p.anchor_ids[int64_t(r) * A + a];
      if (e < 0 || shard_owner(e, G) != q) continue;
      p.anchor_pos[a] = static_cast<int32_t>(p.recv_slot.size());
      p.recv_slot.push_back(a);
      ++p.recv_cnt[q];
    }

  std::vector<uint64_t> keys;
  keys.reserve(static_cast<size_t>(U) * nc / G * 2 + p.send_rows.size());
  auto key = [](int32_t row, int64_t code) {
    return (static_cast<uint64_t>(static_cast<uint32_t>(row)) << 32) |
           static_cast<uint32_t>(code + (1ll << 31));
  };
  for (size_t i = 0; i < p.send_rows.size(); ++i)
    keys.push_back(key(p.send_rows[i], -static_cast<int64_t>(i) - 1));
  p.unit_off.assign(U + 1, 0);
  for (int64_t u = 0; u < U; ++u) {
    const int32_t q = static_cast<int32_t>(u / B);
    const int32_t k = p.unit_k[u];
    if (k < 0 || k > 3) throw ShapeMismatch("unit with more than 3 score slots");
    const int32_t* c = &p.cand[u * nc];
    for (int32_t j = 0; j < nc && k > 0; ++j) {
      if (shard_owner(c[j], G) != r) continue;
      p.owned.push_back(j);
      for (int32_t b = 0; b < k; ++b) {
        const int32_t s = p.unit_slots[u * 3 + b];
        if (s < 0 || s >= S) throw IndexOutOfRange("score slot beyond max_slots");
        keys.push_back(key(shard_local_row(c[j], G), (int64_t(q) * S + s) * nc + j));
      }
    }
    p.unit_off[u + 1] = static_cast<int32_t>(p.owned.size());
  }
  radix_sort_u64(keys);
  p.contrib.resize(keys.size());
  for (size_t i = 0; i < keys.size(); ++i) {
    const int32_t row = static_cast<int32_t>(keys[i] >> 32);
    p.contrib[i] = static_cast<int32_t>(static_cast<int64_t>(keys[i] & 0xffffffffu) - (1ll << 31));
    if (p.rows.empty() || p.rows.back() != row) {
      p.rows.push_back(row);
      p.seg.push_back(static_cast<int32_t>(i));
    }
  }
  p.seg.push_back(static_cast<int32_t>(keys.size()));
  return p;
}

int64_t shard_meta_stride(int32_t batch_cap, int32_t n_candidates) {
  return 4 + 3 * int64_t(batch_cap) + batch_cap + 3 * int64_t(batch_cap) +
         int64_t(batch_cap) * n_candidates;
}

void pack_shard_meta(const StepPlanHost& p, int32_t batch_cap, int32_t* out, int64_t stride) {
  const int32_t nc = p.n_candidates, B = p.n_queries;
  if (stride != shard_meta_stride(batch_cap, nc)) throw ShapeMismatch("shard metadata stride");
  if (B > batch_cap || p.n_anchor_slots > 3 * batch_cap)
    throw ShapeMismatch("step exceeds the metadata record's batch capacity");
  std::fill(out, out + stride, -1);
  out[0] = p.n_anchor_slots;
  out[1] = p.n_score_slots;
  out[2] = B;
  out[3] = nc;
  int32_t* a = out + 4;
  int32_t* k = a + 3 * int64_t(batch_cap);
  int32_t* us = k + batch_cap;
  int32_t* c = us + 3 * int64_t(batch_cap);
  std::copy(p.anchor_ids.begin(), p.anchor_ids.end(), a);
  std::copy(p.unit_k.begin(), p.unit_k.end(), k);
  std::copy(p.unit_slots.begin(), p.unit_slots.end(), us);
  std::copy(p.candidates.begin(), p.candidates.end(), c);
}

ShardPlanHost build_shard_plan_packed(int32_t world, int32_t rank, const int32_t* gathered,
                                      int64_t stride, int32_t batch_cap) {
  if (world < 1 || batch_cap < 1) throw ConfigError("invalid shard spec");
  const int32_t nc = gathered[3];
  if (stride != shard_meta_stride(batch_cap, nc)) throw ShapeMismatch("shard metadata stride");
  int32_t A = 1, S = 1, B = 1;
  for (int32_t q = 0; q < world; ++q) {
    const int32_t* h = gathered + q * stride;
    if (h[3] != nc) throw ShapeMismatch("ranks disagree on n_candidates");
    if (h[0] < 0 || h[0] > 3 * batch_cap || h[2] < 0 || h[2] > batch_cap || h[1] < 0)
      throw ShapeMismatch("shard metadata record out of range");
    A = std::max(A, h[0]);
    S = std::max(S, h[1]);
    B = std::max(B, h[2]);
  }
  const int64_t U = int64_t(world) * B;
  std::vector<int32_t> anc(int64_t(world) * A, -1), uk(U, 0), us(U * 3, -1), cand(U * nc, 0);
  for (int32_t q = 0; q < world; ++q) {
    const int32_t* h = gathered + q * stride;
    const int32_t* ha = h + 4;
    const int32_t* hk = ha + 3 * int64_t(batch_cap);
    const int32_t* hs = hk + batch_cap;
    const int32_t* hc = hs + 3 * int64_t(batch_cap);
    std::copy(ha, ha + h[0], anc.begin() + int64_t(q) * A);
    std::copy(hk, hk + h[2], uk.begin() + int64_t(q) * B);
    std::copy(hs, hs + 3 * int64_t(h[2]), us.begin() + int64_t(q) * B * 3);
    std::copy(hc, hc + int64_t(h[2]) * nc, cand.begin() + int64_t(q) * B * nc);
  }
  const ShardSpec spec{world, rank, B, A, S, nc};
  return build_shard_plan(spec, anc.data(), uk.data(), us.data(), cand.data());
}

}  // namespace ngdb
