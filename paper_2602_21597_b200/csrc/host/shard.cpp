// Owner-side work lists of the row-sharded step (include/ngdb/shard.hpp).
#include "ngdb/shard.hpp"

#include <algorithm>

#include "ngdb/radix.hpp"

#include "ngdb/common.hpp"

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

  std::vector<uint64_t> keys;
  keys.reserve(static_cast<size_t>(U) * nc / G * 2 + A);
  auto key = [](int32_t row, int64_t code) {
    return (static_cast<uint64_t>(static_cast<uint32_t>(row)) << 32) |
           static_cast<uint32_t>(code + (1ll << 31));
  };
  for (int32_t q = 0; q < G; ++q)
    for (int32_t a = 0; a < A; ++a) {
      const int32_t e = p.anchor_ids[int64_t(q) * A + a];
      if (e >= 0 && shard_owner(e, G) == r)
        keys.push_back(key(shard_local_row(e, G), -(int64_t(q) * A + a) - 1));
    }
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

}  // namespace ngdb
