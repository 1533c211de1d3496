// Synthetic KG generator (shapes from PAPER.md:716-720).
#include "ngdb/synth.hpp"

#include <algorithm>
#include <cmath>
#include <unordered_set>

namespace ngdb {

SynthShape synth_shape(const std::string& name) {
  SynthShape s;
  s.name = name;
  if (name == "fb15k-237") {
    s.n_entities = 14505; s.n_relations = 237;
    s.n_train = 272115; s.n_valid = 17526; s.n_test = 20438;
  } else if (name == "nell995") {
    s.n_entities = 63361; s.n_relations = 200;
    s.n_train = 114213; s.n_valid = 14324; s.n_test = 14267;
  } else if (name == "wikikg2") {
    s.n_entities = 2500604; s.n_relations = 535;
    s.n_train = 16109182; s.n_valid = 429456; s.n_test = 598543;
  } else if (name == "tiny") {
    s.n_entities = 100; s.n_relations = 6;
    s.n_train = 600; s.n_valid = 50; s.n_test = 50;
  } else if (name == "small") {
    s.n_entities = 2000; s.n_relations = 20;
    s.n_train = 16000; s.n_valid = 1000; s.n_test = 1000;
  } else {
    throw ConfigError("unknown synthetic shape: " + name);
  }
  return s;
}

SynthTriples synth_triples(const SynthShape& shape, uint64_t seed) {
  const int64_t n = shape.n_entities, r = shape.n_relations;
  const int64_t total = shape.n_train + shape.n_valid + shape.n_test;
  if (n < 2 || r < 1 || total > n * n * r) throw ConfigError("synthetic shape infeasible");
  Rng rng(seed);

  // rank -> entity id (seeded Fisher-Yates)
  std::vector<int32_t> perm(n);
  for (int64_t i = 0; i < n; ++i) perm[i] = static_cast<int32_t>(i);
  for (int64_t i = n - 1; i > 0; --i) std::swap(perm[i], perm[rng.below(i + 1)]);
  // power-law CDF over ranks
  std::vector<double> cdf(n);
  double acc = 0.0;
  for (int64_t k = 0; k < n; ++k) {
    acc += std::pow(static_cast<double>(k + 1), -shape.zipf_exponent);
    cdf[k] = acc;
  }
  auto draw_entity = [&]() {
    const double u = rng.uniform() * acc;
    int64_t k = std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin();
    if (k >= n) k = n - 1;
    return perm[k];
  };

  std::vector<Triple> all;
  all.reserve(total);
  std::unordered_set<uint64_t> seen;
  seen.reserve(static_cast<size_t>(total) * 2);
  while (static_cast<int64_t>(all.size()) < total) {
    const int32_t h = draw_entity();
    const int32_t rel = static_cast<int32_t>(rng.below(r));
    const int32_t t = draw_entity();
    const uint64_t key = (static_cast<uint64_t>(h) * r + rel) * n + t;
    if (seen.insert(key).second) all.push_back({h, rel, t});
  }
  for (int64_t i = total - 1; i > 0; --i) std::swap(all[i], all[rng.below(i + 1)]);

  SynthTriples out;
  out.train.assign(all.begin(), all.begin() + shape.n_train);
  out.valid.assign(all.begin() + shape.n_train, all.begin() + shape.n_train + shape.n_valid);
  out.test.assign(all.begin() + shape.n_train + shape.n_valid, all.end());
  return out;
}

GraphSplit split_from_triples(int32_t n_entities, int32_t n_relations, const SynthTriples& t) {
  GraphSplit s;
  s.train = KnowledgeGraph::from_triples(n_entities, n_relations, t.train);
  s.valid_edges = t.valid;
  s.test_edges = t.test;
  std::vector<Triple> all = t.train;
  all.insert(all.end(), t.valid.begin(), t.valid.end());
  all.insert(all.end(), t.test.begin(), t.test.end());
  s.full = KnowledgeGraph::from_triples(n_entities, n_relations, std::move(all));
  return s;
}

GraphSplit make_synthetic(const SynthShape& shape, uint64_t seed) {
  return split_from_triples(shape.n_entities, shape.n_relations, synth_triples(shape, seed));
}

}  // namespace ngdb
