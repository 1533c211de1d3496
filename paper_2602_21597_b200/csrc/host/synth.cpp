// Synthetic KG generator (shapes from PAPER.md:716-720).
#include "ngdb/synth.hpp"

#include <algorithm>
#include <cmath>
#include <exception>
#include <thread>

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
  // power-law over ranks, sampled in O(1) per draw with Walker's alias table
  // (one uniform: bucket = floor(u n), keep it if frac(u n) < prob[bucket])
  std::vector<double> w(n);
  double acc = 0.0;
  for (int64_t k = 0; k < n; ++k) acc += (w[k] = std::pow(static_cast<double>(k + 1), -shape.zipf_exponent));
  std::vector<double> prob(n);
  std::vector<int32_t> alias(n, 0);
  {
    std::vector<int32_t> small, large;
    for (int64_t k = 0; k < n; ++k) {
      prob[k] = w[k] * static_cast<double>(n) / acc;
      (prob[k] < 1.0 ? small : large).push_back(static_cast<int32_t>(k));
    }
    while (!small.empty() && !large.empty()) {
      const int32_t s = small.back(), l = large.back();
      small.pop_back();
      alias[s] = l;
      prob[l] -= 1.0 - prob[s];
      if (prob[l] < 1.0) {
        large.pop_back();
        small.push_back(l);
      }
    }
    for (int32_t k : small) prob[k] = 1.0;
    for (int32_t k : large) prob[k] = 1.0;
  }
  auto draw_entity = [&]() {
    const double u = rng.uniform() * static_cast<double>(n);
    int64_t k = static_cast<int64_t>(u);
    if (k >= n) k = n - 1;
    return perm[(u - static_cast<double>(k)) < prob[k] ? k : alias[k]];
  };

  // dedup by an open-addressing set of (h, r, t) keys
  size_t cap = 16;
  while (cap < 2 * static_cast<size_t>(total) + 16) cap <<= 1;
  std::vector<uint64_t> seen(cap, ~0ull);
  auto insert = [&](uint64_t key) {
    uint64_t x = key * 0x9e3779b97f4a7c15ull;
    size_t i = (x ^ (x >> 29)) & (cap - 1);
    while (seen[i] != ~0ull) {
      if (seen[i] == key) return false;
      i = (i + 1) & (cap - 1);
    }
    seen[i] = key;
    return true;
  };
  std::vector<Triple> all;
  all.reserve(total);
  while (static_cast<int64_t>(all.size()) < total) {
    const int32_t h = draw_entity();
    const int32_t rel = static_cast<int32_t>(rng.below(r));
    const int32_t t = draw_entity();
    const uint64_t key = (static_cast<uint64_t>(h) * r + rel) * n + t;
    if (insert(key)) all.push_back({h, rel, t});
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
  s.valid_edges = t.valid;
  s.test_edges = t.test;
  std::vector<Triple> all = t.train;
  all.insert(all.end(), t.valid.begin(), t.valid.end());
  all.insert(all.end(), t.test.begin(), t.test.end());
  // the two graphs are independent: build them concurrently
  std::exception_ptr err;
  std::thread full([&] {
    try {
      s.full = KnowledgeGraph::from_triples(n_entities, n_relations, std::move(all));
    } catch (...) {
      err = std::current_exception();
    }
  });
  try {
    s.train = KnowledgeGraph::from_triples(n_entities, n_relations, t.train);
  } catch (...) {
    full.join();
    throw;
  }
  full.join();
  if (err) std::rethrow_exception(err);
  return s;
}

GraphSplit make_synthetic(const SynthShape& shape, uint64_t seed) {
  return split_from_triples(shape.n_entities, shape.n_relations, synth_triples(shape, seed));
}

}  // namespace ngdb
