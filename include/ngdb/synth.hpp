// ngdb/synth.hpp — synthetic knowledge graphs of the benchmark shapes.
//
// The reference lists src/synth.cpp (proj/CMakeLists.txt:28) but no SPEC module
// defines it; SURVEY §8(d) fixes the recipe used here: seeded Rng, relation
// uniform, head and tail from a power law over a seeded permutation of entity
// ids (hub structure), dedup, then a seeded shuffle carves train/valid/test
// with the exact edge counts of the named dataset.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ngdb/kg.hpp"

namespace ngdb {

struct SynthShape {
  std::string name;
  int32_t n_entities = 0;
  int32_t n_relations = 0;
  int64_t n_train = 0;
  int64_t n_valid = 0;
  int64_t n_test = 0;
  double zipf_exponent = 0.6;
};

// Named shapes: "fb15k-237", "nell995", "wikikg2", and small test shapes
// "tiny" (100 entities) / "small" (2000 entities).
SynthShape synth_shape(const std::string& name);

struct SynthTriples {
  std::vector<Triple> train, valid, test;
};
SynthTriples synth_triples(const SynthShape& shape, uint64_t seed);
GraphSplit make_synthetic(const SynthShape& shape, uint64_t seed);
GraphSplit split_from_triples(int32_t n_entities, int32_t n_relations, const SynthTriples& t);

}  // namespace ngdb
