// ngdb/sampler.hpp — online backward-instantiation sampler, adaptive pattern
// distribution and negative sampling.
//
// The draw sequence is part of the bit-exact contract; it is written out step by
// step in DESIGN.md §2.3.
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "ngdb/common.hpp"
#include "ngdb/kg.hpp"
#include "ngdb/query.hpp"

namespace ngdb {

constexpr int kMaxRetries = 64;

struct SamplingDistribution {
  std::array<double, kPatternCount> weights{};  // enum order
  double floor = 0.01;                          // ε

  static SamplingDistribution uniform_over(const std::vector<Pattern>& patterns);
  static SamplingDistribution point_mass(Pattern p);
};

struct DifficultyTracker {
  std::array<double, kPatternCount> ema_loss{};
  std::array<int64_t, kPatternCount> observations{};
  double decay = 0.9;
  double temperature = 1.0;  // η
};

// A sampled training query: the instance plus its walked answer (the positive).
struct SampledQuery {
  QueryInstance query;
  int32_t answer = -1;
};

struct SampleBatch {
  std::vector<SampledQuery> queries;
  int64_t step = 0;
};

// Answer-first instantiation; rejection on negated branches (≤ kMaxRetries).
SampledQuery sample_query(const KnowledgeGraph& g, Pattern p, Rng& rng);
SampleBatch sample_batch(const KnowledgeGraph& g, const SamplingDistribution& pi, int b, Rng& rng);
Pattern draw_pattern(const SamplingDistribution& pi, Rng& rng);

SamplingDistribution update_distribution(const DifficultyTracker& t, double floor = 0.01);
// The same rule restricted to a support (patterns of a configured mix): weights
// outside it stay 0, the floor applies inside it; cold start (a support pattern
// never observed) returns `base`.
SamplingDistribution update_distribution(const DifficultyTracker& t, double floor,
                                         const SamplingDistribution& base);
void record_difficulty(DifficultyTracker& t, Pattern p, double loss);  // throws NonFiniteLoss

// n_neg ids uniform over ℰ \ answers (sorted), with replacement.
std::vector<int32_t> negative_sample(const KnowledgeGraph& g, const QueryInstance& q,
                                     const std::vector<int32_t>& answers, int n_neg, Rng& rng);

// One training batch with negatives, in the exact order the oracle draws them:
// queries first (sample_batch), then per query in batch order negatives against
// answer_query(full, q). Candidate row i = [answer_i, neg_i0 .. neg_i(K-1)].
struct TrainingBatch {
  std::vector<QueryInstance> queries;
  std::vector<int32_t> positives;   // B
  std::vector<int32_t> negatives;   // B * n_neg
  int32_t n_neg = 0;
};
TrainingBatch sample_training_batch(const KnowledgeGraph& train, const KnowledgeGraph& full,
                                    const SamplingDistribution& pi, int b, int n_neg, Rng& rng);

}  // namespace ngdb
