// Online query sampler and negative sampler.
//
// Draw order (bit-exact contract):
//   attempt: t = has_in[below(|has_in|)]  (the answer / positive sample)
//   branches in anchor order; a positive branch walks BACKWARD from its target,
//   last relation first: (r, h) = in_edges(x)[below(|in_edges(x)|)];
//   a negated atom draws a uniform training triple (h, r, *) = triples[below(|T|)];
//   a negated 2-hop branch (pni) then walks forward: out_edges(m)[below(|out|)].
//   An attempt fails (and restarts with a fresh t) when a walk hits an entity
//   without the needed edges, or when the negated branch covers the node it is
//   intersected at. Acceptance == "t is an answer of the instantiated query on
//   the training graph", evaluated with cheap membership checks.
//   After kMaxRetries failed attempts -> ExhaustedRetries.
#include "ngdb/sampler.hpp"

#include <limits>

#include <algorithm>
#include <cmath>

namespace ngdb {
namespace {

struct Walker {
  const KnowledgeGraph& g;
  Rng& rng;

  // one backward hop from x: writes (rel, head); false if x has no in-edges
  bool back(int32_t x, int32_t& rel, int32_t& head) {
    const auto& in = g.in_edges(x);
    if (in.empty()) return false;
    const auto& e = in[rng.below(in.size())];
    rel = e.first;
    head = e.second;
    return true;
  }
  // uniform training triple, used for a negated 1-hop atom (anchor, rel)
  void neg_atom(int32_t& anchor, int32_t& rel) {
    const Triple& t = g.triples()[rng.below(g.triples().size())];
    anchor = t.head;
    rel = t.rel;
  }
  // negated 2-hop branch anchor -r0-> m -r1-> *
  bool neg_path2(int32_t& anchor, int32_t& r0, int32_t& r1) {
    const Triple& t = g.triples()[rng.below(g.triples().size())];
    anchor = t.head;
    r0 = t.rel;
    const auto& out = g.out_edges(t.tail);
    if (out.empty()) return false;
    r1 = out[rng.below(out.size())].first;
    return true;
  }
  // t reachable by anchor -r0-> * -r1-> t ?
  bool reaches2(int32_t anchor, int32_t r0, int32_t r1, int32_t t) {
    for (int32_t m : g.neighbors(anchor, r0))
      if (g.has_triple(m, r1, t)) return true;
    return false;
  }

  // One attempt for pattern p with answer t; fills q on success.
  bool attempt(Pattern p, int32_t t, QueryInstance& q) {
    const PatternInfo& info = pattern_info(p);
    q.pattern = p;
    q.anchors.assign(info.n_anchors, -1);
    q.relations.assign(info.n_relations, -1);
    auto& a = q.anchors;
    auto& r = q.relations;
    int32_t m = -1, m2 = -1;
    switch (p) {
      case Pattern::P1: return back(t, r[0], a[0]);
      case Pattern::P2: return back(t, r[1], m) && back(m, r[0], a[0]);
      case Pattern::P3: return back(t, r[2], m2) && back(m2, r[1], m) && back(m, r[0], a[0]);
      case Pattern::I2:
      case Pattern::U2: return back(t, r[0], a[0]) && back(t, r[1], a[1]);
      case Pattern::I3:
        return back(t, r[0], a[0]) && back(t, r[1], a[1]) && back(t, r[2], a[2]);
      case Pattern::PI: return back(t, r[1], m) && back(m, r[0], a[0]) && back(t, r[2], a[1]);
      case Pattern::IP:
      case Pattern::UP: return back(t, r[2], m) && back(m, r[0], a[0]) && back(m, r[1], a[1]);
      case Pattern::IN2:
        if (!back(t, r[0], a[0])) return false;
        neg_atom(a[1], r[1]);
        return !g.has_triple(a[1], r[1], t);
      case Pattern::IN3:
        if (!back(t, r[0], a[0]) || !back(t, r[1], a[1])) return false;
        neg_atom(a[2], r[2]);
        return !g.has_triple(a[2], r[2], t);
      case Pattern::PIN:
        if (!back(t, r[1], m) || !back(m, r[0], a[0])) return false;
        neg_atom(a[1], r[2]);
        return !g.has_triple(a[1], r[2], t);
      case Pattern::PNI:
        if (!neg_path2(a[0], r[0], r[1])) return false;
        if (!back(t, r[2], a[1])) return false;
        return !reaches2(a[0], r[0], r[1], t);
      case Pattern::INP:
        if (!back(t, r[2], m) || !back(m, r[0], a[0])) return false;
        neg_atom(a[1], r[1]);
        // t stays an answer iff some m' in N(a0,r0) \ N(a1,r1) reaches t by r2
        for (int32_t mm : g.neighbors(a[0], r[0]))
          if (!g.has_triple(a[1], r[1], mm) && g.has_triple(mm, r[2], t)) return true;
        return false;
    }
    return false;
  }
};

}  // namespace

SamplingDistribution SamplingDistribution::uniform_over(const std::vector<Pattern>& patterns) {
  SamplingDistribution d;
  d.weights.fill(0.0);
  if (patterns.empty()) throw ConfigError("empty pattern mix");
  for (Pattern p : patterns) d.weights[static_cast<int>(p)] += 1.0 / patterns.size();
  return d;
}

SamplingDistribution SamplingDistribution::point_mass(Pattern p) {
  SamplingDistribution d;
  d.weights.fill(0.0);
  d.weights[static_cast<int>(p)] = 1.0;
  return d;
}

Pattern draw_pattern(const SamplingDistribution& pi, Rng& rng) {
  const double u = rng.uniform();
  double acc = 0.0;
  int last = -1;
  for (int p = 0; p < kPatternCount; ++p) {
    if (pi.weights[p] <= 0.0) continue;
    acc += pi.weights[p];
    last = p;
    if (u < acc) return static_cast<Pattern>(p);
  }
  if (last < 0) throw ConfigError("sampling distribution has no mass");
  return static_cast<Pattern>(last);
}

SampledQuery sample_query(const KnowledgeGraph& g, Pattern p, Rng& rng) {
  const auto& has_in = g.entities_with_in_edges();
  if (has_in.empty() || g.triples().empty()) throw ExhaustedRetries("graph has no edges");
  Walker w{g, rng};
  SampledQuery out;
  for (int attempt = 0; attempt < kMaxRetries; ++attempt) {
    const int32_t t = has_in[rng.below(has_in.size())];
    if (w.attempt(p, t, out.query)) {
      out.answer = t;
      return out;
    }
  }
  throw ExhaustedRetries(std::string("pattern ") + pattern_info(p).name + " after " +
                         std::to_string(kMaxRetries) + " attempts");
}

SampleBatch sample_batch(const KnowledgeGraph& g, const SamplingDistribution& pi, int b, Rng& rng) {
  if (b < 1) throw ConfigError("batch size must be >= 1");
  SampleBatch batch;
  batch.queries.reserve(b);
  for (int i = 0; i < b; ++i) {
    const Pattern p = draw_pattern(pi, rng);
    batch.queries.push_back(sample_query(g, p, rng));
  }
  return batch;
}

SamplingDistribution update_distribution(const DifficultyTracker& t, double floor) {
  SamplingDistribution all;
  all.weights.fill(1.0 / kPatternCount);
  return update_distribution(t, floor, all);
}

SamplingDistribution update_distribution(const DifficultyTracker& t, double floor,
                                         const SamplingDistribution& base) {
  std::array<bool, kPatternCount> in{};
  int n_in = 0;
  bool cold = false;
  for (int p = 0; p < kPatternCount; ++p) {
    in[p] = base.weights[p] > 0.0;
    n_in += in[p];
    cold |= in[p] && t.observations[p] == 0;
  }
  if (n_in == 0) throw ConfigError("update_distribution: empty support");
  if (n_in * floor > 1.0) throw ConfigError("update_distribution: floor * |support| > 1");
  if (cold) {
    SamplingDistribution d = base;
    d.floor = floor;
    return d;
  }
  SamplingDistribution d;
  d.floor = floor;
  double mx = -std::numeric_limits<double>::infinity();
  for (int p = 0; p < kPatternCount; ++p)
    if (in[p]) mx = std::max(mx, t.ema_loss[p]);
  double sum = 0.0;
  for (int p = 0; p < kPatternCount; ++p) {
    d.weights[p] = in[p] ? std::exp(t.temperature * (t.ema_loss[p] - mx)) : 0.0;
    sum += d.weights[p];
  }
  for (double& w : d.weights) w /= sum;
  // clip below at ε and renormalise the unclipped mass (water-filling)
  std::array<bool, kPatternCount> clipped{};
  for (;;) {
    int n_clipped = 0;
    double free_mass = 0.0;
    bool changed = false;
    for (int p = 0; p < kPatternCount; ++p) {
      if (!in[p]) continue;
      if (!clipped[p] && d.weights[p] < floor) {
        clipped[p] = true;
        changed = true;
      }
      if (clipped[p]) ++n_clipped;
      else free_mass += d.weights[p];
    }
    const double target = 1.0 - n_clipped * floor;
    for (int p = 0; p < kPatternCount; ++p)
      if (in[p]) d.weights[p] = clipped[p] ? floor : d.weights[p] * (target / free_mass);
    if (!changed) break;
  }
  return d;
}

void record_difficulty(DifficultyTracker& t, Pattern p, double loss) {
  if (!std::isfinite(loss) || loss < 0.0) throw NonFiniteLoss("loss " + std::to_string(loss));
  const int i = static_cast<int>(p);
  t.ema_loss[i] = t.decay * t.ema_loss[i] + (1.0 - t.decay) * loss;
  ++t.observations[i];
}

std::vector<int32_t> negative_sample(const KnowledgeGraph& g, const QueryInstance& q,
                                     const std::vector<int32_t>& answers, int n_neg, Rng& rng) {
  (void)q;
  const int64_t n = g.n_entities();
  if (static_cast<int64_t>(answers.size()) >= n) throw NoNegativesAvailable("answers cover all entities");
  std::vector<int32_t> out(n_neg);
  for (int i = 0; i < n_neg; ++i) {
    int32_t x;
    do {
      x = static_cast<int32_t>(rng.below(static_cast<uint64_t>(n)));
    } while (std::binary_search(answers.begin(), answers.end(), x));
    out[i] = x;
  }
  return out;
}

TrainingBatch sample_training_batch(const KnowledgeGraph& train, const KnowledgeGraph& full,
                                    const SamplingDistribution& pi, int b, int n_neg, Rng& rng) {
  SampleBatch sb = sample_batch(train, pi, b, rng);
  TrainingBatch tb;
  tb.n_neg = n_neg;
  tb.queries.reserve(b);
  tb.positives.reserve(b);
  tb.negatives.reserve(static_cast<size_t>(b) * n_neg);
  for (auto& s : sb.queries) {
    auto answers = answer_query(full, s.query);
    auto negs = negative_sample(full, s.query, answers, n_neg, rng);
    tb.negatives.insert(tb.negatives.end(), negs.begin(), negs.end());
    tb.positives.push_back(s.answer);
    tb.queries.push_back(std::move(s.query));
  }
  return tb;
}

}  // namespace ngdb
