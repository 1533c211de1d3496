// ORACLE (test infrastructure only). Restatement of the synthetic benchmark KGs
// (shapes PAPER.md:716-720) so that the CPU reference arm of
// bench.py builds its inputs without the product library: seeded Rng, a seeded
// Fisher-Yates permutation of entity ids (hub identities), head and tail drawn
// from a power law over ranks (weight (k+1)^-0.6) with Vose's alias method,
// relation uniform, duplicates (h, r, t) rejected, then a seeded shuffle carves
// train / valid / test with the dataset's exact edge counts. Pinned against the
// product generator by tests/test_oracle_synth.py (identical triples on every
// shape), so both arms train on the same graph.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <vector>

#include "oracle_internal.hpp"

namespace oracle {

OShape o_shape(const std::string& name) {
  if (name == "fb15k-237") return {14505, 237, 272115, 17526, 20438};
  if (name == "nell995") return {63361, 200, 114213, 14324, 14267};
  if (name == "wikikg2") return {2500604, 535, 16109182, 429456, 598543};
  if (name == "tiny") return {100, 6, 600, 50, 50};
  if (name == "small") return {2000, 20, 16000, 1000, 1000};
  throw std::runtime_error("ConfigError: unknown synthetic shape " + name);
}

std::vector<OTriple> o_synth_triples(const OShape& sh, uint64_t seed) {
  const int64_t n = sh.ne, nr = sh.nr, total = sh.ntr + sh.nva + sh.nte;
  OrRng rng(seed);
  std::vector<int> ids(n);  // rank -> entity id
  for (int64_t i = 0; i < n; ++i) ids[i] = (int)i;
  for (int64_t i = n - 1; i > 0; --i) std::swap(ids[i], ids[rng.below(i + 1)]);
  // Vose alias table over ranks, probabilities scaled to mean 1
  std::vector<double> p(n);
  double z = 0;
  for (int64_t k = 0; k < n; ++k) z += (p[k] = std::pow(double(k + 1), -0.6));
  for (int64_t k = 0; k < n; ++k) p[k] = p[k] * double(n) / z;
  std::vector<int> alias(n, 0), lo, hi;
  for (int64_t k = 0; k < n; ++k) (p[k] < 1.0 ? lo : hi).push_back((int)k);
  while (!lo.empty() && !hi.empty()) {
    const int s = lo.back(), l = hi.back();
    lo.pop_back();
    alias[s] = l;
    p[l] -= 1.0 - p[s];
    if (p[l] < 1.0) {
      hi.pop_back();
      lo.push_back(l);
    }
  }
  for (int k : lo) p[k] = 1.0;
  for (int k : hi) p[k] = 1.0;
  auto entity = [&]() {
    const double u = rng.uniform() * double(n);
    int64_t k = std::min<int64_t>((int64_t)u, n - 1);
    return ids[(u - double(k)) < p[k] ? k : alias[k]];
  };
  std::unordered_set<uint64_t> seen;
  seen.reserve(2 * total);
  std::vector<OTriple> all;
  all.reserve(total);
  while ((int64_t)all.size() < total) {
    const int h = entity();
    const int r = (int)rng.below(nr);
    const int t = entity();
    if (seen.insert(((uint64_t)h * nr + r) * n + t).second) all.push_back({h, r, t});
  }
  for (int64_t i = total - 1; i > 0; --i) std::swap(all[i], all[rng.below(i + 1)]);
  return all;
}

std::vector<float> o_semantic_store(int ne, int dl, uint64_t seed) {
  // PTE rows N(0,1)/sqrt(d_l), Box-Muller from the seeded Rng
  std::vector<float> out((size_t)ne * dl);
  OrRng rng(seed);
  const double sc = 1.0 / std::sqrt(double(dl));
  for (float& v : out) v = float(rng.gaussian() * sc);
  return out;
}

}  // namespace oracle
