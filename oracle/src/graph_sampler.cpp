// ORACLE (test infrastructure only). Graph store, answer semantics, sampler.
//   graph + answer_query: SPEC.md:17-95, kg.hpp:25-89 (set-based, literal)
//   sample_query / sample_batch: SPEC.md:200-217 + the draw order fixed in
//     DESIGN.md §2.3 (SURVEY A-5, A-11)
//   negative_sample: SPEC.md:532-540 (uniform over ℰ \ answers_full, with
//     replacement; rejection redraw)
#include <algorithm>
#include <stdexcept>

#include "oracle_internal.hpp"

namespace oracle {

OGraph OGraph::build(int ne, int nr, std::vector<OTriple> t) {
  OGraph g;
  g.ne = ne;
  g.nr = nr;
  std::set<OTriple> uniq(t.begin(), t.end());
  g.triples.assign(uniq.begin(), uniq.end());
  g.out_edges.assign(ne, {});
  g.in_edges.assign(ne, {});
  for (const auto& x : g.triples) {
    if (x.h < 0 || x.h >= ne || x.t < 0 || x.t >= ne || x.r < 0 || x.r >= nr)
      throw std::runtime_error("IdOutOfRange");
    g.fwd[{x.h, x.r}].insert(x.t);
    g.out_edges[x.h].push_back({x.r, x.t});
    g.in_edges[x.t].push_back({x.r, x.h});
  }
  for (int e = 0; e < ne; ++e) {
    std::sort(g.out_edges[e].begin(), g.out_edges[e].end());
    std::sort(g.in_edges[e].begin(), g.in_edges[e].end());
    if (!g.in_edges[e].empty()) g.has_in.push_back(e);
  }
  return g;
}

std::set<int> OGraph::nbr(int e, int r) const {
  auto it = fwd.find({e, r});
  return it == fwd.end() ? std::set<int>{} : it->second;
}

bool OGraph::has(int h, int r, int t) const {
  auto it = fwd.find({h, r});
  return it != fwd.end() && it->second.count(t) > 0;
}

int o_n_anchors(int p) {
  static const int a[NPAT] = {1, 1, 1, 2, 3, 2, 2, 2, 2, 2, 3, 2, 2, 2};
  return a[p];
}
int o_n_relations(int p) {
  static const int r[NPAT] = {1, 2, 3, 2, 3, 3, 3, 2, 3, 2, 3, 3, 3, 3};
  return r[p];
}

namespace {

using S = std::set<int>;
S img(const OGraph& g, const S& from, int r) {
  S out;
  for (int e : from) {
    S n = g.nbr(e, r);
    out.insert(n.begin(), n.end());
  }
  return out;
}
S cap(const S& a, const S& b) {
  S o;
  for (int x : a)
    if (b.count(x)) o.insert(x);
  return o;
}
S cup(S a, const S& b) {
  a.insert(b.begin(), b.end());
  return a;
}
S diff(const S& a, const S& b) {
  S o;
  for (int x : a)
    if (!b.count(x)) o.insert(x);
  return o;
}

}  // namespace

std::set<int> o_answer(const OGraph& g, const OQuery& q) {
  auto at = [&](int i, int ri) { return g.nbr(q.a[i], q.r[ri]); };
  switch (q.pattern) {
    case P1: return at(0, 0);
    case P2: return img(g, at(0, 0), q.r[1]);
    case P3: return img(g, img(g, at(0, 0), q.r[1]), q.r[2]);
    case I2: return cap(at(0, 0), at(1, 1));
    case I3: return cap(cap(at(0, 0), at(1, 1)), at(2, 2));
    case PI: return cap(img(g, at(0, 0), q.r[1]), at(1, 2));
    case IP: return img(g, cap(at(0, 0), at(1, 1)), q.r[2]);
    case U2: return cup(at(0, 0), at(1, 1));
    case UP: return img(g, cup(at(0, 0), at(1, 1)), q.r[2]);
    case IN2: return diff(at(0, 0), at(1, 1));
    case IN3: return diff(cap(at(0, 0), at(1, 1)), at(2, 2));
    case PIN: return diff(img(g, at(0, 0), q.r[1]), at(1, 2));
    case PNI: return diff(at(1, 2), img(g, at(0, 0), q.r[1]));
    case INP: return img(g, diff(at(0, 0), at(1, 1)), q.r[2]);
  }
  throw std::runtime_error("UnsupportedPattern");
}

namespace {

// One instantiation attempt; the draw order is the contract of DESIGN.md §2.3.
struct Attempt {
  const OGraph& g;
  OrRng& rng;
  bool fail = false;

  // backward hop: a uniformly chosen in-edge of x -> (relation, head)
  std::pair<int, int> back(int x) {
    if (fail) return {-1, -1};
    const auto& in = g.in_edges[x];
    if (in.empty()) {
      fail = true;
      return {-1, -1};
    }
    return in[rng.below(in.size())];
  }
  OTriple triple() { return g.triples[rng.below(g.triples.size())]; }
};

bool instantiate(const OGraph& g, OrRng& rng, int p, int t, OQuery& q) {
  q.pattern = p;
  q.a.assign(o_n_anchors(p), -1);
  q.r.assign(o_n_relations(p), -1);
  Attempt w{g, rng};
  auto set = [&](int ai, int ri, std::pair<int, int> e) {
    q.r[ri] = e.first;
    q.a[ai] = e.second;
  };
  switch (p) {
    case P1: set(0, 0, w.back(t)); return !w.fail;
    case P2: {
      auto e1 = w.back(t);
      if (w.fail) return false;
      q.r[1] = e1.first;
      set(0, 0, w.back(e1.second));
      return !w.fail;
    }
    case P3: {
      auto e2 = w.back(t);
      if (w.fail) return false;
      q.r[2] = e2.first;
      auto e1 = w.back(e2.second);
      if (w.fail) return false;
      q.r[1] = e1.first;
      set(0, 0, w.back(e1.second));
      return !w.fail;
    }
    case I2:
    case U2:
      set(0, 0, w.back(t));
      if (w.fail) return false;
      set(1, 1, w.back(t));
      return !w.fail;
    case I3:
      set(0, 0, w.back(t));
      if (w.fail) return false;
      set(1, 1, w.back(t));
      if (w.fail) return false;
      set(2, 2, w.back(t));
      return !w.fail;
    case PI: {
      auto e1 = w.back(t);
      if (w.fail) return false;
      q.r[1] = e1.first;
      set(0, 0, w.back(e1.second));
      if (w.fail) return false;
      set(1, 2, w.back(t));
      return !w.fail;
    }
    case IP:
    case UP: {
      auto e2 = w.back(t);
      if (w.fail) return false;
      q.r[2] = e2.first;
      set(0, 0, w.back(e2.second));
      if (w.fail) return false;
      set(1, 1, w.back(e2.second));
      return !w.fail;
    }
    case IN2: {
      set(0, 0, w.back(t));
      if (w.fail) return false;
      OTriple x = w.triple();
      q.a[1] = x.h;
      q.r[1] = x.r;
      break;
    }
    case IN3: {
      set(0, 0, w.back(t));
      if (w.fail) return false;
      set(1, 1, w.back(t));
      if (w.fail) return false;
      OTriple x = w.triple();
      q.a[2] = x.h;
      q.r[2] = x.r;
      break;
    }
    case PIN: {
      auto e1 = w.back(t);
      if (w.fail) return false;
      q.r[1] = e1.first;
      set(0, 0, w.back(e1.second));
      if (w.fail) return false;
      OTriple x = w.triple();
      q.a[1] = x.h;
      q.r[2] = x.r;
      break;
    }
    case PNI: {
      OTriple x = w.triple();
      q.a[0] = x.h;
      q.r[0] = x.r;
      const auto& out = g.out_edges[x.t];
      if (out.empty()) return false;
      q.r[1] = out[rng.below(out.size())].first;
      set(1, 2, w.back(t));
      if (w.fail) return false;
      break;
    }
    case INP: {
      auto e2 = w.back(t);
      if (w.fail) return false;
      q.r[2] = e2.first;
      set(0, 0, w.back(e2.second));
      if (w.fail) return false;
      OTriple x = w.triple();
      q.a[1] = x.h;
      q.r[1] = x.r;
      break;
    }
  }
  // negation patterns: accept iff the walked answer survives the negation,
  // i.e. t is an answer of q on this graph (SPEC.md:203 rejection sampling)
  return o_answer(g, q).count(t) > 0;
}

}  // namespace

OBatch o_sample_batch(const OGraph& train, const OGraph& full, const double* w, int b, int k,
                      OrRng& rng) {
  OBatch out;
  out.k = k;
  for (int i = 0; i < b; ++i) {
    // pattern ~ π: first index whose running sum exceeds u (zero weights skipped)
    const double u = rng.uniform();
    double acc = 0.0;
    int p = -1, last = -1;
    for (int j = 0; j < NPAT; ++j) {
      if (w[j] <= 0.0) continue;
      acc += w[j];
      last = j;
      if (u < acc) {
        p = j;
        break;
      }
    }
    if (p < 0) p = last;
    if (p < 0) throw std::runtime_error("ConfigError: empty distribution");
    OQuery q;
    int ans = -1;
    for (int attempt = 0; attempt < 64 && ans < 0; ++attempt) {
      const int t = train.has_in[rng.below(train.has_in.size())];
      if (instantiate(train, rng, p, t, q)) ans = t;
    }
    if (ans < 0) throw std::runtime_error("ExhaustedRetries");
    out.q.push_back(q);
    out.pos.push_back(ans);
  }
  for (int i = 0; i < b; ++i) {
    const std::set<int> answers = o_answer(full, out.q[i]);
    if ((int)answers.size() >= full.ne) throw std::runtime_error("NoNegativesAvailable");
    for (int j = 0; j < k; ++j) {
      int x;
      do {
        x = (int)rng.below((uint64_t)full.ne);
      } while (answers.count(x));
      out.neg.push_back(x);
    }
  }
  return out;
}

}  // namespace oracle
