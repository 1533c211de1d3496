// Knowledge-graph store, loader and symbolic answer oracle.
// Follows /root/reference/proj/include/ngdb/kg.hpp:25-89 and SPEC.md:17-95.
#include "ngdb/kg.hpp"

#include <algorithm>
#include <fstream>
#include <iterator>

namespace ngdb {
namespace {

const std::vector<int32_t> kEmpty;

using Set = std::vector<int32_t>;  // sorted, unique

Set unite(const Set& a, const Set& b) {
  Set out;
  out.reserve(a.size() + b.size());
  std::set_union(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(out));
  return out;
}
Set meet(const Set& a, const Set& b) {
  Set out;
  std::set_intersection(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(out));
  return out;
}
Set minus(const Set& a, const Set& b) {
  Set out;
  std::set_difference(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(out));
  return out;
}

// Relational image of `from` under r.
Set image(const KnowledgeGraph& g, const Set& from, int32_t r) {
  if (from.size() == 1) return g.neighbors(from[0], r);
  Set out;
  for (int32_t e : from) {
    const auto& n = g.neighbors(e, r);
    out.insert(out.end(), n.begin(), n.end());
  }
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}

Set atom(const KnowledgeGraph& g, int32_t anchor, int32_t r) { return g.neighbors(anchor, r); }

void check_ids(const KnowledgeGraph& g, const QueryInstance& q) {
  q.validate();
  for (int32_t a : q.anchors)
    if (a < 0 || a >= g.n_entities()) throw IdOutOfRange("anchor " + std::to_string(a));
  for (int32_t r : q.relations)
    if (r < 0 || r >= g.n_relations()) throw IdOutOfRange("relation " + std::to_string(r));
}

// --- loader helpers -------------------------------------------------------

bool parse_int(const std::string& tok, int64_t& out) {
  if (tok.empty()) return false;
  size_t i = 0;
  bool neg = false;
  if (tok[0] == '-') {
    neg = true;
    i = 1;
    if (tok.size() == 1) return false;
  }
  int64_t v = 0;
  for (; i < tok.size(); ++i) {
    if (tok[i] < '0' || tok[i] > '9') return false;
    v = v * 10 + (tok[i] - '0');
    if (v > (int64_t(1) << 40)) return false;
  }
  out = neg ? -v : v;
  return true;
}

std::vector<std::string> split_tabs(const std::string& line) {
  std::vector<std::string> out;
  size_t start = 0;
  for (;;) {
    size_t tab = line.find('\t', start);
    out.push_back(line.substr(start, tab == std::string::npos ? std::string::npos : tab - start));
    if (tab == std::string::npos) break;
    start = tab + 1;
  }
  if (!out.empty() && !out.back().empty() && out.back().back() == '\r') out.back().pop_back();
  return out;
}

int32_t count_dict(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw MissingFile(path);
  std::string line;
  int64_t n = 0, lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty()) continue;
    auto cols = split_tabs(line);
    int64_t id;
    if (cols.size() < 2 || !parse_int(cols[0], id))
      throw MalformedLine(path + ":" + std::to_string(lineno));
    if (id != n) throw MalformedLine(path + ":" + std::to_string(lineno) + " (ids must be dense)");
    ++n;
  }
  return static_cast<int32_t>(n);
}

std::vector<Triple> read_triples(const std::string& path, int32_t n_ent, int32_t n_rel) {
  std::ifstream in(path);
  if (!in) throw MissingFile(path);
  std::vector<Triple> out;
  std::string line;
  int64_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty()) continue;
    auto cols = split_tabs(line);
    int64_t v[3];
    if (cols.size() != 3) throw MalformedLine(path + ":" + std::to_string(lineno));
    for (int k = 0; k < 3; ++k)
      if (!parse_int(cols[k], v[k])) throw MalformedLine(path + ":" + std::to_string(lineno));
    const int64_t lim[3] = {n_ent, n_rel, n_ent};
    for (int k = 0; k < 3; ++k)
      if (v[k] < 0 || v[k] >= lim[k]) throw IdOutOfRange(cols[k]);
    out.push_back({static_cast<int32_t>(v[0]), static_cast<int32_t>(v[1]),
                   static_cast<int32_t>(v[2])});
  }
  return out;
}

}  // namespace

const uint32_t* KnowledgeGraph::RelIndex::find(int32_t e, int32_t r) const {
  if (e < 0 || static_cast<size_t>(e) + 1 >= off.size()) return nullptr;
  const int32_t* b = rels.data() + off[e];
  const int32_t* en = rels.data() + off[e + 1];
  const int32_t* it = std::lower_bound(b, en, r);
  return (it != en && *it == r) ? &ids[it - rels.data()] : nullptr;
}

namespace {
// Appends the (e, r) runs of `t` (sorted by (e, r, x)) as lists of x; e = E(t),
// x = X(t). Fills the per-entity relation index and per-entity edge lists.
template <class E, class X>
void build_side(const std::vector<Triple>& t, int32_t n_entities, E ent, X other,
                std::vector<std::vector<int32_t>>& lists,
                std::vector<std::vector<std::pair<int32_t, int32_t>>>& edges,
                KnowledgeGraph::RelIndex& idx) {
  const size_t n = t.size();
  idx.off.assign(static_cast<size_t>(n_entities) + 1, 0);
  std::vector<int32_t> deg(n_entities, 0);
  for (size_t i = 0; i < n; ++i) ++deg[ent(t[i])];
  for (int32_t e = 0; e < n_entities; ++e) edges[e].reserve(deg[e]);
  for (size_t i = 0; i < n;) {
    const int32_t e = ent(t[i]), r = t[i].rel;
    size_t j = i;
    while (j < n && ent(t[j]) == e && t[j].rel == r) ++j;
    std::vector<int32_t> l;
    l.reserve(j - i);
    for (size_t k = i; k < j; ++k) {
      l.push_back(other(t[k]));
      edges[e].emplace_back(r, other(t[k]));
    }
    ++idx.off[static_cast<size_t>(e) + 1];
    idx.rels.push_back(r);
    idx.ids.push_back(static_cast<uint32_t>(lists.size()));
    lists.push_back(std::move(l));
    i = j;
  }
  for (int32_t e = 0; e < n_entities; ++e) idx.off[e + 1] += idx.off[e];
}
}  // namespace

KnowledgeGraph KnowledgeGraph::from_triples(int32_t n_entities, int32_t n_relations,
                                            std::vector<Triple> triples) {
  for (const Triple& t : triples) {
    if (t.head < 0 || t.head >= n_entities) throw IdOutOfRange("head " + std::to_string(t.head));
    if (t.tail < 0 || t.tail >= n_entities) throw IdOutOfRange("tail " + std::to_string(t.tail));
    if (t.rel < 0 || t.rel >= n_relations) throw IdOutOfRange("relation " + std::to_string(t.rel));
  }
  std::sort(triples.begin(), triples.end());
  triples.erase(std::unique(triples.begin(), triples.end()), triples.end());

  KnowledgeGraph g;
  g.n_entities_ = n_entities;
  g.n_relations_ = n_relations;
  g.out_edges_.assign(n_entities, {});
  g.in_edges_.assign(n_entities, {});
  // forward side: (h, r, t) order, lists sorted by t
  build_side(triples, n_entities, [](const Triple& t) { return t.head; },
             [](const Triple& t) { return t.tail; }, g.lists_, g.out_edges_, g.fwd_index_);
  // inverse side: (t, r, h) order, lists sorted by h
  std::vector<Triple> inv = triples;
  std::sort(inv.begin(), inv.end(), [](const Triple& x, const Triple& y) {
    if (x.tail != y.tail) return x.tail < y.tail;
    if (x.rel != y.rel) return x.rel < y.rel;
    return x.head < y.head;
  });
  build_side(inv, n_entities, [](const Triple& t) { return t.tail; },
             [](const Triple& t) { return t.head; }, g.lists_, g.in_edges_, g.inv_index_);
  for (int32_t e = 0; e < n_entities; ++e)
    if (!g.in_edges_[e].empty()) g.has_in_.push_back(e);
  g.triples_ = std::move(triples);
  return g;
}

const std::vector<int32_t>& KnowledgeGraph::neighbors(int32_t e, int32_t r) const {
  const uint32_t* v = fwd_index_.find(e, r);
  return v ? lists_[*v] : kEmpty;
}

const std::vector<int32_t>& KnowledgeGraph::inverse_neighbors(int32_t e, int32_t r) const {
  const uint32_t* v = inv_index_.find(e, r);
  return v ? lists_[*v] : kEmpty;
}

bool KnowledgeGraph::has_triple(int32_t h, int32_t r, int32_t t) const {
  const auto& n = neighbors(h, r);
  return std::binary_search(n.begin(), n.end(), t);
}

GraphSplit load_graph(const std::string& dir) {
  const int32_t n_ent = count_dict(dir + "/entities.dict");
  const int32_t n_rel = count_dict(dir + "/relations.dict");
  auto train = read_triples(dir + "/train.txt", n_ent, n_rel);
  auto valid = read_triples(dir + "/valid.txt", n_ent, n_rel);
  auto test = read_triples(dir + "/test.txt", n_ent, n_rel);
  auto dedup = [](std::vector<Triple>& v) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  };
  dedup(valid);
  dedup(test);
  std::vector<Triple> all = train;
  all.insert(all.end(), valid.begin(), valid.end());
  all.insert(all.end(), test.begin(), test.end());
  GraphSplit s;
  s.train = KnowledgeGraph::from_triples(n_ent, n_rel, std::move(train));
  s.valid_edges = std::move(valid);
  s.test_edges = std::move(test);
  s.full = KnowledgeGraph::from_triples(n_ent, n_rel, std::move(all));
  return s;
}

std::vector<int32_t> answer_query(const KnowledgeGraph& g, const QueryInstance& q) {
  check_ids(g, q);
  const auto& a = q.anchors;
  const auto& r = q.relations;
  switch (q.pattern) {
    case Pattern::P1: return atom(g, a[0], r[0]);
    case Pattern::P2: return image(g, atom(g, a[0], r[0]), r[1]);
    case Pattern::P3: return image(g, image(g, atom(g, a[0], r[0]), r[1]), r[2]);
    case Pattern::I2: return meet(atom(g, a[0], r[0]), atom(g, a[1], r[1]));
    case Pattern::I3:
      return meet(meet(atom(g, a[0], r[0]), atom(g, a[1], r[1])), atom(g, a[2], r[2]));
    case Pattern::PI: return meet(image(g, atom(g, a[0], r[0]), r[1]), atom(g, a[1], r[2]));
    case Pattern::IP: return image(g, meet(atom(g, a[0], r[0]), atom(g, a[1], r[1])), r[2]);
    case Pattern::U2: return unite(atom(g, a[0], r[0]), atom(g, a[1], r[1]));
    case Pattern::UP: return image(g, unite(atom(g, a[0], r[0]), atom(g, a[1], r[1])), r[2]);
    case Pattern::IN2: return minus(atom(g, a[0], r[0]), atom(g, a[1], r[1]));
    case Pattern::IN3:
      return minus(meet(atom(g, a[0], r[0]), atom(g, a[1], r[1])), atom(g, a[2], r[2]));
    case Pattern::PIN: return minus(image(g, atom(g, a[0], r[0]), r[1]), atom(g, a[1], r[2]));
    case Pattern::PNI: return minus(atom(g, a[1], r[2]), image(g, atom(g, a[0], r[0]), r[1]));
    case Pattern::INP: return image(g, minus(atom(g, a[0], r[0]), atom(g, a[1], r[1])), r[2]);
  }
  throw UnsupportedPattern("unknown pattern");
}

std::pair<std::vector<int32_t>, std::vector<int32_t>> predictive_answers(const GraphSplit& split,
                                                                         const QueryInstance& q) {
  auto obs = answer_query(split.train, q);
  auto all = answer_query(split.full, q);
  return {obs, minus(all, obs)};
}

}  // namespace ngdb
