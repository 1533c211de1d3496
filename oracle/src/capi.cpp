// ORACLE (test infrastructure only). C ABI for tests / smoke / CPU baseline.
#include <cmath>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "../include/oracle.h"
#include "model_impl.hpp"
#include "oracle_internal.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

struct GraphPair {
  OGraph train, full;
};

std::vector<OTriple> trip(const int32_t* p, int64_t n) {
  std::vector<OTriple> v;
  for (int64_t i = 0; i < n; ++i) v.push_back({p[3 * i], p[3 * i + 1], p[3 * i + 2]});
  return v;
}

std::vector<OQuery> queries_of(int32_t b, const int32_t* patterns, const int32_t* anchors,
                               const int32_t* relations) {
  std::vector<OQuery> qs(b);
  for (int i = 0; i < b; ++i) {
    qs[i].pattern = patterns[i];
    for (int k = 0; k < o_n_anchors(patterns[i]); ++k) qs[i].a.push_back(anchors[3 * i + k]);
    for (int k = 0; k < o_n_relations(patterns[i]); ++k) qs[i].r.push_back(relations[4 * i + k]);
  }
  return qs;
}

struct AnyModel {
  int precision = 64;
  std::unique_ptr<Model<double>> m64;
  std::unique_ptr<Model<float>> m32;
  std::unique_ptr<Model<Dual>> mdv;  // precision 65: f64 values + fp32 deviation bounds
  template <class F>
  void visit(F&& f) {
    if (m64) f(*m64);
    else if (m32) f(*m32);
    else f(*mdv);
  }
  OTrace last;
};

template <class R>
void init_model(Model<R>& md, uint64_t seed) {
  // tensor i of the registry from Rng(seed).fork(i), row-major
  for (size_t i = 0; i < md.names.size(); ++i) {
    const std::string& n = md.names[i];
    OrRng rng = OrRng(seed).fork(i);
    auto [rows, cols] = md.shape[n];
    auto& p = md.P[n];
    const double emb = (md.gamma + 2.0) / md.d;
    const bool bias = n.find("_b") != std::string::npos;
    for (int64_t r = 0; r < rows; ++r)
      for (int64_t c = 0; c < cols; ++c) {
        double v;
        if (bias) v = 0.0;
        else if (!md.sparse[n]) {
          const double b = std::sqrt(6.0 / double(rows + cols));
          v = rng.uniform(-b, b);
        } else if (md.backbone == 1 && n == "relation" && c >= md.d) {
          v = rng.uniform(0.0, emb);
        } else {
          v = rng.uniform(-emb, emb);
        }
        p[r * cols + c] = R(float(v));
      }
  }
}

template <class R>
void get_tensor(Model<R>& md, const char* name, double* out, int64_t n) {
  std::string s(name);
  char kind = 'w';
  if (s.size() > 2 && s[1] == ':') {
    kind = s[0];
    s = s.substr(2);
  }
  if (!md.P.count(s)) throw std::runtime_error("unknown tensor " + s);
  const std::vector<R>& v = kind == 'w' ? md.P[s] : kind == 'g' ? md.G[s] : kind == 'm' ? md.M[s] : md.V[s];
  if ((int64_t)v.size() != n) throw std::runtime_error("size mismatch for " + s);
  for (int64_t i = 0; i < n; ++i) out[i] = double(v[i]);
}

// special functions: NaN (and oracle_last_error) on DomainError
template <class F>
double special(F&& f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    return std::nan("");
  }
}

}  // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

uint64_t oracle_rng_next(uint64_t seed, int64_t fork_tag, int32_t skip) {
  OrRng r(seed);
  if (fork_tag >= 0) r = r.fork((uint64_t)fork_tag);
  for (int i = 0; i < skip; ++i) r.next();
  return r.next();
}

int oracle_rng_below(uint64_t seed, const uint64_t* ns, int32_t count, int32_t reps, uint64_t* out) {
  OrRng r(seed);
  int k = 0;
  for (int i = 0; i < count; ++i)
    for (int j = 0; j < reps; ++j) out[k++] = r.below(ns[i]);
  return 0;
}

int oracle_rng_uniform(uint64_t seed, int32_t n, double lo, double hi, double* out) {
  OrRng r(seed);
  for (int i = 0; i < n; ++i) out[i] = (lo == 0.0 && hi == 1.0) ? r.uniform() : r.uniform(lo, hi);
  return 0;
}

int oracle_rng_gaussian(uint64_t seed, int32_t n, double* out) {
  OrRng r(seed);
  for (int i = 0; i < n; ++i) out[i] = r.gaussian();
  return 0;
}

uint64_t oracle_fnv1a64(const char* s, int64_t n) { return or_fnv1a64(s, (size_t)n); }

int oracle_graph_create(int32_t ne, int32_t nr, const int32_t* train, int64_t n_train,
                        const int32_t* valid, int64_t n_valid, const int32_t* test, int64_t n_test,
                        void** out) {
  return guard([&] {
    auto* g = new GraphPair();
    auto tr = trip(train, n_train);
    auto all = tr;
    auto va = trip(valid, n_valid), te = trip(test, n_test);
    all.insert(all.end(), va.begin(), va.end());
    all.insert(all.end(), te.begin(), te.end());
    g->train = OGraph::build(ne, nr, tr);
    g->full = OGraph::build(ne, nr, all);
    *out = g;
  });
}

int oracle_graph_answer(void* gp, int32_t full, int32_t pattern, const int32_t* anchors,
                        const int32_t* relations, int32_t* out, int64_t cap, int64_t* n) {
  return guard([&] {
    auto* g = static_cast<GraphPair*>(gp);
    OQuery q;
    q.pattern = pattern;
    q.a.assign(anchors, anchors + o_n_anchors(pattern));
    q.r.assign(relations, relations + o_n_relations(pattern));
    auto s = o_answer(full ? g->full : g->train, q);
    *n = (int64_t)s.size();
    int64_t i = 0;
    for (int x : s) {
      if (i >= cap) break;
      out[i++] = x;
    }
  });
}

int oracle_graph_destroy(void* g) {
  delete static_cast<GraphPair*>(g);
  return 0;
}

int oracle_sample_batch(void* gp, const double* w, int32_t b, int32_t k, uint64_t seed,
                        uint64_t tag, int32_t* patterns, int32_t* anchors, int32_t* relations,
                        int32_t* positives, int32_t* negatives) {
  return guard([&] {
    auto* g = static_cast<GraphPair*>(gp);
    OrRng rng = OrRng(seed).fork(tag);
    OBatch bt = o_sample_batch(g->train, g->full, w, b, k, rng);
    for (int i = 0; i < b; ++i) {
      patterns[i] = bt.q[i].pattern;
      for (int j = 0; j < 3; ++j) anchors[3 * i + j] = j < (int)bt.q[i].a.size() ? bt.q[i].a[j] : -1;
      for (int j = 0; j < 4; ++j)
        relations[4 * i + j] = j < (int)bt.q[i].r.size() ? bt.q[i].r[j] : -1;
      positives[i] = bt.pos[i];
    }
    std::memcpy(negatives, bt.neg.data(), bt.neg.size() * sizeof(int32_t));
  });
}

int oracle_build_dag(int32_t b, const int32_t* patterns, const int32_t* anchors,
                     const int32_t* relations, int32_t* out, int64_t cap, int32_t* n, int32_t* nf,
                     int32_t* edges, int64_t edge_cap, int32_t* n_edges) {
  return guard([&] {
    ODag d = o_build_training_dag(queries_of(b, patterns, anchors, relations));
    *n = (int32_t)d.nodes.size();
    *nf = d.nf;
    *n_edges = (int32_t)d.edges.size();
    for (int64_t i = 0; i < (int64_t)d.nodes.size() && (i + 1) * 11 <= cap; ++i) {
      const ONode& x = d.nodes[i];
      int32_t* r = out + i * 11;
      r[0] = x.kind;
      r[1] = x.bwd;
      r[2] = (int32_t)x.in.size();
      for (int k = 0; k < 3; ++k) r[3 + k] = k < (int)x.in.size() ? x.in[k] : -1;
      r[6] = x.payload;
      r[7] = x.query;
      r[8] = x.mirror;
      r[9] = x.consumer;
      r[10] = x.slot;
    }
    for (int64_t i = 0; i < (int64_t)d.edges.size() && 2 * i + 1 < edge_cap; ++i) {
      edges[2 * i] = d.edges[i].first;
      edges[2 * i + 1] = d.edges[i].second;
    }
  });
}

int oracle_model_create(int32_t backbone, int32_t ne, int32_t nr, int32_t dim, int32_t k,
                        double gamma, double alpha, double lr, int32_t precision, void** out) {
  return guard([&] {
    if (backbone < 0 || backbone > 2) throw std::runtime_error("backbone not restated");
    auto* a = new AnyModel();
    a->precision = precision;
    auto setup = [&](auto& md) {
      md.gamma = gamma;
      md.alpha = alpha;
      md.lr = lr;
      md.setup(backbone, ne, nr, dim, k);
    };
    if (precision == 64) {
      a->m64 = std::make_unique<Model<double>>();
      setup(*a->m64);
    } else if (precision == 65) {
      a->mdv = std::make_unique<Model<Dual>>();
      setup(*a->mdv);
    } else {
      a->m32 = std::make_unique<Model<float>>();
      setup(*a->m32);
    }
    *out = a;
  });
}

int oracle_model_set_semantic(void* mp, int32_t dl, const float* store, int64_t n) {
  return guard([&] {
    auto* a = static_cast<AnyModel*>(mp);
    auto set = [&](auto& md) {
      if (md.dl) throw std::runtime_error("semantic store already set");
      if (n != (int64_t)md.ne * dl) throw std::runtime_error("semantic store size");
      md.setup_semantic(dl, store);
    };
    a->visit([&](auto& md) { set(md); });
  });
}

int oracle_model_init(void* mp, uint64_t seed) {
  return guard([&] {
    auto* a = static_cast<AnyModel*>(mp);
    a->visit([&](auto& md) { init_model(md, seed); });
  });
}

int oracle_model_set(void* mp, const char* name, const float* data, int64_t n) {
  return guard([&] {
    auto* a = static_cast<AnyModel*>(mp);
    auto set = [&](auto& md) {
      using R = typename std::remove_reference_t<decltype(md.P[name])>::value_type;
      std::string s(name);
      char kind = 'w';
      if (s.size() > 2 && s[1] == ':') {  // "m:" / "v:" set the Adam moments
        kind = s[0];
        s = s.substr(2);
      }
      auto& v = (kind == 'm' ? md.M : kind == 'v' ? md.V : md.P).at(s);
      if ((int64_t)v.size() != n) throw std::runtime_error("size mismatch");
      for (int64_t i = 0; i < n; ++i) v[i] = R(data[i]);
    };
    a->visit([&](auto& md) { set(md); });
  });
}

int oracle_model_get(void* mp, const char* name, double* out, int64_t n) {
  return guard([&] {
    auto* a = static_cast<AnyModel*>(mp);
    a->visit([&](auto& md) { get_tensor(md, name, out, n); });
  });
}

int oracle_model_step(void* mp, int32_t b, const int32_t* patterns, const int32_t* anchors,
                      const int32_t* relations, const int32_t* positives, const int32_t* negatives,
                      int32_t b_max, int64_t step, int32_t executor, int32_t adam, int32_t eager,
                      double* losses) {
  return guard([&] {
    auto* a = static_cast<AnyModel*>(mp);
    ODag d = o_build_training_dag(queries_of(b, patterns, anchors, relations));
    int dl = 0;
    a->visit([&](auto& md) { dl = md.dl; });
    if (dl)  // FuseSemantic replaces EmbedAnchor
      for (auto& nd : d.nodes)
        if (nd.kind == K_EMB) nd.kind = K_FUSE;
    auto run = [&](auto& md) {
      std::vector<int> cand((size_t)b * (md.k + 1));
      for (int i = 0; i < b; ++i) {
        cand[(size_t)i * (md.k + 1)] = positives[i];
        for (int j = 0; j < md.k; ++j) cand[(size_t)i * (md.k + 1) + 1 + j] = negatives[(size_t)i * md.k + j];
      }
      a->last = o_train_step(md, d, cand, b_max, eager != 0, executor == 1, step, adam == 0,
                             adam >= 0, true);
      for (int i = 0; i < b; ++i) losses[i] = double(md.losses[i]);
    };
    a->visit([&](auto& md) { run(md); });
  });
}

// SURVEY §8(e) parity mode of the row-sharded step: each of n sub-batches (one
// per rank) is scheduled independently, their gradients summed, then ONE Adam.
int oracle_model_step_multi(void* mp, int32_t n, const int32_t* sizes, const int32_t* patterns,
                            const int32_t* anchors, const int32_t* relations,
                            const int32_t* positives, const int32_t* negatives, int32_t b_max,
                            int64_t step, int32_t adam, double* losses) {
  return guard([&] {
    auto* a = static_cast<AnyModel*>(mp);
    auto run = [&](auto& md) {
      int64_t off = 0;
      for (int32_t t = 0; t < n; ++t) {
        const int32_t b = sizes[t];
        ODag d = o_build_training_dag(queries_of(b, patterns + off, anchors + 3 * off,
                                                 relations + 4 * off));
        if (md.dl)  // FuseSemantic replaces EmbedAnchor
          for (auto& nd : d.nodes)
            if (nd.kind == K_EMB) nd.kind = K_FUSE;
        std::vector<int> cand((size_t)b * (md.k + 1));
        for (int i = 0; i < b; ++i) {
          cand[(size_t)i * (md.k + 1)] = positives[off + i];
          for (int j = 0; j < md.k; ++j)
            cand[(size_t)i * (md.k + 1) + 1 + j] = negatives[(off + i) * md.k + j];
        }
        a->last = o_train_step(md, d, cand, b_max, true, false, step, adam == 0,
                               adam >= 0 && t == n - 1, t == 0);
        for (int i = 0; i < b; ++i) losses[off + i] = double(md.losses[i]);
        off += b;
      }
    };
    a->visit([&](auto& md) { run(md); });
  });
}

int oracle_model_margins(void* mp, double* out, int32_t n) {
  return guard([&] {
    auto* a = static_cast<AnyModel*>(mp);
    std::vector<double> m;
    a->visit([&](auto& md) { m = md.margin; });
    if ((int32_t)m.size() != n) throw std::runtime_error("margin count mismatch");
    for (int32_t i = 0; i < n; ++i) out[i] = m[i];
  });
}

int oracle_model_set_dev_tau(void* mp, double tau) {
  return guard([&] {
    auto* a = static_cast<AnyModel*>(mp);
    if (!a->mdv) throw std::runtime_error("deviation bounds need precision 65");
    a->mdv->dev_tau = tau;
  });
}

int oracle_model_dev(void* mp, const char* name, double* out, int64_t n) {
  return guard([&] {
    auto* a = static_cast<AnyModel*>(mp);
    if (!a->mdv) throw std::runtime_error("deviation bounds need precision 65");
    std::string s(name);
    char kind = 'w';
    if (s.size() > 2 && s[1] == ':') {
      kind = s[0];
      s = s.substr(2);
    }
    auto& md = *a->mdv;
    if (!md.P.count(s)) throw std::runtime_error("unknown tensor " + s);
    const auto& v = kind == 'w' ? md.P[s] : kind == 'g' ? md.G[s] : kind == 'm' ? md.M[s] : md.V[s];
    if ((int64_t)v.size() != n) throw std::runtime_error("size mismatch for " + s);
    for (int64_t i = 0; i < n; ++i) out[i] = v[i].d;
  });
}

int oracle_model_qmargins(void* mp, double* out, int32_t n) {
  return guard([&] {
    auto* a = static_cast<AnyModel*>(mp);
    std::vector<double> m;
    a->visit([&](auto& md) { m = md.qmargin; });
    if ((int32_t)m.size() != n) throw std::runtime_error("margin count mismatch");
    for (int32_t i = 0; i < n; ++i) out[i] = m[i];
  });
}

int oracle_model_trace_json(void* mp, int32_t with_nodes, char* buf, int64_t cap, int64_t* len) {
  return guard([&] {
    auto* a = static_cast<AnyModel*>(mp);
    std::string js = a->last.json(with_nodes != 0);
    *len = (int64_t)js.size();
    if (buf && cap > 0) {
      const int64_t k = std::min<int64_t>(cap - 1, *len);
      std::memcpy(buf, js.data(), k);
      buf[k] = 0;
    }
  });
}

int oracle_model_destroy(void* mp) {
  delete static_cast<AnyModel*>(mp);
  return 0;
}

double oracle_q2b_distance(const double* v, const double* c, const double* o, int32_t d,
                           double alpha) {
  Model<double> md;
  md.backbone = 1;
  md.d = d;
  md.alpha = alpha;
  std::vector<double> q(2 * d);
  for (int i = 0; i < d; ++i) {
    q[i] = c[i];
    q[d + i] = o[i];
  }
  return md.dist(q.data(), v);
}

int oracle_synth_shape(const char* name, int32_t* ne, int32_t* nr, int64_t* counts) {
  return guard([&] {
    const OShape sh = o_shape(name);
    *ne = sh.ne;
    *nr = sh.nr;
    counts[0] = sh.ntr;
    counts[1] = sh.nva;
    counts[2] = sh.nte;
  });
}

int oracle_synth_triples(const char* name, uint64_t seed, int32_t* out) {
  return guard([&] {
    const auto all = o_synth_triples(o_shape(name), seed);
    for (size_t i = 0; i < all.size(); ++i) {
      out[3 * i] = all[i].h;
      out[3 * i + 1] = all[i].r;
      out[3 * i + 2] = all[i].t;
    }
  });
}

int oracle_semantic_store(int32_t ne, int32_t dl, uint64_t seed, float* out) {
  return guard([&] {
    const auto v = o_semantic_store(ne, dl, seed);
    std::memcpy(out, v.data(), v.size() * sizeof(float));
  });
}

int oracle_set_threads(int32_t n) {
#ifdef _OPENMP
  omp_set_num_threads(n > 0 ? n : 1);
#endif
  return 0;
}

double oracle_lgamma(double x) { return special([&] { return sp_lgamma(x); }); }
double oracle_digamma(double x) { return special([&] { return sp_digamma(x); }); }
double oracle_trigamma(double x) { return special([&] { return sp_trigamma(x); }); }
double oracle_beta_kl(double a1, double b1, double a2, double b2) {
  return special([&] { return beta_kl(a1, b1, a2, b2); });
}

double oracle_loss(double gamma, double d_pos, const double* d_neg, int32_t k) {
  Model<double> md;
  md.gamma = gamma;
  md.k = k;
  std::vector<double> dists(k + 1), coef(k + 1);
  dists[0] = d_pos;
  for (int j = 0; j < k; ++j) dists[j + 1] = d_neg[j];
  return md.loss_and_coef(dists.data(), coef.data());
}

}  // extern "C"
