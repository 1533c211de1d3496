// ORACLE (test infrastructure only). Literal Alg. 1 executor with a refcounted
// arena and per-node f64/f32 kernels.
//
//   executor      Alg. 1; select_pool Eq. 4 + ledger tie rules
//                 (SPEC.md:463-471, 499-500, 510); pop_cardinality_classes
//                 (SPEC.md:481-489); release Eq. 7
//   arena         alloc/release with size-class free list
//   kernels       GQE SPEC.md:359-376; Q2B SPEC.md:377-385; BetaE SPEC.md:386-403
//                 (forms of SURVEY A-7); union SPEC.md:404-412;
//                 loss SPEC.md:541-549 with psi per SPEC.md:431
//   fusion        fuse_semantic SPEC.md:413-421 (Eq. 12): sigma(W_p [h | F s] + b_p) for
//                 anchors AND candidates; the store s is frozen. BetaE
//                 additionally routes the fused vector through Psi_theta (Eq. 3,
//                 PAPER.md:165-168): a linear map d -> 2d' whose
//                 output is realised by the softplus clamp; h is then d wide
//   adam          SPEC.md:550-558 (dense) and the lazy touched-row variant (A-9)
// Every kernel runs node by node (the "looped" form); batching only changes
// which nodes run together, never the arithmetic of one node.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <deque>
#include <stdexcept>

#include "dual.hpp"
#include "oracle_internal.hpp"
#include "special.hpp"

namespace oracle {

template <class R>
struct Model {
  int backbone = 0;  // 0 GQE, 1 Q2B, 2 BetaE
  int ne = 0, nr = 0, d = 0, k = 0;
  double gamma = 12.0, alpha = 0.02, lr = 1e-4, b1 = 0.9, b2 = 0.999, eps = 1e-8;
  int wq = 0, ew = 0, rw = 0;
  std::vector<std::string> names;
  std::map<std::string, std::pair<int64_t, int64_t>> shape;
  std::map<std::string, bool> sparse;
  std::map<std::string, std::vector<R>> P, M, V, G;  // G: dense grads (all params, zero-filled)
  std::set<int> touchedE, touchedR;
  // semantic fusion: frozen store [ne][dl]; fused
  // candidate rows are cached per step (parameters are fixed within a step) and
  // their gradients accumulated, then pushed through the fusion once per entity
  int dl = 0;
  std::vector<R> sem;
  std::map<int, std::vector<R>> fcache, fgrad;
  std::vector<R> losses;
  std::vector<double> margin;   // per query: min |kink argument| seen in the forward pass
  std::vector<double> qmargin;  // per query: query-level kinks only (those that change dL/dq)
  OTrace trace;
  int trace_elem_bytes = 4;

  void setup(int bb, int ne_, int nr_, int d_, int k_) {
    backbone = bb;
    ne = ne_;
    nr = nr_;
    d = d_;
    k = k_;
    wq = bb == 0 ? d : 2 * d;
    ew = bb == 2 ? 2 * d : d;
    rw = bb == 1 ? 2 * d : d;
    auto add = [&](const std::string& n, int64_t r, int64_t c, bool sp) {
      names.push_back(n);
      shape[n] = {r, c};
      sparse[n] = sp;
      P[n].assign(r * c, R(0));
      M[n].assign(r * c, R(0));
      V[n].assign(r * c, R(0));
      G[n].assign(r * c, R(0));
    };
    add("entity", ne, ew, true);
    add("relation", nr, rw, true);
    if (bb == 0) {
      add("int_w1", d, d, false);
      add("int_w2", d, d, false);
    } else if (bb == 2) {
      // projection MLP [q (2d) | r (d)] -> 2d -> 2d; attention MLP 2d -> 2d -> d
      add("prj_w1", 2 * d, 3 * d, false);
      add("prj_b1", 1, 2 * d, false);
      add("prj_w2", 2 * d, 2 * d, false);
      add("prj_b2", 1, 2 * d, false);
      add("att_w1", 2 * d, 2 * d, false);
      add("att_b1", 1, 2 * d, false);
      add("att_w2", d, 2 * d, false);
      add("att_b2", 1, d, false);
    } else {
      for (const char* n : {"att_w1", "att_b1", "att_w2", "att_b2", "off_w1", "off_b1", "off_w2",
                            "off_b2"})
        add(n, std::string(n).find("_b") != std::string::npos ? 1 : d, d, false);
    }
  }

  void setup_semantic(int dl_, const float* store) {
    dl = dl_;
    sem.assign(store, store + (int64_t)ne * dl);
    auto add = [&](const std::string& n, int64_t r, int64_t c) {
      names.push_back(n);
      shape[n] = {r, c};
      sparse[n] = false;
      for (auto* m : {&P, &M, &V, &G}) (*m)[n].assign(r * c, R(0));
    };
    add("fus_f", d, dl);       // F: d_l -> d, no bias (SURVEY A-7)
    add("fus_wp", d, 2 * d);   // W_p: [h | F s] -> d
    add("fus_bp", 1, d);       // b_p
    if (backbone == 2) {  // Psi_theta: fused d -> pre-activation [alpha | beta] (2d')
      add("fus_psi", 2 * d, d);
      add("fus_psi_b", 1, 2 * d);
      // the structural embedding h is d wide (the entity table of the joint space)
      ew = d;
      shape["entity"] = {ne, ew};
      for (auto* m : {&P, &M, &V, &G}) (*m)["entity"].assign((int64_t)ne * ew, R(0));
    }
  }
  // width of a fused row: d, or the 2d' pre-activation Beta parameters (BetaE)
  int fuse_width() const { return backbone == 2 ? 2 * d : d; }

  // ---- distances -----------------------------------------------------------
  static R softplus(R x) { return x > 0 ? x + mlog1p(mexp(-x)) : mlog1p(mexp(x)); }
  static R sigm(R x) { return x >= 0 ? R(1) / (R(1) + mexp(-x)) : mexp(x) / (R(1) + mexp(x)); }
  static R sgn(R x) { return R((x > 0) - (x < 0)); }
  // BetaE: realised Beta parameter clamp(softplus(x), 0.05, 1e9) (SURVEY A-7)
  static R bclamp(R x) { return std::min(std::max(x, R(0.05)), R(1e9)); }
  static R realize(R x) { return bclamp(softplus(x)); }
  static R drealize(R x) {  // d realize / dx (0 where the clamp binds)
    const R sp = softplus(x);
    return (sp > R(0.05) && sp < R(1e9)) ? sigm(x) : R(0);
  }
  // ---- kink resolution (Dual: deviation bounds; f32/f64: plain selection) ----
  double dev_tau = 0.0;  // > 0 in the deviation-bound model (precision 65)
  // Exact ties (argument exactly 0: identical inputs, e.g. two branches through the
  // same relation) are not kinks an fp32 run can resolve differently — both sides
  // compute the same bits and apply the same tie rule (lowest index, relu'(0) = 0).
  bool near(double m) const { return dev_tau > 0 && m != 0.0 && std::fabs(m) < dev_tau; }
  // relu'(h) * g: g or 0; near the kink either is legitimate
  R relu_k(const R& h, const R& g) const {
    R r = h > R(0) ? g : R(0);
    if (near(val(h))) add_dev(r, std::fabs(val(g)) + dev(g) - dev(r));
    return r;
  }
  // realize'(x): sigma(x) inside the clamp, 0 where it binds
  R drealize_k(const R& x) const {
    R r = drealize(x);
    if (near(val(softplus(x)) - 0.05)) add_dev(r, std::fabs(val(sigm(x))));
    return r;
  }
  // sign(delta): +-1 (0 exactly at 0); near 0 the fp32 side may be either
  R sgn_k(const R& delta) const {
    R r = sgn(delta);
    if (near(val(delta))) add_dev(r, 2.0);
    return r;
  }
  R dist(const R* q, const R* v) const {
    R s = 0;
    if (backbone == 2) {  // sum over dims of KL(entity || query)
      std::vector<double> kl(d);  // per-dim terms in parallel, summed in dim order
#pragma omp parallel for schedule(static) if (d >= 64)
      for (int e = 0; e < d; ++e)
        kl[e] = beta_kl(val(realize(v[e])), val(realize(v[d + e])), val(q[e]), val(q[d + e]));
      for (int e = 0; e < d; ++e) s += R(kl[e]);
      return s;
    }
    if (backbone == 0) {
      for (int e = 0; e < d; ++e) s += mfabs(v[e] - q[e]);
    } else {
      for (int e = 0; e < d; ++e) {
        const R a = mfabs(v[e] - q[e]), o = q[d + e];
        s += std::max(a - o, R(0)) + R(alpha) * std::min(a, o);
      }
    }
    return s;
  }
  // gq += coef * d dist / dq ; gv += coef * d dist / dv
  void ddist(const R* q, const R* v, R coef, R* gq, R* gv) const {
    if (backbone == 2) {  // dims are independent: each writes only its own elements
#pragma omp parallel for schedule(static) if (d >= 64)
      for (int e = 0; e < d; ++e) {
        double g[4];
        beta_kl_grad(val(realize(v[e])), val(realize(v[d + e])), val(q[e]), val(q[d + e]), g);
        if (gv) {
          gv[e] += coef * R(g[0]) * drealize_k(v[e]);
          gv[d + e] += coef * R(g[1]) * drealize_k(v[d + e]);
        }
        if (gq) {
          gq[e] += coef * R(g[2]);
          gq[d + e] += coef * R(g[3]);
        }
      }
      return;
    }
    for (int e = 0; e < d; ++e) {
      const R delta = v[e] - q[e];
      const R s = sgn_k(delta);
      if (backbone == 0) {
        if (gq) gq[e] -= coef * s;
        if (gv) gv[e] += coef * s;
      } else {
        const R a = mfabs(delta), o = q[d + e];
        R io = a > o ? R(1) : R(alpha);             // outside: 1, inside: alpha
        R go = a > o ? R(alpha) - R(1) : R(0);      // d/do
        if (near(val(a) - val(o))) {
          add_dev(io, 1.0 - alpha);
          add_dev(go, 1.0 - alpha);
        }
        const R dv = io * s;
        if (gq) {
          gq[e] -= coef * dv;
          gq[d + e] += coef * go;
        }
        if (gv) gv[e] += coef * dv;
      }
    }
  }
  // loss of one query from its 1+k distances; coef = dloss/dd
  R loss_and_coef(const R* dists, R* coef) const {
    R l = softplus(dists[0] - R(gamma));
    coef[0] = sigm(dists[0] - R(gamma));
    for (int j = 1; j <= k; ++j) {
      l += softplus(R(gamma) - dists[j]) / R(k);
      coef[j] = -sigm(R(gamma) - dists[j]) / R(k);
    }
    return l;
  }
  const R* erow(int e) const { return &P.at("entity")[(int64_t)e * ew]; }
  R* gerow(int e) {
    touchedE.insert(e);
    return &G["entity"][(int64_t)e * ew];
  }
  R* grrow(int r) {
    touchedR.insert(r);
    return &G["relation"][(int64_t)r * rw];
  }

  // ---- small dense algebra: y = W x (+b), W [out][in] -----------------------
  // Row-parallel (OpenMP, SPEC.md:435 allows rowwise parallelism inside kernels):
  // every output element keeps its sequential summation order, so results are
  // bit-identical for any thread count.
  static constexpr int64_t kParMin = int64_t(1) << 16;
  void mv(const std::string& w, const std::string& b, const R* x, R* y) const {
    const auto& W = P.at(w);
    const auto [rows, cols] = shape.at(w);
    const R* bias = b.empty() ? nullptr : P.at(b).data();
#pragma omp parallel for schedule(static) if (rows * cols >= kParMin)
    for (int64_t o = 0; o < rows; ++o) {
      R s = bias ? bias[o] : R(0);
      for (int64_t i = 0; i < cols; ++i) s += W[o * cols + i] * x[i];
      y[o] = s;
    }
  }
  // gx += W^T gy ; gW += gy x^T ; gb += gy  (gx[i] accumulates over o ascending)
  void mv_bwd(const std::string& w, const std::string& b, const R* x, const R* gy, R* gx) {
    const auto& W = P.at(w);
    const auto [rows, cols] = shape.at(w);
    R* gW = G[w].data();
    R* gb = b.empty() ? nullptr : G[b].data();
    if (gb)
      for (int64_t o = 0; o < rows; ++o) gb[o] += gy[o];
#pragma omp parallel for schedule(static) if (rows * cols >= kParMin)
    for (int64_t o = 0; o < rows; ++o)
      for (int64_t i = 0; i < cols; ++i) gW[o * cols + i] += gy[o] * x[i];
    if (!gx) return;
    constexpr int64_t kBlk = 32;
#pragma omp parallel for schedule(static) if (rows * cols >= kParMin)
    for (int64_t i0 = 0; i0 < cols; i0 += kBlk) {
      const int64_t i1 = std::min(cols, i0 + kBlk);
      for (int64_t o = 0; o < rows; ++o)
        for (int64_t i = i0; i < i1; ++i) gx[i] += W[o * cols + i] * gy[o];
    }
  }

  // ---- per-node kernels ------------------------------------------------------
  void gqe_inter_fwd(const std::vector<const R*>& xs, R* out, std::vector<R>* mh = nullptr) {
    const int kk = (int)xs.size();
    std::vector<R> m(d, R(0)), h(d), a(d);
    for (int e = 0; e < d; ++e) {
      for (int l = 0; l < kk; ++l) m[e] += xs[l][e];
      m[e] /= R(kk);
    }
    mv("int_w1", "", m.data(), h.data());
    for (int e = 0; e < d; ++e) a[e] = std::max(h[e], R(0));
    if (out) mv("int_w2", "", a.data(), out);
    if (mh) {
      mh->assign(m.begin(), m.end());
      mh->insert(mh->end(), h.begin(), h.end());
    }
  }
  void gqe_inter_bwd(const std::vector<const R*>& xs, const R* gy, R* gout) {
    const int kk = (int)xs.size();
    std::vector<R> mh;
    gqe_inter_fwd(xs, nullptr, &mh);
    const R* m = mh.data();
    const R* h = mh.data() + d;
    std::vector<R> a(d), ga(d, R(0)), gm(d, R(0));
    for (int e = 0; e < d; ++e) a[e] = std::max(h[e], R(0));
    mv_bwd("int_w2", "", a.data(), gy, ga.data());
    for (int e = 0; e < d; ++e) ga[e] = relu_k(h[e], ga[e]);
    mv_bwd("int_w1", "", m, ga.data(), gm.data());
    for (int l = 0; l < kk; ++l)
      for (int e = 0; e < d; ++e) gout[(int64_t)l * d + e] = gm[e] / R(kk);
  }

  struct Q2bInter {
    std::vector<std::vector<R>> z, s, p;
    std::vector<R> lm, u;
  };
  void q2b_inter_fwd(const std::vector<const R*>& xs, R* out, Q2bInter* keep = nullptr) {
    const int kk = (int)xs.size();
    Q2bInter t;
    t.z.assign(kk, std::vector<R>(d));
    t.s.assign(kk, std::vector<R>(d));
    t.p.assign(kk, std::vector<R>(d));
    t.lm.assign(d, R(0));
    t.u.assign(d, R(0));
    std::vector<R> rz(d);
    for (int l = 0; l < kk; ++l) {
      mv("att_w1", "att_b1", xs[l], t.z[l].data());
      for (int e = 0; e < d; ++e) rz[e] = std::max(t.z[l][e], R(0));
      mv("att_w2", "att_b2", rz.data(), t.s[l].data());
      mv("off_w1", "off_b1", xs[l] + d, t.p[l].data());
      for (int e = 0; e < d; ++e) t.lm[e] += std::max(t.p[l][e], R(0)) / R(kk);
    }
    mv("off_w2", "off_b2", t.lm.data(), t.u.data());
    if (out) {
      for (int e = 0; e < d; ++e) {
        R mx = t.s[0][e];
        for (int l = 1; l < kk; ++l) mx = std::max(mx, t.s[l][e]);
        R z = 0, c = 0, mn = xs[0][d + e];
        for (int l = 0; l < kk; ++l) z += mexp(t.s[l][e] - mx);
        for (int l = 0; l < kk; ++l) {
          c += mexp(t.s[l][e] - mx) / z * xs[l][e];
          mn = std::min(mn, xs[l][d + e]);
        }
        out[e] = c;
        out[d + e] = mn * sigm(t.u[e]);
      }
    }
    if (keep) *keep = t;
  }
  void q2b_inter_bwd(const std::vector<const R*>& xs, const R* gy, R* gout) {
    const int kk = (int)xs.size();
    Q2bInter t;
    q2b_inter_fwd(xs, nullptr, &t);
    std::vector<std::vector<R>> gs(kk, std::vector<R>(d)), gp(kk, std::vector<R>(d));
    std::vector<R> gu(d);
    for (int l = 0; l < kk; ++l)
      for (int e = 0; e < 2 * d; ++e) gout[(int64_t)l * 2 * d + e] = R(0);
    for (int e = 0; e < d; ++e) {
      const R gC = gy[e], gO = gy[d + e];
      R mx = t.s[0][e];
      for (int l = 1; l < kk; ++l) mx = std::max(mx, t.s[l][e]);
      std::vector<R> w(kk);
      R z = 0;
      for (int l = 0; l < kk; ++l) z += (w[l] = mexp(t.s[l][e] - mx));
      R dot = 0;
      for (int l = 0; l < kk; ++l) {
        w[l] /= z;
        dot += w[l] * gC * xs[l][e];
      }
      int arg = 0;
      for (int l = 1; l < kk; ++l)
        if (xs[l][d + e] < xs[arg][d + e]) arg = l;
      const R mn = xs[arg][d + e];
      const R gate = sigm(t.u[e]);
      for (int l = 0; l < kk; ++l) {
        gs[l][e] = w[l] * (gC * xs[l][e] - dot);
        gout[(int64_t)l * 2 * d + e] += gC * w[l];
      }
      const R route = gO * gate;
      gout[(int64_t)arg * 2 * d + d + e] += route;
      for (int l = 0; l < kk; ++l)  // a near-tied offset may take the route instead
        if (l != arg && near(val(xs[l][d + e]) - val(mn))) {
          add_dev(gout[(int64_t)l * 2 * d + d + e], std::fabs(val(route)) + dev(route));
          add_dev(gout[(int64_t)arg * 2 * d + d + e], std::fabs(val(route)));
        }
      gu[e] = gO * mn * gate * (R(1) - gate);
    }
    std::vector<R> glm(d, R(0));
    mv_bwd("off_w2", "off_b2", t.lm.data(), gu.data(), glm.data());
    std::vector<R> tmp(d), rz(d);
    for (int l = 0; l < kk; ++l) {
      for (int e = 0; e < d; ++e) gp[l][e] = relu_k(t.p[l][e], glm[e] / R(kk));
      std::fill(tmp.begin(), tmp.end(), R(0));
      mv_bwd("off_w1", "off_b1", xs[l] + d, gp[l].data(), tmp.data());
      for (int e = 0; e < d; ++e) gout[(int64_t)l * 2 * d + d + e] += tmp[e];
      for (int e = 0; e < d; ++e) rz[e] = std::max(t.z[l][e], R(0));
      std::fill(tmp.begin(), tmp.end(), R(0));
      mv_bwd("att_w2", "att_b2", rz.data(), gs[l].data(), tmp.data());
      for (int e = 0; e < d; ++e) tmp[e] = relu_k(t.z[l][e], tmp[e]);
      std::vector<R> gc(d, R(0));
      mv_bwd("att_w1", "att_b1", xs[l], tmp.data(), gc.data());
      for (int e = 0; e < d; ++e) gout[(int64_t)l * 2 * d + e] += gc[e];
    }
  }

  // ---- BetaE (forms DESIGN.md §3.5) --------------------------
  // project: out = realize(W2 relu(W1 [q | r] + b1) + b2)
  struct BetaProj {
    std::vector<R> x, h, a, z;
  };
  void beta_proj_fwd(const R* in, const R* r, R* out, BetaProj* keep = nullptr) {
    BetaProj t;
    t.x.assign(in, in + 2 * d);
    t.x.insert(t.x.end(), r, r + d);
    t.h.resize(2 * d);
    t.a.resize(2 * d);
    t.z.resize(2 * d);
    mv("prj_w1", "prj_b1", t.x.data(), t.h.data());
    for (int e = 0; e < 2 * d; ++e) t.a[e] = std::max(t.h[e], R(0));
    mv("prj_w2", "prj_b2", t.a.data(), t.z.data());
    if (out)
      for (int e = 0; e < 2 * d; ++e) out[e] = realize(t.z[e]);
    if (keep) *keep = std::move(t);
  }
  void beta_proj_bwd(const R* in, const R* r, const R* gy, R* gin, R* gr) {
    BetaProj t;
    beta_proj_fwd(in, r, nullptr, &t);
    std::vector<R> gz(2 * d), ga(2 * d, R(0)), gx(3 * d, R(0));
    for (int e = 0; e < 2 * d; ++e) gz[e] = gy[e] * drealize_k(t.z[e]);
    mv_bwd("prj_w2", "prj_b2", t.a.data(), gz.data(), ga.data());
    for (int e = 0; e < 2 * d; ++e) ga[e] = relu_k(t.h[e], ga[e]);
    mv_bwd("prj_w1", "prj_b1", t.x.data(), ga.data(), gx.data());
    for (int e = 0; e < 2 * d; ++e) gin[e] = gx[e];
    for (int e = 0; e < d; ++e) gr[e] += gx[2 * d + e];
  }
  // intersect: w = softmax_l(A2 relu(A1 q_l + a1) + a2) per dim;
  // alpha = sum_l w_l alpha_l, beta = sum_l w_l beta_l (a convex combination of
  // clamped values, so the SPEC's re-clamp is the identity)
  struct BetaInter {
    std::vector<std::vector<R>> z, s;
  };
  void beta_inter_fwd(const std::vector<const R*>& xs, R* out, BetaInter* keep = nullptr) {
    const int kk = (int)xs.size();
    BetaInter t;
    t.z.assign(kk, std::vector<R>(2 * d));
    t.s.assign(kk, std::vector<R>(d));
    std::vector<R> rz(2 * d);
    for (int l = 0; l < kk; ++l) {
      mv("att_w1", "att_b1", xs[l], t.z[l].data());
      for (int e = 0; e < 2 * d; ++e) rz[e] = std::max(t.z[l][e], R(0));
      mv("att_w2", "att_b2", rz.data(), t.s[l].data());
    }
    if (out)
      for (int e = 0; e < d; ++e) {
        R mx = t.s[0][e];
        for (int l = 1; l < kk; ++l) mx = std::max(mx, t.s[l][e]);
        R z = 0, al = 0, be = 0;
        for (int l = 0; l < kk; ++l) z += mexp(t.s[l][e] - mx);
        for (int l = 0; l < kk; ++l) {
          const R w = mexp(t.s[l][e] - mx) / z;
          al += w * xs[l][e];
          be += w * xs[l][d + e];
        }
        out[e] = al;
        out[d + e] = be;
      }
    if (keep) *keep = t;
  }
  void beta_inter_bwd(const std::vector<const R*>& xs, const R* gy, R* gout) {
    const int kk = (int)xs.size();
    BetaInter t;
    beta_inter_fwd(xs, nullptr, &t);
    for (int64_t i = 0; i < (int64_t)kk * 2 * d; ++i) gout[i] = R(0);
    std::vector<std::vector<R>> gs(kk, std::vector<R>(d));
    for (int e = 0; e < d; ++e) {
      R mx = t.s[0][e];
      for (int l = 1; l < kk; ++l) mx = std::max(mx, t.s[l][e]);
      std::vector<R> w(kk), gw(kk);
      R z = 0, dot = 0;
      for (int l = 0; l < kk; ++l) z += (w[l] = mexp(t.s[l][e] - mx));
      const R gA = gy[e], gB = gy[d + e];
      for (int l = 0; l < kk; ++l) {
        w[l] /= z;
        gw[l] = gA * xs[l][e] + gB * xs[l][d + e];
        dot += w[l] * gw[l];
      }
      for (int l = 0; l < kk; ++l) {
        gs[l][e] = w[l] * (gw[l] - dot);
        gout[(int64_t)l * 2 * d + e] += gA * w[l];
        gout[(int64_t)l * 2 * d + d + e] += gB * w[l];
      }
    }
    std::vector<R> rz(2 * d), tmp(2 * d), gc(2 * d);
    for (int l = 0; l < kk; ++l) {
      for (int e = 0; e < 2 * d; ++e) rz[e] = std::max(t.z[l][e], R(0));
      std::fill(tmp.begin(), tmp.end(), R(0));
      mv_bwd("att_w2", "att_b2", rz.data(), gs[l].data(), tmp.data());
      for (int e = 0; e < 2 * d; ++e) tmp[e] = relu_k(t.z[l][e], tmp[e]);
      std::fill(gc.begin(), gc.end(), R(0));
      mv_bwd("att_w1", "att_b1", xs[l], tmp.data(), gc.data());
      for (int e = 0; e < 2 * d; ++e) gout[(int64_t)l * 2 * d + e] += gc[e];
    }
  }

  // ---- FuseSemantic -----------------------------------------
  void fuse_fwd(int e, R* out, std::vector<R>* xkeep = nullptr,
                std::vector<R>* ekeep = nullptr) const {
    std::vector<R> x(2 * d), z(d);
    const R* h = erow(e);
    for (int i = 0; i < d; ++i) x[i] = h[i];
    mv("fus_f", "", &sem[(int64_t)e * dl], x.data() + d);
    mv("fus_wp", "fus_bp", x.data(), z.data());
    std::vector<R> ef(d);
    for (int i = 0; i < d; ++i) ef[i] = sigm(z[i]);
    if (backbone == 2) mv("fus_psi", "fus_psi_b", ef.data(), out);  // Psi_theta
    else for (int i = 0; i < d; ++i) out[i] = ef[i];
    if (xkeep) *xkeep = std::move(x);
    if (ekeep) *ekeep = std::move(ef);
  }
  // g = dL/d(fused row): grads to h (entity row), F, W_p, b_p (and Psi_theta for
  // BetaE); never to the store
  void fuse_bwd(int e, const R* g) {
    std::vector<R> x, ef, y(fuse_width()), gz(d), gx(2 * d, R(0));
    fuse_fwd(e, y.data(), &x, &ef);
    std::vector<R> gef(d, R(0));  // dL / d sigma(z)
    if (backbone == 2) mv_bwd("fus_psi", "fus_psi_b", ef.data(), g, gef.data());
    else for (int i = 0; i < d; ++i) gef[i] = g[i];
    for (int i = 0; i < d; ++i) gz[i] = gef[i] * ef[i] * (R(1) - ef[i]);
    mv_bwd("fus_wp", "fus_bp", x.data(), gz.data(), gx.data());
    R* ge = gerow(e);
    for (int i = 0; i < d; ++i) ge[i] += gx[i];
    mv_bwd("fus_f", "", &sem[(int64_t)e * dl], gx.data() + d, nullptr);
  }
  // candidate row (fused when the store is on) and its gradient accumulator
  const R* crow(int e) {
    if (!dl) return erow(e);
    auto& v = fcache[e];
    if (v.empty()) {
      v.resize(fuse_width());
      fuse_fwd(e, v.data());
    }
    return v.data();
  }
  R* cgrow(int e) {
    if (!dl) return gerow(e);
    auto& v = fgrad[e];
    if (v.empty()) v.assign(fuse_width(), R(0));
    return v.data();
  }
  void flush_fused_grads() {
    for (auto& kv : fgrad) fuse_bwd(kv.first, kv.second.data());
    fgrad.clear();
    fcache.clear();
  }

  // ---- Adam -------------------------------------------------
  void adam(int64_t step, bool lazy) {
    const double bc1 = 1.0 - std::pow(b1, (double)step), bc2 = 1.0 - std::pow(b2, (double)step);
    auto upd = [&](const std::string& n, int64_t lo, int64_t hi) {
      auto &p = P[n], &m = M[n], &v = V[n], &g = G[n];
      for (int64_t i = lo; i < hi; ++i) {
        m[i] = R(b1) * m[i] + R(1 - b1) * g[i];
        v[i] = R(b2) * v[i] + R(1 - b2) * g[i] * g[i];
        const R mh = m[i] / R(bc1), vh = v[i] / R(bc2);
        p[i] -= R(lr) * mh / (msqrt(vh) + R(eps));
      }
    };
    for (const auto& n : names) {
      if (sparse[n] && lazy) {
        const std::set<int>& rows = n == "entity" ? touchedE : touchedR;
        const int64_t c = shape[n].second;
        for (int r : rows) upd(n, r * c, (r + 1) * c);
      } else {
        upd(n, 0, (int64_t)P[n].size());
      }
    }
  }
};

// ---------------------------------------------------------------------------
// Executor: Alg. 1 with the refcount arena (or a naive sequential order).
template <class R>
struct Exec {
  Model<R>& md;
  const ODag& g;
  const std::vector<int>& cand;  // [B][1+k]
  int b_max;
  bool eager;

  struct Buf {
    std::vector<R> v;
    int rc = 0;
    int64_t bytes = 0;
  };
  std::vector<Buf> bufs;
  std::map<int64_t, std::vector<int>> free_list;
  int64_t live = 0, peak = 0, hits = 0;
  std::vector<int> T, Gt;
  std::vector<int> release_step, last_use;
  int cur_step = 0;

  int width_fwd(int n) const {
    const int kd = g.nodes[n].kind;
    if (kd == K_SCORE || kd == K_UNION) return md.k + 1;
    if (kd == K_LOSS) return 1;
    return md.wq;
  }
  int alloc(int64_t elems, int rc) {
    if (rc < 1) throw std::runtime_error("ZeroRefcount");
    const int64_t bytes = elems * md.trace_elem_bytes;
    int h;
    auto& fl = free_list[bytes];
    if (!fl.empty()) {
      h = fl.back();
      fl.pop_back();
      ++hits;
    } else {
      h = (int)bufs.size();
      bufs.push_back({});
      release_step.push_back(-1);
      last_use.push_back(-1);
    }
    bufs[h].v.assign(elems, R(0));  // zero-initialised buffer
    bufs[h].rc = rc;
    bufs[h].bytes = bytes;
    live += bytes;
    peak = std::max(peak, live);
    release_step[h] = -1;
    return h;
  }
  int64_t release(int h) {
    Buf& b = bufs[h];
    if (b.rc <= 0) throw std::runtime_error("DoubleRelease");
    last_use[h] = cur_step;
    if (--b.rc > 0) return 0;
    release_step[h] = cur_step;
    if (!eager) return 0;
    free_list[b.bytes].push_back(h);
    live -= b.bytes;
    return b.bytes;
  }
  R* t(int h) {
    if (bufs[h].rc <= 0) throw std::runtime_error("use after reclamation");
    return bufs[h].v.data();
  }
  // Backward kernels that re-read their forward inputs (everything else uses
  // only the upstream gradient); the refcounts keep exactly those alive.
  bool reads_inputs(int kind) const {
    switch (kind) {
      case K_INTER: case K_SCORE: case K_UNION: case K_LOSS: return true;
      case K_PROJ: return md.backbone != 0;
      case K_NEG: return md.backbone == 2;
      default: return false;
    }
  }
  std::vector<int> consumed(int o) const {
    const ONode& x = g.nodes[o];
    std::vector<int> out;
    if (!x.bwd) {
      for (int i : x.in) out.push_back(T[i]);
    } else {
      const ONode& m = g.nodes[x.mirror];
      if (m.consumer >= 0) out.push_back(Gt[g.nf + m.consumer]);
      if (reads_inputs(m.kind))
        for (int i : m.in) out.push_back(T[i]);
      if (m.consumer < 0) out.push_back(T[x.mirror]);  // the Loss sink
    }
    return out;
  }
  void allocate(int o) {
    const ONode& x = g.nodes[o];
    if (!x.bwd) {
      int rc = 1;
      if (x.consumer >= 0 && reads_inputs(g.nodes[x.consumer].kind)) ++rc;
      T[o] = alloc(width_fwd(o), rc);
    } else {
      const ONode& m = g.nodes[x.mirror];
      if (m.in.empty()) return;
      Gt[o] = alloc((int64_t)m.in.size() * width_fwd(m.in[0]), (int)m.in.size());
    }
  }
  bool union_loss(const ONode& x) const { return g.nodes[x.in[0]].kind == K_UNION; }
  const int* cands(int q) const { return &cand[(size_t)q * (md.k + 1)]; }

  // Kink margins (parity certification, tests/parity.py): the distance to the
  // nearest non-differentiable point the query's forward pass touched.
  // kink(): query-level (changes dL/dq); ekink(): gates only an entity element
  template <class X>
  void kink(int q, const X& x) {
    const double v = val(x);
    md.margin[q] = std::min(md.margin[q], std::fabs(v));
    md.qmargin[q] = std::min(md.qmargin[q], std::fabs(v));
  }
  template <class X>
  void ekink(int q, const X& x) {
    md.margin[q] = std::min(md.margin[q], std::fabs(val(x)));
  }
  void dist_kinks(int qi, const R* q, const R* v) {
    if (md.backbone == 2) {  // KL is smooth; only the entity clamp has kinks
      for (int e = 0; e < 2 * md.d; ++e) ekink(qi, double(Model<R>::softplus(v[e])) - 0.05);
      return;
    }
    for (int e = 0; e < md.d; ++e) {
      const double delta = double(v[e]) - double(q[e]);
      kink(qi, delta);                                                       // sign(v - c)
      if (md.backbone == 1) kink(qi, std::fabs(delta) - double(q[md.d + e]));  // inside/outside
    }
  }

  void run_fwd(int o) {
    const ONode& x = g.nodes[o];
    R* out = t(T[o]);
    const int d = md.d;
    switch (x.kind) {
      case K_EMB: {
        const R* e = md.erow(x.payload);
        if (md.backbone == 2) {
          for (int i = 0; i < md.ew; ++i) {
            out[i] = Model<R>::realize(e[i]);
            ekink(x.query, double(Model<R>::softplus(e[i])) - 0.05);
          }
          break;
        }
        for (int i = 0; i < md.ew; ++i) out[i] = e[i];
        break;
      }
      case K_FUSE: {  // fused anchor row; Q2B point box (zero offset); BetaE realised
        const R* e = md.crow(x.payload);
        if (md.backbone == 2) {
          for (int i = 0; i < md.wq; ++i) {
            out[i] = Model<R>::realize(e[i]);
            ekink(x.query, double(Model<R>::softplus(e[i])) - 0.05);
          }
          break;
        }
        for (int i = 0; i < md.wq; ++i) out[i] = i < d ? e[i] : R(0);
        break;
      }
      case K_PROJ: {
        const R* in = t(T[x.in[0]]);
        const R* r = &md.P["relation"][(int64_t)x.payload * md.rw];
        if (md.backbone == 2) {
          typename Model<R>::BetaProj keep;
          md.beta_proj_fwd(in, r, out, &keep);
          for (int e = 0; e < 2 * d; ++e) {
            kink(x.query, keep.h[e]);
            kink(x.query, double(Model<R>::softplus(keep.z[e])) - 0.05);
          }
          break;
        }
        for (int i = 0; i < d; ++i) out[i] = in[i] + r[i];
        if (md.backbone == 1)
          for (int i = 0; i < d; ++i) {
            out[d + i] = std::max(in[d + i] + r[d + i], R(0));
            kink(x.query, in[d + i] + r[d + i]);
          }
        break;
      }
      case K_NEG: {
        const R* in = t(T[x.in[0]]);
        if (md.backbone == 2) {  // (alpha, beta) -> (1/alpha, 1/beta), re-clamped
          for (int i = 0; i < md.wq; ++i) {
            out[i] = Model<R>::bclamp(R(1) / in[i]);
            kink(x.query, double(R(1) / in[i]) - 0.05);
          }
          break;
        }
        for (int i = 0; i < md.wq; ++i) out[i] = i < d ? -in[i] : in[i];
        break;
      }
      case K_INTER: {
        std::vector<const R*> xs;
        for (int i : x.in) xs.push_back(t(T[i]));
        if (md.backbone == 0) {
          std::vector<R> mh;
          md.gqe_inter_fwd(xs, out, &mh);
          for (int e = 0; e < d; ++e) kink(x.query, mh[d + e]);  // relu(W1 m)
        } else if (md.backbone == 2) {
          typename Model<R>::BetaInter keep;
          md.beta_inter_fwd(xs, out, &keep);
          for (size_t l = 0; l < xs.size(); ++l)
            for (int e = 0; e < 2 * d; ++e) kink(x.query, keep.z[l][e]);
        } else {
          typename Model<R>::Q2bInter keep;
          md.q2b_inter_fwd(xs, out, &keep);
          for (size_t l = 0; l < xs.size(); ++l)
            for (int e = 0; e < d; ++e) {
              kink(x.query, keep.z[l][e]);  // relu in the attention MLP
              kink(x.query, keep.p[l][e]);  // relu in the DeepSets MLP
              for (size_t m2 = l + 1; m2 < xs.size(); ++m2)
                kink(x.query, xs[l][d + e] - xs[m2][d + e]);  // min over offsets
            }
        }
        break;
      }
      case K_SCORE: {
        const R* q = t(T[x.in[0]]);
        const int* c = cands(x.query);
        for (int j = 0; j <= md.k; ++j) {
          out[j] = md.dist(q, md.crow(c[j]));
          dist_kinks(x.query, q, md.crow(c[j]));
        }
        break;
      }
      case K_UNION: {
        for (int j = 0; j <= md.k; ++j) {
          R best = t(T[x.in[0]])[j];
          for (size_t l = 1; l < x.in.size(); ++l) best = std::min(best, t(T[x.in[l]])[j]);
          out[j] = best;
          for (size_t l = 0; l < x.in.size(); ++l)  // argmin routing
            for (size_t m2 = l + 1; m2 < x.in.size(); ++m2)
              kink(x.query, t(T[x.in[l]])[j] - t(T[x.in[m2]])[j]);
        }
        break;
      }
      case K_LOSS: {
        std::vector<R> dists(md.k + 1), coef(md.k + 1);
        if (union_loss(x)) {
          const R* in = t(T[x.in[0]]);
          for (int j = 0; j <= md.k; ++j) dists[j] = in[j];
        } else {
          const R* q = t(T[x.in[0]]);
          const int* c = cands(x.query);
          for (int j = 0; j <= md.k; ++j) {
            dists[j] = md.dist(q, md.crow(c[j]));
            dist_kinks(x.query, q, md.crow(c[j]));
          }
        }
        out[0] = md.loss_and_coef(dists.data(), coef.data());
        md.losses[x.query] = out[0];
        break;
      }
      default: throw std::runtime_error("MissingKernel");
    }
  }

  void run_bwd(int o) {
    const ONode& x = g.nodes[o];
    const ONode& m = g.nodes[x.mirror];
    const int d = md.d;
    const R* gin = m.consumer >= 0
                       ? t(Gt[g.nf + m.consumer]) + (int64_t)m.slot * width_fwd(x.mirror)
                       : nullptr;
    R* gout = Gt[o] >= 0 ? t(Gt[o]) : nullptr;
    switch (m.kind) {
      case K_EMB: {
        R* ge = md.gerow(m.payload);
        if (md.backbone == 2) {
          const R* e = md.erow(m.payload);
          for (int i = 0; i < md.ew; ++i) ge[i] += gin[i] * md.drealize_k(e[i]);
          break;
        }
        for (int i = 0; i < md.ew; ++i) ge[i] += gin[i];
        break;
      }
      case K_FUSE:
        if (md.backbone == 2) {  // through the realisation, into the fused row
          const R* e = md.crow(m.payload);
          R* gy = md.cgrow(m.payload);
          for (int i = 0; i < md.wq; ++i) gy[i] += gin[i] * md.drealize_k(e[i]);
          break;
        }
        md.fuse_bwd(m.payload, gin);
        break;
      case K_PROJ: {
        const R* r = &md.P["relation"][(int64_t)m.payload * md.rw];
        R* gr = md.grrow(m.payload);
        if (md.backbone == 2) {
          md.beta_proj_bwd(t(T[m.in[0]]), r, gin, gout, gr);
          break;
        }
        for (int i = 0; i < d; ++i) {
          gout[i] = gin[i];
          gr[i] += gin[i];
        }
        const R* in = md.backbone == 1 ? t(T[m.in[0]]) : nullptr;  // Q2B offset mask
        if (md.backbone == 1)
          for (int i = 0; i < d; ++i) {
            const R gv = md.relu_k(in[d + i] + r[d + i], gin[d + i]);
            gout[d + i] = gv;
            gr[d + i] += gv;
          }
        break;
      }
      case K_NEG:
        if (md.backbone == 2) {
          const R* in = t(T[m.in[0]]);
          for (int i = 0; i < md.wq; ++i) {
            const R inv = R(1) / in[i];
            gout[i] = (inv > R(0.05) && inv < R(1e9)) ? -gin[i] * inv * inv : R(0);
            if (md.near(val(inv) - 0.05)) add_dev(gout[i], std::fabs(val(gin[i] * inv * inv)));
          }
          break;
        }
        for (int i = 0; i < md.wq; ++i) gout[i] = i < d ? -gin[i] : gin[i];
        break;
      case K_INTER: {
        std::vector<const R*> xs;
        for (int i : m.in) xs.push_back(t(T[i]));
        if (md.backbone == 0) md.gqe_inter_bwd(xs, gin, gout);
        else if (md.backbone == 2) md.beta_inter_bwd(xs, gin, gout);
        else md.q2b_inter_bwd(xs, gin, gout);
        break;
      }
      case K_SCORE: {
        const R* q = t(T[m.in[0]]);
        const int* c = cands(m.query);
        for (int i = 0; i < md.wq; ++i) gout[i] = R(0);
        for (int j = 0; j <= md.k; ++j) md.ddist(q, md.crow(c[j]), gin[j], gout, md.cgrow(c[j]));
        break;
      }
      case K_UNION: {
        const int kk = (int)m.in.size();
        for (int j = 0; j <= md.k; ++j) {
          int arg = 0;
          for (int l = 1; l < kk; ++l)
            if (t(T[m.in[l]])[j] < t(T[m.in[arg]])[j]) arg = l;
          for (int l = 0; l < kk; ++l) gout[(int64_t)l * (md.k + 1) + j] = l == arg ? gin[j] : R(0);
          for (int l = 0; l < kk; ++l)  // near-tied branches may take the routed gradient
            if (l != arg && md.near(val(t(T[m.in[l]])[j]) - val(t(T[m.in[arg]])[j]))) {
              add_dev(gout[(int64_t)l * (md.k + 1) + j], std::fabs(val(gin[j])) + dev(gin[j]));
              add_dev(gout[(int64_t)arg * (md.k + 1) + j], std::fabs(val(gin[j])));
            }
        }
        break;
      }
      case K_LOSS: {
        std::vector<R> dists(md.k + 1), coef(md.k + 1);
        if (union_loss(m)) {
          const R* in = t(T[m.in[0]]);
          for (int j = 0; j <= md.k; ++j) dists[j] = in[j];
          md.loss_and_coef(dists.data(), coef.data());
          for (int j = 0; j <= md.k; ++j) gout[j] = coef[j];
        } else {
          const R* q = t(T[m.in[0]]);
          const int* c = cands(m.query);
          for (int j = 0; j <= md.k; ++j) dists[j] = md.dist(q, md.crow(c[j]));
          md.loss_and_coef(dists.data(), coef.data());
          for (int i = 0; i < md.wq; ++i) gout[i] = R(0);
          for (int j = 0; j <= md.k; ++j) md.ddist(q, md.crow(c[j]), coef[j], gout, md.cgrow(c[j]));
        }
        break;
      }
      default: throw std::runtime_error("MissingKernel");
    }
  }

  void exec(int o) {
    if (g.nodes[o].bwd) run_bwd(o);
    else run_fwd(o);
  }

  // sequential=true: naive topological order (fwd ids ascending, then bwd ids
  // descending), one node per step — the SPEC's sequential reference executor.
  OTrace run(bool sequential) {
    const int n = (int)g.nodes.size();
    T.assign(g.nf, -1);
    Gt.assign(n, -1);
    std::vector<std::vector<int>> succ(n);
    std::vector<int> indeg(n, 0);
    for (auto [u, v] : g.edges) {
      succ[u].push_back(v);
      ++indeg[v];
    }
    OTrace tr;
    tr.total_nodes = n;
    auto do_batch = [&](const std::vector<int>& batch, int kind, bool bwd, int cycle) {
      ORecord rec;
      rec.step = cur_step;
      rec.cycle = cycle;
      rec.kind = kind;
      rec.bwd = bwd;
      rec.batch = (int)batch.size();
      rec.nodes = batch;
      for (int o : batch)
        for (int h : consumed(o)) t(h);  // every input must still be referenced
      for (int o : batch) allocate(o);
      if (kind == K_INTER || kind == K_UNION) {
        for (int kk = 2; kk <= 3; ++kk) {
          std::vector<int> cls;
          for (int o : batch)
            if ((int)g.nodes[g.nodes[o].bwd ? g.nodes[o].mirror : o].in.size() == kk) cls.push_back(o);
          if (cls.empty()) continue;
          rec.classes.push_back({kk, (int)cls.size()});
          for (int o : cls) exec(o);
          ++tr.invocations;
        }
      } else {
        for (int o : batch) exec(o);
        ++tr.invocations;
      }
      std::vector<int> newly;
      for (int o : batch) {
        for (int h : consumed(o)) rec.reclaimed += release(h);
        for (int s : succ[o])
          if (--indeg[s] == 0) newly.push_back(s);
      }
      rec.live = live;
      tr.recs.push_back(rec);
      ++cur_step;
      return newly;
    };

    if (sequential) {
      std::vector<int> order;
      for (int i = 0; i < g.nf; ++i) order.push_back(i);
      for (int i = n - 1; i >= g.nf; --i) order.push_back(i);
      for (int o : order) do_batch({o}, g.nodes[o].kind, g.nodes[o].bwd, cur_step);
    } else {
      // pools keyed by type index = bwd*8 + kind; FIFO of (node, enqueue cycle)
      std::vector<std::deque<std::pair<int, int>>> pools(16);
      std::vector<int> ready;
      for (int i = 0; i < n; ++i)
        if (indeg[i] == 0) ready.push_back(i);
      int executed = 0, cycle = 0;
      while (executed < n) {
        for (int v : ready) pools[g.nodes[v].bwd * 8 + g.nodes[v].kind].push_back({v, cycle});
        ready.clear();
        // Eq. 4: rho = |pool| / B_max; argmax, then oldest head, then type order
        int best = -1;
        for (int p = 0; p < 16; ++p) {
          if (pools[p].empty()) continue;
          if (best < 0) {
            best = p;
            continue;
          }
          const double rp = (double)pools[p].size() / b_max, rb = (double)pools[best].size() / b_max;
          if (rp > rb || (rp == rb && pools[p].front().second < pools[best].front().second))
            best = p;
        }
        if (best < 0) throw std::runtime_error("AllPoolsEmpty");
        const int size_at_selection = (int)pools[best].size();
        const int drains = (size_at_selection + b_max - 1) / b_max;
        int left = size_at_selection;
        for (int dr = 0; dr < drains; ++dr) {
          std::vector<int> batch;
          for (int i = 0; i < std::min(left, b_max); ++i) {
            batch.push_back(pools[best].front().first);
            pools[best].pop_front();
          }
          left -= (int)batch.size();
          auto nw = do_batch(batch, best % 8, best >= 8, cycle);
          ready.insert(ready.end(), nw.begin(), nw.end());
          executed += (int)batch.size();
        }
        ++cycle;
      }
    }
    tr.peak = peak;
    tr.hits = hits;
    tr.release_step = release_step;
    tr.last_consumer_step = last_use;
    return tr;
  }
};

// ---- explicit instantiation helpers used by capi.cpp ------------------------
template <class R>
OTrace o_train_step(Model<R>& md, const ODag& g, const std::vector<int>& cand, int b_max,
                    bool eager, bool sequential, int64_t step, bool lazy, bool apply_adam,
                    bool zero_grads) {
  if (zero_grads) {
    for (auto& kv : md.G) std::fill(kv.second.begin(), kv.second.end(), R(0));
    md.touchedE.clear();
    md.touchedR.clear();
  }
  int nq = 0;
  for (const auto& n : g.nodes) nq = std::max(nq, n.query + 1);
  md.losses.assign(nq, R(0));
  md.margin.assign(nq, 1e300);
  md.qmargin.assign(nq, 1e300);
  md.fcache.clear();
  md.fgrad.clear();
  Exec<R> ex{md, g, cand, b_max, eager};
  OTrace tr = ex.run(sequential);
  md.flush_fused_grads();
  if (apply_adam) md.adam(step, lazy);
  md.trace = tr;
  return tr;
}

template struct Model<double>;
template struct Model<float>;
template struct Model<Dual>;
template OTrace o_train_step<double>(Model<double>&, const ODag&, const std::vector<int>&, int,
                                     bool, bool, int64_t, bool, bool, bool);
template OTrace o_train_step<float>(Model<float>&, const ODag&, const std::vector<int>&, int, bool,
                                    bool, int64_t, bool, bool, bool);
template OTrace o_train_step<Dual>(Model<Dual>&, const ODag&, const std::vector<int>&, int, bool,
                                   bool, int64_t, bool, bool, bool);

std::string OTrace::json(bool with_nodes) const {
  static const char* kNames[8] = {"EmbedAnchor", "FuseSemantic", "Project", "Negate",
                                  "Intersect",   "Score",        "UnionScore", "Loss"};
  std::string s = "{\"invocations\":" + std::to_string(invocations) +
                  ",\"peak_bytes\":" + std::to_string(peak) +
                  ",\"free_list_hits\":" + std::to_string(hits) +
                  ",\"total_nodes\":" + std::to_string(total_nodes) + ",\"records\":[";
  for (size_t i = 0; i < recs.size(); ++i) {
    const ORecord& r = recs[i];
    if (i) s += ",";
    s += "{\"step\":" + std::to_string(r.step) + ",\"cycle\":" + std::to_string(r.cycle) +
         ",\"kind\":\"" + kNames[r.kind] + "\",\"dir\":\"" + (r.bwd ? "bwd" : "fwd") +
         "\",\"batch\":" + std::to_string(r.batch) + ",\"classes\":[";
    for (size_t c = 0; c < r.classes.size(); ++c)
      s += (c ? "," : "") + std::string("[") + std::to_string(r.classes[c].first) + "," +
           std::to_string(r.classes[c].second) + "]";
    s += "],\"bytes_reclaimed\":" + std::to_string(r.reclaimed) +
         ",\"live_bytes\":" + std::to_string(r.live);
    if (with_nodes) {
      s += ",\"nodes\":[";
      for (size_t k = 0; k < r.nodes.size(); ++k) s += (k ? "," : "") + std::to_string(r.nodes[k]);
      s += "]";
    }
    s += "}";
  }
  s += "],\"release_step\":[";
  for (size_t i = 0; i < release_step.size(); ++i)
    s += (i ? "," : "") + std::to_string(release_step[i]);
  s += "]}";
  return s;
}

}  // namespace oracle
