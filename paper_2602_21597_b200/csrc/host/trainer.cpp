// Training-step planner and single-GPU trainer (SPEC.md:568-576 train consumer
// loop; Alg. 1; Precomputed Indexing PAPER.md:265-266).
#include "ngdb/trainer.hpp"

#include <algorithm>

#include "ngdb/radix.hpp"
#include <cmath>
#include <cstdio>
#include <cstring>

namespace ngdb {

int32_t query_width(Backbone b, int32_t dim) { return b == Backbone::GQE ? dim : 2 * dim; }
int32_t entity_width(Backbone b, int32_t dim) { return b == Backbone::BETAE ? 2 * dim : dim; }
int32_t relation_width(Backbone b, int32_t dim) { return b == Backbone::Q2B ? 2 * dim : dim; }

std::vector<ParamSpec> param_specs(Backbone b, int32_t n_ent, int32_t n_rel, int32_t dim,
                                   int32_t semantic_dim) {
  const int64_t d = dim;
  std::vector<ParamSpec> s;
  // BetaE with FuseSemantic: the structural embedding h is d wide and Psi_theta
  // maps the fused vector to the 2d' Beta parameters (Eq. 3)
  const bool beta_fused = b == Backbone::BETAE && semantic_dim > 0;
  s.push_back({"entity", n_ent, beta_fused ? d : entity_width(b, dim), true});
  s.push_back({"relation", n_rel, relation_width(b, dim), true});
  if (b == Backbone::GQE) {
    s.push_back({"int_w1", d, d, false});
    s.push_back({"int_w2", d, d, false});
  } else if (b == Backbone::Q2B) {
    for (const char* n : {"att_w1", "att_b1", "att_w2", "att_b2", "off_w1", "off_b1", "off_w2",
                          "off_b2"}) {
      const bool bias = std::string(n).find("_b") != std::string::npos;
      s.push_back({n, bias ? 1 : d, d, false});
    }
  } else {
    // BetaE: projection MLP [q (2d) | r (d)] -> 2d -> 2d,
    // attention MLP 2d -> 2d -> d
    s.push_back({"prj_w1", 2 * d, 3 * d, false});
    s.push_back({"prj_b1", 1, 2 * d, false});
    s.push_back({"prj_w2", 2 * d, 2 * d, false});
    s.push_back({"prj_b2", 1, 2 * d, false});
    s.push_back({"att_w1", 2 * d, 2 * d, false});
    s.push_back({"att_b1", 1, 2 * d, false});
    s.push_back({"att_w2", d, 2 * d, false});
    s.push_back({"att_b2", 1, d, false});
  }
  if (semantic_dim > 0) {
    s.push_back({"fus_f", d, semantic_dim, false});
    s.push_back({"fus_wp", d, 2 * d, false});
    s.push_back({"fus_bp", 1, d, false});
    if (beta_fused) {
      s.push_back({"fus_psi", 2 * d, d, false});
      s.push_back({"fus_psi_b", 1, 2 * d, false});
    }
  }
  return s;
}

std::vector<float> init_param(Backbone b, int32_t n_ent, int32_t n_rel, int32_t dim,
                              const std::string& name, uint64_t seed, double gamma,
                              int32_t semantic_dim) {
  const auto specs = param_specs(b, n_ent, n_rel, dim, semantic_dim);
  for (size_t i = 0; i < specs.size(); ++i) {
    const ParamSpec& p = specs[i];
    if (p.name != name) continue;
    std::vector<float> out(static_cast<size_t>(p.rows * p.cols));
    Rng rng = Rng(seed).fork(i);
    const double emb = (gamma + 2.0) / dim;  // U(-(γ+2)/d, (γ+2)/d), SURVEY §8(d)
    const bool bias = name.size() > 3 && name.find("_b") != std::string::npos;
    if (bias) return out;  // zeros
    if (!p.sparse) {
      const double bound = std::sqrt(6.0 / static_cast<double>(p.rows + p.cols));  // Xavier
      for (float& v : out) v = static_cast<float>(rng.uniform(-bound, bound));
      return out;
    }
    const bool q2b_rel = b == Backbone::Q2B && name == "relation";
    for (int64_t r = 0; r < p.rows; ++r)
      for (int64_t c = 0; c < p.cols; ++c) {
        const bool offset = q2b_rel && c >= dim;  // Q2B offsets U(0, (γ+2)/d)
        out[r * p.cols + c] = static_cast<float>(offset ? rng.uniform(0.0, emb) : rng.uniform(-emb, emb));
      }
    return out;
  }
  throw ConfigError("unknown parameter " + name);
}

std::vector<float> synth_semantic_store(int32_t n_entities, int32_t dim, uint64_t seed) {
  // PTE rows N(0,1)/sqrt(d_l); gaussian() uses libm, so the bits
  // are those of this host (tests hand the same store to both sides)
  std::vector<float> out(static_cast<size_t>(n_entities) * dim);
  Rng rng(seed);
  const double scale = 1.0 / std::sqrt(static_cast<double>(dim));
  for (float& v : out) v = static_cast<float>(rng.gaussian() * scale);
  return out;
}

void write_ngse(const std::string& path, const float* data, int64_t count, int32_t dim) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw ConfigError("cannot open " + path);
  const uint32_t version = 1, d = static_cast<uint32_t>(dim);
  const uint64_t n = static_cast<uint64_t>(count);
  bool ok = std::fwrite("NGSE", 1, 4, f) == 4 && std::fwrite(&version, 4, 1, f) == 1 &&
            std::fwrite(&n, 8, 1, f) == 1 && std::fwrite(&d, 4, 1, f) == 1;
  const size_t elems = static_cast<size_t>(count) * dim;
  ok = ok && std::fwrite(data, sizeof(float), elems, f) == elems;  // host is little-endian
  std::fclose(f);
  if (!ok) throw ConfigError("short write to " + path);
}

std::vector<float> read_ngse(const std::string& path, int64_t* count, int32_t* dim) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw ConfigError("cannot open " + path);
  char magic[4];
  uint32_t version = 0, d = 0;
  uint64_t n = 0;
  const bool hdr = std::fread(magic, 1, 4, f) == 4 && std::fread(&version, 4, 1, f) == 1 &&
                   std::fread(&n, 8, 1, f) == 1 && std::fread(&d, 4, 1, f) == 1;
  if (!hdr || std::memcmp(magic, "NGSE", 4) != 0 || version != 1 || d == 0) {
    std::fclose(f);
    throw ShapeMismatch("not an NGSE v1 file: " + path);
  }
  std::vector<float> out(static_cast<size_t>(n) * d);
  const bool body = std::fread(out.data(), sizeof(float), out.size(), f) == out.size();
  std::fclose(f);
  if (!body) throw ShapeMismatch("truncated NGSE file: " + path);
  *count = static_cast<int64_t>(n);
  *dim = static_cast<int32_t>(d);
  return out;
}

ngdb_step_plan StepPlanHost::view() const {
  ngdb_step_plan p{};
  p.n_queries = n_queries;
  p.n_candidates = n_candidates;
  p.candidates = candidates.data();
  p.n_pools = static_cast<int32_t>(pools.size());
  p.pools = pools.data();
  p.n_nodes = static_cast<int32_t>(nodes.size());
  p.nodes = nodes.data();
  p.arena_elems = arena_elems;
  p.n_score_slots = n_score_slots;
  p.n_anchor_slots = n_anchor_slots;
  p.n_project_slots = n_project_slots;
  p.n_entity_rows = static_cast<int32_t>(entity_rows.size());
  p.entity_rows = entity_rows.data();
  p.entity_seg = entity_seg.data();
  p.entity_contrib = entity_contrib.data();
  p.n_relation_rows = static_cast<int32_t>(relation_rows.size());
  p.relation_rows = relation_rows.data();
  p.relation_seg = relation_seg.data();
  p.relation_contrib = relation_contrib.data();
  if (pool_dep_off.size() == pools.size() + 1) {
    p.pool_dep_off = pool_dep_off.data();
    p.pool_deps = pool_deps.data();
  }
  return p;
}

namespace {

// (row, code) pairs -> CSR with rows ascending and codes ascending within a row.
// The caller emits the keys with codes ascending in input order, so a stable
// sort by row alone yields the (row, code) order.
void build_csr(std::vector<uint64_t>& keys, std::vector<int32_t>& rows, std::vector<int32_t>& seg,
               std::vector<int32_t>& contrib) {
  radix_sort_u64(keys, 32);
  rows.clear();
  seg.clear();
  contrib.resize(keys.size());
  for (size_t i = 0; i < keys.size(); ++i) {
    const int32_t row = static_cast<int32_t>(keys[i] >> 32);
    contrib[i] = static_cast<int32_t>(static_cast<int64_t>(keys[i] & 0xffffffffu) - (1ll << 31));
    if (rows.empty() || rows.back() != row) {
      rows.push_back(row);
      seg.push_back(static_cast<int32_t>(i));
    }
  }
  seg.push_back(static_cast<int32_t>(keys.size()));
}

uint64_t pack_key(int32_t row, int32_t code) {
  return (static_cast<uint64_t>(static_cast<uint32_t>(row)) << 32) |
         static_cast<uint32_t>(static_cast<int64_t>(code) + (1ll << 31));
}

}  // namespace

StepPlanHost plan_training_step(const TrainingBatch& tb, const TrainConfig& cfg) {
  const int32_t B = static_cast<int32_t>(tb.queries.size());
  if (B == 0) throw ConfigError("empty batch");
  if (tb.n_neg != cfg.n_neg) throw ShapeMismatch("batch negatives != config n_neg");
  const int32_t nc = 1 + tb.n_neg;
  const int32_t wq = query_width(cfg.backbone, cfg.dim);

  FusedDag f = build_training_dag(tb.queries, cfg.semantic);
  const int32_t nf = f.n_fwd;

  StepPlanHost plan;
  plan.n_queries = B;
  plan.n_candidates = nc;
  plan.candidates.resize(static_cast<size_t>(B) * nc);
  for (int32_t i = 0; i < B; ++i) {
    plan.candidates[static_cast<size_t>(i) * nc] = tb.positives[i];
    std::copy(tb.negatives.begin() + static_cast<size_t>(i) * tb.n_neg,
              tb.negatives.begin() + static_cast<size_t>(i + 1) * tb.n_neg,
              plan.candidates.begin() + static_cast<size_t>(i) * nc + 1);
  }

  // Slots of the persistent per-step staging buffers, in forward-id order.
  std::vector<int32_t> aux(nf, -1);
  int32_t n_intersect = 0;
  std::vector<uint64_t> ekeys, akeys, rkeys;
  ekeys.reserve(static_cast<size_t>(B) * nc * 2 + 4 * B);
  akeys.reserve(4 * static_cast<size_t>(B));
  rkeys.reserve(4 * static_cast<size_t>(B));
  for (int32_t i = 0; i < nf; ++i) {
    const OperatorNode& x = f.nodes[i];
    switch (x.op.kind) {
      case OpKind::EmbedAnchor:
      case OpKind::FuseSemantic:
        aux[i] = plan.n_anchor_slots++;
        akeys.push_back(pack_key(x.payload, -aux[i] - 1));
        break;
      case OpKind::Project:
        aux[i] = plan.n_project_slots++;
        rkeys.push_back(pack_key(x.payload, aux[i]));
        break;
      case OpKind::Intersect:
        // stash slot: the forward kernel keeps its MLP intermediates there for
        // the mirror (at most one Intersect per query, query.hpp:14-29)
        aux[i] = n_intersect++;
        break;
      case OpKind::Score:
      case OpKind::Loss: {
        if (x.op.kind == OpKind::Loss && f.nodes[x.inputs[0]].op.kind == OpKind::UnionScore) break;
        const int32_t s = aux[i] = plan.n_score_slots++;
        const int32_t* row = &plan.candidates[static_cast<size_t>(x.query) * nc];
        for (int32_t j = 0; j < nc; ++j) ekeys.push_back(pack_key(row[j], s * nc + j));
        break;
      }
      default: break;
    }
  }
  // anchor codes -aux-1 descend in slot order: reversed, they precede the
  // ascending scoring codes
  ekeys.insert(ekeys.begin(), akeys.rbegin(), akeys.rend());
  build_csr(ekeys, plan.entity_rows, plan.entity_seg, plan.entity_contrib);
  build_csr(rkeys, plan.relation_rows, plan.relation_seg, plan.relation_contrib);

  plan.anchor_ids.assign(plan.n_anchor_slots, -1);
  plan.unit_k.assign(B, 0);
  plan.unit_slots.assign(static_cast<size_t>(B) * 3, -1);
  for (int32_t i = 0; i < nf; ++i) {
    const OperatorNode& x = f.nodes[i];
    if (x.op.kind == OpKind::EmbedAnchor || x.op.kind == OpKind::FuseSemantic)
      plan.anchor_ids[aux[i]] = x.payload;
    if (x.op.kind != OpKind::Loss) continue;
    const OperatorNode& in = f.nodes[x.inputs[0]];
    int32_t* us = &plan.unit_slots[static_cast<size_t>(x.query) * 3];
    if (in.op.kind == OpKind::UnionScore) {
      plan.unit_k[x.query] = in.n_inputs;
      for (int k = 0; k < in.n_inputs; ++k) us[k] = aux[in.inputs[k]];
    } else {
      plan.unit_k[x.query] = 1;
      us[0] = aux[i];
    }
  }

  SchedulerConfig sc;
  sc.backbone = cfg.backbone;
  sc.b_max = cfg.b_max;
  sc.query_width = wq;
  sc.n_candidates = nc;
  sc.elem_bytes = 4;
  sc.device_reuse = !cfg.sharded && cfg.device_reuse;
  sc.query_level = cfg.query_level;
  Planner planner(sc);
  const TensorModel tm{wq, nc};
  auto elems = [](int64_t bytes) { return static_cast<int32_t>(bytes / 4); };

  plan.nodes.reserve(f.nodes.size());
  auto emit = [&](const Invocation& inv) {
    ngdb_pool_desc pd;
    pd.kind = static_cast<int32_t>(inv.type.kind);
    pd.dir = static_cast<int32_t>(inv.type.dir);
    pd.k = inv.k;
    pd.first = static_cast<int32_t>(plan.nodes.size());
    pd.count = inv.n;
    pd.cycle = inv.cycle;
    plan.pools.push_back(pd);
    for (int32_t t = 0; t < inv.n; ++t) {
      const int32_t o = inv.nodes[t];
      const OperatorNode& x = f.nodes[o];
      const bool fwd = x.op.dir == Direction::Fwd;
      const int32_t mi = fwd ? o : x.mirror;
      const OperatorNode& m = f.nodes[mi];
      ngdb_node_desc d;
      d.out = fwd ? elems(planner.fwd_slot(o))
                  : (planner.bwd_slot(o) >= 0 ? elems(planner.bwd_slot(o)) : -1);
      for (int k = 0; k < 3; ++k) d.in[k] = k < m.n_inputs ? elems(planner.fwd_slot(m.inputs[k])) : -1;
      d.grad = -1;
      d.self = -1;
      if (!fwd) {
        d.self = elems(planner.fwd_slot(mi));
        if (m.consumer >= 0)
          d.grad = elems(planner.bwd_slot(nf + m.consumer)) +
                   m.consumer_slot * static_cast<int32_t>(tm.fwd_elems(f, m));
      }
      const bool scoring = m.op.kind == OpKind::Score || m.op.kind == OpKind::Loss;
      d.id = scoring ? m.query : m.payload;
      d.aux = aux[mi];
      plan.nodes.push_back(d);
    }
  };
  plan.trace = planner.run(f, emit);
  plan.arena_elems = planner.arena_bytes() / 4;
  plan.pool_dep_off = planner.inv_dep_off();
  plan.pool_deps = planner.inv_deps();
  return plan;
}

void check_status(int rc) {
  if (rc == NGDB_OK) return;
  const std::string msg = ngdb_last_error();
  switch (rc) {
    case NGDB_ERR_SHAPE_MISMATCH: throw ShapeMismatch(msg);
    case NGDB_ERR_INDEX_OUT_OF_RANGE: throw IndexOutOfRange(msg);
    case NGDB_ERR_PARAM_OUT_OF_RANGE: throw ParamOutOfRange(msg);
    case NGDB_ERR_DOMAIN: throw DomainError(msg);
    case NGDB_ERR_MISSING_KERNEL: throw MissingKernel(msg);
    case NGDB_ERR_NON_FINITE: throw NonFinite(msg);
    case NGDB_ERR_CONFIG: throw ConfigError(msg);
    default: throw Error("CUDA: " + msg);
  }
}

Trainer::Trainer(const TrainConfig& cfg, int32_t n_entities, int32_t n_relations, int device)
    : cfg_(cfg) {
  ngdb_model_desc d{};
  d.backbone = static_cast<int32_t>(cfg.backbone);
  d.n_entities = n_entities;
  d.n_relations = n_relations;
  d.dim = cfg.dim;
  d.n_neg = cfg.n_neg;
  d.semantic_dim = cfg.semantic ? cfg.semantic_dim : 0;
  d.gamma = static_cast<float>(cfg.gamma);
  d.alpha_box = static_cast<float>(cfg.alpha_box);
  d.lr = static_cast<float>(cfg.lr);
  d.beta1 = 0.9f;
  d.beta2 = 0.999f;
  d.eps_adam = 1e-8f;
  d.max_batch = cfg.b_max;
  d.max_queries = cfg.batch;
  check_status(ngdb_ctx_create(&d, device, &ctx_));
  const int32_t sd = cfg.semantic ? cfg.semantic_dim : 0;
  for (const auto& p : param_specs(cfg.backbone, n_entities, n_relations, cfg.dim, sd)) {
    auto v = init_param(cfg.backbone, n_entities, n_relations, cfg.dim, p.name, cfg.seed_params,
                        cfg.gamma, sd);
    check_status(ngdb_param_upload(ctx_, p.name.c_str(), v.data(), static_cast<int64_t>(v.size())));
  }
}

Trainer::~Trainer() { ngdb_ctx_destroy(ctx_); }

double Trainer::run_planned(const StepPlanHost& plan, std::vector<float>* per_query_loss) {
  const ngdb_step_plan view = plan.view();
  check_status(ngdb_step_begin(ctx_, &view));
  for (const auto& p : plan.pools) check_status(ngdb_exec_pool(ctx_, &p));
  check_status(ngdb_optimizer_step(ctx_, ++step_));
  double loss = 0.0;
  int32_t nonfinite = 0;
  float* out = nullptr;
  if (per_query_loss) {
    per_query_loss->resize(plan.n_queries);
    out = per_query_loss->data();
  }
  check_status(ngdb_step_end(ctx_, out, plan.n_queries, &loss, &nonfinite));
  if (nonfinite) throw NonFinite("non-finite loss at step " + std::to_string(step_));
  return loss;
}

double Trainer::step(const TrainingBatch& batch, std::vector<float>* per_query_loss) {
  return run_planned(plan_training_step(batch, cfg_), per_query_loss);
}

}  // namespace ngdb
