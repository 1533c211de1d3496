// C ABI over the host engine (include/ngdb/ngdb_host.h).
#include "ngdb/ngdb_host.h"

#include <cstring>
#include <exception>
#include <string>

#include <array>

#include "ngdb/kg.hpp"
#include "ngdb/sampler.hpp"
#include "ngdb/scheduler.hpp"
#include "ngdb/shard.hpp"
#include "ngdb/shard_loop.hpp"
#include "ngdb/synth.hpp"
#include "ngdb/trainer.hpp"
#include "ngdb/train_loop.hpp"

namespace ngdb_internal {
void set_last_error(const std::string& msg);  // ctx.cu
}

struct ngdb_graph {
  ngdb::GraphSplit split;
};
struct ngdb_batch {
  ngdb::TrainingBatch tb;
};
struct ngdb_step {
  ngdb::StepPlanHost plan;
};
struct ngdb_shard {
  ngdb::ShardPlanHost plan;
};

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return NGDB_OK;
  } catch (const ngdb::ShapeMismatch& e) {
    ngdb_internal::set_last_error(e.what());
    return NGDB_ERR_SHAPE_MISMATCH;
  } catch (const ngdb::IndexOutOfRange& e) {
    ngdb_internal::set_last_error(e.what());
    return NGDB_ERR_INDEX_OUT_OF_RANGE;
  } catch (const ngdb::IdOutOfRange& e) {
    ngdb_internal::set_last_error(e.what());
    return NGDB_ERR_INDEX_OUT_OF_RANGE;
  } catch (const ngdb::MissingKernel& e) {
    ngdb_internal::set_last_error(e.what());
    return NGDB_ERR_MISSING_KERNEL;
  } catch (const ngdb::NonFinite& e) {
    ngdb_internal::set_last_error(e.what());
    return NGDB_ERR_NON_FINITE;
  } catch (const ngdb::NonFiniteLoss& e) {
    ngdb_internal::set_last_error(std::string("NonFiniteLoss: ") + e.what());
    return NGDB_ERR_NON_FINITE;
  } catch (const ngdb::Error& e) {
    ngdb_internal::set_last_error(std::string(e.what()));
    return NGDB_ERR_CONFIG;
  } catch (const std::exception& e) {
    ngdb_internal::set_last_error(e.what());
    return NGDB_ERR_CONFIG;
  }
}

std::vector<ngdb::Triple> triples_of(const int32_t* p, int64_t n) {
  std::vector<ngdb::Triple> out(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) out[i] = {p[3 * i], p[3 * i + 1], p[3 * i + 2]};
  return out;
}

ngdb::QueryInstance query_of(int32_t pattern, const int32_t* anchors, const int32_t* relations) {
  if (pattern < 0 || pattern >= ngdb::kPatternCount)
    throw ngdb::UnsupportedPattern("pattern index " + std::to_string(pattern));
  ngdb::QueryInstance q;
  q.pattern = static_cast<ngdb::Pattern>(pattern);
  const auto& info = ngdb::pattern_info(q.pattern);
  q.anchors.assign(anchors, anchors + info.n_anchors);
  q.relations.assign(relations, relations + info.n_relations);
  q.validate();
  return q;
}

}  // namespace

extern "C" {

int ngdb_graph_synthetic(const char* shape, uint64_t seed, ngdb_graph** out) {
  return guarded([&] {
    auto* g = new ngdb_graph();
    g->split = ngdb::make_synthetic(ngdb::synth_shape(shape), seed);
    *out = g;
  });
}

int ngdb_graph_from_triples(int32_t n_entities, int32_t n_relations, const int32_t* train,
                            int64_t n_train, const int32_t* valid, int64_t n_valid,
                            const int32_t* test, int64_t n_test, ngdb_graph** out) {
  return guarded([&] {
    ngdb::SynthTriples t;
    t.train = triples_of(train, n_train);
    t.valid = triples_of(valid, n_valid);
    t.test = triples_of(test, n_test);
    auto* g = new ngdb_graph();
    g->split = ngdb::split_from_triples(n_entities, n_relations, t);
    *out = g;
  });
}

int ngdb_graph_load(const char* dir, ngdb_graph** out) {
  return guarded([&] {
    auto* g = new ngdb_graph();
    g->split = ngdb::load_graph(dir);
    *out = g;
  });
}

int ngdb_graph_info(const ngdb_graph* g, int32_t* n_entities, int32_t* n_relations,
                    int64_t* n_train, int64_t* n_valid, int64_t* n_test) {
  return guarded([&] {
    if (n_entities) *n_entities = g->split.full.n_entities();
    if (n_relations) *n_relations = g->split.full.n_relations();
    if (n_train) *n_train = static_cast<int64_t>(g->split.train.triples().size());
    if (n_valid) *n_valid = static_cast<int64_t>(g->split.valid_edges.size());
    if (n_test) *n_test = static_cast<int64_t>(g->split.test_edges.size());
  });
}

int ngdb_graph_triples(const ngdb_graph* g, int32_t split, int32_t* out, int64_t n) {
  return guarded([&] {
    const std::vector<ngdb::Triple>* v = split == 0   ? &g->split.train.triples()
                                         : split == 1 ? &g->split.valid_edges
                                                      : &g->split.test_edges;
    if (static_cast<int64_t>(v->size()) != n) throw ngdb::ShapeMismatch("triple count");
    for (int64_t i = 0; i < n; ++i) {
      out[3 * i] = (*v)[i].head;
      out[3 * i + 1] = (*v)[i].rel;
      out[3 * i + 2] = (*v)[i].tail;
    }
  });
}

int ngdb_graph_answer(const ngdb_graph* g, int32_t full, int32_t pattern, const int32_t* anchors,
                      const int32_t* relations, int32_t* out, int64_t cap, int64_t* n) {
  return guarded([&] {
    auto ans = ngdb::answer_query(full ? g->split.full : g->split.train,
                                  query_of(pattern, anchors, relations));
    *n = static_cast<int64_t>(ans.size());
    const int64_t k = std::min<int64_t>(cap, *n);
    if (k > 0) std::memcpy(out, ans.data(), k * sizeof(int32_t));
  });
}

int ngdb_graph_predictive_answers(const ngdb_graph* g, int32_t pattern, const int32_t* anchors,
                                  const int32_t* relations, int32_t* obs, int64_t obs_cap,
                                  int64_t* n_obs, int32_t* miss, int64_t miss_cap, int64_t* n_miss) {
  return guarded([&] {
    const auto [o, m] = ngdb::predictive_answers(g->split, query_of(pattern, anchors, relations));
    *n_obs = static_cast<int64_t>(o.size());
    *n_miss = static_cast<int64_t>(m.size());
    const int64_t ko = std::min<int64_t>(obs_cap, *n_obs), km = std::min<int64_t>(miss_cap, *n_miss);
    if (ko > 0) std::memcpy(obs, o.data(), ko * sizeof(int32_t));
    if (km > 0) std::memcpy(miss, m.data(), km * sizeof(int32_t));
  });
}

int ngdb_graph_destroy(ngdb_graph* g) {
  delete g;
  return NGDB_OK;
}

int ngdb_batch_sample(const ngdb_graph* g, const double* w, int32_t b, int32_t n_neg, uint64_t seed,
                      uint64_t tag, ngdb_batch** out) {
  return guarded([&] {
    ngdb::SamplingDistribution pi;
    for (int i = 0; i < ngdb::kPatternCount; ++i) pi.weights[i] = w[i];
    ngdb::Rng rng = ngdb::Rng(seed).fork(tag);
    auto* bt = new ngdb_batch();
    bt->tb = ngdb::sample_training_batch(g->split.train, g->split.full, pi, b, n_neg, rng);
    *out = bt;
  });
}

int ngdb_batch_from_arrays(int32_t b, const int32_t* patterns, const int32_t* anchors,
                           const int32_t* relations, const int32_t* positives, int32_t n_neg,
                           const int32_t* negatives, ngdb_batch** out) {
  return guarded([&] {
    auto* bt = new ngdb_batch();
    bt->tb.n_neg = n_neg;
    for (int32_t i = 0; i < b; ++i) {
      bt->tb.queries.push_back(query_of(patterns[i], anchors + 3 * i, relations + 4 * i));
      bt->tb.positives.push_back(positives[i]);
    }
    bt->tb.negatives.assign(negatives, negatives + static_cast<int64_t>(b) * n_neg);
    *out = bt;
  });
}

int ngdb_batch_info(const ngdb_batch* bt, int32_t* b, int32_t* n_neg) {
  return guarded([&] {
    *b = static_cast<int32_t>(bt->tb.queries.size());
    *n_neg = bt->tb.n_neg;
  });
}

int ngdb_batch_arrays(const ngdb_batch* bt, int32_t* patterns, int32_t* anchors,
                      int32_t* relations, int32_t* positives, int32_t* negatives) {
  return guarded([&] {
    const auto& tb = bt->tb;
    for (size_t i = 0; i < tb.queries.size(); ++i) {
      const auto& q = tb.queries[i];
      if (patterns) patterns[i] = static_cast<int32_t>(q.pattern);
      for (int k = 0; k < 3; ++k)
        if (anchors) anchors[3 * i + k] = k < static_cast<int>(q.anchors.size()) ? q.anchors[k] : -1;
      for (int k = 0; k < 4; ++k)
        if (relations)
          relations[4 * i + k] = k < static_cast<int>(q.relations.size()) ? q.relations[k] : -1;
      if (positives) positives[i] = tb.positives[i];
    }
    if (negatives) std::memcpy(negatives, tb.negatives.data(), tb.negatives.size() * sizeof(int32_t));
  });
}

int ngdb_batch_destroy(ngdb_batch* bt) {
  delete bt;
  return NGDB_OK;
}

int ngdb_step_build(const ngdb_batch* bt, int32_t backbone, int32_t dim, int32_t b_max,
                    int32_t semantic, ngdb_step** out) {
  return guarded([&] {
    ngdb::TrainConfig cfg;
    cfg.backbone = static_cast<ngdb::Backbone>(backbone);
    cfg.dim = dim;
    cfg.n_neg = bt->tb.n_neg;
    cfg.b_max = b_max;
    cfg.semantic = semantic != 0;
    auto* s = new ngdb_step();
    s->plan = ngdb::plan_training_step(bt->tb, cfg);
    *out = s;
  });
}

int ngdb_step_build_ex(const ngdb_batch* bt, int32_t backbone, int32_t dim, int32_t b_max,
                       int32_t flags, ngdb_step** out) {
  return guarded([&] {
    ngdb::TrainConfig cfg;
    cfg.backbone = static_cast<ngdb::Backbone>(backbone);
    cfg.dim = dim;
    cfg.n_neg = bt->tb.n_neg;
    cfg.b_max = b_max;
    cfg.semantic = (flags & 1) != 0;
    cfg.sharded = (flags & 2) != 0;
    cfg.query_level = (flags & 4) != 0;
    cfg.device_reuse = (flags & 8) != 0;
    auto* s = new ngdb_step();
    s->plan = ngdb::plan_training_step(bt->tb, cfg);
    *out = s;
  });
}

int ngdb_step_view(const ngdb_step* s, ngdb_step_plan* view) {
  return guarded([&] { *view = s->plan.view(); });
}

int ngdb_step_trace_json(const ngdb_step* s, int32_t with_nodes, char* buf, int64_t cap,
                         int64_t* len) {
  return guarded([&] {
    std::string js = s->plan.trace.to_json();
    if (with_nodes) {
      // append {"nodes":[[...],...]} as a sibling document after a newline
      js += "\n[";
      for (size_t i = 0; i < s->plan.trace.records.size(); ++i) {
        if (i) js += ',';
        js += '[';
        const auto& nodes = s->plan.trace.records[i].nodes;
        for (size_t k = 0; k < nodes.size(); ++k) {
          if (k) js += ',';
          js += std::to_string(nodes[k]);
        }
        js += ']';
      }
      js += ']';
    }
    *len = static_cast<int64_t>(js.size());
    if (buf && cap > 0) {
      const int64_t k = std::min<int64_t>(cap - 1, *len);
      std::memcpy(buf, js.data(), k);
      buf[k] = '\0';
    }
  });
}

int ngdb_step_destroy(ngdb_step* s) {
  delete s;
  return NGDB_OK;
}

uint64_t ngdb_rng_next(uint64_t seed, int64_t fork_tag, int32_t skip) {
  ngdb::Rng r(seed);
  if (fork_tag >= 0) r = r.fork(static_cast<uint64_t>(fork_tag));
  for (int32_t i = 0; i < skip; ++i) r.next();
  return r.next();
}

int ngdb_rng_below(uint64_t seed, const uint64_t* ns, int32_t count, int32_t reps, uint64_t* out) {
  return guarded([&] {
    ngdb::Rng r(seed);
    int64_t k = 0;
    for (int32_t i = 0; i < count; ++i)
      for (int32_t j = 0; j < reps; ++j) out[k++] = r.below(ns[i]);
  });
}

int ngdb_select_pool(const int64_t* counts, const int64_t* heads, int32_t* pool) {
  return guarded([&] {
    std::array<int64_t, ngdb::kPoolCount> c{}, h{};
    for (int i = 0; i < ngdb::kPoolCount; ++i) {
      c[i] = counts[i];
      h[i] = heads[i];
    }
    *pool = ngdb::select_pool(c, h);
  });
}

int ngdb_jsonl_roundtrip(const char* line, char* out, int64_t cap) {
  return guarded([&] {
    const std::string s = ngdb::to_jsonl(ngdb::parse_jsonl(line));
    if (static_cast<int64_t>(s.size()) + 1 > cap) throw ngdb::ShapeMismatch("buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
  });
}

int ngdb_param_init(int32_t backbone, int32_t n_entities, int32_t n_relations, int32_t dim,
                    const char* name, uint64_t seed, float* out, int64_t n) {
  return guarded([&] {
    auto v = ngdb::init_param(static_cast<ngdb::Backbone>(backbone), n_entities, n_relations, dim,
                              name, seed);
    if (static_cast<int64_t>(v.size()) != n) throw ngdb::ShapeMismatch("param size");
    std::memcpy(out, v.data(), n * sizeof(float));
  });
}

int ngdb_param_init_ex(int32_t backbone, int32_t n_entities, int32_t n_relations, int32_t dim,
                       int32_t semantic_dim, const char* name, uint64_t seed, float* out,
                       int64_t n) {
  return guarded([&] {
    auto v = ngdb::init_param(static_cast<ngdb::Backbone>(backbone), n_entities, n_relations, dim,
                              name, seed, 12.0, semantic_dim);
    if (static_cast<int64_t>(v.size()) != n) throw ngdb::ShapeMismatch("param size");
    std::memcpy(out, v.data(), n * sizeof(float));
  });
}

int ngdb_semantic_synth(int32_t n_entities, int32_t dim, uint64_t seed, float* out) {
  return guarded([&] {
    auto v = ngdb::synth_semantic_store(n_entities, dim, seed);
    std::memcpy(out, v.data(), v.size() * sizeof(float));
  });
}

int ngdb_ngse_write(const char* path, const float* data, int64_t count, int32_t dim) {
  return guarded([&] { ngdb::write_ngse(path, data, count, dim); });
}

int ngdb_ngse_read(const char* path, float* out, int64_t cap, int64_t* count, int32_t* dim) {
  return guarded([&] {
    auto v = ngdb::read_ngse(path, count, dim);
    if (out) {
      if (cap < static_cast<int64_t>(v.size())) throw ngdb::ShapeMismatch("buffer too small");
      std::memcpy(out, v.data(), v.size() * sizeof(float));
    }
  });
}

int ngdb_step_shard_info(const ngdb_step* s, int32_t* n_anchor_slots, int32_t* n_score_slots,
                         int32_t* batch, int32_t* n_candidates) {
  return guarded([&] {
    *n_anchor_slots = s->plan.n_anchor_slots;
    *n_score_slots = s->plan.n_score_slots;
    *batch = s->plan.n_queries;
    *n_candidates = s->plan.n_candidates;
  });
}

int ngdb_step_shard_meta(const ngdb_step* s, int32_t* anchor_ids, int32_t* unit_k,
                         int32_t* unit_slots, int32_t* cand) {
  return guarded([&] {
    const auto& p = s->plan;
    std::memcpy(anchor_ids, p.anchor_ids.data(), p.anchor_ids.size() * sizeof(int32_t));
    std::memcpy(unit_k, p.unit_k.data(), p.unit_k.size() * sizeof(int32_t));
    std::memcpy(unit_slots, p.unit_slots.data(), p.unit_slots.size() * sizeof(int32_t));
    std::memcpy(cand, p.candidates.data(), p.candidates.size() * sizeof(int32_t));
  });
}

int ngdb_shard_build(int32_t world, int32_t rank, int32_t batch, int32_t max_anchors,
                     int32_t max_slots, int32_t n_candidates, const int32_t* anchor_ids_all,
                     const int32_t* unit_k_all, const int32_t* unit_slots_all,
                     const int32_t* cand_all, ngdb_shard** out) {
  return guarded([&] {
    ngdb::ShardSpec spec{world, rank, batch, max_anchors, max_slots, n_candidates};
    auto* s = new ngdb_shard();
    s->plan = ngdb::build_shard_plan(spec, anchor_ids_all, unit_k_all, unit_slots_all, cand_all);
    *out = s;
  });
}

int ngdb_shard_view(const ngdb_shard* s, ngdb_shard_plan* v) {
  return guarded([&] {
    const auto& p = s->plan;
    *v = ngdb_shard_plan{};
    v->world = p.spec.world;
    v->rank = p.spec.rank;
    v->batch = p.spec.batch;
    v->max_anchors = p.spec.max_anchors;
    v->max_slots = p.spec.max_slots;
    v->n_candidates = p.spec.n_candidates;
    v->anchor_ids = p.anchor_ids.data();
    v->unit_k = p.unit_k.data();
    v->unit_slots = p.unit_slots.data();
    v->cand = p.cand.data();
    v->unit_off = p.unit_off.data();
    v->owned = p.owned.data();
    v->n_rows = static_cast<int32_t>(p.rows.size());
    v->rows = p.rows.data();
    v->seg = p.seg.data();
    v->contrib = p.contrib.data();
    v->send_cnt = p.send_cnt.data();
    v->recv_cnt = p.recv_cnt.data();
    v->n_send = static_cast<int32_t>(p.send_rows.size());
    v->n_recv = static_cast<int32_t>(p.recv_slot.size());
    v->send_rows = p.send_rows.data();
    v->recv_slot = p.recv_slot.data();
    v->n_anchor_pos = static_cast<int32_t>(p.anchor_pos.size());
    v->anchor_pos = p.anchor_pos.data();
  });
}

int64_t ngdb_shard_meta_stride(int32_t batch_cap, int32_t n_candidates) {
  return ngdb::shard_meta_stride(batch_cap, n_candidates);
}

int ngdb_step_shard_pack(const ngdb_step* s, int32_t batch_cap, int32_t* out, int64_t stride) {
  return guarded([&] { ngdb::pack_shard_meta(s->plan, batch_cap, out, stride); });
}

int ngdb_shard_build_packed(int32_t world, int32_t rank, const int32_t* gathered, int64_t stride,
                            int32_t batch_cap, ngdb_shard** out) {
  return guarded([&] {
    auto* s = new ngdb_shard();
    try {
      s->plan = ngdb::build_shard_plan_packed(world, rank, gathered, stride, batch_cap);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

int ngdb_shard_destroy(ngdb_shard* s) {
  delete s;
  return NGDB_OK;
}

int ngdb_param_init_shard(int32_t backbone, int32_t n_entities, int32_t n_relations, int32_t dim,
                          const char* name, uint64_t seed, int32_t world, int32_t rank,
                          float* out, int64_t n) {
  return guarded([&] {
    auto v = ngdb::init_param(static_cast<ngdb::Backbone>(backbone), n_entities, n_relations, dim,
                              name, seed);
    const auto specs = ngdb::param_specs(static_cast<ngdb::Backbone>(backbone), n_entities,
                                         n_relations, dim);
    int64_t cols = 0;
    for (const auto& p : specs)
      if (p.name == name) cols = p.cols;
    const int64_t rows = static_cast<int64_t>(v.size()) / cols;
    int64_t k = 0;
    for (int64_t r = rank; r < rows; r += world) {
      if ((k + 1) * cols > n) throw ngdb::ShapeMismatch("shard buffer too small");
      std::memcpy(out + k * cols, v.data() + r * cols, cols * sizeof(float));
      ++k;
    }
    if (k * cols != n) throw ngdb::ShapeMismatch("shard size");
  });
}

int ngdb_run_step(ngdb_ctx* ctx, const ngdb_step* s, int64_t step, float* per_query_loss,
                  double* loss_sum) {
  return guarded([&] {
    const ngdb_step_plan view = s->plan.view();
    ngdb::check_status(ngdb_step_begin(ctx, &view));
    for (const auto& p : s->plan.pools) ngdb::check_status(ngdb_exec_pool(ctx, &p));
    ngdb::check_status(ngdb_optimizer_step(ctx, step));
    int32_t nonfinite = 0;
    ngdb::check_status(
        ngdb_step_end(ctx, per_query_loss, s->plan.n_queries, loss_sum, &nonfinite));
    if (nonfinite) throw ngdb::NonFinite("non-finite loss at step " + std::to_string(step));
  });
}

int ngdb_train_step(ngdb_ctx* ctx, const ngdb_batch* bt, int32_t b_max, int64_t step,
                    float* per_query_loss, double* loss_sum) {
  return guarded([&] {
    ngdb_model_desc d;
    ngdb::check_status(ngdb_ctx_desc(ctx, &d));
    ngdb::TrainConfig cfg;
    cfg.backbone = static_cast<ngdb::Backbone>(d.backbone);
    cfg.dim = d.dim;
    cfg.n_neg = bt->tb.n_neg;
    cfg.b_max = b_max;
    cfg.semantic = d.semantic_dim > 0;
    cfg.semantic_dim = d.semantic_dim;
    ngdb_step s;
    s.plan = ngdb::plan_training_step(bt->tb, cfg);
    ngdb::check_status(ngdb_run_step(ctx, &s, step, per_query_loss, loss_sum));
  });
}

int ngdb_train_run_ex(ngdb_ctx* ctx, const ngdb_graph* g, const ngdb_train_opts* o,
                      const ngdb_train_feedback* fb, int64_t first_step, int32_t n_steps,
                      double* loss_per_step, float* per_query_loss, double* timings) {
  return guarded([&] {
    if (!ctx || !g || !o || !o->pattern_weights) throw ngdb::ConfigError("null argument");
    ngdb::TrainLoopConfig cfg;
    for (int i = 0; i < ngdb::kPatternCount; ++i) cfg.pi.weights[i] = o->pattern_weights[i];
    cfg.batch = o->batch;
    cfg.n_neg = o->n_neg;
    cfg.b_max = o->b_max;
    cfg.n_producers = o->n_producers;
    cfg.queue_depth = o->queue_depth;
    cfg.seed = o->seed;
    cfg.first_tag = o->first_tag;
    if (o->in_flight > 0) cfg.in_flight = o->in_flight;
    cfg.graphs = (o->flags & NGDB_TRAIN_NO_GRAPHS) == 0;
    cfg.steady_from = o->steady_from;
    ngdb::DifficultyTracker tracker;
    if (fb) {
      cfg.adaptive = fb->adaptive != 0;
      if (fb->refresh_every > 0) cfg.refresh_every = fb->refresh_every;
      if (fb->decay > 0) tracker.decay = fb->decay;
      if (fb->eta > 0) tracker.temperature = fb->eta;
      if (fb->floor > 0) cfg.floor = fb->floor;
      if (fb->ema_loss && fb->observations)
        for (int p = 0; p < ngdb::kPatternCount; ++p) {
          tracker.ema_loss[p] = fb->ema_loss[p];
          tracker.observations[p] = fb->observations[p];
        }
      cfg.pi_per_step = fb->pi_per_step;
      if (fb->metrics_path) cfg.metrics_path = fb->metrics_path;
      if (fb->checkpoint_path) cfg.checkpoint_path = fb->checkpoint_path;
      cfg.checkpoint_every = fb->checkpoint_every;
      cfg.config_hash = fb->config_hash;
    }
    cfg.tracker = &tracker;
    const auto st = ngdb::run_train_loop(ctx, g->split, cfg, first_step, n_steps, loss_per_step,
                                         per_query_loss);
    if (fb && fb->ema_loss && fb->observations)
      for (int p = 0; p < ngdb::kPatternCount; ++p) {
        fb->ema_loss[p] = tracker.ema_loss[p];
        fb->observations[p] = tracker.observations[p];
      }
    if (timings) {
      timings[0] = st.plan_wait_s;
      timings[1] = st.submit_s;
      timings[2] = st.collect_wait_s;
      timings[3] = st.begin_s;
      timings[4] = st.pools_s;
      timings[5] = st.optim_s;
      if (o->steady_from > 0) timings[6] = st.steady_s;
    }
  });
}

int ngdb_train_run(ngdb_ctx* ctx, const ngdb_graph* g, const ngdb_train_opts* o,
                   int64_t first_step, int32_t n_steps, double* loss_per_step,
                   float* per_query_loss, double* timings) {
  return ngdb_train_run_ex(ctx, g, o, nullptr, first_step, n_steps, loss_per_step,
                           per_query_loss, timings);
}

int ngdb_shard_train_run(ngdb_ctx* ctx, const ngdb_graph* g, const ngdb_train_opts* o,
                         int64_t first_step, int32_t n_steps, double* loss_per_step,
                         double* timings) {
  return guarded([&] {
    if (!ctx || !g || !o || !o->pattern_weights) throw ngdb::ConfigError("null argument");
    ngdb::ShardLoopConfig cfg;
    for (int i = 0; i < ngdb::kPatternCount; ++i) cfg.pi.weights[i] = o->pattern_weights[i];
    cfg.batch = o->batch;
    cfg.n_neg = o->n_neg;
    cfg.b_max = o->b_max;
    cfg.n_producers = o->n_producers;
    cfg.queue_depth = o->queue_depth;
    cfg.seed = o->seed;
    cfg.first_tag = o->first_tag;
    if (o->in_flight > 0) cfg.in_flight = o->in_flight;
    cfg.steady_from = o->steady_from;
    const auto st = ngdb::run_shard_train_loop(ctx, g->split, cfg, first_step, n_steps, loss_per_step);
    if (timings) {
      timings[0] = st.plan_wait_s;
      timings[1] = st.submit_s;
      timings[2] = st.collect_wait_s;
      timings[3] = st.exchange_s;
      timings[4] = st.begin_s;  // (owner lists are built on the producers: no build time)
      timings[5] = st.producers;
      if (o->steady_from > 0) {  // timings then needs 8 entries
        timings[6] = st.steady_s;
        timings[7] = st.exec_s;
      }
    }
  });
}

int ngdb_record_difficulty(double* ema_loss, int64_t* observations, double decay, int32_t pattern,
                           double loss) {
  return guarded([&] {
    if (pattern < 0 || pattern >= ngdb::kPatternCount) throw ngdb::ConfigError("pattern index");
    ngdb::DifficultyTracker t;
    t.decay = decay;
    t.ema_loss[pattern] = ema_loss[pattern];
    t.observations[pattern] = observations[pattern];
    ngdb::record_difficulty(t, static_cast<ngdb::Pattern>(pattern), loss);
    ema_loss[pattern] = t.ema_loss[pattern];
    observations[pattern] = t.observations[pattern];
  });
}

int ngdb_update_distribution(const double* ema_loss, const int64_t* observations, double eta,
                             double floor, const double* base, double* weights_out) {
  return guarded([&] {
    ngdb::DifficultyTracker t;
    t.temperature = eta;
    for (int p = 0; p < ngdb::kPatternCount; ++p) {
      t.ema_loss[p] = ema_loss[p];
      t.observations[p] = observations[p];
    }
    ngdb::SamplingDistribution b;
    for (int p = 0; p < ngdb::kPatternCount; ++p) b.weights[p] = base ? base[p] : 1.0 / ngdb::kPatternCount;
    const auto d = ngdb::update_distribution(t, floor, b);
    for (int p = 0; p < ngdb::kPatternCount; ++p) weights_out[p] = d.weights[p];
  });
}

}  // extern "C"
