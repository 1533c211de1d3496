// Producer/consumer training loop (include/ngdb/train_loop.hpp).
#include "ngdb/train_loop.hpp"

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <deque>
#include <exception>
#include <fstream>
#include <mutex>
#include <optional>
#include <sstream>
#include <thread>

namespace ngdb {

namespace {

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

struct PlannedSlot {
  std::optional<StepPlanHost> plan;
  int64_t packed_n = 0;          // the plan packed into the pinned ring slot of its index
  std::vector<int8_t> patterns;  // per query (difficulty feedback)
  SamplingDistribution pi;       // the π the batch was sampled with
  std::exception_ptr error;
  bool ready = false;
};

// A launched step awaiting its losses.
struct Pending {
  int32_t index;
  int64_t ticket;
  std::vector<int8_t> patterns;
  int64_t peak_bytes;
};

void json_array(std::ostringstream& o, const std::array<double, kPatternCount>& v) {
  o << '[';
  for (int p = 0; p < kPatternCount; ++p) o << (p ? "," : "") << v[p];
  o << ']';
}

}  // namespace

TrainLoopStats run_train_loop(ngdb_ctx* ctx, const GraphSplit& graph, const TrainLoopConfig& cfg,
                              int64_t first_step, int32_t n_steps, double* loss_per_step,
                              float* per_query_loss) {
  TrainLoopStats stats;
  if (n_steps <= 0) return stats;
  if (cfg.batch <= 0 || cfg.n_neg <= 0 || cfg.b_max <= 0) throw ConfigError("invalid train loop config");
  ngdb_model_desc d{};
  check_status(ngdb_ctx_desc(ctx, &d));
  if (d.world > 1) throw ConfigError("row-sharded context: the sharded step has its own driver");
  if (cfg.n_neg != d.n_neg) throw ShapeMismatch("train loop n_neg != context n_neg");
  TrainConfig tc;
  tc.backbone = static_cast<Backbone>(d.backbone);
  tc.dim = d.dim;
  tc.batch = cfg.batch;
  tc.n_neg = cfg.n_neg;
  tc.b_max = cfg.b_max;
  tc.semantic = d.semantic_dim > 0;
  tc.semantic_dim = d.semantic_dim;

  int32_t P = cfg.n_producers;
  if (P <= 0) P = std::max(1, static_cast<int32_t>(std::thread::hardware_concurrency()) - 1);
  // the pinned plan ring is sized from the configured depth (not the clamped
  // one) so a short warm-up call allocates what later calls reuse
  const int32_t depth_cfg = std::max(cfg.queue_depth > 0 ? cfg.queue_depth : 2 * P, 1);
  P = std::min(P, n_steps);
  const int32_t depth = std::max(cfg.queue_depth > 0 ? cfg.queue_depth : 2 * P, 1);
  stats.producers = P;
  // the context keeps 4 result slots (ngdb_step_end_async)
  const int32_t in_flight = std::clamp(cfg.in_flight, 1, 3);

  std::vector<PlannedSlot> ring(depth);
  std::mutex mu;
  std::condition_variable cv_ready, cv_space;
  int64_t next_claim = 0, consumed = 0;
  bool stop = false;
  // π of refresh v (adaptive): batch i waits for refresh i / R
  const int32_t R = std::max(cfg.refresh_every, 1);
  std::vector<SamplingDistribution> pis{cfg.pi};
  DifficultyTracker own_tracker;
  DifficultyTracker& tracker = cfg.tracker ? *cfg.tracker : own_tracker;
  std::ofstream metrics;
  if (!cfg.metrics_path.empty()) {
    metrics.open(cfg.metrics_path, std::ios::app);
    if (!metrics) throw MissingFile("cannot open metrics log " + cfg.metrics_path);
  }

  // pinned ring of packed plans: producers pack batch i into slot i % RP; a
  // producer may claim i only while i < consumed + depth, and batch i - RP was
  // collected by then (in_flight <= 3), so its H2D has long completed
  // (one context-owned allocation, reused by later calls; a plan larger than
  // its slot is packed by the consumer instead)
  const int32_t RP = std::max(depth, depth_cfg) + 4;
  const int64_t slot_ints = int64_t(cfg.batch) * (1 + cfg.n_neg) * 3 + int64_t(cfg.batch) * 512 + 65536;
  int32_t* ring_base = nullptr;
  check_status(ngdb_ctx_pinned_ring(ctx, slot_ints * RP, &ring_base));
  auto slot_ptr = [&](int64_t i) { return ring_base + (i % RP) * slot_ints; };

  auto producer = [&] {
    for (;;) {
      int64_t i;
      SamplingDistribution pi;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv_space.wait(lk, [&] { return stop || next_claim >= n_steps || next_claim < consumed + depth; });
        if (stop || next_claim >= n_steps) return;
        i = next_claim++;
        const size_t v = cfg.adaptive ? static_cast<size_t>(i / R) : 0;
        cv_space.wait(lk, [&] { return stop || pis.size() > v; });
        if (stop) return;
        pi = pis[v];
      }
      PlannedSlot out;
      out.pi = pi;
      try {
        Rng rng = Rng(cfg.seed).fork(cfg.first_tag + static_cast<uint64_t>(i));
        const TrainingBatch tb =
            sample_training_batch(graph.train, graph.full, pi, cfg.batch, cfg.n_neg, rng);
        out.patterns.reserve(tb.queries.size());
        for (const auto& q : tb.queries) out.patterns.push_back(static_cast<int8_t>(q.pattern));
        out.plan.emplace(plan_training_step(tb, tc));
        const ngdb_step_plan v = out.plan->view();
        const int64_t need = ngdb_plan_packed_size(&v);
        if (need <= slot_ints) {
          check_status(ngdb_plan_pack(&v, slot_ptr(i), slot_ints));
          out.packed_n = need;
        }
      } catch (...) {
        out.error = std::current_exception();
      }
      {
        std::lock_guard<std::mutex> lk(mu);
        PlannedSlot& s = ring[i % depth];
        s.plan = std::move(out.plan);
        s.packed_n = out.packed_n;
        s.patterns = std::move(out.patterns);
        s.pi = out.pi;
        s.error = out.error;
        s.ready = true;
      }
      cv_ready.notify_all();
    }
  };
  std::vector<std::thread> threads;
  threads.reserve(P);
  for (int32_t t = 0; t < P; ++t) threads.emplace_back(producer);
  auto shutdown = [&] {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv_space.notify_all();
    for (auto& t : threads) t.join();
  };

  std::deque<Pending> pending;
  std::vector<float> losses(cfg.batch);
  auto t_last = std::chrono::steady_clock::now();
  auto collect = [&] {
    const Pending pd = std::move(pending.front());
    pending.pop_front();
    const int32_t i = pd.index;
    double loss = 0.0;
    int32_t nonfinite = 0;
    float* out = per_query_loss ? per_query_loss + static_cast<int64_t>(i) * cfg.batch
                                : losses.data();
    const int32_t nq = static_cast<int32_t>(pd.patterns.size());
    const auto t0 = std::chrono::steady_clock::now();
    check_status(ngdb_step_wait(ctx, pd.ticket, out, nq, &loss, &nonfinite));
    stats.collect_wait_s += seconds_since(t0);
    if (nonfinite) throw NonFinite("non-finite loss at step " + std::to_string(first_step + i + 1));
    if (loss_per_step) loss_per_step[i] = loss;
    // difficulty feedback: mean per-query loss of each pattern present, in pattern order
    std::array<double, kPatternCount> sum{};
    std::array<int32_t, kPatternCount> cnt{};
    for (int32_t q = 0; q < nq; ++q) {
      sum[pd.patterns[q]] += out[q];
      ++cnt[pd.patterns[q]];
    }
    for (int p = 0; p < kPatternCount; ++p)
      if (cnt[p]) record_difficulty(tracker, static_cast<Pattern>(p), sum[p] / cnt[p]);
    if (metrics) {
      const auto now = std::chrono::steady_clock::now();
      const double dt = std::chrono::duration<double>(now - t_last).count();
      t_last = now;
      std::ostringstream o;
      o.precision(17);
      o << "{\"step\": " << first_step + i + 1 << ", \"loss\": " << loss << ", \"ema\": ";
      json_array(o, tracker.ema_loss);
      o << ", \"queries_per_s\": " << (dt > 0 ? nq / dt : 0.0)
        << ", \"peak_bytes\": " << pd.peak_bytes << "}\n";
      metrics << o.str();
      metrics.flush();
    }
  };
  auto drain = [&] {
    while (!pending.empty()) collect();
  };
  std::chrono::steady_clock::time_point t_steady{};
  try {
    for (int32_t i = 0; i < n_steps; ++i) {
      if (cfg.steady_from > 0 && i == cfg.steady_from) t_steady = std::chrono::steady_clock::now();
      if (cfg.adaptive && i > 0 && i % R == 0) {
        // refresh boundary: every earlier step's losses are in the tracker
        drain();
        {
          std::lock_guard<std::mutex> lk(mu);
          pis.push_back(update_distribution(tracker, cfg.floor, cfg.pi));
        }
        cv_space.notify_all();
      }
      StepPlanHost plan;
      int64_t packed_n = 0;
      Pending pd;
      pd.index = i;
      {
        std::unique_lock<std::mutex> lk(mu);
        PlannedSlot& s = ring[i % depth];
        const auto t0 = std::chrono::steady_clock::now();
        cv_ready.wait(lk, [&] { return s.ready; });
        stats.plan_wait_s += seconds_since(t0);
        if (s.error) std::rethrow_exception(s.error);
        plan = std::move(*s.plan);
        packed_n = s.packed_n;
        pd.patterns = std::move(s.patterns);
        if (cfg.pi_per_step)
          std::copy(s.pi.weights.begin(), s.pi.weights.end(), cfg.pi_per_step + int64_t(i) * kPatternCount);
        s = PlannedSlot{};
        consumed = i + 1;
      }
      cv_space.notify_all();
      pd.peak_bytes = plan.trace.peak_bytes;
      const auto t_submit = std::chrono::steady_clock::now();
      const ngdb_step_plan view = plan.view();
      // the producer packed the plan into pinned memory: one H2D; the step
      // prologue goes into the graph
      const int32_t bflags = cfg.graphs ? NGDB_BEGIN_DEFER_PROLOGUE : 0;
      if (packed_n > 0) check_status(ngdb_step_begin_packed(ctx, &view, slot_ptr(i), packed_n, bflags));
      else check_status(ngdb_step_begin_ex(ctx, &view, bflags));
      const auto t_pools = std::chrono::steady_clock::now();
      stats.begin_s += std::chrono::duration<double>(t_pools - t_submit).count();
      const int64_t step_no = first_step + i + 1;
      check_status(ngdb_step_launch(ctx, step_no, cfg.graphs ? 1 : 0));
      stats.pools_s += seconds_since(t_pools);
      check_status(ngdb_step_end_async(ctx, &pd.ticket));
      pending.push_back(std::move(pd));
      stats.submit_s += seconds_since(t_submit);
      if (cfg.checkpoint_every > 0 && !cfg.checkpoint_path.empty() &&
          step_no % cfg.checkpoint_every == 0) {
        drain();  // parameters of exactly `step_no` steps
        const std::string tmp = cfg.checkpoint_path + ".tmp";
        check_status(ngdb_checkpoint_save(ctx, tmp.c_str(), cfg.config_hash, step_no));
        if (std::rename(tmp.c_str(), cfg.checkpoint_path.c_str()) != 0)
          throw MissingFile("cannot rename checkpoint to " + cfg.checkpoint_path);
      }
      // the oldest step's losses, read back while the newer ones run on the device
      while (static_cast<int32_t>(pending.size()) >= in_flight) collect();
    }
    drain();
    if (cfg.steady_from > 0 && cfg.steady_from < n_steps) stats.steady_s = seconds_since(t_steady);
  } catch (...) {
    shutdown();
    for (const auto& pd : pending) ngdb_step_wait(ctx, pd.ticket, nullptr, 0, nullptr, nullptr);
    ngdb_sync(ctx);  // no H2D may still read the ring
    throw;
  }
  shutdown();
  ngdb_sync(ctx);
  return stats;
}

}  // namespace ngdb
