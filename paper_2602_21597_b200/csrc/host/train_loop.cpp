// Producer/consumer training loop (include/ngdb/train_loop.hpp).
#include "ngdb/train_loop.hpp"

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <exception>
#include <mutex>
#include <optional>
#include <thread>

namespace ngdb {

namespace {

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

struct PlannedSlot {
  std::optional<StepPlanHost> plan;
  std::exception_ptr error;
  bool ready = false;
};

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

  auto producer = [&] {
    for (;;) {
      int64_t i;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv_space.wait(lk, [&] { return stop || next_claim >= n_steps || next_claim < consumed + depth; });
        if (stop || next_claim >= n_steps) return;
        i = next_claim++;
      }
      PlannedSlot out;
      try {
        Rng rng = Rng(cfg.seed).fork(cfg.first_tag + static_cast<uint64_t>(i));
        const TrainingBatch tb =
            sample_training_batch(graph.train, graph.full, cfg.pi, cfg.batch, cfg.n_neg, rng);
        out.plan.emplace(plan_training_step(tb, tc));
      } catch (...) {
        out.error = std::current_exception();
      }
      {
        std::lock_guard<std::mutex> lk(mu);
        PlannedSlot& s = ring[i % depth];
        s.plan = std::move(out.plan);
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

  std::deque<std::pair<int32_t, int64_t>> pending;  // (step index, ticket)
  auto collect = [&] {
    const auto [i, ticket] = pending.front();
    pending.pop_front();
    double loss = 0.0;
    int32_t nonfinite = 0;
    float* out = per_query_loss ? per_query_loss + static_cast<int64_t>(i) * cfg.batch : nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    check_status(ngdb_step_wait(ctx, ticket, out, out ? cfg.batch : 0, &loss, &nonfinite));
    stats.collect_wait_s += seconds_since(t0);
    if (nonfinite) throw NonFinite("non-finite loss at step " + std::to_string(first_step + i + 1));
    if (loss_per_step) loss_per_step[i] = loss;
  };
  try {
    for (int32_t i = 0; i < n_steps; ++i) {
      StepPlanHost plan;
      {
        std::unique_lock<std::mutex> lk(mu);
        PlannedSlot& s = ring[i % depth];
        const auto t0 = std::chrono::steady_clock::now();
        cv_ready.wait(lk, [&] { return s.ready; });
        stats.plan_wait_s += seconds_since(t0);
        if (s.error) std::rethrow_exception(s.error);
        plan = std::move(*s.plan);
        s = PlannedSlot{};
        consumed = i + 1;
      }
      cv_space.notify_all();
      const auto t_submit = std::chrono::steady_clock::now();
      const ngdb_step_plan view = plan.view();
      // packs into pinned staging + one H2D; the step prologue goes into the graph
      check_status(ngdb_step_begin_ex(ctx, &view, cfg.graphs ? NGDB_BEGIN_DEFER_PROLOGUE : 0));
      const auto t_pools = std::chrono::steady_clock::now();
      stats.begin_s += std::chrono::duration<double>(t_pools - t_submit).count();
      check_status(ngdb_step_launch(ctx, first_step + i + 1, cfg.graphs ? 1 : 0));
      stats.pools_s += seconds_since(t_pools);
      int64_t ticket = -1;
      check_status(ngdb_step_end_async(ctx, &ticket));
      pending.emplace_back(i, ticket);
      stats.submit_s += seconds_since(t_submit);
      // the oldest step's losses, read back while the newer ones run on the device
      while (static_cast<int32_t>(pending.size()) >= in_flight) collect();
    }
    while (!pending.empty()) collect();
  } catch (...) {
    shutdown();
    for (const auto& [i, ticket] : pending) ngdb_step_wait(ctx, ticket, nullptr, 0, nullptr, nullptr);
    throw;
  }
  shutdown();
  return stats;
}

}  // namespace ngdb
