// The row-sharded trainer loop (include/ngdb/shard_loop.hpp):
// the sharded counterpart of run_train_loop, all in C++ so every host stage
// runs in parallel threads without an interpreter in between.
//
//   producers (P threads)  sample batch i of this rank, plan it (sharded: private
//                          slabs, the phase-ordered step) and pack its metadata
//                          record; and — first, when one is waiting — build the
//                          owner work lists of an exchanged step (several steps'
//                          lists are built in parallel) and pack the step's
//                          device plan and owner lists into its pinned slot
//   exchange (1 thread)    in step order: all-gather the records over the
//                          context's metadata communicator (ngdb_comm_allgather_i32:
//                          its own NCCL communicator and stream, so it runs ahead
//                          of the step collectives)
//   consumer (caller)      in step order: ngdb_shard_begin + ngdb_shard_step_exec
//                          (stages + NCCL collectives + Adam on the context
//                          stream), then read step i's losses while i+1 runs
#include "ngdb/shard_loop.hpp"

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <exception>
#include <mutex>
#include <optional>
#include <thread>

#include "ngdb/shard.hpp"

namespace ngdb {

namespace {

// the C view of a rank's owner work lists (points into `s`)
ngdb_shard_plan shard_view(const ShardPlanHost& s) {
  ngdb_shard_plan sv{};
  sv.world = s.spec.world;
  sv.rank = s.spec.rank;
  sv.batch = s.spec.batch;
  sv.max_anchors = s.spec.max_anchors;
  sv.max_slots = s.spec.max_slots;
  sv.n_candidates = s.spec.n_candidates;
  sv.anchor_ids = s.anchor_ids.data();
  sv.unit_k = s.unit_k.data();
  sv.unit_slots = s.unit_slots.data();
  sv.cand = s.cand.data();
  sv.unit_off = s.unit_off.data();
  sv.owned = s.owned.data();
  sv.n_rows = static_cast<int32_t>(s.rows.size());
  sv.rows = s.rows.data();
  sv.seg = s.seg.data();
  sv.contrib = s.contrib.data();
  sv.send_cnt = s.send_cnt.data();
  sv.recv_cnt = s.recv_cnt.data();
  sv.n_send = static_cast<int32_t>(s.send_rows.size());
  sv.n_recv = static_cast<int32_t>(s.recv_slot.size());
  sv.send_rows = s.send_rows.data();
  sv.recv_slot = s.recv_slot.data();
  sv.n_anchor_pos = static_cast<int32_t>(s.anchor_pos.size());
  sv.anchor_pos = s.anchor_pos.data();
  return sv;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

struct Pinned {  // a producer-packed pinned slot: [device plan | owner lists]
  int64_t plan_n = 0, shard_n = 0;  // 0: too large for the slot, packed by the consumer
};

struct Slot {
  std::optional<StepPlanHost> plan;
  std::vector<int32_t> record;         // this rank's packed metadata
  std::vector<int32_t> all;            // every rank's records (after the exchange)
  std::optional<ShardPlanHost> shard;  // owner work lists (built by a producer)
  std::exception_ptr error;
  bool planned = false, gathered = false, exchanged = false;
};

}  // namespace

ShardLoopStats run_shard_train_loop(ngdb_ctx* ctx, const GraphSplit& graph,
                                    const ShardLoopConfig& cfg, int64_t first_step,
                                    int32_t n_steps, double* loss_per_step) {
  ShardLoopStats stats;
  if (n_steps <= 0) return stats;
  ngdb_model_desc d{};
  check_status(ngdb_ctx_desc(ctx, &d));
  const int32_t world = std::max(d.world, 1), rank = d.rank;
  if (cfg.batch <= 0 || cfg.n_neg != d.n_neg || cfg.b_max <= 0)
    throw ConfigError("invalid sharded train loop config");
  TrainConfig tc;
  tc.backbone = static_cast<Backbone>(d.backbone);
  tc.dim = d.dim;
  tc.batch = cfg.batch;
  tc.n_neg = cfg.n_neg;
  tc.b_max = cfg.b_max;
  tc.sharded = true;
  tc.semantic = d.semantic_dim > 0;
  tc.semantic_dim = d.semantic_dim;
  const int32_t cap = std::max(cfg.batch, d.max_queries);
  const int64_t stride = shard_meta_stride(cap, cfg.n_neg + 1);

  int32_t P = cfg.n_producers;
  if (P <= 0) P = std::max(1, static_cast<int32_t>(std::thread::hardware_concurrency()) - 2);
  P = std::min(P, n_steps);
  const int32_t depth = std::max(cfg.queue_depth > 0 ? cfg.queue_depth : 2 * P, 2);
  stats.producers = P;
  const int32_t in_flight = std::clamp(cfg.in_flight, 1, 3);

  std::vector<Slot> ring(depth);
  // pinned slot of step i: i % RP. A producer packs step j only while
  // j < consumed + depth, so the slot's previous step (j - RP) was submitted at
  // least 4 steps earlier and — with at most 3 steps in flight — collected:
  // its H2D copies are long done.
  // (one context-owned pinned allocation, reused by later calls: allocating
  // pinned memory while the other threads issue CUDA calls stalls them)
  const int32_t RP = depth + 4;
  std::vector<Pinned> pinned(RP);
  const int64_t nc = cfg.n_neg + 1, U = int64_t(world) * cap;
  const int64_t slot_ints = int64_t(cap) * nc * 3 + int64_t(cap) * 512 + 65536  // device plan
                            + U * nc + 4 * int64_t(cap) * nc + 8 * U + 65536;     // owner lists
  int32_t* ring_base = nullptr;
  check_status(ngdb_ctx_pinned_ring(ctx, slot_ints * RP, &ring_base));
  auto slot_ptr = [&](int64_t i) { return ring_base + (i % RP) * slot_ints; };
  std::mutex mu;
  std::condition_variable cv;
  int64_t next_claim = 0, consumed = 0, next_build = 0, gathered_upto = 0;
  bool stop = false;

  auto build = [&](int64_t i) {  // owner lists of exchanged step i (outside the lock)
    std::vector<int32_t> all;
    {
      std::lock_guard<std::mutex> lk(mu);
      all = std::move(ring[i % depth].all);
    }
    std::optional<ShardPlanHost> sp;
    std::exception_ptr err;
    try {
      sp.emplace(build_shard_plan_packed(world, rank, all.data(), stride, cap));
      // the device plan and the owner lists, packed here (off the consumer)
      const ngdb_step_plan view = ring[i % depth].plan->view();
      const ngdb_shard_plan sv = shard_view(*sp);
      Pinned& pk = pinned[i % RP];
      pk.plan_n = ngdb_plan_packed_size(&view);
      pk.shard_n = ngdb_shard_packed_size(&sv);
      if (pk.plan_n + pk.shard_n <= slot_ints) {
        int32_t* p = slot_ptr(i);
        check_status(ngdb_plan_pack(&view, p, pk.plan_n));
        check_status(ngdb_shard_pack(&sv, p + pk.plan_n, pk.shard_n));
      } else {
        pk.plan_n = pk.shard_n = 0;
      }
    } catch (...) {
      err = std::current_exception();
    }
    {
      std::lock_guard<std::mutex> lk(mu);
      Slot& s = ring[i % depth];
      s.shard = std::move(sp);
      if (err) s.error = err;
      s.exchanged = true;
    }
    cv.notify_all();
  };

  auto producer = [&] {
    for (;;) {
      int64_t i = -1, b = -1;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] {
          return stop || next_build < gathered_upto ||
                 (next_claim < n_steps && next_claim < consumed + depth) ||
                 (next_claim >= n_steps && next_build >= n_steps);
        });
        if (stop) return;
        if (next_build < gathered_upto) {
          b = next_build++;
        } else if (next_claim < n_steps && next_claim < consumed + depth) {
          i = next_claim++;
        } else {
          return;  // everything sampled and built
        }
      }
      if (b >= 0) {
        build(b);
        continue;
      }
      Slot out;
      try {
        const uint64_t tag = (cfg.first_tag + static_cast<uint64_t>(i)) * world + rank;
        Rng rng = Rng(cfg.seed).fork(tag);
        const TrainingBatch tb =
            sample_training_batch(graph.train, graph.full, cfg.pi, cfg.batch, cfg.n_neg, rng);
        out.plan.emplace(plan_training_step(tb, tc));
        out.record.resize(stride);
        pack_shard_meta(*out.plan, cap, out.record.data(), stride);
      } catch (...) {
        out.error = std::current_exception();
      }
      {
        std::lock_guard<std::mutex> lk(mu);
        Slot& s = ring[i % depth];
        s.plan = std::move(out.plan);
        s.record = std::move(out.record);
        s.error = out.error;
        s.planned = true;
      }
      cv.notify_all();
    }
  };

  // the exchange: collectives in step order on every rank
  auto exchange = [&] {
    for (int64_t i = 0; i < n_steps; ++i) {
      std::vector<int32_t> rec;
      bool failed = false;
      {
        std::unique_lock<std::mutex> lk(mu);
        Slot& s = ring[i % depth];
        cv.wait(lk, [&] { return stop || s.planned; });
        if (stop) return;
        failed = static_cast<bool>(s.error);
        if (!failed) rec = s.record;
      }
      std::vector<int32_t> all;
      std::exception_ptr err;
      if (!failed) {
        try {
          all.resize(stride * world);
          const auto t0 = std::chrono::steady_clock::now();
          check_status(ngdb_comm_allgather_i32(ctx, rec.data(), stride, all.data()));
          stats.exchange_s += seconds_since(t0);
        } catch (...) {
          err = std::current_exception();
        }
      }
      {
        std::lock_guard<std::mutex> lk(mu);
        Slot& s = ring[i % depth];
        if (err) s.error = err;
        if (failed || err) {
          s.exchanged = true;  // the consumer rethrows
        } else {
          s.all = std::move(all);
          s.gathered = true;
          gathered_upto = i + 1;
        }
      }
      cv.notify_all();
      if (failed || err) return;  // every rank stops at the same step
    }
  };

  std::vector<std::thread> threads;
  threads.reserve(P + 1);
  for (int32_t t = 0; t < P; ++t) threads.emplace_back(producer);
  threads.emplace_back(exchange);
  auto shutdown = [&] {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : threads) t.join();
  };

  std::deque<std::pair<int32_t, int64_t>> pending;  // (step index, ticket)
  std::vector<float> losses(cfg.batch);
  auto collect = [&] {
    const auto [i, ticket] = pending.front();
    pending.pop_front();
    double loss = 0.0;
    int32_t nonfinite = 0;
    const auto t0 = std::chrono::steady_clock::now();
    check_status(ngdb_step_wait(ctx, ticket, losses.data(), cfg.batch, &loss, &nonfinite));
    stats.collect_wait_s += seconds_since(t0);
    if (nonfinite) throw NonFinite("non-finite loss at step " + std::to_string(first_step + i + 1));
    if (loss_per_step) loss_per_step[i] = loss;
  };
  std::chrono::steady_clock::time_point t_steady{};
  try {
    for (int32_t i = 0; i < n_steps; ++i) {
      if (cfg.steady_from > 0 && i == cfg.steady_from) t_steady = std::chrono::steady_clock::now();
      StepPlanHost plan;
      ShardPlanHost shard;
      {
        std::unique_lock<std::mutex> lk(mu);
        Slot& s = ring[i % depth];
        const auto t0 = std::chrono::steady_clock::now();
        cv.wait(lk, [&] { return s.exchanged || (s.planned && s.error); });
        stats.plan_wait_s += seconds_since(t0);
        if (s.error) std::rethrow_exception(s.error);
        plan = std::move(*s.plan);
        shard = std::move(*s.shard);
        s = Slot{};
        consumed = i + 1;
      }
      cv.notify_all();
      const auto t_submit = std::chrono::steady_clock::now();
      const ngdb_step_plan view = plan.view();
      const ngdb_shard_plan sv = shard_view(shard);
      const Pinned& pk = pinned[i % RP];
      if (pk.plan_n > 0)
        check_status(ngdb_shard_begin_packed(ctx, &view, slot_ptr(i), pk.plan_n, &sv,
                                             slot_ptr(i) + pk.plan_n, pk.shard_n, nullptr));
      else
        check_status(ngdb_shard_begin(ctx, &view, &sv, nullptr));
      const auto t_exec = std::chrono::steady_clock::now();
      stats.begin_s += std::chrono::duration<double>(t_exec - t_submit).count();
      check_status(ngdb_shard_step_exec(ctx, first_step + i + 1));
      stats.exec_s += seconds_since(t_exec);
      int64_t ticket = -1;
      check_status(ngdb_step_end_async(ctx, &ticket));
      pending.emplace_back(i, ticket);
      stats.submit_s += seconds_since(t_submit);
      while (static_cast<int32_t>(pending.size()) >= in_flight) collect();
    }
    while (!pending.empty()) collect();
    if (cfg.steady_from > 0 && cfg.steady_from < n_steps) stats.steady_s = seconds_since(t_steady);
  } catch (...) {
    shutdown();
    for (const auto& [i, ticket] : pending) ngdb_step_wait(ctx, ticket, nullptr, 0, nullptr, nullptr);
    ngdb_sync(ctx);
    throw;
  }
  shutdown();
  ngdb_sync(ctx);  // no H2D may still read a pinned slot
  return stats;
}

}  // namespace ngdb
