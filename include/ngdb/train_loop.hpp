// ngdb/train_loop.hpp — the trainer's producer/consumer loop (SPEC.md:568-576
// train consumer loop, SPEC.md:591 producers never touch kernels).
//
// Producers sample batch i from Rng(seed).fork(first_tag + i) and plan it
// (DAG, Max-Fillness trace, device plan: all pure host work on the batch); the
// consumer thread takes the plans strictly in index order, uploads each one
// (one H2D), launches its pools and the optimizer, and collects the losses of
// step i after it has launched step i+1 (ngdb_step_end_async), so host
// planning, launch and the device step overlap. Batch contents, plans and the
// parameter update order are exactly those of the sequential
// sample -> ngdb_train_step loop; only the host work is spread over threads.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ngdb/kg.hpp"
#include "ngdb/ngdb_cuda.h"
#include "ngdb/sampler.hpp"
#include "ngdb/trainer.hpp"

namespace ngdb {

struct TrainLoopConfig {
  SamplingDistribution pi;
  int32_t batch = 512;
  int32_t n_neg = 128;
  int32_t b_max = 512;
  uint64_t seed = 3;        // sampler seed (seeds kg 1, params 2, sampler 3)
  uint64_t first_tag = 0;   // batch i uses Rng(seed).fork(first_tag + i)
  int32_t n_producers = 0;  // 0: hardware threads - 1 (at least 1)
  int32_t queue_depth = 0;  // planned batches buffered ahead of the consumer; 0: 2 * producers
  bool graphs = true;       // launch each step as one CUDA graph (ngdb_step_launch)
  int32_t in_flight = 3;    // steps on the device before the oldest one's losses are read back
                            // (C2 steady state: 2 -> 1.15 M q/s, 3 -> 1.25 M)
  int32_t steady_from = 0;  // > 0: TrainLoopStats::steady_s times steps [steady_from, n_steps)

  // -- adaptive sampling feedback (SURVEY A-10) ---------
  // After every step the consumer records, per pattern present in the batch,
  // the mean per-query loss into the DifficultyTracker (pattern order). When
  // `adaptive`, π is refreshed every `refresh_every` steps from the tracker
  // (update_distribution over the support of `pi`) and batch i is sampled with
  // the π of refresh floor(i / refresh_every): producers wait for it, so the
  // batches (and the run) do not depend on the producer count.
  bool adaptive = false;
  int32_t refresh_every = 100;
  double floor = 0.01;          // ε
  DifficultyTracker* tracker = nullptr;  // in/out; nullptr: a fresh tracker
  double* pi_per_step = nullptr;         // [n_steps][14]: π batch i was sampled with
  // -- metrics log and checkpoints ---------------------
  std::string metrics_path;     // JSON-lines, one record per step (appended)
  std::string checkpoint_path;  // written every `checkpoint_every` steps (atomic rename)
  int32_t checkpoint_every = 0; // 0: off (SPEC default cadence 1,000)
  uint64_t config_hash = 0;
};

struct TrainLoopStats {
  double plan_wait_s = 0.0;     // consumer waiting for a planned batch
  double submit_s = 0.0;        // consumer uploading + launching steps, of which:
  double begin_s = 0.0;         //   ngdb_step_begin (pack + H2D + step prologue)
  double pools_s = 0.0;         //   ngdb_exec_pool calls
  double optim_s = 0.0;         //   ngdb_optimizer_step
  double collect_wait_s = 0.0;  // consumer waiting for a step's losses
  double steady_s = 0.0;        // consumer at step steady_from -> last losses read back
  int32_t producers = 0;
};

// Runs n_steps training steps on ctx; step numbers first_step + 1 .. first_step
// + n_steps (1-based Adam step). loss_per_step[i] = Σ_q ℓ_q of step i;
// per_query_loss (optional) is [n_steps][batch]. Throws the ngdb::Error of the
// first failure (a producer's error surfaces at its step).
TrainLoopStats run_train_loop(ngdb_ctx* ctx, const GraphSplit& graph, const TrainLoopConfig& cfg,
                              int64_t first_step, int32_t n_steps, double* loss_per_step,
                              float* per_query_loss);

}  // namespace ngdb
