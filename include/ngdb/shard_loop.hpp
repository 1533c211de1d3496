// ngdb/shard_loop.hpp — the row-sharded trainer loop: host
// producer threads sample + plan + pack, one exchange thread all-gathers the
// packed metadata records in step order over the context's metadata
// communicator and builds the owner work lists, the calling thread launches
// each step (stages + NCCL collectives + Adam) and reads step i's losses back
// while step i+1 runs. Requires ngdb_comm_init on the context.
#pragma once

#include <cstdint>

#include "ngdb/kg.hpp"
#include "ngdb/ngdb_cuda.h"
#include "ngdb/sampler.hpp"
#include "ngdb/trainer.hpp"

namespace ngdb {

struct ShardLoopConfig {
  SamplingDistribution pi;
  int32_t batch = 512;      // queries per rank
  int32_t n_neg = 128;
  int32_t b_max = 512;
  uint64_t seed = 3;
  uint64_t first_tag = 0;   // batch i of rank r: Rng(seed).fork((first_tag + i) * world + r)
  int32_t n_producers = 0;  // 0: hardware threads - 2
  int32_t queue_depth = 0;  // 0: 2 * producers
  int32_t in_flight = 3;  // (C5 N=1 steady state: 2 -> 0.77 M q/s, 3 -> 0.79 M)
  int32_t steady_from = 0;  // > 0: ShardLoopStats::steady_s times steps [steady_from, n_steps)
};

struct ShardLoopStats {
  double plan_wait_s = 0.0, submit_s = 0.0, collect_wait_s = 0.0;
  double exchange_s = 0.0;  // on the exchange thread (all-gathers)
  double build_s = 0.0;     // unused: owner lists are built by the producers
  double begin_s = 0.0;     // of submit_s: ngdb_shard_begin (pack + H2D of plan and owner lists)
  double exec_s = 0.0;      // of submit_s: ngdb_shard_step_exec (stages + collectives enqueued)
  double steady_s = 0.0;    // consumer at step steady_from -> last losses read back
  int32_t producers = 0;
};

ShardLoopStats run_shard_train_loop(ngdb_ctx* ctx, const GraphSplit& graph,
                                    const ShardLoopConfig& cfg, int64_t first_step,
                                    int32_t n_steps, double* loss_per_step);

}  // namespace ngdb
