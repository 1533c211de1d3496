// The row-sharded training step driven from C++ alone (no Python, no
// framework): one process per GPU, NCCL owned by libngdb_b200 (DESIGN.md §6,
// INTEGRATION.md §2). Rank 0 writes the NCCL unique id to a file the other
// ranks read (any channel works: MPI, a TCP store ...).
//
//   sharded_train <world> <rank> <device> <id_file> <shape> <steps> <batch> <n_neg> <dim>
//
// Step s of rank r trains on the batch sampled from Rng(3).fork((s+1)*world + r)
// (the bench / test convention); prints "step <s> <loss sum of this rank>".
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include "ngdb/ngdb_host.h"
#include "ngdb/trainer.hpp"

namespace {
void ok(int rc, const char* what) {
  if (rc != NGDB_OK) {
    std::fprintf(stderr, "%s failed (%d): %s\n", what, rc, ngdb_last_error());
    std::exit(1);
  }
}
}  // namespace

int main(int argc, char** argv) {
  if (argc != 10) {
    std::fprintf(stderr, "usage: %s world rank device id_file shape steps batch n_neg dim\n", argv[0]);
    return 2;
  }
  const int world = std::atoi(argv[1]), rank = std::atoi(argv[2]), device = std::atoi(argv[3]);
  const std::string id_file = argv[4], shape = argv[5];
  const int steps = std::atoi(argv[6]), batch = std::atoi(argv[7]), n_neg = std::atoi(argv[8]),
            dim = std::atoi(argv[9]);

  ngdb_graph* g = nullptr;
  ok(ngdb_graph_synthetic(shape.c_str(), 1, &g), "ngdb_graph_synthetic");
  int32_t ne, nr;
  int64_t ntr, nva, nte;
  ok(ngdb_graph_info(g, &ne, &nr, &ntr, &nva, &nte), "ngdb_graph_info");

  const ngdb_model_desc d{NGDB_Q2B, ne, nr, dim, n_neg, 0, 12.f, 0.02f, 1e-4f, 0.9f, 0.999f,
                          1e-8f, 512, batch, world, rank};
  ngdb_ctx* ctx = nullptr;
  ok(ngdb_ctx_create(&d, device, &ctx), "ngdb_ctx_create");
  for (const auto& p : ngdb::param_specs(ngdb::Backbone::Q2B, ne, nr, dim)) {
    const bool ent = p.name == "entity";
    const int64_t rows = ent ? (ne - rank + world - 1) / world : p.rows;
    std::vector<float> v(rows * p.cols);
    if (ent)
      ok(ngdb_param_init_shard(NGDB_Q2B, ne, nr, dim, p.name.c_str(), 2, world, rank, v.data(),
                               v.size()), "ngdb_param_init_shard");
    else
      ok(ngdb_param_init_ex(NGDB_Q2B, ne, nr, dim, 0, p.name.c_str(), 2, v.data(), v.size()),
         "ngdb_param_init_ex");
    ok(ngdb_param_upload(ctx, p.name.c_str(), v.data(), v.size()), "ngdb_param_upload");
  }

  // NCCL id: rank 0 -> file -> every rank
  uint8_t id[NGDB_COMM_ID_BYTES];
  if (rank == 0) {
    ok(ngdb_comm_unique_id(id), "ngdb_comm_unique_id");
    const std::string tmp = id_file + ".tmp";
    std::ofstream(tmp, std::ios::binary).write(reinterpret_cast<char*>(id), sizeof(id));
    std::rename(tmp.c_str(), id_file.c_str());
  } else {
    for (;;) {
      std::ifstream f(id_file, std::ios::binary);
      if (f && f.read(reinterpret_cast<char*>(id), sizeof(id))) break;
      std::this_thread::sleep_for(std::chrono::milliseconds(20));
    }
  }
  ok(ngdb_comm_init(ctx, id), "ngdb_comm_init");

  std::vector<double> w(14, 1.0 / 14);
  const int64_t stride = ngdb_shard_meta_stride(batch, n_neg + 1);
  std::vector<int32_t> rec(stride), all(stride * world);
  std::vector<float> losses(batch);
  for (int s = 0; s < steps; ++s) {
    ngdb_batch* bt = nullptr;
    ok(ngdb_batch_sample(g, w.data(), batch, n_neg, 3, uint64_t(s + 1) * world + rank, &bt),
       "ngdb_batch_sample");
    ngdb_step* st = nullptr;
    ok(ngdb_step_build_ex(bt, NGDB_Q2B, dim, 512, /*sharded*/ 2, &st), "ngdb_step_build_ex");
    // packed metadata record -> all ranks -> this rank's owner work lists
    ok(ngdb_step_shard_pack(st, batch, rec.data(), stride), "ngdb_step_shard_pack");
    ok(ngdb_comm_allgather_i32(ctx, rec.data(), stride, all.data()), "ngdb_comm_allgather_i32");
    ngdb_shard* sh = nullptr;
    ok(ngdb_shard_build_packed(world, rank, all.data(), stride, batch, &sh),
       "ngdb_shard_build_packed");
    ngdb_step_plan plan;
    ngdb_shard_plan splan;
    ok(ngdb_step_view(st, &plan), "ngdb_step_view");
    ok(ngdb_shard_view(sh, &splan), "ngdb_shard_view");
    ok(ngdb_shard_begin(ctx, &plan, &splan, nullptr), "ngdb_shard_begin");
    ok(ngdb_shard_step_exec(ctx, s + 1), "ngdb_shard_step_exec");  // stages + NCCL + Adam
    double sum = 0;
    int32_t nonfinite = 0;
    ok(ngdb_step_end(ctx, losses.data(), plan.n_queries, &sum, &nonfinite), "ngdb_step_end");
    std::printf("step %d %.17g\n", s + 1, sum);
    ngdb_shard_destroy(sh);
    ngdb_step_destroy(st);
    ngdb_batch_destroy(bt);
  }
  ngdb_ctx_destroy(ctx);
  ngdb_graph_destroy(g);
  return 0;
}
