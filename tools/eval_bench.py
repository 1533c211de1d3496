"""Evaluator measurement (GPU box): ngdb_eval_ranks on the C2 shape (63,361
entities, d = 400, Q2B and GQE), 512 queries per call, filters of 100 entities.
Reports queries/s end to end (host query/target/filter upload, 2-3 kernels,
rank read-back) and the count kernel's (entity, query, dimension) rate."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_21597_b200 as m  # noqa: E402

n_ent, dim, nq, reps = 63361, 400, 512, 10
rng = np.random.default_rng(1)
for bb in ("gqe", "q2b"):
    eng = m.Engine(bb, n_ent, 200, dim=dim, n_neg=4, max_queries=64)
    wq = dim if bb == "gqe" else 2 * dim
    q = rng.uniform(-0.035, 0.035, size=(nq, wq)).astype(np.float32)
    q[:, dim:] = np.abs(q[:, dim:])
    t = rng.integers(0, n_ent, size=nq).astype(np.int32)
    f = [[int(x) for x in rng.integers(0, n_ent, size=100) if x != t[i]] for i in range(nq)]
    off = np.zeros(nq + 1, dtype=np.int32)
    off[1:] = np.cumsum([len(x) for x in f])
    ids = np.concatenate([np.asarray(x, dtype=np.int32) for x in f])
    for _ in range(3):
        eng.eval_ranks_csr(q, t, off, ids)
    t0 = time.perf_counter()
    for _ in range(reps):
        r = eng.eval_ranks_csr(q, t, off, ids)
    dt = (time.perf_counter() - t0) / reps
    print(json.dumps({"evaluator": bb, "entities": n_ent, "dim": dim, "queries_per_call": nq,
                      "ms_per_call": dt * 1e3, "queries_per_s": nq / dt,
                      "pair_dims_per_s": nq * n_ent * dim / dt,
                      "mrr_random_model": m.rank_metrics(r)["mrr"]}), flush=True)
