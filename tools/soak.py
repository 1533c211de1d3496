"""Soak run (GPU box): long trainer-loop runs of every config through the public
API, checking finite losses and steady throughput; one JSON line per config."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2602_21597_b200 as m  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
for cfg in ("c1", "c2", "c3", "c4"):
    backbone, shape, mix, dim, batch, n_neg = bench.CONFIGS[cfg]
    graph = m.Graph.synthetic(shape, 1)
    info = graph.info()
    sdim = bench.SEMANTIC_DIM.get(cfg, 0)
    store = m.semantic_store(info["n_entities"], sdim, seed=5) if sdim else None
    eng = m.Engine(backbone, info["n_entities"], info["n_relations"], dim=dim, n_neg=n_neg,
                   b_max=512, max_queries=batch, semantic=store)
    w = m.pattern_weights(bench.MIXES[mix])
    t0 = time.perf_counter()
    sums = eng.train(graph, w, steps, batch=batch, n_neg=n_neg, seed=3, first_tag=7_000_000,
                     steady_from=50)
    dt = time.perf_counter() - t0
    q = batch * (steps - 50) / eng.last_timings["steady_s"]
    dec = [float(np.mean(sums[i:i + steps // 10])) for i in range(0, steps, steps // 10)]
    print(json.dumps({"config": cfg, "steps": steps, "finite": bool(np.all(np.isfinite(sums))),
                      "steady_qps": round(q), "wall_s": round(dt, 2),
                      "mean_loss_per_decile": [round(x, 1) for x in dec]}), flush=True)
