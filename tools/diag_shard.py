"""Diagnose the sharded step: world_size 1 (gloo) sharded vs the plain engine
on the same batch; prints per-tensor max relative gradient differences."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
import torch.distributed as dist  # noqa: E402

import paper_2602_21597_b200 as m  # noqa: E402
from paper_2602_21597_b200.sharded import Comm, ShardedEngine  # noqa: E402

dist.init_process_group("gloo", rank=0, world_size=1)
mix = sys.argv[1].split(",") if len(sys.argv) > 1 else ["2i"]
bb = sys.argv[2] if len(sys.argv) > 2 else "q2b"
g = m.Graph.synthetic("small", 1)
info = g.info()
b, k, dim = int(sys.argv[3]) if len(sys.argv) > 3 else 16, 4, 8
tag = int(sys.argv[4]) if len(sys.argv) > 4 else 1
batch = m.Batch.sample(g, m.pattern_weights(mix), b, k, seed=3, tag=tag)
plain = m.Engine(bb, info["n_entities"], info["n_relations"], dim=dim, n_neg=k, max_queries=b, debug=True)
lp = plain.train_step(batch)
sh = ShardedEngine(Comm(), bb, info["n_entities"], info["n_relations"], dim=dim, n_neg=k,
                   max_queries=b, debug=True)
ls = sh.train_step(batch)
print("loss maxdiff", np.max(np.abs(lp - ls)))
print("per-query", [(m.PATTERNS[p], round(float(x), 4)) for p, x in zip(batch.arrays().patterns, np.abs(lp - ls))])
for name, *_ in m.param_specs(bb, info["n_entities"], info["n_relations"], dim):
    a, c = plain.download("g:" + name), sh.download("g:" + name)
    d = np.max(np.abs(a - c)) / max(np.max(np.abs(a)), 1e-12)
    print(f"{name:10s} grad rel diff {d:.3e}  |g| {np.max(np.abs(a)):.3e} vs {np.max(np.abs(c)):.3e}")
dist.destroy_process_group()
