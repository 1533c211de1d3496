"""world_size 2 (gloo, one GPU) sharded step vs the oracle sub-batch mode;
per-tensor gradient differences for a given pattern mix."""
import os
import pickle
import socket
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch.multiprocessing as mp

    import oracle as O
    import paper_2602_21597_b200 as m
    import shard_workers
    mix = sys.argv[1].split(",")
    bb = sys.argv[2] if len(sys.argv) > 2 else "q2b"
    b, k, dim = 8, 4, 8
    sizes = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [b, b]
    g = m.Graph.synthetic("small", 1)
    info = g.info()
    ne, nr = info["n_entities"], info["n_relations"]
    tmp = tempfile.mkdtemp()
    arrs = []
    for r in range(2):
        bt = m.Batch.sample(g, m.pattern_weights(mix), sizes[r], k, seed=3, tag=2 + r)
        arrs.append(bt.arrays())
        pickle.dump(arrs[-1], open(os.path.join(tmp, f"batch_1_{r}.pkl"), "wb"))
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    mp.spawn(shard_workers.gpu_step_worker, args=(2, port, tmp, "small", mix, b, k, dim, 1, bb),
             nprocs=2, join=True)
    outs = [pickle.load(open(os.path.join(tmp, f"gpu{r}.pkl"), "rb")) for r in range(2)]
    om = O.OracleModel(bb, ne, nr, dim, k)
    om.init(2)
    refs = om.step_multi(arrs, step=1)
    for r in range(2):
        print("rank", r, "loss maxdiff", np.max(np.abs(outs[r]["loss"][0] - refs[r])))
        dd = np.abs(outs[r]["loss"][0] - refs[r])
        print("   per-query", [(m.PATTERNS[p], round(float(x), 4)) for p, x in zip(arrs[r].patterns, dd)])
    for name, rows, cols, _ in m.param_specs(bb, ne, nr, dim):
        if name == "entity":
            t = np.zeros((rows, cols), np.float32)
            for r in range(2):
                t[r::2] = outs[r]["grads"][name]
        else:
            t = outs[0]["grads"][name]
        ref = om.get("g:" + name, (rows, cols))
        d = np.abs(t - ref)
        bad = np.argwhere(d > 1e-4 * max(np.max(np.abs(ref)), 1e-9))
        print(f"{name:10s} maxdiff {d.max():.3e} |ref| {np.max(np.abs(ref)):.3e} bad rows {sorted(set(bad[:, 0].tolist()))[:12]}")
    # single-rank oracle grads to see if product = one rank only
    for r in range(2):
        o1 = O.OracleModel(bb, ne, nr, dim, k)
        o1.init(2)
        o1.step(arrs[r].patterns, arrs[r].anchors, arrs[r].relations, arrs[r].positives,
                arrs[r].negatives, adam=-1)
        for name in ("relation",):
            ref1 = o1.get("g:" + name, (nr, dim * (2 if bb == "q2b" else 1)))
            print(f"rank {r} alone: relation rows {sorted(set(np.argwhere(np.abs(ref1) > 0)[:, 0].tolist()))}")
    print("anchors", [a.anchors.tolist() for a in arrs])
    print("relations", [a.relations.tolist() for a in arrs])


if __name__ == "__main__":
    main()
