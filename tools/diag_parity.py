"""Diagnostic: where do product and oracle gradients differ (GPU)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
import paper_2602_21597_b200 as m
import oracle as O
from parity import run_pair, rel_close, rms

ALL = m.PATTERNS
g = m.Graph.synthetic("small", 1)
info = g.info()
og = O.OracleGraph(info["n_entities"], info["n_relations"], g.triples(0), g.triples(1), g.triples(2))
backbone = sys.argv[1] if len(sys.argv) > 1 else "gqe"
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 32
mix = ALL if (len(sys.argv) <= 3 or sys.argv[3] == "all") else sys.argv[3].split(",")
res = run_pair(g, og, backbone, mix, b=128, k=32, dim=dim)
for loss, ref in res["loss"]:
    print("loss maxrel", np.max(np.abs(loss - ref) / np.abs(ref)))
for name, (gg, r) in res["grads"].items():
    ok, nbad, worst = rel_close(gg, r)
    d = np.abs(gg - r)
    s = max(rms(r), 1e-30)
    print(f"{name}: bad {nbad}/{r.size} worst {worst:.2e} rms_ref {rms(r):.3e} rms_diff {rms(gg-r):.3e}")
    if nbad and gg.ndim == 2 and gg.shape[0] <= 800:
        rows = np.where((d > 1e-4 * np.maximum(np.abs(r), s)).any(axis=1))[0]
        cols = np.where((d > 1e-4 * np.maximum(np.abs(r), s)).any(axis=0))[0]
        print("   bad rows", rows[:20], len(rows), "bad cols", cols[:20], len(cols))
