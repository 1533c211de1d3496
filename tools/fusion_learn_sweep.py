"""Acceptance 10, second half: with an informative synthetic
semantic store, fusion-enabled training vs structural-only at equal steps on
the compositional KG of tests/test_gpu_learning.py (relation r_k: h -> h + s_k).
Prints held-out 1p filtered MRR per store design."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2602_21597_b200 as m

N, SHIFTS = 200, [1, 2, 3, 5, 8]
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 400
triples = np.array([(h, r, h + s) for r, s in enumerate(SHIFTS) for h in range(N) if h + s < N], np.int32)
rng = np.random.default_rng(0)
idx = rng.permutation(len(triples))
test, train = triples[idx[:60]], triples[idx[60:]]
g = m.Graph.from_triples(N, len(SHIFTS), train, None, test)


def store_cluster(dl=32):  # one-hot of a contiguous position bucket
    s = np.zeros((N, dl), np.float32)
    s[np.arange(N), np.arange(N) * dl // N] = 1.0
    return s


def store_thermo(dl=32):  # thermometer code of the position
    return (np.arange(dl)[None, :] < (np.arange(N)[:, None] * dl / N)).astype(np.float32)


def store_random(dl=32):  # uninformative control
    return np.random.default_rng(1).standard_normal((N, dl)).astype(np.float32) / np.sqrt(dl)


def run(store):
    eng = m.Engine("gqe", N, len(SHIFTS), dim=dim, n_neg=128, max_queries=512, semantic=store)
    sums = eng.train(g, m.pattern_weights(["1p", "2p", "3p"]), steps, batch=512, n_neg=128, seed=3,
                     first_tag=0)
    n = len(test)
    arrs = m.BatchArrays(np.zeros(n, np.int32),
                         np.stack([test[:, 0], -np.ones(n), -np.ones(n)], 1).astype(np.int32),
                         np.concatenate([test[:, 1:2], -np.ones((n, 3))], 1).astype(np.int32),
                         test[:, 2].astype(np.int32), np.zeros((n, 128), np.int32))
    emb, _ = eng.query_embeddings(m.PlannedStep(m.Batch.from_arrays(arrs), "gqe", dim,
                                                semantic=store is not None))
    q = np.stack([emb[i][0] for i in range(n)]).astype(np.float32)
    ranks = eng.eval_ranks(q, test[:, 2], [[] for _ in range(n)])
    return m.rank_metrics(ranks)["mrr"], float(sums[0]), float(sums[-1])


for name, st in (("structural", None), ("cluster", store_cluster()), ("thermo", store_thermo()),
                 ("random", store_random())):
    mrr, l0, l1 = run(st)
    print(f"{name:10s} MRR {mrr:.4f} loss {l0:.1f} -> {l1:.1f}", flush=True)
