import sys; sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2602_21597_b200 as m
N = 200
for shifts in ([1, 2, 3, 5, 8], [1, 3, 7, 11, 17, 29]):
    triples = np.array([(h, r, h + s) for r, s in enumerate(shifts) for h in range(N) if h + s < N], np.int32)
    rng = np.random.default_rng(0)
    idx = rng.permutation(len(triples))
    test, train = triples[idx[:60]], triples[idx[60:]]
    g = m.Graph.from_triples(N, len(shifts), train, None, test)
    for mix in (["1p","2p","3p","2i","3i"], ["1p","2p","3p"], ["1p"]):
        for dim in (400, 64):
            eng = m.Engine("gqe", N, len(shifts), dim=dim, n_neg=128, max_queries=512)
            sums = eng.train(g, m.pattern_weights(mix), 2000, batch=512, n_neg=128, seed=3, first_tag=0)
            n = len(test)
            arrs = m.BatchArrays(np.zeros(n, np.int32), np.stack([test[:, 0], -np.ones(n), -np.ones(n)], 1).astype(np.int32),
                                 np.concatenate([test[:, 1:2], -np.ones((n, 3))], 1).astype(np.int32), test[:, 2].astype(np.int32), np.zeros((n, 128), np.int32))
            emb, _ = eng.query_embeddings(m.PlannedStep(m.Batch.from_arrays(arrs), "gqe", dim))
            q = np.stack([emb[i][0] for i in range(n)]).astype(np.float32)
            ranks = eng.eval_ranks(q, test[:, 2], [[] for _ in range(n)])
            print(shifts, mix, dim, m.rank_metrics(ranks), sums[0], sums[-1], flush=True)
