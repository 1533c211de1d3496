"""Evaluator query encoder: the forward pools of a planned
batch alone give each query's embedding (ngdb_read_score_queries); they
reproduce the step's per-query losses (Eq. 6 recomputed in f64 from the
embeddings and the entity table), leave the parameters untouched, and feed
ngdb_eval_ranks, whose ranks match the oracle bit for bit."""
import numpy as np
import pytest

import oracle
import paper_2602_21597_b200 as m

pytestmark = pytest.mark.gpu

NON_UNION = ["1p", "2p", "3p", "2i", "3i", "pi", "ip", "2in", "3in", "pin", "pni", "inp"]


def _softplus(x):
    return np.logaddexp(0.0, x)


@pytest.mark.parametrize("backbone", ["gqe", "q2b"])
def test_forward_embeddings_reproduce_losses_and_rank(small_graph, backbone):
    info = small_graph.info()
    dim, k, b = 32, 16, 96
    mix = NON_UNION + ["2u", "up"]
    bt = m.Batch.sample(small_graph, m.pattern_weights(mix), b, k, seed=3, tag=31)
    arr = bt.arrays()
    eng = m.Engine(backbone, info["n_entities"], info["n_relations"], dim=dim, n_neg=k,
                   max_queries=b)
    ent0 = eng.download("entity")
    emb, losses = eng.query_embeddings(m.PlannedStep(bt, backbone, dim))
    np.testing.assert_array_equal(eng.download("entity"), ent0)  # no update
    assert sorted(emb) == list(range(b))
    ent = ent0.astype(np.float64)
    cand = np.concatenate([arr.positives[:, None], arr.negatives], axis=1)
    for q in range(b):
        e = emb[q].astype(np.float64)  # [branches][wq]
        v = ent[cand[q]][:, None, :dim]  # [1+K][1][d]
        t = np.abs(v - e[None, :, :dim])
        if backbone == "gqe":
            d = t.sum(-1)
        else:
            o = e[None, :, dim:]
            d = np.maximum(t - o, 0).sum(-1) + 0.02 * np.minimum(t, o).sum(-1)
        d = d.min(axis=1)  # union: nearest branch (UnionScore)
        want = _softplus(d[0] - 12.0) + _softplus(12.0 - d[1:]).mean()
        assert abs(losses[q] - want) <= 1e-4 * max(abs(want), 1.0), (q, losses[q], want)
    qs = [q for q in range(b) if emb[q].shape[0] == 1]
    qv = np.stack([emb[q][0] for q in qs])
    t = arr.positives[qs].astype(np.int32)
    f = [[int(x) for x in arr.negatives[q][:5] if x != arr.positives[q]] for q in qs]
    np.testing.assert_array_equal(eng.eval_ranks(qv, t, f),
                                  oracle.eval_ranks(backbone, ent0, qv, t, f, dim))


@pytest.mark.parametrize("backbone", ["gqe", "q2b"])
def test_union_queries_rank_by_nearest_branch(small_graph, backbone):
    # the full 14-pattern evaluation path: forward embeddings (unions with two
    # branches) -> ngdb_eval_ranks_multi, bit-exact against the oracle
    info = small_graph.info()
    dim, k, b = 32, 8, 80
    bt = m.Batch.sample(small_graph, m.pattern_weights(m.PATTERNS), b, k, seed=3, tag=41)
    arr = bt.arrays()
    eng = m.Engine(backbone, info["n_entities"], info["n_relations"], dim=dim, n_neg=k,
                   max_queries=b)
    emb, _ = eng.query_embeddings(m.PlannedStep(bt, backbone, dim))
    assert any(emb[q].shape[0] == 2 for q in range(b))  # unions present
    embs = [emb[q] for q in range(b)]
    t = arr.positives.astype(np.int32)
    f = [[int(x) for x in arr.negatives[q][:4] if x != arr.positives[q]] for q in range(b)]
    ent = eng.download("entity")
    np.testing.assert_array_equal(eng.eval_ranks_multi(embs, t, f),
                                  oracle.eval_ranks_multi(backbone, ent, embs, t, f, dim))
    # synthetic branch counts 1..8 straddling the 8-slot groups (the
    # count pass must take the min over all of a query's branch slots)
    rng = np.random.default_rng(5)
    wq = dim if backbone == "gqe" else 2 * dim
    embs = []
    for i in range(40):
        e = rng.uniform(-0.04, 0.04, size=(1 + (i * 5) % 8, wq)).astype(np.float32)
        e[:, dim:] = np.abs(e[:, dim:])
        embs.append(e)
    t = rng.integers(0, info["n_entities"], size=40).astype(np.int32)
    f = [[int(x) for x in rng.integers(0, info["n_entities"], size=6) if x != t[i]]
         for i in range(40)]
    np.testing.assert_array_equal(eng.eval_ranks_multi(embs, t, f),
                                  oracle.eval_ranks_multi(backbone, ent, embs, t, f, dim))
