"""Evaluator on the BetaE and fusion backbones (SURVEY §8(f)
rank 2). BetaE ranks by KL(entity || query) through the step prologue's entity
side (T_e, C_e) over all entities; GQE + FuseSemantic ranks by L1 against the
fused rows sigma(W_p [h | F s] + b_p) of every entity. Two-level parity: the
device entity tables against the f64 oracle (1e-4 relative), and the integer
ranks bit-exact against the oracle's fp32 restatement over those tables."""
import numpy as np
import pytest

import oracle as O
import paper_2602_21597_b200 as m
from parity import rel_close

pytestmark = pytest.mark.gpu
ALL = m.engine.PATTERNS


def _train(eng, graph, steps=2, b=64, k=16):
    w = m.pattern_weights(ALL)
    for s in range(steps):
        eng.train_step(m.Batch.sample(graph, w, b, k, seed=3, tag=40 + s))


def _queries(rng, n, n_ent, width, beta):
    if beta:
        q = rng.uniform(0.05, 4.0, size=(n, width)).astype(np.float32)
    else:
        q = rng.uniform(0.2, 0.8, size=(n, width)).astype(np.float32)
    t = rng.integers(0, n_ent, size=n).astype(np.int32)
    f = [[int(x) for x in rng.integers(0, n_ent, size=7) if x != t[i]] for i in range(n)]
    return q, t, f


@pytest.mark.parametrize("shape,dim", [("small", 32), ("fb15k-237", 400)])
def test_betae_ranks(shape, dim):
    g = m.Graph.synthetic(shape, 1)
    info = g.info()
    eng = m.Engine("betae", info["n_entities"], info["n_relations"], dim=dim, n_neg=16,
                   max_queries=64)
    _train(eng, g)
    T, Cst = eng.eval_entity_table()
    T64, C64 = O.beta_eval_table(eng.download("entity").astype(np.float64), dim)
    ok, nbad, worst = rel_close(T, T64)
    assert ok, f"T: {nbad} beyond 1e-4 (worst {worst:.3e})"
    ok, nbad, worst = rel_close(Cst, C64)
    assert ok, f"C: {nbad} beyond 1e-4 (worst {worst:.3e})"
    rng = np.random.default_rng(5)
    q, t, f = _queries(rng, 48, info["n_entities"], 2 * dim, True)
    got = eng.eval_ranks(q, t, f)
    want = O.eval_ranks("betae", T, q, t, f, dim, consts=Cst)
    assert np.array_equal(got, want)
    # union queries: nearest branch (1..3 branches per query)
    nb = rng.integers(1, 4, size=16)
    units = [rng.uniform(0.05, 4.0, size=(k, 2 * dim)).astype(np.float32) for k in nb]
    got = eng.eval_ranks_multi(units, t[:16], f[:16])
    want = O.eval_ranks_multi("betae", T, units, t[:16], f[:16], dim, consts=Cst)
    assert np.array_equal(got, want)
    # the ranking is by KL: with the f64 table the nearest entity of a query is
    # the argmin of the closed-form KL (checked on a few queries)
    a = O.beta_realize(eng.download("entity")[:, :dim].astype(np.float64))
    b = O.beta_realize(eng.download("entity")[:, dim:].astype(np.float64))
    for i in range(3):
        A, B = q[i, :dim].astype(np.float64), q[i, dim:].astype(np.float64)
        kl = O.beta_kl(a, b, A[None], B[None]).sum(1)
        lin = C64 + T64 @ np.concatenate([A, B])
        assert np.argmin(kl) == np.argmin(lin)


@pytest.mark.parametrize("shape,dim,dl", [("small", 32, 48), ("fb15k-237", 400, 768)])
def test_fusion_ranks(shape, dim, dl):
    g = m.Graph.synthetic(shape, 1)
    info = g.info()
    store = m.semantic_store(info["n_entities"], dl, seed=5)
    eng = m.Engine("gqe", info["n_entities"], info["n_relations"], dim=dim, n_neg=16,
                   max_queries=64, semantic=store)
    _train(eng, g)
    rows, consts = eng.eval_entity_table()
    assert consts is None
    want64 = O.fused_table(eng.download("entity"), store, eng.download("fus_f"),
                           eng.download("fus_wp"), eng.download("fus_bp"))
    ok, nbad, worst = rel_close(rows, want64)
    assert ok, f"fused rows: {nbad} beyond 1e-4 (worst {worst:.3e})"
    rng = np.random.default_rng(6)
    q, t, f = _queries(rng, 48, info["n_entities"], dim, False)
    got = eng.eval_ranks(q, t, f)
    want = O.eval_ranks("gqe", rows, q, t, f, dim)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("dim,dl", [(32, 48), (400, 768)])
def test_betae_psi_fusion_ranks(small_graph, dim, dl):
    # BetaE + FuseSemantic: KL against the Beta parameters Psi_theta makes from
    # the fused rows (Eq. 3)
    info = small_graph.info()
    store = m.semantic_store(info["n_entities"], dl, seed=5)
    eng = m.Engine("betae", info["n_entities"], info["n_relations"], dim=dim, n_neg=16,
                   max_queries=64, semantic=store)
    _train(eng, small_graph)
    T, Cst = eng.eval_entity_table()
    E = O.fused_table(eng.download("entity"), store, eng.download("fus_f"),
                      eng.download("fus_wp"), eng.download("fus_bp"))
    Y = E @ eng.download("fus_psi").astype(np.float64).T + eng.download("fus_psi_b").astype(
        np.float64).reshape(1, -1)
    T64, C64 = O.beta_eval_table(Y, dim)
    ok, nbad, worst = rel_close(T, T64)
    assert ok, f"T: {nbad} beyond 1e-4 (worst {worst:.3e})"
    ok, nbad, worst = rel_close(Cst, C64)
    assert ok, f"C: {nbad} beyond 1e-4 (worst {worst:.3e})"
    rng = np.random.default_rng(7)
    q, t, f = _queries(rng, 48, info["n_entities"], 2 * dim, True)
    assert np.array_equal(eng.eval_ranks(q, t, f), O.eval_ranks("betae", T, q, t, f, dim,
                                                                 consts=Cst))
