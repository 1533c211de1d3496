"""The oracle's own correctness (it is the parity reference, so it is checked
first): central finite differences on every gradient,
Alg. 1 scheduling == the sequential per-node executor,
Eq. 7 eager reclamation peak vs end-of-DAG release, and
lazy Adam leaving untouched rows unchanged (SURVEY A-9)."""
import numpy as np
import pytest

import oracle as O
import paper_2602_21597_b200 as m

P = m.PATTERNS


@pytest.fixture(scope="module")
def tiny():
    g = m.Graph.synthetic("tiny", 1)
    return g, g.info()


def _batch(g, mix, b, k, tag=1):
    return m.Batch.sample(g, m.pattern_weights(mix), b, k, seed=3, tag=tag).arrays()


def _loss(om, a):
    return om.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives, adam=-1).sum()


@pytest.mark.parametrize("backbone,dl", [("gqe", 0), ("q2b", 0), ("betae", 0), ("gqe", 8),
                                         ("q2b", 8), ("betae", 8)])
def test_finite_difference_gradients(tiny, backbone, dl):
    g, info = tiny
    d, k = 4, 3
    a = _batch(g, P, 20, k)
    om = O.OracleModel(backbone, info["n_entities"], info["n_relations"], d, k, precision=64)
    if dl:
        om.set_semantic(m.semantic_store(info["n_entities"], dl, seed=5))
    om.init(2)
    _loss(om, a)
    specs = m.param_specs(backbone, info["n_entities"], info["n_relations"], d, dl)
    grads = {n: om.get("g:" + n, (r, c)) for n, r, c, _ in specs}
    rng = np.random.default_rng(1)
    h = 1e-5
    checked = 0
    for name, rows, cols, sparse in specs:
        base = om.get(name, (rows, cols))
        cand = np.argwhere(np.abs(grads[name]) > 1e-3)
        if len(cand) == 0:
            continue
        for idx in cand[rng.choice(len(cand), size=min(6, len(cand)), replace=False)]:
            i, j = int(idx[0]), int(idx[1])
            # params are stored as f32 in the oracle's f64 model via set(); use
            # exact f64 perturbations through a float64 round trip of the tensor
            pert = base.copy()
            pert[i, j] += h
            om.set(name, pert.astype(np.float32))
            lp = _loss(om, a)
            pert[i, j] -= 2 * h
            om.set(name, pert.astype(np.float32))
            lm = _loss(om, a)
            om.set(name, base.astype(np.float32))
            # f32 storage of the perturbed value: use the realised step
            hp = float(np.float32(base[i, j] + h)) - float(np.float32(base[i, j] - h))
            fd = (lp - lm) / hp
            an = grads[name][i, j]
            assert abs(fd - an) <= 2e-3 * max(abs(an), 1e-3), (name, i, j, fd, an)
            checked += 1
    assert checked >= 10


@pytest.mark.parametrize("backbone", ["gqe", "q2b", "betae"])
def test_scheduled_equals_sequential(tiny, backbone):
    g, info = tiny
    a = _batch(g, P, 60, 4)
    res = []
    for executor in (0, 1):
        om = O.OracleModel(backbone, info["n_entities"], info["n_relations"], 8, 4, precision=64)
        om.init(2)
        loss = om.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives,
                       executor=executor, adam=-1)
        specs = m.param_specs(backbone, info["n_entities"], info["n_relations"], 8)
        res.append((loss, {n: om.get("g:" + n, (r, c)) for n, r, c, _ in specs}))
    assert np.max(np.abs(res[0][0] - res[1][0])) < 1e-10
    for n in res[0][1]:
        assert np.max(np.abs(res[0][1][n] - res[1][1][n])) < 1e-10, n


def test_eager_reclamation_peak(small_graph):
    # 3p-heavy batch of 512: eager peak <= 0.6 x end-of-DAG peak
    info = small_graph.info()
    a = _batch(small_graph, ["3p"], 512, 2)
    peaks = []
    for eager in (True, False):
        om = O.OracleModel("gqe", info["n_entities"], info["n_relations"], 8, 2, precision=32)
        om.init(2)
        om.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives, adam=-1, eager=eager)
        peaks.append(om.trace()["peak_bytes"])
    assert peaks[0] <= 0.6 * peaks[1]


def test_lazy_adam_untouched_rows(tiny):
    g, info = tiny
    a = _batch(g, ["1p"], 4, 2)
    om = O.OracleModel("gqe", info["n_entities"], info["n_relations"], 4, 2)
    om.init(2)
    before = om.get("entity", (info["n_entities"], 4))
    om.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives, adam=0)
    after = om.get("entity", (info["n_entities"], 4))
    touched = set(a.anchors[:, 0].tolist()) | set(a.positives.tolist()) | set(
        a.negatives.ravel().tolist())
    for e in range(info["n_entities"]):
        if e not in touched:
            assert (after[e] == before[e]).all()
        else:
            # first Adam step moves each coordinate by at most lr
            assert np.max(np.abs(after[e] - before[e])) <= 1e-4 * 1.0001
