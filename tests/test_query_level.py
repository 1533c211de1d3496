"""Query-level baseline executor (module `bench`): queries
grouped by pattern, groups executed one after another with their own kernel
invocations, on the same kernels as the operator-level (Max-Fillness) run.
CPU: the SPEC's machine-independent invocation-count claims. GPU: the
query-level step against the CPU oracle (losses, gradients and post-Adam
parameters at the 1e-4 bar, like the operator-level parity tests), and against
the operator-level step."""
import numpy as np
import pytest

import paper_2602_21597_b200 as m

ALL = ["1p", "2p", "3p", "2i", "3i", "pi", "ip", "2u", "up", "2in", "3in", "pin", "pni", "inp"]


def _sub(arrs, idx):
    return m.BatchArrays(arrs.patterns[idx], arrs.anchors[idx], arrs.relations[idx],
                         arrs.positives[idx], arrs.negatives[idx])


def _inv(batch, backbone="q2b", query_level=False, b_max=512):
    return m.PlannedStep(batch, backbone, 16, b_max, query_level=query_level).trace()["invocations"]


def test_homogeneous_batch_same_invocations(small_graph):
    # 512 x 1p: no fragmentation, identical invocation count
    bt = m.Batch.sample(small_graph, m.pattern_weights(["1p"]), 512, 8, seed=3, tag=5)
    assert _inv(bt, query_level=True) == _inv(bt)


@pytest.mark.parametrize("backbone", ["gqe", "q2b", "betae"])
def test_invocations_are_sum_over_pattern_groups(small_graph, backbone):
    # query-level invocations = sum over the pattern groups of the
    # group's own (single-pattern) invocations
    arrs = m.Batch.sample(small_graph, m.pattern_weights(ALL), 14 * 8, 8, seed=3, tag=6).arrays()
    full = m.Batch.from_arrays(arrs)
    want = 0
    for p in np.unique(arrs.patterns):
        want += _inv(m.Batch.from_arrays(_sub(arrs, np.nonzero(arrs.patterns == p)[0])), backbone)
    assert _inv(full, backbone, query_level=True) == want


def test_invocation_ratio_on_uniform_mixture(small_graph):
    # query-level / operator-level invocations >= 3 on the 14-pattern mix
    bt = m.Batch.sample(small_graph, m.pattern_weights(ALL), 512, 8, seed=3, tag=7)
    ql, ol = _inv(bt, query_level=True), _inv(bt)
    assert ql >= 3 * ol, (ql, ol)


@pytest.mark.gpu
@pytest.mark.parametrize("backbone", ["gqe", "q2b", "betae"])
def test_query_level_step_matches_operator_level(small_graph, backbone):
    bt = m.Batch.sample(small_graph, m.pattern_weights(ALL), 128, 16, seed=3, tag=9)
    info = small_graph.info()
    out = []
    for ql in (False, True):
        eng = m.Engine(backbone, info["n_entities"], info["n_relations"], dim=32, n_neg=16,
                       max_queries=128)
        st = m.PlannedStep(bt, backbone, 32, 512, query_level=ql)
        losses = eng.run_step(st, 128)
        out.append((losses, {k: eng.download(k) for k in ("entity", "relation")}))
    (l0, p0), (l1, p1) = out
    np.testing.assert_allclose(l1, l0, rtol=1e-4, atol=1e-5)
    for k in p0:
        scale = max(float(np.sqrt(np.mean(p0[k] ** 2))), 1e-12)
        assert np.max(np.abs(p1[k] - p0[k])) <= 1e-4 * scale, k


@pytest.mark.gpu
@pytest.mark.parametrize("backbone", ["gqe", "q2b", "betae"])
@pytest.mark.parametrize("dim,b,k,steps", [(32, 128, 32, 2), (400, 128, 32, 1)])
def test_query_level_step_matches_oracle(small_graph, small_oracle_graph, backbone, dim, b, k,
                                         steps):
    from parity import check_all, run_pair
    res = run_pair(small_graph, small_oracle_graph, backbone, ALL, b=b, k=k, dim=dim,
                   steps=steps, query_level=True)
    check_all(res, allow_frac=0.0, steps=steps)
