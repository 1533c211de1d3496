"""The per-element kink masks of tests/parity.py, validated without a GPU.

An independent fp32 execution (the oracle's own f32 mode: the same formulas in
fp32 rounding) against the f64 oracle's deviation-bound mode (precision 65,
oracle/src/dual.hpp) on full 512-query, 128-negative batches of the benchmark
KG shapes. Every gradient and post-Adam parameter element outside the mask must
agree within 1e-4 (no allowance); every element that differs by more than the
tolerance must be explained by its deviation bound; and the mask must leave
>= 90 % of the live gradient elements compared — the bar the GPU tests hold
(test_gpu_parity_shapes.py)."""
import numpy as np
import pytest

import oracle as O
import paper_2602_21597_b200 as m
from parity import RTOL, TAU, compare_masked, grad_scale, kink_mask, rel_close, rms, weak_mask

ALL = m.PATTERNS
C1_MIX = ["1p", "2p", "3p", "2i", "3i"]
C3_MIX = ["2in", "3in", "inp", "pin", "pni"]


@pytest.fixture(scope="module")
def fb15k():
    return m.Graph.synthetic("fb15k-237", 1)


@pytest.mark.parametrize("backbone,mix,dim", [("gqe", C1_MIX, 64), ("q2b", ALL, 64),
                                              ("betae", C3_MIX, 16)])
def test_f32_execution_matches_f64_outside_masks(fb15k, backbone, mix, dim):
    info = fb15k.info()
    ne, nr = info["n_entities"], info["n_relations"]
    a = m.Batch.sample(fb15k, m.pattern_weights(mix), 512, 128, seed=3, tag=1).arrays()
    sides = []
    for prec in (32, 65):
        om = O.OracleModel(backbone, ne, nr, dim, 128, precision=prec)
        om.init(2)
        if prec == 65:
            om.set_dev_tau(TAU)
        sides.append((om, om.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives)))
    (o32, l32), (odv, ldv) = sides
    ok, nbad, worst = rel_close(l32, ldv)
    assert ok, f"loss {nbad} bad, worst {worst:.3e}"
    specs = m.param_specs(backbone, ne, nr, dim)
    grads = {n: (o32.get("g:" + n, (r, c)), odv.get("g:" + n, (r, c))) for n, r, c, _ in specs}
    compared = live = 0
    for n, r, c, _ in specs:
        g32, g64 = grads[n]
        dev = odv.dev("g:" + n, (r, c))
        sc = grad_scale(n, grads)
        mask = kink_mask(g64, dev, sc)
        ok, nbad, worst, nc, nl = compare_masked(n, g32, g64, mask, sc)
        assert ok, f"grad {n}: {nbad} of {nc} beyond 1e-4 (worst {worst:.3e})"
        compared, live = compared + nc, live + nl
        # soundness: whatever differs beyond the tolerance is covered by its bound
        tol = RTOL * np.maximum(np.abs(g64), max(rms(g64), sc))
        err = np.abs(g32 - g64)
        assert np.all((err <= tol) | (err <= dev + tol)), f"grad {n}: deviation beyond its bound"
        p32, p64 = o32.get(n, (r, c)), odv.get(n, (r, c))
        pmask = mask | weak_mask(n, grads) | kink_mask(p64, odv.dev(n, (r, c)))
        ok, nbad, worst, _, _ = compare_masked(n, p32, p64, pmask, rms(p64))
        assert ok, f"param {n}: {nbad} beyond 1e-4 (worst {worst:.3e})"
    assert compared / live >= 0.9, f"only {compared}/{live} live gradient elements compared"


def test_deviation_mode_values_equal_f64(small_graph):
    info = small_graph.info()
    a = m.Batch.sample(small_graph, m.pattern_weights(ALL), 96, 8, seed=3, tag=2).arrays()
    out = []
    for prec in (64, 65):
        om = O.OracleModel("q2b", info["n_entities"], info["n_relations"], 16, 8, precision=prec)
        om.init(2)
        if prec == 65:
            om.set_dev_tau(TAU)
        out.append((om, om.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives)))
    assert np.array_equal(out[0][1], out[1][1])
    for n, r, c, _ in m.param_specs("q2b", info["n_entities"], info["n_relations"], 16):
        for pre in ("", "g:", "m:", "v:"):
            assert np.array_equal(out[0][0].get(pre + n, (r, c)), out[1][0].get(pre + n, (r, c)))


def test_deviation_bounds_zero_without_kinks(small_graph):
    # tau = 0: no kink injects a bound -> every deviation is exactly zero
    info = small_graph.info()
    a = m.Batch.sample(small_graph, m.pattern_weights(ALL), 64, 8, seed=3, tag=3).arrays()
    om = O.OracleModel("q2b", info["n_entities"], info["n_relations"], 16, 8, precision=65)
    om.init(2)
    om.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives)
    for n, r, c, _ in m.param_specs("q2b", info["n_entities"], info["n_relations"], 16):
        assert not om.dev("g:" + n, (r, c)).any()
    # a huge tau makes every kink a source: the MLP weights get nonzero bounds
    om.set_dev_tau(1e300)
    om.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives, step=2)
    assert om.dev("g:att_w1", (16, 16)).all()
