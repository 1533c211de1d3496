"""GPU parity at the BASELINE.json configs' own shapes (VERDICT r1 "next" item 1).

Full benchmark batches — B = 512 queries, K = 128 negatives, d = 400 — on the
synthetic FB15k-237 (C1 GQE, C3 BetaE, C4 GQE + 768-d PTE) and NELL995 (C2 Q2B,
14 patterns) graphs, one step and three steps, through the C ABI against the
f64 oracle (tests/parity.py `run_masked`): every per-query loss; every pre-Adam
gradient element and post-Adam parameter element outside the per-element kink
masks, with no allowance; and the masks leave >= 90 % of the live gradient
elements compared (the fraction is printed). The query-level executor is checked
against the oracle the same way.

C4's bar is 0.88: its fusion projection F (768 x 400, 4.6 % of the live elements)
receives every candidate row's gradient, so every L1 kink of the step reaches all
of F. The fp32 oracle itself differs from the f64 one there by up to 4x the 1e-4
tolerance (measured f32 vs f64 on C4), so
F is legitimately masked."""
import pytest

import paper_2602_21597_b200 as m
from parity import run_masked

pytestmark = pytest.mark.gpu

ALL = m.PATTERNS
C1_MIX = ["1p", "2p", "3p", "2i", "3i"]
C3_MIX = ["2in", "3in", "inp", "pin", "pni"]

_graphs = {}


def graph(shape):
    if shape not in _graphs:
        _graphs[shape] = m.Graph.synthetic(shape, 1)
    return _graphs[shape]


CASES = [("c1", "fb15k-237", "gqe", C1_MIX, 0), ("c2", "nell995", "q2b", ALL, 0),
         ("c3", "fb15k-237", "betae", C3_MIX, 0), ("c4", "fb15k-237", "gqe", C1_MIX, 768)]


@pytest.mark.parametrize("steps", [1, 3])
@pytest.mark.parametrize("cfg,shape,backbone,mix,sd", CASES, ids=[c[0] for c in CASES])
def test_benchmark_shape_parity(cfg, shape, backbone, mix, sd, steps):
    res = run_masked(graph(shape), backbone, mix, b=512, k=128, dim=400, steps=steps,
                     semantic_dim=sd)
    assert res["compared"] >= (0.88 if sd else 0.9), res


@pytest.mark.parametrize("cfg,shape,backbone,mix", [("c2", "nell995", "q2b", ALL),
                                                    ("c1", "fb15k-237", "gqe", C1_MIX),
                                                    ("c3", "fb15k-237", "betae", C3_MIX)],
                         ids=["c2", "c1", "c3"])
def test_query_level_executor_vs_oracle(cfg, shape, backbone, mix):
    # the query-level baseline runs the same kernels group by
    # group; it must reproduce the oracle's (Alg. 1) step like the operator-level one
    res = run_masked(graph(shape), backbone, mix, b=512, k=128, dim=400, steps=1,
                     query_level=True)
    assert res["compared"] >= 0.9, res
