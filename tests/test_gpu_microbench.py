"""operator_microbench and acceptance 6: the
cardinality-class batched Intersect and UnionScore are >= 3x faster than the
per-op loop at n=1024, k=2, d=400, with outputs verified bitwise equal before
timing; n=1 gives a speedup of about 1 (within 50%)."""
import json

import pytest

import paper_2602_21597_b200 as m
from paper_2602_21597_b200.microbench import operator_microbench

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("op,k", [("Intersect", 2), ("UnionScore", 2)])
def test_acceptance_6(small_graph, op, k):
    r = operator_microbench(small_graph, op, n=1024, k=k, dim=400)
    print(json.dumps(r))
    assert r["outputs_equal"]
    assert r["default_split_rel_dev"] <= 1e-6
    assert r["speedup"] >= 3.0, r


@pytest.mark.parametrize("op,k", [("Intersect", 3), ("Project", 1), ("EmbedAnchor", 1)])
def test_other_operators(small_graph, op, k):
    r = operator_microbench(small_graph, op, n=1024, k=k, dim=400)
    print(json.dumps(r))
    assert r["outputs_equal"] and r["speedup"] > 1.0, r


def test_single_node_no_batching_benefit(small_graph):
    r = operator_microbench(small_graph, "Intersect", n=1, k=2, dim=400, reps=9)
    print(json.dumps(r))
    assert r["outputs_equal"] and 0.5 <= r["speedup"] <= 1.5, r
