"""Bit-exact host contract at the BASELINE.json KG shapes (north_star: "sampled
indices, operator grouping and schedule, DAG order bit-exact"): on the
synthetic FB15k-237, NELL995 and ogbl-wikikg2-shaped graphs, full 512-query /
128-negative batches of each config's mix sample identically in the product and
the oracle, and the Max-Fillness trace of the planned step (pops, cardinality
classes, node ids, reclaimed / live / peak bytes, free-list hits) is identical."""
import numpy as np
import pytest

import oracle as O
import paper_2602_21597_b200 as m

ALL = m.PATTERNS
C1_MIX = ["1p", "2p", "3p", "2i", "3i"]
C3_MIX = ["2in", "3in", "inp", "pin", "pni"]
KEYS = ["step", "cycle", "kind", "dir", "batch", "classes", "bytes_reclaimed", "live_bytes",
        "nodes"]

# (config, shape, backbone, mix, dim used for the trace's byte counts)
CONFIGS = [("c1", "fb15k-237", "gqe", C1_MIX, 400), ("c2", "nell995", "q2b", ALL, 400),
           ("c3", "fb15k-237", "betae", C3_MIX, 400), ("c5", "wikikg2", "q2b", ALL, 8)]

_graphs = {}


def graphs(shape):
    # wikikg2: ~25 s (product) + ~50 s / 13 GB (oracle's set-based KG) to build
    if shape not in _graphs:
        _graphs.clear()
        g = m.Graph.synthetic(shape, 1)
        info = g.info()
        og = O.OracleGraph(info["n_entities"], info["n_relations"], g.triples(0), g.triples(1),
                           g.triples(2))
        _graphs[shape] = (g, og)
    return _graphs[shape]


@pytest.mark.slow
@pytest.mark.parametrize("cfg,shape,backbone,mix,dim", CONFIGS, ids=[c[0] for c in CONFIGS])
def test_benchmark_shape_batches_and_trace(cfg, shape, backbone, mix, dim):
    g, og = graphs(shape)
    info = g.info()
    w = m.pattern_weights(mix)
    for tag in (1, 2, 17):
        bt = m.Batch.sample(g, w, 512, 128, seed=3, tag=tag)
        a = bt.arrays()
        pat, anc, rel, pos, neg = og.sample(w, 512, 128, seed=3, tag=tag)
        for x, y in ((a.patterns, pat), (a.anchors, anc), (a.relations, rel), (a.positives, pos),
                     (a.negatives, neg)):
            assert np.array_equal(x, y), (cfg, tag)
    # schedule of the last batch: product planner vs the oracle's literal Alg. 1
    tr = m.PlannedStep(bt, backbone, dim, 512).trace(with_nodes=True)
    om = O.OracleModel(backbone, info["n_entities"], info["n_relations"], dim, 128, precision=32)
    om.init(2)
    om.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives, b_max=512, adam=-1)
    ot = om.trace(with_nodes=True)
    for key in ("invocations", "peak_bytes", "free_list_hits", "total_nodes"):
        assert tr[key] == ot[key], (cfg, key)
    assert len(tr["records"]) == len(ot["records"])
    for x, y in zip(tr["records"], ot["records"]):
        assert {k: x[k] for k in KEYS} == {k: y[k] for k in KEYS}
