"""Bit-exact host contract (north_star): sampled indices, DAG order and the
Max-Fillness schedule/trace of the product's host engine equal the oracle's
independent restatement on identical seeds and inputs. Also answer_query vs a
brute-force enumeration over all bindings."""
import itertools

import numpy as np
import pytest

import oracle as O
import paper_2602_21597_b200 as m

P = m.PATTERNS
MIXES = [P, ["1p", "2p", "3p", "2i", "3i"], ["2in", "3in", "inp", "pin", "pni"], ["2u", "up"]]


@pytest.mark.parametrize("mix", range(len(MIXES)))
@pytest.mark.parametrize("tag", [0, 7, 123])
def test_sampled_batches_identical(small_graph, small_oracle_graph, mix, tag):
    w = m.pattern_weights(MIXES[mix])
    a = m.Batch.sample(small_graph, w, 200, 16, seed=3, tag=tag).arrays()
    pat, anc, rel, pos, neg = small_oracle_graph.sample(w, 200, 16, seed=3, tag=tag)
    assert (a.patterns == pat).all()
    assert (a.anchors == anc).all()
    assert (a.relations == rel).all()
    assert (a.positives == pos).all()
    assert (a.negatives == neg).all()


KEYS = ["step", "cycle", "kind", "dir", "batch", "classes", "bytes_reclaimed", "live_bytes",
        "nodes"]


@pytest.mark.parametrize("backbone,dim", [("gqe", 16), ("q2b", 16), ("q2b", 400)])
@pytest.mark.parametrize("b_max", [512, 64, 7])
def test_schedule_trace_identical(small_graph, backbone, dim, b_max):
    info = small_graph.info()
    w = m.pattern_weights(P)
    bt = m.Batch.sample(small_graph, w, 256, 8, seed=3, tag=1)
    a = bt.arrays()
    tr = m.PlannedStep(bt, backbone, dim, b_max).trace(with_nodes=True)
    om = O.OracleModel(backbone, info["n_entities"], info["n_relations"], dim, 8, precision=32)
    om.init(2)
    om.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives, b_max=b_max, adam=-1)
    ot = om.trace(with_nodes=True)
    assert tr["invocations"] == ot["invocations"]
    assert tr["peak_bytes"] == ot["peak_bytes"]
    assert tr["free_list_hits"] == ot["free_list_hits"]
    assert tr["total_nodes"] == ot["total_nodes"]
    assert len(tr["records"]) == len(ot["records"])
    for x, y in zip(tr["records"], ot["records"]):
        assert {k: x[k] for k in KEYS} == {k: y[k] for k in KEYS}


def test_trace_invariants(small_graph):
    bt = m.Batch.sample(small_graph, m.pattern_weights(P), 300, 4, seed=3, tag=2)
    tr = m.PlannedStep(bt, "q2b", 16, 512).trace(with_nodes=True)
    # Σ batch sizes = node count; every node exactly once; pops respect deps
    seen = [n for r in tr["records"] for n in r["nodes"]]
    assert len(seen) == tr["total_nodes"] == len(set(seen))
    assert sum(r["batch"] for r in tr["records"]) == tr["total_nodes"]
    # all intermediates reclaimed at the end (SPEC.md:314 conservation)
    assert tr["records"][-1]["live_bytes"] == 0


def test_initial_params_identical():
    for backbone in ("gqe", "q2b"):
        p = m.init_params(backbone, 50, 5, 12)
        om = O.OracleModel(backbone, 50, 5, 12, 4)
        om.init(2)
        for name, v in p.items():
            assert (om.get(name, v.shape) == v.astype(np.float64)).all(), name


# --- brute-force denotation ------------------------------------

def brute_answer(ne, edges, pattern, a, r):
    adj = set(map(tuple, edges))

    def hop(x, rel, y):
        return (x, rel, y) in adj
    ents = range(ne)
    out = set()
    for y in ents:
        if pattern == "1p":
            ok = hop(a[0], r[0], y)
        elif pattern == "2p":
            ok = any(hop(a[0], r[0], v) and hop(v, r[1], y) for v in ents)
        elif pattern == "3p":
            ok = any(hop(a[0], r[0], v) and hop(v, r[1], u) and hop(u, r[2], y)
                     for v, u in itertools.product(ents, ents))
        elif pattern == "2i":
            ok = hop(a[0], r[0], y) and hop(a[1], r[1], y)
        elif pattern == "3i":
            ok = hop(a[0], r[0], y) and hop(a[1], r[1], y) and hop(a[2], r[2], y)
        elif pattern == "pi":
            ok = any(hop(a[0], r[0], v) and hop(v, r[1], y) for v in ents) and hop(a[1], r[2], y)
        elif pattern == "ip":
            ok = any(hop(a[0], r[0], v) and hop(a[1], r[1], v) and hop(v, r[2], y) for v in ents)
        elif pattern == "2u":
            ok = hop(a[0], r[0], y) or hop(a[1], r[1], y)
        elif pattern == "up":
            ok = any((hop(a[0], r[0], v) or hop(a[1], r[1], v)) and hop(v, r[2], y) for v in ents)
        elif pattern == "2in":
            ok = hop(a[0], r[0], y) and not hop(a[1], r[1], y)
        elif pattern == "3in":
            ok = hop(a[0], r[0], y) and hop(a[1], r[1], y) and not hop(a[2], r[2], y)
        elif pattern == "pin":
            ok = any(hop(a[0], r[0], v) and hop(v, r[1], y) for v in ents) and not hop(a[1], r[2], y)
        elif pattern == "pni":
            ok = hop(a[1], r[2], y) and not any(hop(a[0], r[0], v) and hop(v, r[1], y) for v in ents)
        elif pattern == "inp":
            ok = any(hop(a[0], r[0], v) and not hop(a[1], r[1], v) and hop(v, r[2], y) for v in ents)
        if ok:
            out.add(y)
    return sorted(out)


def test_answer_query_brute_force():
    ne, nr = 20, 3
    rng = np.random.default_rng(0)
    edges = np.unique(np.stack([rng.integers(0, ne, 90), rng.integers(0, nr, 90),
                                rng.integers(0, ne, 90)], 1), axis=0).astype(np.int32)
    g = m.Graph.from_triples(ne, nr, edges)
    og = O.OracleGraph(ne, nr, edges)
    for pi, pattern in enumerate(P):
        na, nrel = m.PATTERN_ARITY[pattern]
        for _ in range(6):
            a = rng.integers(0, ne, na).tolist()
            r = rng.integers(0, nr, nrel).tolist()
            want = brute_answer(ne, edges.tolist(), pattern, a, r)
            assert g.answer(pattern, a, r).tolist() == want, (pattern, a, r)
            assert og.answer(pi, a, r).tolist() == want, (pattern, a, r)


def test_sampled_queries_have_answers(small_graph):
    # SPEC.md:208 validity sweep (desk-scale): the walked answer is an answer
    bt = m.Batch.sample(small_graph, m.pattern_weights(P), 700, 1, seed=3, tag=77).arrays()
    for i in range(700):
        pat = P[bt.patterns[i]]
        na, nrel = m.PATTERN_ARITY[pat]
        ans = small_graph.answer(pat, bt.anchors[i, :na], bt.relations[i, :nrel])
        assert bt.positives[i] in set(ans.tolist())


def test_predictive_answers_partition(small_graph):
    # obs = train-graph answers, miss = full-graph answers not in
    # obs, obs ⊎ miss = full-graph answers — for every sampled query, with the
    # full-graph answers checked against the oracle's independent graph
    info = small_graph.info()
    full = np.concatenate([small_graph.triples(s) for s in (0, 1, 2)])
    og = O.OracleGraph(info["n_entities"], info["n_relations"], full)
    bt = m.Batch.sample(small_graph, m.pattern_weights(P), 300, 1, seed=3, tag=78).arrays()
    n_miss = 0
    for i in range(300):
        pat = P[bt.patterns[i]]
        na, nrel = m.PATTERN_ARITY[pat]
        a, r = bt.anchors[i, :na], bt.relations[i, :nrel]
        obs, miss = small_graph.predictive_answers(pat, a, r)
        assert obs.tolist() == small_graph.answer(pat, a, r).tolist()
        assert not set(obs.tolist()) & set(miss.tolist())
        both = sorted(obs.tolist() + miss.tolist())
        assert both == small_graph.answer(pat, a, r, full=True).tolist()
        assert both == og.answer(int(bt.patterns[i]), a.tolist(), r.tolist()).tolist()
        n_miss += len(miss)
    assert n_miss > 0  # the held-out edges do produce missing answers


def test_sampler_validity_10k_and_scaling(small_graph):
    # SPEC acceptance 8: 10,000 online-sampled queries across all
    # patterns all have non-empty train-graph answer sets (the sampled positive
    # is an answer per the traversal oracle), and batch sampling time scales
    # sub-linearly-bounded: time(2048) / time(512) <= 8
    import time
    bt = m.Batch.sample(small_graph, m.pattern_weights(P), 10000, 1, seed=3, tag=91).arrays()
    assert len(set(bt.patterns.tolist())) == len(P)
    for i in range(10000):
        pat = P[bt.patterns[i]]
        na, nrel = m.PATTERN_ARITY[pat]
        ans = small_graph.answer(pat, bt.anchors[i, :na], bt.relations[i, :nrel])
        assert ans.size > 0 and bt.positives[i] in set(ans.tolist()), i

    def best_of(b, reps=5):
        ts = []
        for r in range(reps):
            t0 = time.perf_counter()
            m.Batch.sample(small_graph, m.pattern_weights(P), b, 128, seed=3, tag=1000 + r)
            ts.append(time.perf_counter() - t0)
        return min(ts)
    ratio = best_of(2048) / best_of(512)
    assert ratio <= 8.0, ratio
