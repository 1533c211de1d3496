"""Known-answer examples from /root/reference/SPEC.md on the training-step
path ([TRIVIAL] / [DERIVED] tags), checked on the product host engine and on
the oracle. Values marked mpmath were recomputed at arbitrary precision
(SURVEY Appendix B)."""
import ctypes as C
import math

import numpy as np
import pytest

import oracle as O
import paper_2602_21597_b200 as m
from paper_2602_21597_b200._native import NgdbError, lib

P = m.PATTERNS


def graph(n_ent, n_rel, triples):
    return m.Graph.from_triples(n_ent, n_rel, np.array(triples, dtype=np.int32))


# --- query model (query.hpp:14-45) -----------------------------

def test_pattern_table():
    assert len(P) == 14
    assert P[:5] == ["1p", "2p", "3p", "2i", "3i"]


@pytest.mark.parametrize("pattern,fwd_nodes", [("1p", 3), ("2p", 4), ("3p", 5), ("2i", 6),
                                               ("3i", 8), ("pi", 7), ("ip", 7), ("2u", 8),
                                               ("up", 10), ("2in", 7), ("3in", 9), ("pin", 8),
                                               ("pni", 8), ("inp", 8)])
def test_training_dag_sizes(pattern, fwd_nodes):
    # 1p -> 3, 3i -> 8 forward nodes; union patterns append a
    # Loss after UnionScore (SURVEY A-1). Gradient mirrors double the count.
    na, nr = m.PATTERN_ARITY[pattern]
    pat = np.array([P.index(pattern)], np.int32)
    anc = np.array([[0, 1, 2][:na] + [-1] * (3 - na)], np.int32)
    rel = np.array([[0, 1, 2][:nr] + [-1] * (4 - nr)], np.int32)
    nodes, nf, _ = O.build_dag(pat, anc, rel)
    assert nf == fwd_nodes and len(nodes) == 2 * fwd_nodes


def test_fuse_counts():
    # fuse {1p, 2i} -> 3 + 8 nodes in eval form; 3 + 6 training fwd
    pat = np.array([0, 3], np.int32)
    anc = np.array([[0, -1, -1], [1, 2, -1]], np.int32)
    rel = np.array([[0, -1, -1, -1], [0, 1, -1, -1]], np.int32)
    nodes, nf, edges = O.build_dag(pat, anc, rel)
    assert nf == 3 + 6 and len(nodes) == 18


def test_jsonl_roundtrip():
    line = ('{"pattern":"2in","anchors":[3,9],"relations":[1,4],'
            '"answers_obs":[5,7],"answers_miss":[]}')
    buf = C.create_string_buffer(512)
    assert lib.ngdb_jsonl_roundtrip(line.encode(), buf, 512) == 0
    assert buf.value.decode() == line
    with pytest.raises(NgdbError):
        from paper_2602_21597_b200._native import check
        check(lib.ngdb_jsonl_roundtrip(b'{"pattern":"2in","anchors":[3],"relations":[1,4]}',
                                       buf, 512))


# --- kg store / answer_query -----------------------------------

def test_neighbors_and_dedup():
    g = graph(3, 2, [[0, 0, 1], [1, 1, 2], [0, 0, 1]])
    assert g.info()["n_train"] == 2          # duplicate triple stored once
    assert g.answer("1p", [0], [0]).tolist() == [1]


def test_id_out_of_range():
    with pytest.raises(NgdbError):
        graph(3, 2, [[0, 0, 3]])


def test_answer_examples():
    a, b, c, d = 0, 1, 2, 3
    g = graph(4, 3, [[a, 1, b], [c, 2, b], [c, 2, d]])
    assert g.answer("1p", [a], [1]).tolist() == [b]
    assert g.answer("2i", [a, c], [1, 2]).tolist() == [b]
    assert g.answer("2in", [a, c], [1, 2]).tolist() == []


# --- sampler --------------------------------------------------

def test_path_graph_2p():
    # a -r1-> b -r2-> c: pattern 2p always yields (a, r1, r2) with answer c
    a, b, c = 0, 1, 2
    g = graph(3, 3, [[a, 1, b], [b, 2, c]])
    bt = m.Batch.sample(g, m.pattern_weights(["2p"]), 16, 1, seed=5)
    arr = bt.arrays()
    assert (arr.anchors[:, 0] == a).all()
    assert (arr.relations[:, :2] == [1, 2]).all()
    assert (arr.positives == c).all()


def test_exhausted_retries():
    # every negated atom covers the only answer -> 2in cannot be instantiated
    g = graph(3, 2, [[0, 0, 2], [1, 1, 2]])
    with pytest.raises(NgdbError, match="attempts|ExhaustedRetries|pattern"):
        m.Batch.sample(g, m.pattern_weights(["2in"]), 1, 1, seed=1)


def test_negatives_exclude_answers(small_graph):
    bt = m.Batch.sample(small_graph, m.pattern_weights(P), 64, 32, seed=3, tag=9)
    a = bt.arrays()
    for i in range(64):
        na, nr = m.PATTERN_ARITY[P[a.patterns[i]]]
        ans = set(small_graph.answer(P[a.patterns[i]], a.anchors[i, :na], a.relations[i, :nr],
                                     full=True).tolist())
        assert a.positives[i] in set(small_graph.answer(P[a.patterns[i]], a.anchors[i, :na],
                                                        a.relations[i, :nr]).tolist())
        assert not (set(a.negatives[i].tolist()) & ans)


def test_no_negatives_available():
    # entity 0 reaches every entity by relation 0: every 1p answer set is all of E
    g = graph(2, 1, [[0, 0, 0], [0, 0, 1]])
    with pytest.raises(NgdbError, match="answers cover all entities"):
        m.Batch.sample(g, m.pattern_weights(["1p"]), 8, 4, seed=1)


# --- scheduler -----------------------------------------------

def _pools(d):
    counts = np.zeros(16, np.int64)
    heads = np.zeros(16, np.int64)
    for k, (cnt, ts) in d.items():
        counts[k] = cnt
        heads[k] = ts
    out = C.c_int32()
    rc = lib.ngdb_select_pool(counts.ctypes.data_as(C.POINTER(C.c_int64)),
                              heads.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(out))
    return rc, out.value


def test_select_pool_argmax():
    # {Project: 300, Intersect: 40, EmbedAnchor: 500} -> EmbedAnchor
    rc, p = _pools({2: (300, 0), 4: (40, 0), 0: (500, 0)})
    assert rc == 0 and p == 0


def test_select_pool_fifo_tie():
    rc, p = _pools({2: (512, 3), 4: (512, 1)})  # equal fill: older head wins
    assert p == 4
    rc, p = _pools({2: (512, 1), 4: (512, 1)})  # then fixed type order
    assert p == 2


def test_select_pool_all_empty():
    rc, _ = _pools({})
    assert rc != 0


def _trace_of(patterns, anchors, relations, b_max=512, k=2, dim=8):
    n = len(patterns)
    arr = m.BatchArrays(np.array(patterns, np.int32), np.array(anchors, np.int32),
                        np.array(relations, np.int32), np.zeros(n, np.int32),
                        np.ones((n, k), np.int32))
    return m.PlannedStep(m.Batch.from_arrays(arr), "gqe", dim, b_max).trace()


def test_single_1p_three_forward_steps():
    tr = _trace_of([0], [[0, -1, -1]], [[0, -1, -1, -1]])
    fwd = [r for r in tr["records"] if r["dir"] == "fwd"]
    assert [r["batch"] for r in fwd] == [1, 1, 1]


def test_512_homogeneous_1p_three_invocations():
    n = 512
    tr = _trace_of([0] * n, [[i % 7, -1, -1] for i in range(n)], [[0, -1, -1, -1]] * n)
    fwd = [r for r in tr["records"] if r["dir"] == "fwd"]
    assert len(fwd) == 3 and all(r["batch"] == 512 for r in fwd)


def test_cardinality_classes():
    # pool {2i, 2i, 3i} -> classes C2 (2 nodes), C3 (1 node): 2 kernel calls
    tr = _trace_of([3, 3, 4], [[0, 1, -1], [2, 3, -1], [4, 5, 6]],
                   [[0, 1, -1, -1], [1, 0, -1, -1], [0, 1, 0, -1]])
    inter = [r for r in tr["records"] if r["kind"] == "Intersect" and r["dir"] == "fwd"]
    assert len(inter) == 1 and inter[0]["classes"] == [[2, 2], [3, 1]]


def test_bmax_drains_consecutively():
    n = 40
    tr = _trace_of([0] * n, [[i, -1, -1] for i in range(n)], [[0, -1, -1, -1]] * n, b_max=16)
    first = tr["records"][:3]
    assert [r["batch"] for r in first] == [16, 16, 8]
    assert len({r["cycle"] for r in first}) == 1  # one selection, three pops


# --- kernels / loss ---------------------------------

def test_q2b_distance_examples():
    assert O.q2b_distance([3.0], [0.0], [1.0], 0.02) == pytest.approx(2.02, abs=1e-15)
    assert O.q2b_distance([0.7, -2.0], [0.7, -2.0], [1.0, 0.3], 0.02) == 0.0


def test_loss_examples():
    # d_pos = d_neg = gamma -> ln 2 per term (positive + mean of negatives)
    assert O.loss(12.0, 12.0, [12.0, 12.0]) == pytest.approx(2 * math.log(2), abs=1e-15)
    # gamma=12, d_pos=2, d_neg=[14,15] -> 0.0878030802075741 (mpmath)
    assert O.loss(12.0, 2.0, [14.0, 15.0]) == pytest.approx(0.0878030802075741, abs=1e-13)


def test_synthetic_shapes():
    for shape, counts in [("tiny", (100, 6, 600, 50, 50)), ("small", (2000, 20, 16000, 1000, 1000))]:
        info = m.Graph.synthetic(shape, 1).info()
        assert (info["n_entities"], info["n_relations"], info["n_train"], info["n_valid"],
                info["n_test"]) == counts


@pytest.mark.slow
def test_benchmark_shape_counts():
    info = m.Graph.synthetic("nell995", 1).info()
    assert (info["n_entities"], info["n_relations"], info["n_train"], info["n_valid"],
            info["n_test"]) == (63361, 200, 114213, 14324, 14267)


# ---- BetaE special functions and KL ----------------------------

def test_special_function_known_answers():
    assert abs(O.lgamma(1.0)) < 1e-12 and abs(O.lgamma(2.0)) < 1e-12
    assert abs(O.digamma(1.0) - (-0.5772156649015329)) < 1e-10
    for x in (0.1, 1.0, 10.0, 100.0):  # recurrence identity
        assert abs(O.digamma(x + 1) - O.digamma(x) - 1.0 / x) < 1e-10
        assert abs(O.trigamma(x) - O.trigamma(x + 1) - 1.0 / (x * x)) < 1e-10 * max(1, 1 / x**2)
    assert math.isnan(O.lgamma(0.0)) and math.isnan(O.digamma(-1.0))


def test_special_functions_vs_scipy():
    sp = pytest.importorskip("scipy.special")
    xs = np.concatenate([np.linspace(0.05, 8, 300), np.logspace(0.5, 6, 100)])
    for x in xs:
        assert abs(O.lgamma(x) - sp.gammaln(x)) < 1e-10 * max(1.0, abs(sp.gammaln(x)))
        assert abs(O.digamma(x) - sp.digamma(x)) < 1e-10 * max(1.0, abs(sp.digamma(x)))
        assert abs(O.trigamma(x) - sp.polygamma(1, x)) < 1e-10 * max(1.0, sp.polygamma(1, x))


def test_beta_kl_examples():
    assert abs(O.beta_kl(1, 1, 1, 1)) < 1e-14
    # mpmath-verified closed form; SPEC.md:394 quotes ~0.1251
    assert abs(O.beta_kl(2, 2, 1, 1) - 0.125092802561388) < 1e-12
    rng = np.random.default_rng(0)
    for a1, b1, a2, b2 in rng.uniform(0.05, 20, size=(50, 4)):
        assert O.beta_kl(a1, b1, a2, b2) >= -1e-12  # KL >= 0



# ---- FuseSemantic and the NGSE store -----

def _fusion_pair(small_graph, backbone, dl, wp=None, store=None):
    info = small_graph.info()
    ne, nr, d, k = info["n_entities"], info["n_relations"], 8, 4
    a = m.Batch.sample(small_graph, m.pattern_weights(["1p", "2p", "2i"]), 24, k, seed=3,
                       tag=1).arrays()
    fused = O.OracleModel(backbone, ne, nr, d, k)
    fused.set_semantic(store if store is not None else m.semantic_store(ne, dl, seed=5))
    fused.init(2)
    if wp is not None:
        fused.set("fus_wp", wp)
    return fused, a, (ne, nr, d, k)


def test_fuse_semantic_identity_block(small_graph):
    # W_p = [I | 0], b_p = 0 -> e_fused = sigma(h): a structural-only model whose
    # entity table is sigma(h) scores identically
    d = 8
    wp = np.concatenate([np.eye(d), np.zeros((d, d))], axis=1).astype(np.float32)
    fused, a, (ne, nr, d, k) = _fusion_pair(small_graph, "gqe", 12, wp=wp)
    lf = fused.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives, adam=-1)
    plain = O.OracleModel("gqe", ne, nr, d, k)
    plain.init(2)
    h = fused.get("entity", (ne, d))
    plain.set("entity", (1.0 / (1.0 + np.exp(-h))).astype(np.float32))
    for n in ("relation", "int_w1", "int_w2"):
        plain.set(n, fused.get(n, (nr, d) if n == "relation" else (d, d)).astype(np.float32))
    lp = plain.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives, adam=-1)
    # sigma(h) is rounded to f32 in the plain model: agreement to f32 resolution
    assert np.max(np.abs(lf - lp) / np.maximum(np.abs(lp), 1e-6)) < 1e-5


def test_fuse_semantic_zero_store_ignores_F(small_graph):
    # zero semantic rows: the result does not depend on F
    info = small_graph.info()
    zero = np.zeros((info["n_entities"], 12), np.float32)
    o1, a, (ne, nr, d, k) = _fusion_pair(small_graph, "gqe", 12, store=zero)
    l1 = o1.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives, adam=-1)
    o2, _, _ = _fusion_pair(small_graph, "gqe", 12, store=zero)
    o2.set("fus_f", np.full((d, 12), 3.0, np.float32))
    l2 = o2.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives, adam=-1)
    assert np.array_equal(l1, l2)
    assert not np.any(o1.get("g:fus_f", (d, 12)))  # dF = dFs^T S = 0 for a zero store


def test_ngse_roundtrip(tmp_path):
    st = m.semantic_store(37, 12, seed=9)
    path = tmp_path / "store.ngse"
    m.ngse_write(path, st)
    raw = path.read_bytes()
    assert raw[:4] == b"NGSE" and int.from_bytes(raw[4:8], "little") == 1
    assert int.from_bytes(raw[8:16], "little") == 37 and int.from_bytes(raw[16:20], "little") == 12
    assert len(raw) == 20 + 37 * 12 * 4
    back = m.ngse_read(path)
    assert back.shape == (37, 12) and np.array_equal(back, st)
    bad = tmp_path / "bad.ngse"
    bad.write_bytes(b"NGSX" + raw[4:])
    with pytest.raises(NgdbError):
        m.ngse_read(bad)


def test_semantic_store_statistics():
    st = m.semantic_store(2000, 768, seed=5)
    assert abs(float(st.std()) - 1 / np.sqrt(768)) < 2e-3 / np.sqrt(768) * 10
