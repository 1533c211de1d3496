"""The packed device plan's sparse-gradient CSR (built with the radix sort of
include/ngdb/radix.hpp) and the Intersect stash slots, checked on the host
against a direct restatement: entity rows ascending, contribution codes
ascending within a row, every anchor slot and every (score slot, candidate)
pair exactly once under the right entity; relation rows likewise over the
Project slots; every Intersect node a distinct stash slot."""
import numpy as np
import pytest

import paper_2602_21597_b200 as m

ALL = m.engine.PATTERNS


def _arr(ptr, n):
    return np.ctypeslib.as_array(ptr, (max(n, 1),))[:n].copy()


def _expected_entity_pairs(v):
    nc = v.n_candidates
    nodes = _arr(v.nodes, v.n_nodes) if v.n_nodes else None
    cand = _arr(v.candidates, v.n_queries * nc).reshape(v.n_queries, nc)
    pairs = set()
    seen_anchor, seen_score = set(), set()
    for p in range(v.n_pools):
        pool = v.pools[p]
        if pool.dir != 0:
            continue
        for t in range(pool.first, pool.first + pool.count):
            d = v.nodes[t]
            if pool.kind in (0, 1):  # EmbedAnchor / FuseSemantic
                if d.aux not in seen_anchor:
                    seen_anchor.add(d.aux)
                    pairs.add((d.id, -d.aux - 1))
            elif pool.kind in (5, 7) and d.aux >= 0:  # Score / non-union Loss
                if d.aux not in seen_score:
                    seen_score.add(d.aux)
                    for j in range(nc):
                        pairs.add((int(cand[d.id, j]), d.aux * nc + j))
    del nodes
    return pairs


@pytest.mark.parametrize("shape,backbone,mix", [("small", "q2b", ALL), ("small", "gqe", ALL[:5]),
                                                ("small", "betae", ALL), ("nell995", "q2b", ALL)])
def test_entity_and_relation_csr(shape, backbone, mix):
    g = m.Graph.synthetic(shape, 1)
    b = m.Batch.sample(g, m.pattern_weights(mix), 256, 32, seed=3, tag=5)
    st = m.PlannedStep(b, backbone, 32)
    v = st.view()
    n = v.n_entity_rows
    rows = _arr(v.entity_rows, n)
    seg = _arr(v.entity_seg, n + 1)
    con = _arr(v.entity_contrib, int(seg[-1]) if n else 0)
    assert np.all(np.diff(rows) > 0)
    got = set()
    for r in range(n):
        codes = con[seg[r]:seg[r + 1]]
        assert len(codes) > 0 and np.all(np.diff(codes) > 0)
        got.update((int(rows[r]), int(c)) for c in codes)
    assert len(got) == len(con)
    assert got == _expected_entity_pairs(v)
    # relations: one contribution per Project slot, under its relation id
    nr = v.n_relation_rows
    rrows = _arr(v.relation_rows, nr)
    rseg = _arr(v.relation_seg, nr + 1)
    rcon = _arr(v.relation_contrib, int(rseg[-1]) if nr else 0)
    assert np.all(np.diff(rrows) > 0)
    proj = {}
    for p in range(v.n_pools):
        pool = v.pools[p]
        if pool.kind == 2 and pool.dir == 0:
            for t in range(pool.first, pool.first + pool.count):
                proj[v.nodes[t].aux] = v.nodes[t].id
    assert sorted(rcon.tolist()) == sorted(proj)
    for r in range(nr):
        codes = rcon[rseg[r]:rseg[r + 1]]
        assert np.all(np.diff(codes) > 0)
        assert all(proj[int(c)] == rrows[r] for c in codes)


def test_intersect_stash_slots_distinct():
    g = m.Graph.synthetic("small", 1)
    b = m.Batch.sample(g, m.pattern_weights(ALL), 512, 8, seed=3, tag=9)
    v = m.PlannedStep(b, "q2b", 16).view()
    fwd, bwd = {}, {}
    for p in range(v.n_pools):
        pool = v.pools[p]
        if pool.kind != 4:  # Intersect
            continue
        for t in range(pool.first, pool.first + pool.count):
            d = v.nodes[t]
            (fwd if pool.dir == 0 else bwd)[d.aux] = (tuple(d.in_), pool.k)
    assert fwd and len(fwd) == sum(1 for p in range(v.n_pools) for _ in range(
        v.pools[p].count) if v.pools[p].kind == 4 and v.pools[p].dir == 0)
    assert min(fwd) == 0 and max(fwd) == len(fwd) - 1 < 512  # one slot per node, <= 1 per query
    assert fwd == bwd  # the mirror reads the slot its forward wrote
