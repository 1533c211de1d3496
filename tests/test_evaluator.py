"""Evaluator hot path: filtered_rank / MRR known answers on
the CPU oracle, and the sm_100a full-entity ranking (ngdb_eval_ranks) against it
on the GPU — bit-exact integer ranks (the oracle reproduces the kernel's
sequential fp32 distance sums, so even exact ties agree)."""
import numpy as np
import pytest

import oracle
from paper_2602_21597_b200 import rank_metrics


# ---- CPU: the oracle against the SPEC's examples ------------------------------
def test_spec_rank_examples():
    assert oracle.filtered_rank([1.0, 9.0, 3.0], 1, []) == 1  # strictly best
    # scores [5,4,3,2], target idx 2, filter {0}: competitors {1,3}, one above -> 2
    assert oracle.filtered_rank([5.0, 4.0, 3.0, 2.0], 2, [0]) == 2
    with pytest.raises(oracle.TargetFiltered):
        oracle.filtered_rank([1.0, 2.0], 0, [0])


def test_mean_rank_ties():
    # 4 equal competitors: rank 1 + 0 + floor(4/2) = 3; filtering two of them -> 2
    s = [1.0, 1.0, 1.0, 1.0, 1.0, 0.0]
    assert oracle.filtered_rank(s, 0, []) == 3
    assert oracle.filtered_rank(s, 0, [1, 2]) == 2


def test_spec_mrr_example():
    m = rank_metrics([1, 2, 4])  # MRR = (1 + 0.5 + 0.25)/3
    assert abs(m["mrr"] - 0.5833333333) < 1e-9
    assert m["hits@1"] <= m["hits@3"] <= m["hits@10"]


def test_rank_vs_full_sort_oracle():
    rng = np.random.default_rng(7)
    for _ in range(50):  # 50 random score vectors
        s = rng.integers(0, 6, size=40).astype(np.float64)  # many ties
        t = int(rng.integers(0, 40))
        f = [int(x) for x in rng.choice(40, size=8, replace=False) if x != t]
        assert oracle.filtered_rank(s, t, f) == oracle.filtered_rank_sorted(s, t, f)


def test_filter_monotonicity():
    rng = np.random.default_rng(8)
    s = rng.integers(0, 10, size=60).astype(np.float64)
    t = 3
    f1 = [5, 9]
    f2 = f1 + [11, 20, 33]
    assert oracle.filtered_rank(s, t, f2) <= oracle.filtered_rank(s, t, f1)


# ---- GPU: ngdb_eval_ranks vs the oracle ------------------------------------------
def _case(backbone, n_ent, dim, nq, seed, integer=False, n_filter=12):
    import paper_2602_21597_b200 as m
    rng = np.random.default_rng(seed)
    eng = m.Engine(backbone, n_ent, 8, dim=dim, n_neg=4, max_queries=64)
    ent = eng.download("entity")
    if integer:  # small integers: exact distances, many exact ties
        ent = rng.integers(-2, 3, size=ent.shape).astype(np.float32)
        eng.upload("entity", ent)
    wq = dim if backbone == "gqe" else 2 * dim
    if integer:
        q = rng.integers(-2, 3, size=(nq, wq)).astype(np.float32)
        if backbone == "q2b":
            q[:, dim:] = np.abs(q[:, dim:])
    else:
        q = rng.uniform(-0.04, 0.04, size=(nq, wq)).astype(np.float32)
        if backbone == "q2b":
            q[:, dim:] = np.abs(q[:, dim:])
    targets = rng.integers(0, n_ent, size=nq).astype(np.int32)
    filters = []
    for i in range(nq):
        f = [int(x) for x in rng.integers(0, n_ent, size=n_filter) if x != targets[i]]
        filters.append(f + f[:2])  # duplicates are ignored (sets)
    return eng, ent, q, targets, filters


@pytest.mark.gpu
@pytest.mark.parametrize("backbone", ["gqe", "q2b"])
@pytest.mark.parametrize("dim,integer", [(40, False), (400, False), (36, True), (400, True)])
def test_gpu_ranks_match_oracle(backbone, dim, integer):
    eng, ent, q, t, f = _case(backbone, 1000, dim, 70, seed=dim + integer, integer=integer)
    got = eng.eval_ranks(q, t, f)
    want = oracle.eval_ranks(backbone, ent, q, t, f, dim)
    np.testing.assert_array_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("backbone", ["gqe", "q2b"])
def test_gpu_ranks_full_size(backbone):
    # NELL995 entity count, d = 400 (C2 shape)
    eng, ent, q, t, f = _case(backbone, 63361, 400, 40, seed=11, n_filter=200)
    got = eng.eval_ranks(q, t, f)
    want = oracle.eval_ranks(backbone, ent, q, t, f, 400)
    np.testing.assert_array_equal(got, want)


@pytest.mark.gpu
def test_gpu_rank_edge_cases():
    import paper_2602_21597_b200 as m
    from paper_2602_21597_b200._native import NgdbError
    eng, ent, q, t, f = _case("gqe", 300, 16, 5, seed=3)
    assert eng.eval_ranks(q[:0], t[:0], []).shape == (0,)
    # a query equal to its target's row: distance 0, rank 1 unless other rows tie at 0
    q2 = ent[t[:1], :16].copy()
    r = eng.eval_ranks(q2, t[:1], [[]])
    assert r[0] == oracle.eval_ranks("gqe", ent, q2, t[:1], [[]], 16)[0]
    with pytest.raises(NgdbError) as e:  # SPEC TargetFiltered
        eng.eval_ranks(q[:1], t[:1], [[int(t[0])]])
    assert e.value.kind == "DomainError"
    with pytest.raises(NgdbError) as e:
        eng.eval_ranks(q[:1], np.array([300], dtype=np.int32), [[]])
    assert e.value.kind == "IndexOutOfRange"
    # a non-positive Beta query parameter is accepted (no finiteness check on
    # queries): only shape / index errors are raised


def test_beta_linearised_kl_matches_closed_form():
    # DESIGN.md §3.5 / §3.7: KL(Beta(a,b) || Beta(A,B)) summed over the dims =
    # lnB(q) + C_e + <q, T_e> with the entity side of oracle.beta_eval_table
    from scipy.special import betaln
    rng = np.random.default_rng(3)
    d = 16
    raw = rng.normal(0, 2, size=(20, 2 * d))
    T, C = oracle.beta_eval_table(raw, d)
    a, b = oracle.beta_realize(raw[:, :d]), oracle.beta_realize(raw[:, d:])
    for _ in range(5):
        A, B = rng.uniform(0.05, 6, d), rng.uniform(0.05, 6, d)
        kl = oracle.beta_kl(a, b, A[None], B[None]).sum(1)
        lin = betaln(A, B).sum() + C + T @ np.concatenate([A, B])
        np.testing.assert_allclose(lin, kl, rtol=1e-10, atol=1e-10)
    # KL(Beta(2,2) || Beta(1,1)) = 0.125092802561388
    assert abs(oracle.beta_kl(2.0, 2.0, 1.0, 1.0) - 0.125092802561388) < 1e-12
