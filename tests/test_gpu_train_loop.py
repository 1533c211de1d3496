"""The producer/consumer trainer loop (ngdb_train_run) runs
exactly the sequential loop: batch i from Rng(seed).fork(first_tag + i),
planned and executed in index order. Per-query losses and the parameters after
the run are bit-identical to sampling + ngdb_train_step step by step, for any
producer count; the first step is also checked against the CPU oracle."""
import numpy as np
import pytest

import paper_2602_21597_b200 as m
from parity import rel_close

pytestmark = pytest.mark.gpu

ALL = m.engine.PATTERNS


def _engine(graph, backbone, dim, k, b):
    info = graph.info()
    return m.Engine(backbone, info["n_entities"], info["n_relations"], dim=dim, n_neg=k,
                    max_queries=b)


@pytest.mark.parametrize("backbone", ["gqe", "q2b", "betae"])
@pytest.mark.parametrize("producers", [1, 3])
def test_loop_matches_sequential(small_graph, backbone, producers):
    b, k, dim, steps = 128, 16, 32, 5
    w = m.pattern_weights(ALL)
    seq = _engine(small_graph, backbone, dim, k, b)
    ref = []
    for i in range(steps):
        batch = m.Batch.sample(small_graph, w, b, k, seed=3, tag=7 + i)
        ref.append(seq.train_step(batch))
    loop = _engine(small_graph, backbone, dim, k, b)
    sums, pq = loop.train(small_graph, w, steps, batch=b, n_neg=k, seed=3, first_tag=7,
                          n_producers=producers, queue_depth=2, per_query=True)
    for i in range(steps):
        np.testing.assert_array_equal(pq[i], ref[i])
        assert sums[i] == pytest.approx(float(np.sum(ref[i], dtype=np.float64)), rel=1e-12)
    for name in ("entity", "relation"):
        np.testing.assert_array_equal(loop.download(name), seq.download(name))
    assert loop.step_count == seq.step_count == steps


def test_loop_continues_step_numbering(small_graph):
    # two runs of 2 + 3 steps == one run of 5 (Adam bias correction uses the global step)
    b, k, dim = 64, 8, 16
    w = m.pattern_weights(ALL)
    one = _engine(small_graph, "q2b", dim, k, b)
    s1 = one.train(small_graph, w, 5, batch=b, n_neg=k, first_tag=0, n_producers=2)
    two = _engine(small_graph, "q2b", dim, k, b)
    s2 = np.concatenate([two.train(small_graph, w, 2, batch=b, n_neg=k, first_tag=0),
                         two.train(small_graph, w, 3, batch=b, n_neg=k, first_tag=2)])
    np.testing.assert_array_equal(s1, s2)
    np.testing.assert_array_equal(one.download("entity"), two.download("entity"))


def test_loop_first_step_vs_oracle(small_graph, small_oracle_graph):
    import oracle as O
    b, k, dim = 128, 16, 32
    info = small_graph.info()
    w = m.pattern_weights(ALL)
    eng = _engine(small_graph, "q2b", dim, k, b)
    _, pq = eng.train(small_graph, w, 1, batch=b, n_neg=k, seed=3, first_tag=11, per_query=True)
    a = m.Batch.sample(small_graph, w, b, k, seed=3, tag=11).arrays()
    om = O.OracleModel("q2b", info["n_entities"], info["n_relations"], dim, k, precision=64)
    om.init(2)
    ref = om.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives, b_max=512, step=1)
    ok, nbad, worst = rel_close(pq[0], np.asarray(ref))
    assert ok, f"{nbad} bad, worst {worst:.3e}"


def test_loop_errors_surface(small_graph):
    b, k, dim = 32, 8, 16
    eng = _engine(small_graph, "gqe", dim, k, b)
    w = m.pattern_weights(ALL)
    from paper_2602_21597_b200._native import NgdbError
    with pytest.raises(NgdbError) as e:  # n_neg differs from the context's
        eng.train(small_graph, w, 2, batch=b, n_neg=k + 1)
    assert e.value.kind == "ShapeMismatch"
    # a failed run leaves the context usable
    sums = eng.train(small_graph, w, 2, batch=b, n_neg=k)
    assert np.all(np.isfinite(sums))


@pytest.mark.parametrize("in_flight,graphs", [(1, True), (3, True), (2, False)])
def test_loop_depth_and_launch_mode(small_graph, in_flight, graphs):
    # ngdb_train_opts.in_flight / NGDB_TRAIN_NO_GRAPHS change only how far the
    # host runs ahead and how steps are launched: results stay bit-identical
    b, k, dim, steps = 96, 8, 32, 4
    w = m.pattern_weights(ALL)
    base = _engine(small_graph, "q2b", dim, k, b)
    ref = base.train(small_graph, w, steps, batch=b, n_neg=k, seed=3, first_tag=21,
                     n_producers=2, per_query=True)[1]
    eng = _engine(small_graph, "q2b", dim, k, b)
    pq = eng.train(small_graph, w, steps, batch=b, n_neg=k, seed=3, first_tag=21, n_producers=2,
                   per_query=True, in_flight=in_flight, graphs=graphs)[1]
    np.testing.assert_array_equal(pq, ref)
    for name in ("entity", "relation"):
        np.testing.assert_array_equal(eng.download(name), base.download(name))


@pytest.mark.parametrize("producers", [1, 3])
def test_adaptive_feedback_loop(small_graph, tmp_path, producers):
    # ngdb_train_run_ex with adaptive pi, the metrics
    # log and the checkpoint cadence: every
    # batch is the sampler's batch under the pi in force at its refresh, pi
    # follows the oracle's restatement of the tracker over the returned
    # per-query losses, and runs do not depend on the producer count
    import json

    import oracle as O
    b, k, dim, steps, R = 96, 16, 32, 30, 10
    w = m.pattern_weights(ALL)
    eng = _engine(small_graph, "q2b", dim, k, b)
    tr = m.DifficultyTracker()
    ck = tmp_path / "run.ngck"
    sums, pq, pis = eng.train(small_graph, w, steps, batch=b, n_neg=k, seed=3, first_tag=100,
                              n_producers=producers, per_query=True, adaptive=True,
                              refresh_every=R, tracker=tr, metrics_path=str(tmp_path / "m.jsonl"),
                              checkpoint_path=str(ck), checkpoint_every=12, pi_per_step=True)
    ema, obs = np.zeros(14), np.zeros(14, np.int64)
    pi = w.copy()
    for i in range(steps):
        if i and i % R == 0:
            pi = O.update_distribution(ema, obs, 1.0, 0.01, w)
        np.testing.assert_allclose(pis[i], pi, rtol=1e-12, atol=1e-15)
        pats = m.Batch.sample(small_graph, pis[i], b, k, seed=3, tag=100 + i).arrays().patterns
        for p, x in O.batch_pattern_losses(pats, pq[i]):
            O.record_difficulty(ema, obs, p, x)
    assert not np.allclose(pis[-1], w)  # pi moved away from uniform
    np.testing.assert_allclose(tr.ema_loss, ema, rtol=1e-12)
    assert np.array_equal(tr.observations, obs)
    # metrics log: one record per step
    recs = [json.loads(x) for x in (tmp_path / "m.jsonl").read_text().splitlines()]
    assert [r["step"] for r in recs] == list(range(1, steps + 1))
    assert all(r["queries_per_s"] > 0 and r["peak_bytes"] > 0 for r in recs)
    np.testing.assert_allclose([r["loss"] for r in recs], sums, rtol=1e-15)
    # checkpoint cadence 12 -> the last blob holds step 24; resuming it and
    # replaying steps 25..30 with the recorded pi reproduces the run
    res = _engine(small_graph, "q2b", dim, k, b)
    assert res.load_checkpoint(str(ck)) == 24
    for i in range(24, steps):
        res.train_step(m.Batch.sample(small_graph, pis[i], b, k, seed=3, tag=100 + i))
    for name in ("entity", "relation"):
        np.testing.assert_array_equal(res.download(name), eng.download(name))
    # producer-count independence
    other = _engine(small_graph, "q2b", dim, k, b)
    s2 = other.train(small_graph, w, steps, batch=b, n_neg=k, seed=3, first_tag=100,
                     n_producers=4 - producers, adaptive=True, refresh_every=R)
    np.testing.assert_array_equal(s2, sums)


@pytest.mark.parametrize("backbone,mix", [("q2b", ALL), ("betae", ALL), ("gqe", ALL)])
def test_concurrent_pools_match_serial(small_graph, monkeypatch, backbone, mix):
    # resident plans replayed as graphs whose independent pools run on side
    # streams (planner dependencies) update the parameters exactly as the
    # serial pool order does (NGDB_SERIAL_POOLS=1)
    import ctypes as C

    from paper_2602_21597_b200._native import check, lib
    b, k, dim = 128, 16, 32
    w = m.pattern_weights(mix)
    steps = [m.PlannedStep(m.Batch.sample(small_graph, w, b, k, seed=3, tag=50 + i), backbone,
                           dim, 512) for i in range(4)]
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("NGDB_SERIAL_POOLS", mode)
        eng = _engine(small_graph, backbone, dim, k, b)
        plans = []
        for st in steps:
            v = st.view()
            assert v.pool_dep_off  # the planner ships dependencies
            h = C.c_void_p()
            check(lib.ngdb_plan_create(eng.handle, C.byref(v), C.byref(h)))
            check(lib.ngdb_plan_prepare(eng.handle, h))
            plans.append(h)
        for i, h in enumerate(plans):
            check(lib.ngdb_plan_run(eng.handle, h, i + 1))
        check(lib.ngdb_sync(eng.handle))
        info = small_graph.info()
        out[mode] = {n: eng.download(n) for n, *_ in m.param_specs(
            backbone, info["n_entities"], info["n_relations"], dim)}
        for h in plans:
            check(lib.ngdb_plan_destroy(h))
    for name in out["1"]:
        np.testing.assert_array_equal(out["0"][name], out["1"][name])


def test_seeded_runs_are_bitwise_reproducible(small_graph, tmp_path):
    # SPEC acceptance 11: identical seed + single-threaded mode
    # (one producer) -> bitwise-identical checkpoints and metrics logs across
    # two runs (the log's wall-clock throughput field excluded: it is a timing)
    import json
    b, k, dim, steps = 96, 16, 32, 12
    w = m.pattern_weights(ALL)
    logs, blobs = [], []
    for run in range(2):
        eng = _engine(small_graph, "q2b", dim, k, b)
        ck, ml = tmp_path / f"run{run}.ngck", tmp_path / f"m{run}.jsonl"
        eng.train(small_graph, w, steps, batch=b, n_neg=k, seed=3, first_tag=500, n_producers=1,
                  adaptive=True, refresh_every=5, metrics_path=str(ml), checkpoint_path=str(ck),
                  checkpoint_every=steps)
        blobs.append(ck.read_bytes())
        recs = [json.loads(x) for x in ml.read_text().splitlines()]
        for r in recs:
            r.pop("queries_per_s")
        logs.append(json.dumps(recs, sort_keys=True))
    assert blobs[0] == blobs[1]
    assert logs[0] == logs[1]


def test_steady_state_window(small_graph):
    # steady_from = W: the loop times steps W..n-1 itself (the bench's e2e);
    # the window is positive and shorter than the whole call, and the run's
    # results do not depend on it
    import time
    b, k, dim, steps = 64, 16, 32, 20
    w = m.pattern_weights(ALL)
    eng = _engine(small_graph, "q2b", dim, k, b)
    t0 = time.perf_counter()
    sums = eng.train(small_graph, w, steps, batch=b, n_neg=k, seed=3, first_tag=900,
                     steady_from=5)
    whole = time.perf_counter() - t0
    win = eng.last_timings["steady_s"]
    assert 0.0 < win < whole
    other = _engine(small_graph, "q2b", dim, k, b)
    s2 = other.train(small_graph, w, steps, batch=b, n_neg=k, seed=3, first_tag=900)
    np.testing.assert_array_equal(sums, s2)
    assert other.last_timings["steady_s"] == 0.0  # not requested
