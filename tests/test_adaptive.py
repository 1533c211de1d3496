"""Adaptive sampling (acceptance SPEC.md:753): the product's
DifficultyTracker / update_distribution against the SPEC examples and the
oracle's numpy restatement, and the steered-difficulty property (a pattern
whose loss spikes becomes the most likely pattern within 500 steps)."""
import math

import numpy as np
import pytest

import oracle as O
import paper_2602_21597_b200 as m


def _tracker(ema, obs=None, eta=1.0, floor=0.01):
    t = m.DifficultyTracker(eta=eta, floor=floor)
    t.ema_loss[:] = ema
    t.observations[:] = 1 if obs is None else obs
    return t


def test_spec_update_examples():
    # all ema equal -> uniform
    w = _tracker(np.full(14, 0.7)).distribution()
    np.testing.assert_allclose(w, np.full(14, 1 / 14), rtol=0, atol=1e-15)
    # ema = [1,0,...], eta=1, eps=0 -> w(p1)/w(p2) = e
    e = np.zeros(14)
    e[0] = 1.0
    w = _tracker(e, floor=0.0).distribution()
    assert abs(w[0] / w[1] - math.e) < 1e-12
    # eps=0.01 and one extreme loss -> min weight 0.01 after clipping, sum 1
    e = np.zeros(14)
    e[3] = 50.0
    w = _tracker(e).distribution()
    assert abs(w.min() - 0.01) < 1e-15 and abs(w.sum() - 1) < 1e-12
    assert abs(w[3] - (1 - 13 * 0.01)) < 1e-12


def test_spec_record_examples():
    t = m.DifficultyTracker(decay=0.9)
    t.ema_loss[0], t.observations[0] = 1.0, 1
    t.record(0, 2.0)  # prior 1.0, loss 2.0 -> 1.1
    assert abs(t.ema_loss[0] - 1.1) < 1e-15
    for _ in range(500):  # constant loss c converges to c
        t.record(1, 3.5)
    assert abs(t.ema_loss[1] - 3.5) < 1e-12
    # step response: 95% of the target within ceil(log 0.05 / log decay) updates
    n = math.ceil(math.log(0.05) / math.log(0.9))
    t2 = m.DifficultyTracker(decay=0.9)
    for _ in range(n):
        t2.record(2, 1.0)
    assert t2.ema_loss[2] >= 0.95
    from paper_2602_21597_b200._native import NgdbError
    for bad in (float("nan"), float("inf"), -1.0):  # NonFiniteLoss
        with pytest.raises(NgdbError) as e:
            t2.record(2, bad)
        assert e.value.code == 6 and "NonFiniteLoss" in str(e.value)


def test_cold_start_and_support():
    base = m.pattern_weights(["1p", "2p", "3p", "2i", "3i"])
    t = m.DifficultyTracker()
    t.ema_loss[:5] = [1, 2, 3, 4, 5]
    t.observations[:4] = 1  # 3i never observed -> the base distribution
    np.testing.assert_array_equal(t.distribution(base), base)
    t.observations[4] = 1
    w = t.distribution(base)
    assert (w[5:] == 0).all() and abs(w.sum() - 1) < 1e-12 and (w[:5] >= 0.01).all()
    assert np.argmax(w) == 4


@pytest.mark.parametrize("seed", range(6))
def test_product_matches_oracle(seed):
    rng = np.random.default_rng(seed)
    for _ in range(20):
        ema = rng.uniform(0, 8, 14) * (rng.uniform(size=14) < 0.8)
        obs = rng.integers(0, 3, 14)
        base = rng.uniform(size=14) * (rng.uniform(size=14) < 0.7)
        if base.sum() == 0:
            base[0] = 1
        base /= base.sum()
        eta, floor = rng.uniform(0.2, 3), rng.choice([0.0, 0.01, 0.05])
        got = _tracker(ema, obs, eta, floor).distribution(base)
        want = O.update_distribution(ema, obs, eta, floor, base)
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-15)
    # tracker updates agree bit for bit
    t = m.DifficultyTracker()
    e, o = np.zeros(14), np.zeros(14, np.int64)
    for _ in range(200):
        p, x = int(rng.integers(14)), float(rng.uniform(0, 5))
        t.record(p, x)
        O.record_difficulty(e, o, p, x)
    assert np.array_equal(t.ema_loss, e) and np.array_equal(t.observations, o)


def test_steered_difficulty_spike():
    # acceptance: a pattern whose loss spikes becomes the maximum
    # of pi within 500 steps of the spike. Desk-scale steering:
    # every 1,500 steps one pattern's loss is raised; the tracker records each
    # step's per-pattern mean loss and pi refreshes every 100 steps.
    rng = np.random.default_rng(0)
    base_loss = rng.uniform(0.5, 1.5, 14)
    t = m.DifficultyTracker()
    pi = np.full(14, 1 / 14)
    for spike, p_star in enumerate([5, 11, 2]):
        start = 1500 * (spike + 1)
        losses = base_loss.copy()
        losses[p_star] += 2.0
        became_max = None
        for step in range(start - 1500 if spike == 0 else start, start + 1500):
            cur = losses if step >= start else base_loss
            counts = rng.multinomial(512, pi)
            for p in range(14):
                if counts[p]:
                    t.record(p, float(cur[p] * rng.uniform(0.95, 1.05)))
            if (step + 1) % 100 == 0:
                pi = t.distribution()
            if step >= start and became_max is None and np.argmax(pi) == p_star:
                became_max = step - start
        assert became_max is not None and became_max <= 500, (p_star, became_max)
        base_loss = losses  # the spike persists until the next one
        base_loss[p_star] -= 2.0
