"""Shared helpers: run the product (GPU) and the oracle (CPU, f64) on identical
seeded inputs and compare with the tolerance the north_star states.

Two ways to handle kinks (see below): `run_pair` certifies whole queries
(tie_free; small batches), `run_masked` compares every gradient / parameter
element except those the oracle's per-element kink taint marks (full
benchmark-shape batches; allow_frac = 0 on everything compared).

Tolerance: |a - b| <= rtol * max(|b|, s) with s the RMS
of the reference tensor, rtol = 1e-4 for fp32 vs the f64 oracle.

L1 / box distances have sign() in their (sub)gradients. An element whose
coordinate difference |v - q| is within fp32 rounding of zero can take the
other side of the kink in fp32 than in f64; those isolated elements are the
measure-zero ties of SPEC.md:412/433 and are reported, bounded (< 1e-3 of the
elements), and excluded from the elementwise bound.
"""
from __future__ import annotations

import numpy as np

RTOL = 1e-4


def rms(x):
    x = np.asarray(x, dtype=np.float64)
    return float(np.sqrt(np.mean(x * x))) if x.size else 0.0


def rel_close(a, b, rtol=RTOL, allow_frac=0.0, scale=0.0):
    """Elementwise |a-b| <= rtol*max(|b|, s), s = max(rms(b), scale)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    assert a.shape == b.shape, (a.shape, b.shape)
    if b.size == 0:
        return True, 0, 0.0
    s = max(rms(b), scale)
    tol = rtol * np.maximum(np.abs(b), s) + 1e-12
    bad = np.abs(a - b) > tol
    nbad = int(bad.sum())
    worst = float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(b), s), 1e-30)))
    return nbad <= allow_frac * b.size, nbad, worst


def grad_scale(name, grads):
    """Scale floor for a gradient tensor. A bias shares its upstream signal with
    its weight matrix; Q2B's attention bias att_b2 has an identically-zero
    gradient (softmax is shift-invariant over the k inputs), so fp32 leaves
    rounding noise ~1e-7 * |dL/dS| there — judged against dL/dW's scale."""
    if "_b" in name:
        partner = name.replace("_b", "_w")
        if partner in grads:
            return rms(grads[partner][1])
    return 0.0


def weak_mask(name, grads):
    """Elements whose oracle gradient is below the fp32 noise of its tensor."""
    g_ref = grads[name][1]
    noise = 1e-5 * max(rms(g_ref), grad_scale(name, grads))
    return np.abs(g_ref) <= noise


def check_all(res, lr=1e-4, allow_frac=0.0, steps=1):
    """Assert losses, gradients and post-Adam parameters agree (see module doc)."""
    msgs = []
    for loss, ref in res["loss"]:
        ok, nbad, worst = rel_close(loss, ref)
        if not ok:
            msgs.append(f"loss: {nbad} bad, worst rel {worst:.3e}")
    grads = res["grads"]
    for name, (g, r) in grads.items():
        ok, nbad, worst = rel_close(g, r, allow_frac=allow_frac, scale=grad_scale(name, grads))
        if not ok:
            msgs.append(f"grad {name}: {nbad}/{r.size} beyond 1e-4 (worst {worst:.3e})")
    for name, (p, r) in res["params"].items():
        # Adam turns |g| >> eps into -lr*sign(g). Where the oracle gradient is
        # below fp32 noise of its tensor the update direction is not defined by
        # the data; those elements are held to the Adam step bound lr*steps.
        if name in res.get("weak", {}):
            weak = res["weak"][name]  # weak at ANY step of a multi-step run
        elif name in grads:
            weak = weak_mask(name, grads)
        else:
            weak = np.zeros(r.shape, dtype=bool)
        strong = ~weak
        ok, nbad, worst = rel_close(p[strong], r[strong], allow_frac=allow_frac, scale=rms(r))
        if not ok:
            msgs.append(f"param {name}: {nbad}/{strong.sum()} beyond 1e-4 (worst {worst:.3e})")
        if weak.any():
            d = float(np.max(np.abs(p[weak] - r[weak])))
            # each side moves at most lr per step, in either direction
            if d > 2 * lr * steps * 1.0001 + 1e-9:
                msgs.append(f"param {name}: weak-gradient elements differ {d:.3e} > 2*lr*steps")
    assert not msgs, "; ".join(msgs)


TAU = 1e-6  # kink margin certified for gradient parity (>= 25x the fp32 forward error)


def tie_free(batch, om, b_max, step, tau=TAU):
    """Drop the queries whose forward pass comes within tau of a kink (L1/box
    sign, inside/outside, ReLU input, argmin/min routing). At a kink fp32 and
    f64 may legitimately pick different subgradients; away from kinks the
    gradient is a smooth function of the inputs and 1e-4 parity is well posed.
    Returns (filtered batch, kept fraction)."""
    import paper_2602_21597_b200 as m
    a = batch.arrays()
    om.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives, b_max=b_max, step=step,
            adam=-1)  # forward + backward only, no optimizer step
    keep = om.margins(len(a.patterns)) > tau
    if keep.all():
        return batch, 1.0
    sub = m.BatchArrays(a.patterns[keep], a.anchors[keep], a.relations[keep], a.positives[keep],
                        a.negatives[keep])
    return m.Batch.from_arrays(sub), float(keep.mean())


def compare_masked(name, a, b, mask, scale=0.0):
    """|a-b| <= 1e-4*max(|b|, s) on every element outside `mask`, no allowance.
    Returns (ok, n_bad, worst, n_compared, n_live) with n_live = elements whose
    oracle value is nonzero (the ones a step actually produced)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    keep = ~mask
    s = max(rms(b), scale)
    tol = RTOL * np.maximum(np.abs(b), s) + 1e-12
    bad = (np.abs(a - b) > tol) & keep
    live = b != 0
    worst = float(np.max(np.where(keep, np.abs(a - b) / np.maximum(np.maximum(np.abs(b), s), 1e-30),
                                  0.0))) if b.size else 0.0
    return (not bad.any(), int(bad.sum()), worst, int((keep & live).sum()), int(live.sum()))


def kink_mask(ref, dev, scale=0.0, frac=0.1):
    """Elements whose fp32 deviation bound (oracle precision 65, oracle/src/dual.hpp)
    exceeds frac of the 1e-4 tolerance: there a kink resolved the other way in fp32
    could move the value by more than the comparison allows. Everything else must
    match within 1e-4 with the bound's remainder inside the tolerance."""
    s = max(rms(ref), scale)
    return dev > frac * RTOL * np.maximum(np.abs(ref), s)


def run_masked(graph, backbone, mix, b, k, dim, steps=1, b_max=512, seed_tag=0, semantic_dim=0,
               tau=TAU, resync=True, query_level=False, log=print):
    """Benchmark-shape parity with per-element kink masks.

    Every step: the GPU step and the oracle step (f64 values + first-order fp32
    deviation bounds, precision 65) on the same batch; per-query losses compared
    on ALL queries; pre-Adam gradients of every parameter and the post-Adam
    parameters compared element by element with no allowance everywhere
    outside `kink_mask` (a kink within tau of its switch point, where fp32 and
    f64 may legitimately take different subgradients, bounds the element's
    possible deviation above a tenth of the tolerance). Post-Adam parameters
    additionally skip elements whose oracle gradient is below fp32 noise (Adam's
    direction is undefined there; held to the 2*lr step bound instead).

    resync: before steps 2.., the oracle takes the GPU's parameters and Adam
    moments, so every step is compared from an identical state (a masked
    element's +-lr Adam move would otherwise shift later forwards).
    query_level: the GPU runs the query-level baseline executor
    while the oracle runs Alg. 1 — same per-node arithmetic, different order.
    Returns {"compared": fraction of live gradient elements compared, ...}."""
    import oracle as O
    import paper_2602_21597_b200 as m

    info = graph.info()
    ne, nr = info["n_entities"], info["n_relations"]
    w = m.pattern_weights(mix)
    store = m.semantic_store(ne, semantic_dim, seed=5) if semantic_dim else None
    eng = m.Engine(backbone, ne, nr, dim=dim, n_neg=k, b_max=b_max, max_queries=b, debug=True,
                   semantic=store)
    om = O.OracleModel(backbone, ne, nr, dim, k, precision=65)
    if semantic_dim:
        om.set_semantic(store)
    om.init(2)
    om.set_dev_tau(tau)
    specs = m.param_specs(backbone, ne, nr, dim, semantic_dim)
    msgs, compared, live, per = [], 0, 0, {}
    for step in range(1, steps + 1):
        batch = m.Batch.sample(graph, w, b, k, seed=3, tag=seed_tag + step)
        a = batch.arrays()
        if query_level:
            plan = m.PlannedStep(batch, backbone, dim, b_max, semantic=bool(semantic_dim),
                                 query_level=True)
            eng_loss = eng.run_step(plan, b)
        else:
            eng_loss = eng.train_step(batch)
        ref = om.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives, b_max=b_max,
                      step=step)
        ok, nbad, worst = rel_close(eng_loss, ref)
        if not ok:
            msgs.append(f"step {step} loss: {nbad}/{len(ref)} bad, worst rel {worst:.3e}")
        grads = {}
        for name, rows, cols, _ in specs:
            grads[name] = (eng.download("g:" + name), om.get("g:" + name, (rows, cols)))
        for name, rows, cols, _ in specs:
            g, r = grads[name]
            gmask = kink_mask(r, om.dev("g:" + name, (rows, cols)), grad_scale(name, grads))
            ok, nbad, worst, nc, nl = compare_masked(name, g, r, gmask, grad_scale(name, grads))
            compared += nc
            live += nl
            c0, l0 = per.get(name, (0, 0))
            per[name] = (c0 + nc, l0 + nl)
            if not ok:
                msgs.append(f"step {step} grad {name}: {nbad} of {nc} compared beyond 1e-4 "
                            f"(worst {worst:.3e})")
            p, pr = eng.download(name), om.get(name, (rows, cols))
            weak = weak_mask(name, grads)
            pmask = gmask | weak | kink_mask(pr, om.dev(name, (rows, cols)))
            ok, nbad, worst, _, _ = compare_masked(name, p, pr, pmask, rms(pr))
            if not ok:
                msgs.append(f"step {step} param {name}: {nbad} beyond 1e-4 (worst {worst:.3e})")
            wk = weak & ~gmask
            if wk.any():
                d = float(np.max(np.abs(p[wk] - pr[wk])))
                if d > 2 * 1e-4 * 1.0001 + 1e-9:
                    msgs.append(f"step {step} param {name}: weak-gradient elements differ {d:.3e}")
        if resync and step < steps:
            for name, rows, cols, _ in specs:
                for pre in ("", "m:", "v:"):
                    om.set(pre + name, eng.download(pre + name))
    frac = compared / max(live, 1)
    log(f"parity[{backbone} b={b} k={k} d={dim} steps={steps}"
        f"{' query-level' if query_level else ''}]: compared {compared}/{live} live gradient "
        f"elements ({frac:.4f}); per tensor " +
        ", ".join(f"{n} {c / max(l, 1):.3f}" for n, (c, l) in per.items()))
    assert not msgs, "; ".join(msgs)
    return {"compared": frac, "per_tensor": {n: c / max(l, 1) for n, (c, l) in per.items()}}


def run_pair(graph, ograph, backbone, mix, b, k, dim, b_max=512, steps=1, seed_tag=0,
             compare_grads=True, certify=True, semantic_dim=0, query_level=False):
    """One or more training steps on both sides; returns a dict of comparisons.
    semantic_dim > 0: FuseSemantic with a synthetic frozen store of that width.
    query_level: the GPU side runs the query-level baseline executor's plan
     instead of the Max-Fillness one."""
    import oracle as O
    import paper_2602_21597_b200 as m

    info = graph.info()
    ne, nr = info["n_entities"], info["n_relations"]
    w = m.pattern_weights(mix)
    store = m.semantic_store(ne, semantic_dim, seed=5) if semantic_dim else None
    eng = m.Engine(backbone, ne, nr, dim=dim, n_neg=k, b_max=b_max, max_queries=b, debug=True,
                   semantic=store)
    om = O.OracleModel(backbone, ne, nr, dim, k, precision=64)
    if semantic_dim:
        om.set_semantic(store)
    om.init(2)
    specs = m.param_specs(backbone, ne, nr, dim, semantic_dim)
    out = {"loss": [], "grads": {}, "params": {}, "kept": [], "weak": {}}
    for step in range(1, steps + 1):
        batch = m.Batch.sample(graph, w, b, k, seed=3, tag=seed_tag + step)
        if certify:
            batch, kept = tie_free(batch, om, b_max, step)
            out["kept"].append(kept)
        a = batch.arrays()
        if query_level:
            st = m.PlannedStep(batch, backbone, dim, b_max, semantic=bool(semantic_dim),
                               query_level=True)
            loss = eng.run_step(st, len(a.patterns))
        else:
            loss = eng.train_step(batch)
        ref = om.step(a.patterns, a.anchors, a.relations, a.positives, a.negatives, b_max=b_max,
                      step=step)
        out["loss"].append((loss, ref))
        if steps > 1 and step < steps:
            # Adam maps a sub-noise gradient at ANY step to an arbitrary +-lr move
            g = {name: (None, om.get("g:" + name, (rows, cols))) for name, rows, cols, _ in specs}
            for name in g:
                wk = weak_mask(name, g)
                out["weak"][name] = out["weak"].get(name, np.zeros_like(wk)) | wk
    if compare_grads:
        for name, rows, cols, sparse in specs:
            out["grads"][name] = (eng.download("g:" + name), om.get("g:" + name, (rows, cols)))
    if steps > 1:
        g = {name: (None, om.get("g:" + name, (rows, cols))) for name, rows, cols, _ in specs}
        for name in g:
            out["weak"][name] = out["weak"].get(name, np.zeros(g[name][1].shape, bool)) | weak_mask(name, g)
    for name, rows, cols, sparse in specs:
        out["params"][name] = (eng.download(name), om.get(name, (rows, cols)))
    return out
