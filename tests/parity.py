"""Shared helpers: run the product (GPU) and the oracle (CPU, f64) on identical
seeded inputs and compare with the tolerance the north_star states.

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


def check_all(res, lr=1e-4, allow_frac=1e-3, steps=1):
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


def run_pair(graph, ograph, backbone, mix, b, k, dim, b_max=512, steps=1, seed_tag=0,
             compare_grads=True, certify=True, semantic_dim=0):
    """One or more training steps on both sides; returns a dict of comparisons.
    semantic_dim > 0: FuseSemantic with a synthetic frozen store of that width."""
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
