"""operator_microbench (acceptance 6; the paper's
Appendix E.1 per-operator table).

One operator type, n nodes of one cardinality class k, d-wide rows: the SAME
planned invocation is timed as one batched kernel call (ngdb_exec_pool over all
n nodes — what the Max-Fillness scheduler issues) and as a loop of n per-node
calls (one invocation per operator, the unbatched baseline), on the device
stream with CUDA events. Before timing, both paths run with the GEMMs' split-K
fixed to 1 (ngdb_set_gemm_split) so every row's arithmetic is the same in both,
and the outputs are compared bit for bit (the SPEC's "identical to 1e-12"
precheck; at the per-launch split-K the batched GEMMs may sum K in another
order, so the timed default path is additionally held to 1e-6 relative).

The inputs are those of a real planned step: n queries of the operator's
simplest pattern (Intersect k: 2i / 3i, UnionScore: 2u, Project / EmbedAnchor:
1p) sampled from the graph, and every forward pool before the operator's run
once to fill its input slots in the arena.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict

import numpy as np

from ._native import PoolDesc, check, lib
from .engine import OP_KINDS, Batch, Engine, Graph, PlannedStep, pattern_weights

PATTERN_OF = {("Intersect", 2): "2i", ("Intersect", 3): "3i", ("UnionScore", 2): "2u",
              ("Project", 1): "1p", ("EmbedAnchor", 1): "1p"}


def _time(eng: Engine, fn, reps: int, warmup: int) -> float:
    ms = C.c_float()
    for _ in range(warmup):
        fn()
    check(lib.ngdb_sync(eng.handle))
    out = []
    for _ in range(reps):
        check(lib.ngdb_timer_start(eng.handle))
        fn()
        check(lib.ngdb_timer_stop(eng.handle, C.byref(ms)))
        out.append(ms.value)
    return float(np.median(out))


def operator_microbench(graph: Graph, op: str, n: int = 1024, k: int = 2, dim: int = 400,
                        backbone: str = "q2b", n_neg: int = 16, reps: int = 5,
                        warmup: int = 2, seed_tag: int = 77) -> Dict[str, object]:
    """Loop vs batched device time of n `op` nodes (median of `reps` after
    `warmup`), with the outputs of both paths verified equal first."""
    key = (op, k if op in ("Intersect", "UnionScore") else 1)
    if key not in PATTERN_OF:
        raise ValueError(f"operator_microbench: unsupported {op} k={k}")
    if n < 1:
        raise ValueError("operator_microbench: n >= 1")
    info = graph.info()
    eng = Engine(backbone, info["n_entities"], info["n_relations"], dim=dim, n_neg=n_neg,
                 b_max=max(n, 1), max_queries=n)
    batch = Batch.sample(graph, pattern_weights([PATTERN_OF[key]]), n, n_neg, seed=3,
                         tag=seed_tag)
    ps = PlannedStep(batch, backbone, dim, max(n, 1))
    v = ps.view()
    kind = OP_KINDS.index(op)
    pools = [v.pools[i] for i in range(v.n_pools)]
    target = next(i for i, p in enumerate(pools)
                  if p.dir == 0 and p.kind == kind and (op not in ("Intersect", "UnionScore")
                                                        or p.k == k))
    tp = pools[target]
    if tp.count != n:
        raise RuntimeError(f"operator_microbench: {op} pool holds {tp.count} nodes, not {n}")
    h = eng.handle
    check(lib.ngdb_step_begin(h, C.byref(v)))
    for p in pools[:target]:
        if p.dir == 0:
            check(lib.ngdb_exec_pool(h, C.byref(p)))
    check(lib.ngdb_exec_flush(h))
    width = n_neg + 1 if op == "UnionScore" else (dim if backbone == "gqe" else 2 * dim)
    outs = np.array([v.nodes[tp.first + i].out for i in range(n)], dtype=np.int64)
    lo, hi = int(outs.min()), int(outs.max()) + width

    def read():
        buf = np.zeros(hi - lo, dtype=np.float32)
        check(lib.ngdb_read_arena(h, lo, hi - lo, buf.ctypes.data_as(C.POINTER(C.c_float))))
        return np.stack([buf[o - lo:o - lo + width] for o in outs])

    def batched():
        check(lib.ngdb_exec_pool(h, C.byref(tp)))
        check(lib.ngdb_exec_flush(h))

    one = [PoolDesc(tp.kind, tp.dir, tp.k, tp.first + i, 1, tp.cycle) for i in range(n)]

    def loop():
        for p in one:
            check(lib.ngdb_exec_pool(h, C.byref(p)))
        check(lib.ngdb_exec_flush(h))

    try:
        # precheck: identical arithmetic per row (split-K 1), bitwise equal outputs
        check(lib.ngdb_set_gemm_split(1))
        batched()
        a = read()
        loop()
        b = read()
        equal = bool(np.array_equal(a, b))
        if not equal:
            raise AssertionError(f"operator_microbench {op}: loop and batched outputs differ")
    finally:
        check(lib.ngdb_set_gemm_split(0))
    # the default (per-launch split-K) path, timed
    batched()
    c = read()
    scale = max(float(np.sqrt(np.mean(a.astype(np.float64) ** 2))), 1e-30)
    dev = float(np.max(np.abs(c.astype(np.float64) - a)) / scale) if a.size else 0.0
    t_batched = _time(eng, batched, reps, warmup)
    t_loop = _time(eng, loop, reps, warmup)
    losses = np.zeros(n, dtype=np.float32)
    total, bad = C.c_double(), C.c_int32()
    check(lib.ngdb_step_end(h, losses.ctypes.data_as(C.POINTER(C.c_float)), n, C.byref(total),
                            C.byref(bad)))
    return {"op": op, "n": n, "k": k, "d": dim, "backbone": backbone,
            "loop_ms": t_loop, "batched_ms": t_batched, "speedup": t_loop / t_batched,
            "outputs_equal": equal, "default_split_rel_dev": dev,
            "launches": "1 invocation vs n invocations through ngdb_exec_pool"}
