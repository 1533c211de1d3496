"""Operator-level (Max-Fillness) vs query-level baseline executor on the same
sm_100a kernels (SPEC.md:673-681 throughput_bench; the paper's 1.8-6.8x claim,
PAPER.md abstract / §5.2). C2 workload (Q2B, NELL995 shape, 14 patterns, 512
queries, 128 negatives, d = 400); each step a resident plan replayed as a CUDA
graph, device time over K steps (CUDA events on the context stream).
Usage (GPU box): python tools/query_level_bench.py [config] [steps]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2602_21597_b200 as m  # noqa: E402
from paper_2602_21597_b200._native import check, lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
warm = 3
backbone, shape, mix, dim, batch, n_neg = bench.CONFIGS[cfg]
graph = m.Graph.synthetic(shape, 1)
info = graph.info()
batches = bench.make_batches(graph, mix, batch, n_neg, warm + steps, 1)
res = {"config": cfg, "workload": f"{backbone} {shape} {mix} mix, batch {batch}, K {n_neg}, d {dim}"}
for ql in (False, True):
    eng = m.Engine(backbone, info["n_entities"], info["n_relations"], dim=dim, n_neg=n_neg,
                   b_max=512, max_queries=batch, device=0)
    ctx = eng.handle
    pl = [m.PlannedStep(b, backbone, dim, 512, query_level=ql) for b in batches]
    inv = sum(p.trace()["invocations"] for p in pl[warm:]) / steps
    plans = []
    for s in pl:
        v = s.view()
        h = C.c_void_p()
        check(lib.ngdb_plan_create(ctx, C.byref(v), C.byref(h)))
        check(lib.ngdb_plan_prepare(ctx, h))
        plans.append(h)
    step = 0
    for i in range(warm):
        step += 1
        check(lib.ngdb_plan_run(ctx, plans[i], step))
    check(lib.ngdb_sync(ctx))
    l0 = lib.ngdb_launch_count(ctx)
    ms = C.c_float()
    check(lib.ngdb_timer_start(ctx))
    for i in range(steps):
        step += 1
        check(lib.ngdb_plan_run(ctx, plans[warm + i], step))
    check(lib.ngdb_timer_stop(ctx, C.byref(ms)))
    launches = (lib.ngdb_launch_count(ctx) - l0) / steps
    key = "query_level" if ql else "operator_level"
    res[key] = {"ms_per_step": ms.value / steps, "queries_per_s": batch * steps / (ms.value / 1e3),
                "invocations_per_step": inv, "launches_per_step": launches}
    for h in plans:
        check(lib.ngdb_plan_destroy(h))
    del eng
res["speedup"] = res["operator_level"]["queries_per_s"] / res["query_level"]["queries_per_s"]
res["invocation_ratio"] = (res["query_level"]["invocations_per_step"] /
                           res["operator_level"]["invocations_per_step"])
print(json.dumps(res), flush=True)
