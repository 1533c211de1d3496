"""e2e trainer-loop sweep (GPU box): C2 q/s for in-flight depth x step graphs x producers.
Usage: python tools/e2e_sweep.py [steps]"""
import itertools
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import bench  # noqa: E402
from paper_2602_21597_b200._native import check, lib  # noqa: E402
import paper_2602_21597_b200 as m  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
backbone, shape, mix, dim, batch, n_neg = bench.CONFIGS["c2"]
graph = m.Graph.synthetic(shape, 1)
info = graph.info()
eng = m.Engine(backbone, info["n_entities"], info["n_relations"], dim=dim, n_neg=n_neg,
               b_max=512, max_queries=batch, device=0)
w = m.pattern_weights(bench.MIXES[mix])
ncpu = os.cpu_count() or 2
tag = 1_000_000
combos = list(itertools.product([1, 2, 3], [True, False], [ncpu - 1, max(1, ncpu // 2)]))
if os.environ.get("SWEEP_DEFAULT_ONLY"):
    combos = [(int(x), True, ncpu - 1) for x in os.environ.get("SWEEP_IN_FLIGHT", "2,2,2").split(",")]
for fl, gr, pr in combos:
    eng.train(graph, w, 5, batch=batch, n_neg=n_neg, first_tag=tag, n_producers=pr,
              in_flight=fl, graphs=gr)
    tag += 5
    t0 = time.perf_counter()
    eng.train(graph, w, steps, batch=batch, n_neg=n_neg, first_tag=tag, n_producers=pr,
              in_flight=fl, graphs=gr)
    dt = time.perf_counter() - t0
    tag += steps
    tim = {k: round(v / steps * 1e3, 4) for k, v in eng.last_timings.items()}
    busy, gap, ns = C.c_double(), C.c_double(), C.c_int64()
    check(lib.ngdb_step_timeline(eng.handle, C.byref(busy), C.byref(gap), C.byref(ns)))
    if ns.value:
        tim["device_busy_ms_per_step"] = round(busy.value / ns.value, 4)
        tim["device_gap_ms_per_step"] = round(gap.value / ns.value, 4)
    print(json.dumps({"in_flight": fl, "graphs": gr, "producers": pr,
                      "qps": round(batch * steps / dt), "ms_per_step": round(dt / steps * 1e3, 4),
                      "consumer_ms": tim}), flush=True)

# resident plans (the bench `value` path) under the same timeline
batches = bench.make_batches(graph, mix, batch, n_neg, 40, 5_000_000)
plans, keep = [], []
for b in batches:
    keep.append(m.PlannedStep(b, backbone, dim, 512))
    v = keep[-1].view()
    h = C.c_void_p()
    check(lib.ngdb_plan_create(eng.handle, C.byref(v), C.byref(h)))
    check(lib.ngdb_plan_prepare(eng.handle, h))
    plans.append(h)
step = eng.step_count
for h in plans:
    step += 1
    check(lib.ngdb_plan_run(eng.handle, h, step))
busy, gap, ns = C.c_double(), C.c_double(), C.c_int64()
check(lib.ngdb_step_timeline(eng.handle, C.byref(busy), C.byref(gap), C.byref(ns)))
if ns.value:
    print(json.dumps({"resident_plans": ns.value,
                      "device_busy_ms_per_step": round(busy.value / ns.value, 4),
                      "device_gap_ms_per_step": round(gap.value / ns.value, 4)}), flush=True)
for h in plans:
    check(lib.ngdb_plan_destroy(h))
