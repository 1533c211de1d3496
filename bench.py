#!/usr/bin/env python
"""Benchmark of the operator-level training step (BASELINE.json metric:
training queries/sec, mixed query types).

Workload (N=1 line): configs[1] — Query2Box on a synthetic NELL995-shaped KG
(63,361 entities, 200 relations, 114k/14k/14k edges), the full 14-type query
mix, 512 queries/step, 128 negatives, d=400, fp32, Adam lr 1e-4.

  value  device-timed q/s over K steps with the step plans already resident in
         HBM (host planning excluded; every kernel of every step is launched
         inside the timed region).
  e2e    q/s through the public C ABI call ngdb_train_step with HOST buffers:
         planning on the host, H2D of the packed plan, all kernels, D2H of the
         per-query losses, every step.
  roofline  the dominant kernel family, algorithmic bytes / CUDA-event time.
  cpu_baseline  the CPU oracle (f32, 1 thread) on a bounded sample.

`--impl reference` times the reference's CPU implementation of the path. The
reference ships no implementation, so this is the oracle port of
it (oracle/), with its own JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (backbone, shape, mix, dim, batch, n_neg)  -- BASELINE.json configs
    "c1": ("gqe", "fb15k-237", "c1", 400, 512, 128),
    "c2": ("q2b", "nell995", "all", 400, 512, 128),
    "c3": ("betae", "fb15k-237", "c3", 400, 512, 128),
    "c4": ("gqe", "fb15k-237", "c1", 400, 512, 128),  # + 768-d frozen PTE store
    "c5": ("q2b", "wikikg2", "all", 400, 512, 128),   # entity table row-sharded over ranks
}
SEMANTIC_DIM = {"c4": 768}
MIXES = {"all": ["1p", "2p", "3p", "2i", "3i", "pi", "ip", "2u", "up", "2in", "3in", "pin", "pni",
                 "inp"],
         "c1": ["1p", "2p", "3p", "2i", "3i"],
         "c3": ["2in", "3in", "inp", "pin", "pni"]}
METRIC = "training queries/sec (mixed query types)"


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled by NVML every ~1 ms on a host
    thread while the timed region runs on the device."""

    REASONS = {"hw_slowdown": 0x8, "sw_power_cap": 0x4, "hw_thermal_slowdown": 0x40,
               "sw_thermal_slowdown": 0x20, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device=0):
        self.device = device
        self.samples, self.reason_bits = [], 0
        self.stop_flag = threading.Event()
        self.thread = None
        self.error = None

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
        except Exception as e:  # noqa: BLE001 - reported in the JSON line
            self.error = f"nvml unavailable: {e}"
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        N, h = self.N, self.h
        while not self.stop_flag.is_set():
            try:
                self.samples.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
                self.reason_bits |= int(N.nvmlDeviceGetCurrentClocksEventReasons(h))
            except Exception as e:  # noqa: BLE001
                self.error = str(e)
                return
            time.sleep(0.001)

    def stop(self):
        if self.thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.error or "no sampler"],
                    "samples": 0}
        self.stop_flag.set()
        self.thread.join(timeout=2)
        reasons = sorted(k for k, b in self.REASONS.items() if self.reason_bits & b)
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


def roofline(fams, config=None):
    """Roofline of the dominant kernel family (largest share of the profiled
    step): GEMM families against the measured dense tensor peak (bf16 cuBLAS,
    the only measured tensor figure; our contractions are 3xTF32 on tcgen05),
    bandwidth families against measured HBM. Also the top HBM-bound family.
    `traffic` = DRAM bytes per launch from the committed ncu capture of this
    config (profiles/ncu_traffic.json), when there is one."""
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (
        ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    tensor = float(peaks.get("bf16_tflops", 1590.0))
    kind = "measured" if peaks else "fallback"
    total = sum(v["ms_per_step"] for v in fams.values())
    name, f = max(fams.items(), key=lambda kv: kv[1]["ms_per_step"])
    tf = ROOT / "profiles" / "ncu_traffic.json"
    traffic = json.loads(tf.read_text()).get(config, {}) if tf.exists() and config else {}

    def traffic_of(n, v):
        t = traffic.get(n)
        if not t:
            return None
        alg = v["bytes_per_step"] / max(v["launches_per_step"], 1e-9)
        return {"dram_bytes_per_launch": t["bytes_per_launch"],
                "algorithmic_bytes_per_launch": alg, "kernel": t["kernel"], "source": t["source"]}

    def hbm_entry(n, v):
        t = traffic_of(n, v)
        return {"bound": "hbm", "kernel": n, "achieved": v["gbs"], "peak": hbm, "unit": "GB/s",
                "frac": v["gbs"] / hbm, "traffic": t["dram_bytes_per_launch"] if t else None,
                "traffic_detail": t, "peak_kind": kind, "share_of_step": v["ms_per_step"] / total}

    if f["flops_per_step"] > 0:
        roof = {"bound": "tensor", "kernel": name, "achieved": f["tflops"], "peak": tensor,
                "unit": "TFLOP/s", "frac": f["tflops"] / tensor,
                "traffic": (traffic_of(name, f) or {}).get("dram_bytes_per_launch"),
                "traffic_detail": traffic_of(name, f),
                "peak_kind": kind + " (bf16 dense; kernels are 3xTF32)",
                "share_of_step": f["ms_per_step"] / total}
    else:
        roof = hbm_entry(name, f)
    bw = {k: v for k, v in fams.items() if v["flops_per_step"] == 0}
    if bw:
        n2, f2 = max(bw.items(), key=lambda kv: kv[1]["ms_per_step"])
        roof["hbm_kernel"] = hbm_entry(n2, f2)
    return roof


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_batches(graph, mix, batch, n_neg, count, base_tag):
    import paper_2602_21597_b200 as m
    w = m.pattern_weights(MIXES[mix])
    return [m.Batch.sample(graph, w, batch, n_neg, seed=3, tag=base_tag + i) for i in range(count)]


# entity / relation counts of the synthetic shapes
SHAPES = {"fb15k-237": (14505, 237), "nell995": (63361, 200), "wikikg2": (2500604, 535)}


def config_dict(cfg, world):
    """The `config` object of the JSON line — identical in both arms (ours and
    --impl reference) for the same --config and N."""
    backbone, shape, mix, dim, batch, n_neg = CONFIGS[cfg]
    ne, nr = SHAPES[shape]
    sdim = SEMANTIC_DIM.get(cfg, 0)
    ent_cols = 2 * dim if backbone == "betae" else dim
    out = {"workload": f"{backbone} on {shape}-shaped synthetic KG ({ne} entities, {nr} "
                       f"relations), {mix}-pattern mix"
                       + (f", FuseSemantic over a frozen {sdim}-d PTE store" if sdim else "")
                       + (", entity table row-sharded" if sharded(cfg, world) else ""),
           "config": cfg, "global_batch": batch * world, "n_neg": n_neg, "dim": dim}
    table_mb = 3 * ne * ent_cols * 4 / 1e6 / (world if sharded(cfg, world) else 1)
    if sharded(cfg, world):
        out["parallelism"] = f"rowshard{world}+dp{world}"
        out["l2"] = (f"inputs larger than L2: local entity table + Adam moments "
                     f"{table_mb / 1e3:.1f} GB per rank")
    else:
        out["parallelism"] = "single"
        out["l2"] = (f"L2 flushed (512 MB write) before every timed step; entity table + Adam "
                     f"moments {table_mb:.0f} MB" if l2_flush(cfg) else
                     f"inputs larger than L2: entity table + Adam moments {table_mb:.0f} MB; "
                     f"no flush between steps")
    return out


def sharded(cfg, world):
    """The row-sharded step runs C5 at every N and C1 / C2 at N > 1."""
    return cfg == "c5" or world > 1


def l2_flush(cfg):
    backbone, shape, mix, dim, batch, n_neg = CONFIGS[cfg]
    ent_cols = 2 * dim if backbone == "betae" else dim
    return 3 * SHAPES[shape][0] * ent_cols * 4 / 1e6 < 2 * 126  # L2 is 126 MB


# ---- the CPU reference (oracle/ only: never the product library) -------------
_REF = {}


def _oracle_worker(job):
    """One host process of the CPU reference: the oracle's own sampler and model
    on the oracle's graph (built before the fork); `warmup` untimed steps, then
    up to `steps` timed steps, each = sample a batch + one training step (the
    reference's train loop body), one OpenMP thread."""
    backbone, dim, n_neg, batch, mix_w, wid, warmup, steps, budget, threads = job
    import oracle as O
    O.set_threads(threads)
    g, info, store = _REF["graph"], _REF["info"], _REF["store"]
    om = O.OracleModel(backbone, info["n_entities"], info["n_relations"], dim, n_neg,
                       precision=32)
    if store is not None:
        om.set_semantic(store)
    om.init(2)
    tag = 10_000_000 + 1000 * wid

    def one(i):
        a = g.sample(mix_w, batch, n_neg, seed=3, tag=tag + i)
        om.step(*a, b_max=512, step=i + 1)
    for i in range(warmup):
        one(i)
    t0 = time.perf_counter()
    done = 0
    while done < steps:
        one(warmup + done)
        done += 1
        if budget and time.perf_counter() - t0 >= budget:
            break
    return done * batch, time.perf_counter() - t0


def cpu_reference(cfg, workers, warmup, steps_total, budget=None, threads=1):
    """The CPU reference (the oracle port: graph, sampler, Alg. 1 step, Adam; f32)
    on `workers` forked host processes in parallel (data-parallel replicas of
    `threads` OpenMP threads each: an upper bound for any shared-model CPU run).
    Loads only oracle/. Returns (aggregate q/s, workers, steps done, seconds)."""
    import multiprocessing as mp

    import oracle as O
    backbone, shape, mix, dim, batch, n_neg = CONFIGS[cfg]
    if _REF.get("shape") != shape or _REF.get("cfg") != cfg:
        info = O.synth_info(shape)
        sdim = SEMANTIC_DIM.get(cfg, 0)
        _REF.update(shape=shape, cfg=cfg, info=info, graph=O.OracleGraph.synthetic(shape, 1),
                    store=O.semantic_store(info["n_entities"], sdim, seed=5) if sdim else None)
    info = _REF["info"]
    w = np.zeros(len(MIXES["all"]), np.float64)
    for p in MIXES[mix]:
        w[MIXES["all"].index(p)] = 1.0
    w /= w.sum()
    # bounded by host memory: each process holds its own model (θ, m, v, grad in f32)
    ent_w = 2 * dim if backbone == "betae" else dim
    per_worker = 5 * 4 * info["n_entities"] * ent_w + (1 << 29)
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 16 << 30
    workers = max(1, min(workers, int(0.6 * avail // per_worker)))
    per = max(1, -(-steps_total // workers))
    jobs = [(backbone, dim, n_neg, batch, w, i, warmup, per, budget, threads)
            for i in range(workers)]
    if workers == 1:
        res = [_oracle_worker(jobs[0])]
    else:
        with mp.get_context("fork").Pool(workers) as pool:
            res = pool.map(_oracle_worker, jobs)
    q = sum(r[0] for r in res)
    el = max(r[1] for r in res)
    return q / el, workers, q // batch, el


def cpu_baseline_entry(cfg, steps_total, budget):
    """cpu_baseline of the JSON line: all host cores (forked replicas) and one
    core (--threads nproc and --threads 1)."""
    batch = CONFIGS[cfg][4]
    qps, workers, done, el = cpu_reference(cfg, host_workers(), 1, steps_total, budget)
    q1, _, done1, el1 = cpu_reference(cfg, 1, 1, max(1, steps_total // workers), budget)
    return {"value": qps, "unit": "queries/s", "cores": workers, "kind": "port",
            "sample": f"{done} full {batch}-query steps (oracle sampler + Alg. 1 step + Adam, "
                      f"f32) on {workers} forked host processes (1 thread each), {el:.1f}s; "
                      f"the reference ships no implementation (SURVEY §0), so this is the "
                      f"oracle port of it (oracle/ only)",
            "single_core": {"value": q1, "unit": "queries/s", "cores": 1,
                            "sample": f"{done1} steps on 1 process / 1 thread, {el1:.1f}s"}}


QL_STEPS = 20


def executor_comparison(m, lib, check, ctx, batches, backbone, dim, batch, sdim, step_no):
    """Device time per step of the same batches planned by Max-Fillness
    (operator-level) and by the query-level baseline executor,
    each step a resident plan replayed as a CUDA graph on this context."""
    import ctypes as C
    out = {}
    bs = batches[:QL_STEPS]
    for ql in (False, True):
        steps = [m.PlannedStep(b, backbone, dim, 512, semantic=bool(sdim), query_level=ql)
                 for b in bs]
        inv = sum(s.trace()["invocations"] for s in steps) / len(steps)
        plans = []
        for s in steps:
            v = s.view()
            h = C.c_void_p()
            check(lib.ngdb_plan_create(ctx, C.byref(v), C.byref(h)))
            check(lib.ngdb_plan_prepare(ctx, h))
            plans.append(h)
        step_no += 1
        check(lib.ngdb_plan_run(ctx, plans[0], step_no))  # warm the graph path
        check(lib.ngdb_sync(ctx))
        ms = C.c_float()
        check(lib.ngdb_timer_start(ctx))
        for h in plans:
            step_no += 1
            check(lib.ngdb_plan_run(ctx, h, step_no))
        check(lib.ngdb_timer_stop(ctx, C.byref(ms)))
        for h in plans:
            check(lib.ngdb_plan_destroy(h))
        out["query_level" if ql else "operator_level"] = {
            "queries_per_s": batch * len(plans) / (ms.value / 1e3),
            "ms_per_step": ms.value / len(plans), "invocations_per_step": inv}
    out["operator_over_query_level"] = (out["operator_level"]["queries_per_s"] /
                                        out["query_level"]["queries_per_s"])
    out["steps"] = len(bs)
    return out


def evaluator_measure(eng, info, dim, backbone, nq=512, reps=5):
    """ngdb_eval_ranks: nq random query embeddings ranked against every entity
    of the trained table (filters of 100 entities), end to end per call."""
    rng = np.random.default_rng(1)
    n_ent = info["n_entities"]
    wq = dim if backbone == "gqe" else 2 * dim
    if backbone == "betae":  # (alpha | beta) > 0
        q = rng.uniform(0.05, 3.0, size=(nq, wq)).astype(np.float32)
    else:
        q = rng.uniform(-0.035, 0.035, size=(nq, wq)).astype(np.float32)
        q[:, dim:] = np.abs(q[:, dim:])
    t = rng.integers(0, n_ent, size=nq).astype(np.int32)
    ids = rng.integers(0, n_ent, size=(nq, 100)).astype(np.int32)
    ids[ids == t[:, None]] = (ids[ids == t[:, None]] + 1) % n_ent
    off = np.arange(0, 100 * nq + 1, 100, dtype=np.int32)
    eng.eval_ranks_csr(q, t, off, ids.ravel())
    t0 = time.perf_counter()
    for _ in range(reps):
        eng.eval_ranks_csr(q, t, off, ids.ravel())
    dt = (time.perf_counter() - t0) / reps
    return {"queries_per_s": nq / dt, "ms_per_call": dt * 1e3, "queries_per_call": nq,
            "entities": n_ent, "api": "ngdb_eval_ranks (host queries/targets/filters, ranks back)"}


def host_workers():
    return max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity")
               else (os.cpu_count() or 1))


def reference_arm(args):
    """--impl reference: the reference's CPU implementation of the path (the
    oracle port) on every host core, same config / metric / unit as
    our arm. Imports only oracle/ — the product library is never loaded here."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = args.config
    batch = CONFIGS[cfg][4]
    base = cpu_baseline_entry(cfg, args.steps, args.cpu_budget * 3)
    qps = base["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": qps, "unit": "queries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * batch / qps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(cfg, max(1, args.gpus)),
        "cpu_baseline": base,
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    # the arm's contract: nothing of the product was imported or mapped
    assert "paper_2602_21597_b200" not in sys.modules
    with open("/proc/self/maps") as f:
        assert "libngdb_b200" not in f.read()
    print(json.dumps(line), flush=True)


def bench_sharded(args):
    """Row-sharded step (configs[4]: Q2B on the wikikg2 shape; also C1/C2 when
    N > 1): entity table row-sharded over the ranks, one process per GPU, 512
    queries per rank (weak scaling). The device collectives run on the
    context's own NCCL communicator inside libngdb (uneven all-to-alls of owned
    rows, all-gather, reduce-scatter, all-reduce — captured with the stages in
    one CUDA graph per step); torch.distributed (gloo) carries only the packed
    int32 metadata records, the NCCL id and the barrier / max-over-ranks timing."""
    import torch
    import torch.distributed as dist

    import paper_2602_21597_b200 as m
    from paper_2602_21597_b200._native import check, lib
    from paper_2602_21597_b200.sharded import Comm, ShardedEngine, plan_shard_step

    rank, world, local = dist_env()
    os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep stdout to the one JSON line
    if "MASTER_ADDR" not in os.environ:  # single process: a one-rank group
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = Comm(transport="nccl")

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    backbone, shape, mix, dim, batch, n_neg = CONFIGS[args.config]
    t_setup = time.perf_counter()
    graph = m.Graph.synthetic(shape, 1)
    info = graph.info()
    w = m.pattern_weights(MIXES[mix])
    n_steps = args.warmup + args.steps
    # rank r's batch of step s: Rng(3).fork(s * world + r)
    batches = [m.Batch.sample(graph, w, batch, n_neg, seed=3, tag=(1 + s) * world + rank)
               for s in range(n_steps)]
    sdim = SEMANTIC_DIM.get(args.config, 0)
    store = m.semantic_store(info["n_entities"], sdim, seed=5) if sdim else None
    eng = ShardedEngine(comm, backbone, info["n_entities"], info["n_relations"], dim=dim,
                        n_neg=n_neg, max_queries=batch, device=local, semantic=store)
    plans = [plan_shard_step(comm, b, backbone, dim, batch_cap=batch, semantic=bool(sdim))
             for b in batches]
    setup_s = time.perf_counter() - t_setup
    ctx = eng.handle
    step_no = 0
    for i in range(args.warmup):
        step_no += 1
        eng.run(plans[i], step_no)
    torch.cuda.synchronize()
    dist.barrier()
    launches0 = lib.ngdb_launch_count(ctx)
    clocks = ClockSampler(local)
    clocks.start()
    import ctypes as C
    ms = C.c_float()
    # resident steps: each step's stages + NCCL collectives captured once into
    # a CUDA graph (before the timed region) and replayed, like the resident
    # plans of the single-GPU bench
    graphs = eng.capture(plans[args.warmup:])
    torch.cuda.synchronize()
    dist.barrier()
    check(lib.ngdb_timer_start(ctx))
    for i in range(args.steps):
        step_no += 1
        graphs[i].replay(step_no)
    check(lib.ngdb_timer_stop(ctx, C.byref(ms)))
    clk = clocks.stop()
    launches = lib.ngdb_launch_count(ctx) - launches0
    torch.cuda.synchronize()
    dist.barrier()
    ms_step = max_over_ranks(ms.value / args.steps)
    value = batch * world / (ms_step / 1000.0)
    # per-family CUDA-event times on a profiled replay of a few steps
    check(lib.ngdb_profile_enable(ctx, 1))
    n_prof = min(args.profile_steps, args.steps)
    for i in range(n_prof):
        step_no += 1
        eng.run(plans[args.warmup + i], step_no)
    torch.cuda.synchronize()
    fams = {}
    for f in range(lib.ngdb_profile_families()):
        fms, fl, fb, ff = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
        check(lib.ngdb_profile_read(ctx, f, C.byref(fms), C.byref(fl), C.byref(fb)))
        check(lib.ngdb_profile_flops(ctx, f, C.byref(ff)))
        if fl.value:
            fams[lib.ngdb_profile_family_name(f).decode()] = {
                "ms_per_step": fms.value / n_prof, "launches_per_step": fl.value / n_prof,
                "gbs": fb.value / (fms.value / 1000.0) / 1e9 if fms.value > 0 else 0.0,
                "tflops": ff.value / (fms.value / 1000.0) / 1e12 if fms.value > 0 else 0.0,
                "bytes_per_step": fb.value / n_prof, "flops_per_step": ff.value / n_prof}
    check(lib.ngdb_profile_enable(ctx, 0))
    # e2e: host planning (sampling, DAG, Max-Fillness, metadata all-gather, owner
    # lists) + every stage and collective, per step
    # e2e: the pipelined sharded trainer loop — sampling + planning on host
    # threads, metadata all-gather, owner lists, every stage and collective,
    # losses read back per step
    # this rank's share of the host cores (minus the launching and exchange threads)
    producers = max(2, host_workers() // world - 2)
    # one trainer-loop call: W warm-up steps, then the K timed ones (window
    # measured inside the loop, as in the single-GPU e2e)
    eng.step_count = step_no
    b0, d0 = C.c_int64(), C.c_int64()
    check(lib.ngdb_transfer_bytes(ctx, C.byref(b0), C.byref(d0)))
    dist.barrier()
    n_call = args.warmup + args.steps
    t0 = time.perf_counter()
    eng.train_native(graph, w, n_call, batch, n_neg, first_tag=1 + n_steps, producers=producers,
                     steady_from=args.warmup)
    torch.cuda.synchronize()
    call_s = time.perf_counter() - t0
    e2e_s = eng.last_timings["steady_s"]
    b1, d1 = C.c_int64(), C.c_int64()
    check(lib.ngdb_transfer_bytes(ctx, C.byref(b1), C.byref(d1)))
    step_no = eng.step_count
    e2e = batch * world * args.steps / max_over_ranks(e2e_s)
    e2e_call = batch * world * n_call / max_over_ranks(call_s)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": config_dict(args.config, world),
            "roofline": roofline(fams, args.config) if fams else None,
            "cpu_baseline": None,
            "e2e": {"value": e2e, "unit": "queries/s",
                    "h2d_bytes_per_step": int((b1.value - b0.value) / n_call),
                    "window": f"steps {args.warmup}..{n_call - 1} of one {n_call}-step "
                              "ngdb_shard_train_run call (timed inside the loop)",
                    "whole_call": {"value": e2e_call, "steps": n_call,
                                   "note": "thread start-up and pipeline fill included"},
                    "api": "ngdb_shard_train_run (producer threads sample + plan + pack, "
                           "exchange thread all-gathers the packed metadata over the "
                           "metadata communicator and builds owner lists, stages + NCCL "
                           "collectives + Adam, loss read-back per step)",
                    "consumer": getattr(eng, "last_timings", None),
                    "d2h_bytes_per_step": 4 * batch + 16},
            "families": fams,
            "gpu_launches": int(launches),
            "clocks": clk,
            "setup_s": setup_s,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: c2 at N=1, c5 (row-sharded wikikg2) at N>1")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=5)
    ap.add_argument("--quiet", action="store_true")
    ap.add_argument("--producers", type=int, default=0, help="e2e host producer threads (0: cores-1)")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the query-level executor and evaluator side measurements")
    ap.add_argument("--in-flight", type=int, default=0,
                    help="e2e steps on the device before the oldest one's losses are read (0: 3)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `--gpus N` without a launcher: one process per GPU via torchrun
        if args.impl == "ours":
            import torch
            if torch.cuda.device_count() < args.gpus:
                raise SystemExit(f"bench.py: --gpus {args.gpus} but {torch.cuda.device_count()} "
                                 "visible GPU(s)")
        port = 29400 + os.getpid() % 500
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
        os.execv(sys.executable, cmd)
    if world > 1 and world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.config is None:
        args.config = "c5" if world > 1 else "c2"

    if args.impl == "reference":
        return reference_arm(args)
    if args.config == "c5" or world > 1:
        return bench_sharded(args)
    dist = None

    import ctypes as C

    import paper_2602_21597_b200 as m
    from paper_2602_21597_b200._native import check, lib

    backbone, shape, mix, dim, batch, n_neg = CONFIGS[args.config]
    t_setup = time.perf_counter()
    graph = m.Graph.synthetic(shape, 1)
    info = graph.info()
    n_steps = args.warmup + args.steps
    # each rank draws its own batches: Rng(3).fork(step * world + rank)
    batches = make_batches(graph, mix, batch, n_neg, n_steps, 1 + rank * 100000)
    sdim = SEMANTIC_DIM.get(args.config, 0)
    store = m.semantic_store(info["n_entities"], sdim, seed=5) if sdim else None
    eng = m.Engine(backbone, info["n_entities"], info["n_relations"], dim=dim, n_neg=n_neg,
                   b_max=512, max_queries=batch, device=local, semantic=store)
    ctx = eng.handle
    steps = [m.PlannedStep(b, backbone, dim, 512, semantic=bool(sdim)) for b in batches]
    plans = []
    for s in steps:
        v = s.view()
        h = C.c_void_p()
        check(lib.ngdb_plan_create(ctx, C.byref(v), C.byref(h)))
        plans.append(h)
    for h in plans:  # capture every step's CUDA graph up front (resident plans)
        check(lib.ngdb_plan_prepare(ctx, h))
    setup_s = time.perf_counter() - t_setup

    def barrier():
        if dist is not None:
            dist.barrier()

    step_no = 0

    def run_plan(i):
        nonlocal step_no
        step_no += 1
        check(lib.ngdb_plan_run(ctx, plans[i], step_no))

    # ---- value: device-timed, plans resident in HBM --------------------------
    for i in range(args.warmup):
        run_plan(i)
    check(lib.ngdb_sync(ctx))
    barrier()
    launches0 = lib.ngdb_launch_count(ctx)
    clocks = ClockSampler(local)
    if not os.environ.get("BENCH_NO_CLOCKS"):
        clocks.start()
    flush = l2_flush(args.config)  # entity table + Adam m, v vs the 126 MB L2
    ms = C.c_float()
    if flush:
        # each step timed on its own (CUDA events on the ctx stream) after a
        # 512 MB write that evicts L2; the per-step times are summed
        total_ms = 0.0
        for i in range(args.steps):
            check(lib.ngdb_flush_l2(ctx))
            check(lib.ngdb_timer_start(ctx))
            run_plan(args.warmup + i)
            check(lib.ngdb_timer_stop(ctx, C.byref(ms)))
            total_ms += ms.value
        ms.value = total_ms
    else:
        check(lib.ngdb_timer_start(ctx))
        for i in range(args.steps):
            run_plan(args.warmup + i)
        check(lib.ngdb_timer_stop(ctx, C.byref(ms)))
    clk = clocks.stop()
    launches = lib.ngdb_launch_count(ctx) - launches0
    barrier()
    ms_step = ms.value / args.steps
    if dist is not None:
        import torch
        t = torch.tensor([ms_step], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    value = batch * world / (ms_step / 1000.0)

    # ---- roofline: per-family CUDA-event times on a profiled replay ----------
    check(lib.ngdb_profile_enable(ctx, 1))
    for i in range(args.profile_steps):
        run_plan(args.warmup + (i % args.steps))
    check(lib.ngdb_sync(ctx))
    fams = {}
    for f in range(lib.ngdb_profile_families()):
        fms, fl, fb, ff = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
        check(lib.ngdb_profile_read(ctx, f, C.byref(fms), C.byref(fl), C.byref(fb)))
        check(lib.ngdb_profile_flops(ctx, f, C.byref(ff)))
        if fl.value:
            fams[lib.ngdb_profile_family_name(f).decode()] = {
                "ms_per_step": fms.value / args.profile_steps,
                "launches_per_step": fl.value / args.profile_steps,
                "gbs": fb.value / (fms.value / 1000.0) / 1e9 if fms.value > 0 else 0.0,
                "tflops": ff.value / (fms.value / 1000.0) / 1e12 if fms.value > 0 else 0.0,
                "bytes_per_step": fb.value / args.profile_steps,
                "flops_per_step": ff.value / args.profile_steps}
    check(lib.ngdb_profile_enable(ctx, 0))
    roof = roofline(fams, args.config)
    # the resident plans (and their captured graphs) are released before the
    # e2e leg, which streams fresh plans
    check(lib.ngdb_sync(ctx))
    for h in plans:
        check(lib.ngdb_plan_destroy(h))
    plans.clear()

    # ---- e2e: public C ABI call with host buffers ----------------------------
    # The trainer loop (ngdb_train_run): host producer threads sample and plan
    # every step's batch, the calling thread uploads each plan (one H2D from
    # pinned staging), launches its pools + optimizer and reads the step's
    # per-query losses back (D2H) while the next step runs. Sampling, planning,
    # copies and kernels of every step are inside the timed region.
    w = m.pattern_weights(MIXES[mix])
    tag0 = 1_000_000 + rank * 100_000

    # ONE trainer-loop call runs the W warm-up steps and then the K timed
    # steps (a training run is one call): the timed window starts when the
    # consumer reaches step W (that step's plan wait included) and ends when
    # step W+K-1's losses are back on the host (steady_s, measured inside the
    # loop). The whole call, thread start-up and pipeline fill included, is
    # reported beside it.
    b0, d0 = C.c_int64(), C.c_int64()
    check(lib.ngdb_transfer_bytes(ctx, C.byref(b0), C.byref(d0)))
    barrier()
    eng.step_count = step_no
    t0 = time.perf_counter()
    eng.train(graph, w, args.warmup + args.steps, batch=batch, n_neg=n_neg, seed=3,
              first_tag=tag0, n_producers=args.producers, in_flight=args.in_flight,
              steady_from=args.warmup)
    call_s = time.perf_counter() - t0
    e2e_s = eng.last_timings["steady_s"]
    n_call = args.warmup + args.steps
    step_no += n_call
    b1, d1 = C.c_int64(), C.c_int64()
    check(lib.ngdb_transfer_bytes(ctx, C.byref(b1), C.byref(d1)))
    gu, gi = C.c_int64(), C.c_int64()
    check(lib.ngdb_graph_stats(ctx, C.byref(gu), C.byref(gi)))
    tim = eng.last_timings
    if dist is not None:
        import torch
        t = torch.tensor([e2e_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
        t = torch.tensor([call_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        call_s = float(t.item())
    e2e = batch * world * args.steps / e2e_s
    e2e_call = batch * world * n_call / call_s
    producers = args.producers if args.producers > 0 else max(1, (os.cpu_count() or 2) - 1)
    # the same public API one step at a time, no overlap (ngdb_train_step on
    # pre-sampled batches): what a synchronous caller gets
    losses = np.zeros(batch, dtype=np.float32)
    total = C.c_double()
    n_seq = min(args.steps, 20)
    t0 = time.perf_counter()
    for i in range(n_seq):
        step_no += 1
        check(lib.ngdb_train_step(ctx, batches[args.warmup + i]._h, 512, step_no,
                                  losses.ctypes.data_as(C.POINTER(C.c_float)), C.byref(total)))
    seq_qps = batch * n_seq / (time.perf_counter() - t0)

    # ---- side measurements: operator-level vs the query-level
    # baseline executor on the same kernels and batches, and the evaluator's
    # full-entity filtered ranking. Reported beside the headline; a failure
    # here is recorded in the line instead of aborting it.
    extras = {}
    if not args.no_extras:
        try:
            extras["query_level"] = executor_comparison(m, lib, check, ctx, batches[args.warmup:],
                                                        backbone, dim, batch, sdim, step_no)
            step_no += 2 * len(batches[args.warmup:][:QL_STEPS]) + 2
        except Exception as exc:  # noqa: BLE001
            extras["query_level"] = {"error": repr(exc)}
        if not (backbone == "betae" and sdim):
            try:
                extras["evaluator"] = evaluator_measure(eng, info, dim, backbone)
            except Exception as exc:  # noqa: BLE001
                extras["evaluator"] = {"error": repr(exc)}
        if backbone in ("gqe", "q2b"):
            # SPEC.md:682-690 operator_microbench at acceptance 6's shape
            # (n=1024, k=2, d=400), on this config's graph and backbone
            from paper_2602_21597_b200.microbench import operator_microbench
            mb = {}
            for op, k in (("Intersect", 2), ("UnionScore", 2), ("Project", 1),
                          ("EmbedAnchor", 1)):
                try:
                    r = operator_microbench(graph, op, n=1024, k=k, dim=dim, backbone=backbone)
                    mb[f"{op}_k{k}"] = {x: r[x] for x in ("loop_ms", "batched_ms", "speedup",
                                                           "outputs_equal")}
                except Exception as exc:  # noqa: BLE001
                    mb[f"{op}_k{k}"] = {"error": repr(exc)}
            extras["operator_microbench"] = mb

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_entry(args.config, 10 ** 6, args.cpu_budget)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": config_dict(args.config, world),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "queries/s",
                    "h2d_bytes_per_step": int((b1.value - b0.value) / n_call),
                    "d2h_bytes_per_step": int((d1.value - d0.value) / n_call),
                    "api": "ngdb_train_run (sampling + planning on host producer threads, "
                           "plan H2D, kernels, loss D2H per step)",
                    "window": f"steps {args.warmup}..{n_call - 1} of one {n_call}-step "
                              "ngdb_train_run call (timed inside the loop)",
                    "whole_call": {"value": e2e_call, "steps": n_call,
                                   "note": "thread start-up and pipeline fill included"},
                    "producers": producers,
                    "consumer_ms_per_step": {k[:-2]: 1000 * v / n_call for k, v in tim.items()
                                             if k != "steady_s"},
                    "sequential_train_step": seq_qps,
                    "step_graphs": {"updated": gu.value, "instantiated": gi.value}},
            "gpu_launches": int(launches),
            "clocks": clk,
            "families": fams if not args.quiet else None,
            "setup_s": setup_s,
        }
        line.update(extras)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
