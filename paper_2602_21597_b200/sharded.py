"""Row-sharded training step over torch.distributed (
BASELINE.json configs[4]: Query2Box on the ogbl-wikikg2 shape, 2/4/8 B200).

One process per GPU. Entity e lives on rank e mod G (local row e div G);
relations and MLPs are replicated and their gradients all-reduced. Each rank
plans its own batch with the host Max-Fillness planner (bit-exact per-rank
trace); the device work runs in stages of ngdb_shard_run with the collectives
between them, all on the framework stream the context is bound to:

  anchors    reduce-scatter  owned rows of every rank's anchor ids
  forward    local pools (all but Score / UnionScore / Loss)
  scoring    all-gather of the score-slot queries; every rank scores the
             candidates it owns for every rank's queries; reduce-scatter of
             the partial dL/dq and losses back to the query's rank
  backward   local pools
  gradients  all-to-all of anchor-gradient rows to their owners, all-reduce
             of dense + relation gradients, then owner-local Adam

`Comm` maps these onto NCCL device collectives; with the gloo backend (tests:
two processes sharing one GPU) the same calls are staged through host memory.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np

from ._native import SHARD_BUFFERS, ModelDesc, ShardBuffers, ShardPlan, StepPlan, check, lib
from .engine import BACKBONES, Batch, PlannedStep, param_specs

FORWARD_STAGES = {"anchor_pack": 0, "forward": 1, "query_pack": 2, "score": 3, "score_done": 4,
                  "backward": 5, "grad_pack": 6}


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class Comm:
    """The five collectives of the sharded step over a torch.distributed group.

    NCCL: device tensors straight into the NCCL collectives (NVLink/NVSwitch).
    gloo: host-staged equivalents (used by the tests, where two ranks share one
    GPU). Host metadata always travels over a gloo group."""

    def __init__(self, group=None, meta_group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nccl = dist.get_backend(group) == "nccl"
        self.meta_group = meta_group if meta_group is not None else (
            dist.new_group(backend="gloo") if self.nccl else group)

    # -- device tensors ---------------------------------------------------------
    def all_gather(self, out, inp):
        if self.nccl:
            self.dist.all_gather_into_tensor(out, inp, group=self.group)
            return
        parts = self._gather_host(inp)
        out.copy_(self.torch.cat(parts).to(out.device))

    def reduce_scatter(self, out, inp):
        if self.nccl:
            self.dist.reduce_scatter_tensor(out, inp, group=self.group)
            return
        n = out.numel()
        parts = self._gather_host(inp)
        acc = parts[0][self.rank * n:(self.rank + 1) * n].clone()
        for q in range(1, self.world):  # rank order (deterministic)
            acc += parts[q][self.rank * n:(self.rank + 1) * n]
        out.copy_(acc.to(out.device))

    def all_to_all(self, out, inp):
        if self.nccl:
            self.dist.all_to_all_single(out, inp, group=self.group)
            return
        n = out.numel() // self.world
        parts = self._gather_host(inp)
        out.copy_(self.torch.cat([parts[q][self.rank * n:(self.rank + 1) * n]
                                  for q in range(self.world)]).to(out.device))

    def all_reduce(self, t):
        if self.nccl:
            self.dist.all_reduce(t, group=self.group)
            return
        parts = self._gather_host(t)
        acc = parts[0].clone()
        for q in range(1, self.world):
            acc += parts[q]
        t.copy_(acc.to(t.device))

    def _gather_host(self, t):
        h = t.detach().to("cpu")
        parts = [self.torch.empty_like(h) for _ in range(self.world)]
        self.dist.all_gather(parts, h, group=self.group)
        return parts

    # -- host metadata ----------------------------------------------------------
    def all_gather_object(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.meta_group)
        return out


def _device_view(torch, ptr, n):
    """Zero-copy torch view of a context-owned float32 device buffer."""
    class _CAI:
        __cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f4",
                                    "data": (int(ptr), False), "version": 3, "strides": None}
    return torch.as_tensor(_CAI(), device="cuda")


class ShardStep:
    """A rank's planned step plus the owner work lists of the shard plan."""

    def __init__(self, planned: PlannedStep, shard_handle, n_queries: int):
        self.planned, self._h, self.n_queries = planned, shard_handle, n_queries

    def views(self):
        v = self.planned.view()
        s = ShardPlan()
        check(lib.ngdb_shard_view(self._h, C.byref(s)))
        return v, s

    def __del__(self):
        if getattr(self, "_h", None):
            lib.ngdb_shard_destroy(self._h)
            self._h = None


def _local_meta(ps: PlannedStep):
    """This rank's scoring metadata of a planned step (host arrays)."""
    na, ns, b, nc = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    check(lib.ngdb_step_shard_info(ps._h, C.byref(na), C.byref(ns), C.byref(b), C.byref(nc)))
    anchors = np.zeros(na.value, np.int32)
    unit_k = np.zeros(b.value, np.int32)
    unit_slots = np.zeros(b.value * 3, np.int32)
    cand = np.zeros(b.value * nc.value, np.int32)
    check(lib.ngdb_step_shard_meta(ps._h, _p(anchors, C.c_int32), _p(unit_k, C.c_int32),
                                   _p(unit_slots, C.c_int32), _p(cand, C.c_int32)))
    return (anchors, unit_k, unit_slots, cand, ns.value), b.value, nc.value


def _gather_meta(comm: Comm, local):
    """All-gather the ranks' scoring metadata (gloo, ordered per step) and pad
    it into the dense [G][...] arrays of ngdb_shard_build."""
    mine, b, nc = local
    meta = comm.all_gather_object(mine)
    G = comm.world
    A = max(1, max(m[0].size for m in meta))
    S = max(1, max(m[4] for m in meta))
    B = max(m[1].size for m in meta)
    anc_all = np.full((G, A), -1, np.int32)
    k_all = np.zeros((G, B), np.int32)
    slots_all = np.full((G, B, 3), -1, np.int32)
    cand_all = np.zeros((G, B, nc), np.int32)
    for q, (an, uk, us, ca, _) in enumerate(meta):
        bq = uk.size
        anc_all[q, :an.size] = an
        k_all[q, :bq] = uk
        slots_all[q, :bq] = us.reshape(bq, 3)
        cand_all[q, :bq] = ca.reshape(bq, nc)
    return (G, comm.rank, B, A, S, nc, anc_all, k_all, slots_all, cand_all), b


def _build_shard_step(ps: PlannedStep, gathered) -> ShardStep:
    """Owner work lists of this rank (C++; releases the GIL)."""
    (G, rank, B, A, S, nc, anc_all, k_all, slots_all, cand_all), b = gathered
    h = C.c_void_p()
    check(lib.ngdb_shard_build(G, rank, B, A, S, nc, _p(anc_all, C.c_int32),
                               _p(k_all, C.c_int32), _p(slots_all, C.c_int32),
                               _p(cand_all, C.c_int32), C.byref(h)))
    return ShardStep(ps, h, b)


def _finish_shard_step(comm: Comm, ps: PlannedStep, local) -> ShardStep:
    """Exchange the metadata (gloo all-gather) and build the owner work lists."""
    return _build_shard_step(ps, _gather_meta(comm, local))


def plan_shard_step(comm: Comm, batch: Batch, backbone: str, dim: int, b_max: int = 512) -> ShardStep:
    """Plan this rank's batch, exchange the metadata, build the owner work lists."""
    ps = PlannedStep(batch, backbone, dim, b_max, sharded=True)
    return _finish_shard_step(comm, ps, _local_meta(ps))


class ShardedEngine:
    """One rank's context of the row-sharded step."""

    def __init__(self, comm: Comm, backbone: str, n_entities: int, n_relations: int,
                 dim: int = 400, n_neg: int = 128, b_max: int = 512, max_queries: int = 512,
                 gamma: float = 12.0, lr: float = 1e-4, alpha_box: float = 0.02,
                 device: int = 0, seed: int = 2, debug: bool = False):
        import torch
        if backbone not in ("gqe", "q2b"):
            raise NotImplementedError("row-sharded step: GQE / Q2B")
        self.torch, self.comm = torch, comm
        self.backbone, self.dim, self.b_max = backbone, dim, b_max
        self.n_entities, self.n_relations = n_entities, n_relations
        G, r = comm.world, comm.rank
        d = ModelDesc(BACKBONES[backbone], n_entities, n_relations, dim, n_neg, 0, gamma,
                      alpha_box, lr, 0.9, 0.999, 1e-8, b_max, max_queries, G, r)
        self._h = C.c_void_p()
        check(lib.ngdb_ctx_create(C.byref(d), device, C.byref(self._h)))
        torch.cuda.set_device(device)
        # one explicit stream carries the context's kernels AND the collectives
        # (the legacy default stream would not order against the context)
        self.stream = torch.cuda.Stream(device=device)
        check(lib.ngdb_ctx_set_stream(self._h, C.c_void_p(self.stream.cuda_stream)))
        self.n_local = (n_entities - r + G - 1) // G
        for name, rows, cols, _ in param_specs(backbone, n_entities, n_relations, dim):
            if name == "entity":
                a = np.zeros((self.n_local, cols), np.float32)
                check(lib.ngdb_param_init_shard(BACKBONES[backbone], n_entities, n_relations, dim,
                                                name.encode(), seed, G, r, _p(a, C.c_float),
                                                a.size))
            else:  # replicated tensors: identical deterministic init on every rank
                a = np.zeros((rows, cols), np.float32)
                check(lib.ngdb_param_init_ex(BACKBONES[backbone], n_entities, n_relations, dim, 0,
                                             name.encode(), seed, _p(a, C.c_float), a.size))
            self.upload(name, a)
        if debug:
            check(lib.ngdb_set_debug(self._h, 1))
        self.step_count = 0

    def upload(self, name, value):
        a = np.ascontiguousarray(value, dtype=np.float32)
        check(lib.ngdb_param_upload(self._h, name.encode(), _p(a, C.c_float), a.size))

    def download(self, name: str) -> np.ndarray:
        base = name.split(":")[-1]
        spec = {s[0]: s for s in param_specs(self.backbone, self.n_entities, self.n_relations,
                                             self.dim)}[base]
        rows = self.n_local if base == "entity" else spec[1]
        out = np.zeros((rows, spec[2]), dtype=np.float32)
        check(lib.ngdb_param_download(self._h, name.encode(), _p(out, C.c_float), out.size))
        return out

    def plan(self, batch: Batch) -> ShardStep:
        return plan_shard_step(self.comm, batch, self.backbone, self.dim, self.b_max)

    def run(self, step: ShardStep, step_no: Optional[int] = None) -> np.ndarray:
        """All stages + collectives of one step; returns this rank's per-query losses."""
        if step_no is None:
            self.step_count += 1
            step_no = self.step_count
        with self.torch.cuda.stream(self.stream):
            return self._run(step, step_no)

    def _run(self, step: ShardStep, step_no: int) -> np.ndarray:
        v, s = step.views()
        b = ShardBuffers()
        check(lib.ngdb_shard_begin(self._h, C.byref(v), C.byref(s), C.byref(b)))
        t = {n: _device_view(self.torch, getattr(b, n), getattr(b, "n_" + n)) for n in SHARD_BUFFERS}
        _stages(self, t)
        check(lib.ngdb_shard_optimizer(self._h, step_no))
        losses = np.zeros(step.n_queries, np.float32)
        total, nonfinite = C.c_double(), C.c_int32()
        check(lib.ngdb_step_end(self._h, _p(losses, C.c_float), step.n_queries, C.byref(total),
                                C.byref(nonfinite)))
        if nonfinite.value:
            raise FloatingPointError(f"non-finite loss at step {step_no}")
        return losses

    def train_step(self, batch: Batch) -> np.ndarray:
        return self.run(self.plan(batch))

    def _launch(self, step: ShardStep, step_no: int) -> int:
        """All stages + collectives of one step, enqueued; returns the ticket of
        its asynchronous loss read-back (ngdb_step_end_async)."""
        with self.torch.cuda.stream(self.stream):
            v, s = step.views()
            b = ShardBuffers()
            check(lib.ngdb_shard_begin(self._h, C.byref(v), C.byref(s), C.byref(b)))
            t = {n: _device_view(self.torch, getattr(b, n), getattr(b, "n_" + n)) for n in SHARD_BUFFERS}
            _stages(self, t)
            check(lib.ngdb_shard_optimizer(self._h, step_no))
            ticket = C.c_int64()
            check(lib.ngdb_step_end_async(self._h, C.byref(ticket)))
        return ticket.value

    def train(self, graph, weights, n_steps: int, batch: int, n_neg: int, tag_of,
              producers: int = 8) -> np.ndarray:
        """Pipelined sharded trainer loop (the sharded counterpart of
        ngdb_train_run): host threads sample + plan upcoming batches (the C++
        calls release the GIL), the calling thread exchanges each step's
        metadata, builds its owner lists, enqueues its stages and collectives,
        and reads step i's losses back while step i+1 runs. Batch of step s is
        Rng(3).fork(tag_of(s)). Returns the per-step loss sums of this rank."""
        import concurrent.futures as cf

        def prep(s):
            b = Batch.sample(graph, weights, batch, n_neg, seed=3, tag=tag_of(s))
            ps = PlannedStep(b, self.backbone, self.dim, self.b_max, sharded=True)
            return ps, _local_meta(ps)

        sums = np.zeros(n_steps, np.float64)
        losses = np.zeros(batch, np.float32)
        pending = []
        ahead = 2 * producers

        def collect():
            i, ticket, _step = pending.pop(0)
            total, nonfinite = C.c_double(), C.c_int32()
            check(lib.ngdb_step_wait(self._h, ticket, _p(losses, C.c_float), batch,
                                     C.byref(total), C.byref(nonfinite)))
            if nonfinite.value:
                raise FloatingPointError(f"non-finite loss at step {i}")
            sums[i] = total.value

        # three stages ahead of the launching thread: sample + plan (pool), the
        # ordered metadata all-gather (one thread: collectives run in step
        # order on every rank), owner lists (pool)
        with cf.ThreadPoolExecutor(producers) as pool, cf.ThreadPoolExecutor(1) as exch:
            def gather(s, prep_fut):
                ps, local = prep_fut.result()
                return ps, _gather_meta(self.comm, local)

            def build(gather_fut):
                ps, gathered = gather_fut.result()
                return _build_shard_step(ps, gathered)

            futs = {}

            def submit(s):
                pf = pool.submit(prep, s)
                gf = exch.submit(gather, s, pf)
                futs[s] = pool.submit(build, gf)

            for s in range(min(n_steps, ahead)):
                submit(s)
            for s in range(n_steps):
                step = futs.pop(s).result()
                if s + ahead < n_steps:
                    submit(s + ahead)
                self.step_count += 1
                pending.append((s, self._launch(step, self.step_count), step))
                while len(pending) > 1:
                    collect()
            while pending:
                collect()
        return sums

    def capture(self, steps: List[ShardStep]) -> List["ShardGraph"]:
        """Resident copies of `steps` whose stages AND collectives replay as one
        CUDA graph each (NCCL only; the communicator must have run eagerly
        first). Every resident step is created — and the context's buffers
        sized for all of them — before the first capture, so no later growth
        invalidates a captured graph."""
        handles = []
        for st in steps:
            v, s = st.views()
            h = C.c_void_p()
            check(lib.ngdb_shard_step_create(self._h, C.byref(v), C.byref(s), C.byref(h)))
            handles.append((h, st.n_queries))
        return [ShardGraph(self, h, nq) for h, nq in handles]

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.ngdb_ctx_destroy(self._h)
            self._h = None


class ShardGraph:
    """A resident sharded step (ngdb_shard_step_create: plan + owner lists in
    device memory, buffers sized up front) captured with its NCCL collectives
    into one CUDA graph on the engine's stream. replay(step_no) sets the Adam
    step scalars and launches the graph: no host work per stage."""

    def __init__(self, eng: ShardedEngine, handle, n_queries: int):
        self._h = handle  # owned from here on (destroyed with the graph)
        if not eng.comm.nccl:
            raise RuntimeError("graph capture of the sharded step needs the NCCL backend")
        torch = eng.torch
        self.eng = eng
        self.n_queries = n_queries
        self.graph = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(self.graph, stream=eng.stream):
            b = ShardBuffers()
            check(lib.ngdb_shard_step_begin(eng._h, self._h, C.byref(b)))
            t = {n: _device_view(torch, getattr(b, n), getattr(b, "n_" + n)) for n in SHARD_BUFFERS}
            _stages(eng, t)
            check(lib.ngdb_shard_optimizer(eng._h, 0))

    def replay(self, step_no: int) -> None:
        check(lib.ngdb_set_step(self.eng._h, step_no))
        with self.eng.torch.cuda.stream(self.eng.stream):
            self.graph.replay()

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.ngdb_shard_step_destroy(self._h)
            self._h = None


def _stages(eng: ShardedEngine, t) -> None:
    """The device stages of a sharded step with the collectives between them."""
    run = lambda stage: check(lib.ngdb_shard_run(eng._h, FORWARD_STAGES[stage]))  # noqa: E731
    comm = eng.comm
    run("anchor_pack")
    comm.reduce_scatter(t["anchor_rows"], t["anchor_send"])
    run("forward")
    run("query_pack")
    comm.all_gather(t["query_all"], t["query_mine"])
    run("score")
    comm.reduce_scatter(t["dq_mine"], t["dq_part"])
    comm.reduce_scatter(t["loss_mine"], t["loss_part"])
    run("score_done")
    run("backward")
    run("grad_pack")
    comm.all_to_all(t["grad_all"], t["grad_send"])
    comm.all_reduce(t["reduce"])


def gather_entity_table(comm: Comm, local: np.ndarray, n_entities: int) -> Optional[np.ndarray]:
    """Reassemble the full entity table (rank 0 gets it; others None)."""
    parts = comm.all_gather_object(local)
    if comm.rank != 0:
        return None
    out = np.zeros((n_entities, local.shape[1]), np.float32)
    for q, p in enumerate(parts):
        out[q::comm.world] = p
    return out


def ranks_batches(graph, weights, b: int, n_neg: int, world: int, step: int,
                  seed: int = 3) -> List[Batch]:
    """Rank r's batch of step `step`: Rng(seed).fork(step * world + r)."""
    return [Batch.sample(graph, weights, b, n_neg, seed=seed, tag=step * world + r)
            for r in range(world)]
