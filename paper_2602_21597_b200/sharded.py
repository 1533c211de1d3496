"""Row-sharded training step (BASELINE.json
configs[4]: Query2Box on the ogbl-wikikg2 shape, 2/4/8 B200).

One process per GPU. Entity e lives on rank e mod G (local row e div G);
relations and MLPs are replicated and their gradients all-reduced. Each rank
plans its own batch with the host Max-Fillness planner (bit-exact per-rank
trace) and publishes ONE packed int32 metadata record (ngdb_step_shard_pack);
the records are all-gathered and every rank builds its owner work lists
(ngdb_shard_build_packed). The device step, in stages with the collectives
between them:

  lookups    uneven all-to-all: each owner sends a rank exactly the rows of
             that rank's anchors it owns
  forward    local pools (all but Score / UnionScore / Loss)
  scoring    all-gather of the score-slot queries; every rank scores the
             candidates it owns for every rank's queries; ONE reduce-scatter
             returns the partial dL/dq and partial losses to the query's rank
  backward   local pools
  gradients  the lookup all-to-all reversed (anchor-gradient rows to their
             owners), all-reduce of dense + relation gradients, owner-local Adam

Transports (`Comm.transport`):
  "nccl"  the context's own NCCL communicator (libngdb: ngdb_comm_init; the
          stages + collectives + optimizer run inside ngdb_shard_step_exec or
          a captured CUDA graph) — no framework collective on the data path;
  "host"  the same collectives staged through host memory over the gloo group
          (tests: two ranks sharing one GPU, where NCCL cannot run).
torch.distributed (gloo) only carries the host metadata, the NCCL unique id
and the benchmark's barrier / max-over-ranks timing.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np

from ._native import SHARD_BUFFERS, ModelDesc, ShardBuffers, ShardPlan, StepPlan, check, lib
from .engine import BACKBONES, Batch, PlannedStep, param_specs

FORWARD_STAGES = {"anchor_pack": 0, "forward": 1, "query_pack": 2, "score": 3, "score_done": 4,
                  "backward": 5, "grad_pack": 6, "fuse_bwd": 7}
NCCL_ID_BYTES = 128


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class Comm:
    """Host side of the sharded step over a torch.distributed process group.

    transport "nccl" (default when the default group is NCCL, or when asked):
    device collectives run on the context's own NCCL communicator inside
    libngdb; "host": host-staged equivalents over the gloo group (tests).
    Host metadata always travels over a gloo group as packed int32 records."""

    def __init__(self, group=None, transport: Optional[str] = None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        backend = dist.get_backend(group)
        self.transport = transport or ("nccl" if backend == "nccl" else "host")
        if self.transport not in ("nccl", "host"):
            raise ValueError(f"unknown transport {self.transport!r}")
        self.meta_group = group if backend == "gloo" else dist.new_group(backend="gloo")

    @property
    def nccl(self) -> bool:
        return self.transport == "nccl"

    # -- host-staged device collectives (transport "host") ----------------------
    def all_gather(self, out, inp):
        parts = self._gather_host(inp)
        out.copy_(self.torch.cat(parts).to(out.device))

    def reduce_scatter(self, out, inp):
        n = out.numel()
        parts = self._gather_host(inp)
        acc = parts[0][self.rank * n:(self.rank + 1) * n].clone()
        for q in range(1, self.world):  # rank order (deterministic)
            acc += parts[q][self.rank * n:(self.rank + 1) * n]
        out.copy_(acc.to(out.device))

    def all_to_all_v(self, out, inp, send_counts, recv_counts):
        """Uneven all-to-all: send_counts[q] elements of `inp` (rank-major) go
        to rank q; recv_counts[q] elements from rank q land in `out`."""
        sc = [int(x) for x in send_counts]
        rc = [int(x) for x in recv_counts]
        cap = int(self.all_gather_i32(np.asarray([sum(sc)], np.int32)).max())
        buf = self.torch.zeros(max(1, cap), dtype=self.torch.float32)
        buf[:sum(sc)] = inp.detach().view(-1)[:sum(sc)].to("cpu")
        parts = [self.torch.empty_like(buf) for _ in range(self.world)]
        self.dist.all_gather(parts, buf, group=self.meta_group)
        counts = self.all_gather_i32(np.asarray(sc, np.int32)).reshape(self.world, self.world)
        pieces = []
        for q in range(self.world):  # rank q's block addressed to me
            if int(counts[q, self.rank]) != rc[q]:
                raise RuntimeError("all_to_all_v: send/receive counts disagree")
            off = int(counts[q, :self.rank].sum())
            pieces.append(parts[q][off:off + rc[q]])
        res = self.torch.cat(pieces)
        if res.numel():
            out.view(-1)[:res.numel()].copy_(res.to(out.device))

    def all_reduce(self, t):
        parts = self._gather_host(t)
        acc = parts[0].clone()
        for q in range(1, self.world):
            acc += parts[q]
        t.copy_(acc.to(t.device))

    def _gather_host(self, t):
        h = t.detach().to("cpu")
        parts = [self.torch.empty_like(h) for _ in range(self.world)]
        self.dist.all_gather(parts, h, group=self.meta_group)
        return parts

    # -- host metadata ----------------------------------------------------------
    def all_gather_i32(self, rec: np.ndarray) -> np.ndarray:
        """All-gather one fixed-size int32 record per rank -> [world * n] (rank-major)."""
        t = self.torch.from_numpy(np.ascontiguousarray(rec, np.int32))
        parts = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t, group=self.meta_group)
        return self.torch.cat(parts).numpy()

    def broadcast_bytes(self, data: bytes, n: int) -> bytes:
        t = self.torch.zeros(n, dtype=self.torch.uint8)
        if self.rank == 0:
            t[:] = self.torch.frombuffer(bytearray(data), dtype=self.torch.uint8)
        self.dist.broadcast(t, 0, group=self.meta_group)
        return bytes(t.numpy().tobytes())


def _device_view(torch, ptr, n):
    """Zero-copy torch view of a context-owned float32 device buffer."""
    class _CAI:
        __cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f4",
                                    "data": (int(ptr), False), "version": 3, "strides": None}
    return torch.as_tensor(_CAI(), device="cuda")


def _arr(ptr, n):
    return np.ctypeslib.as_array(ptr, (max(int(n), 1),))[:int(n)].copy() if n else \
        np.zeros(0, np.int32)


class ShardStep:
    """A rank's planned step plus the owner work lists of the shard plan."""

    def __init__(self, planned: PlannedStep, shard_handle, n_queries: int):
        self.planned, self._h, self.n_queries = planned, shard_handle, n_queries

    def views(self):
        v = self.planned.view()
        s = ShardPlan()
        check(lib.ngdb_shard_view(self._h, C.byref(s)))
        return v, s

    def counts(self):
        """(send_cnt, recv_cnt) rows of the lookup all-to-all, per rank."""
        _, s = self.views()
        return _arr(s.send_cnt, s.world), _arr(s.recv_cnt, s.world)

    def __del__(self):
        if getattr(self, "_h", None):
            lib.ngdb_shard_destroy(self._h)
            self._h = None


def _local_meta(ps: PlannedStep, batch_cap: int):
    """This rank's packed metadata record (ngdb_step_shard_pack)."""
    nc = ps.view().n_candidates
    stride = int(lib.ngdb_shard_meta_stride(batch_cap, nc))
    rec = np.empty(stride, np.int32)
    check(lib.ngdb_step_shard_pack(ps._h, batch_cap, _p(rec, C.c_int32), stride))
    return rec, batch_cap


def _gather_meta(comm: Comm, local):
    """All-gather the ranks' packed records (gloo, one int32 tensor per rank)."""
    rec, batch_cap = local
    return comm.all_gather_i32(rec), rec.size, batch_cap, comm.world, comm.rank


def _build_shard_step(ps: PlannedStep, gathered) -> ShardStep:
    """Owner work lists of this rank (C++; releases the GIL)."""
    allrec, stride, batch_cap, world, rank = gathered
    h = C.c_void_p()
    check(lib.ngdb_shard_build_packed(world, rank, _p(allrec, C.c_int32), stride, batch_cap,
                                      C.byref(h)))
    return ShardStep(ps, h, ps.view().n_queries)


def plan_shard_step(comm: Comm, batch: Batch, backbone: str, dim: int, b_max: int = 512,
                    batch_cap: Optional[int] = None, semantic: bool = False) -> ShardStep:
    """Plan this rank's batch, exchange the packed metadata, build the owner lists.
    batch_cap (the record's query capacity) must be the same on every rank."""
    ps = PlannedStep(batch, backbone, dim, b_max, semantic=semantic, sharded=True)
    cap = batch_cap or ps.view().n_queries
    return _build_shard_step(ps, _gather_meta(comm, _local_meta(ps, cap)))


class ShardedEngine:
    """One rank's context of the row-sharded step."""

    def __init__(self, comm: Comm, backbone: str, n_entities: int, n_relations: int,
                 dim: int = 400, n_neg: int = 128, b_max: int = 512, max_queries: int = 512,
                 gamma: float = 12.0, lr: float = 1e-4, alpha_box: float = 0.02,
                 device: int = 0, seed: int = 2, debug: bool = False,
                 semantic: Optional[np.ndarray] = None):
        """semantic: the frozen store [n_entities][d_l] (FuseSemantic); this rank
        uploads its own rows (entity e = rank + world * local row)."""
        import torch
        if backbone not in ("gqe", "q2b", "betae"):
            raise NotImplementedError(f"row-sharded step: {backbone}")
        self.torch, self.comm = torch, comm
        self.backbone, self.dim, self.b_max = backbone, dim, b_max
        self.max_queries = max_queries
        self.n_entities, self.n_relations = n_entities, n_relations
        G, r = comm.world, comm.rank
        sd = 0 if semantic is None else int(semantic.shape[1])
        self.semantic_dim = sd
        d = ModelDesc(BACKBONES[backbone], n_entities, n_relations, dim, n_neg, sd, gamma,
                      alpha_box, lr, 0.9, 0.999, 1e-8, b_max, max_queries, G, r)
        self._h = C.c_void_p()
        check(lib.ngdb_ctx_create(C.byref(d), device, C.byref(self._h)))
        torch.cuda.set_device(device)
        # one explicit stream carries the context's kernels (and, for the host
        # transport, the torch copies staging the collectives)
        self.stream = torch.cuda.Stream(device=device)
        check(lib.ngdb_ctx_set_stream(self._h, C.c_void_p(self.stream.cuda_stream)))
        if comm.nccl:  # the context's own communicator: rank 0's id over gloo
            uid = (C.c_uint8 * NCCL_ID_BYTES)()
            if r == 0:
                check(lib.ngdb_comm_unique_id(uid))
            got = comm.broadcast_bytes(bytes(uid), NCCL_ID_BYTES)
            uid = (C.c_uint8 * NCCL_ID_BYTES).from_buffer_copy(got)
            check(lib.ngdb_comm_init(self._h, uid))
        self.n_local = (n_entities - r + G - 1) // G
        if semantic is not None:
            st = np.ascontiguousarray(semantic[r::G], dtype=np.float32)
            check(lib.ngdb_semantic_upload(self._h, _p(st, C.c_float), st.size))
        for name, rows, cols, _ in param_specs(backbone, n_entities, n_relations, dim, sd):
            if name == "entity" and sd:  # (the fused BetaE entity row is d wide)
                full = np.zeros((rows, cols), np.float32)
                check(lib.ngdb_param_init_ex(BACKBONES[backbone], n_entities, n_relations, dim, sd,
                                             name.encode(), seed, _p(full, C.c_float), full.size))
                a = np.ascontiguousarray(full[r::G])
            elif name == "entity":
                a = np.zeros((self.n_local, cols), np.float32)
                check(lib.ngdb_param_init_shard(BACKBONES[backbone], n_entities, n_relations, dim,
                                                name.encode(), seed, G, r, _p(a, C.c_float),
                                                a.size))
            else:  # replicated tensors: identical deterministic init on every rank
                a = np.zeros((rows, cols), np.float32)
                check(lib.ngdb_param_init_ex(BACKBONES[backbone], n_entities, n_relations, dim, sd,
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
                                             self.dim, self.semantic_dim)}[base]
        rows = self.n_local if base == "entity" else spec[1]
        out = np.zeros((rows, spec[2]), dtype=np.float32)
        check(lib.ngdb_param_download(self._h, name.encode(), _p(out, C.c_float), out.size))
        return out

    def plan(self, batch: Batch) -> ShardStep:
        return plan_shard_step(self.comm, batch, self.backbone, self.dim, self.b_max,
                               self.max_queries, semantic=self.semantic_dim > 0)

    def _enqueue(self, step: ShardStep, step_no: int) -> None:
        """begin + stages + collectives + optimizer of one step, enqueued."""
        v, s = step.views()
        b = ShardBuffers()
        with self.torch.cuda.stream(self.stream):
            check(lib.ngdb_shard_begin(self._h, C.byref(v), C.byref(s), C.byref(b)))
            if self.comm.nccl:
                check(lib.ngdb_shard_step_exec(self._h, step_no))
            else:
                _host_stages(self, b, _arr(s.send_cnt, s.world), _arr(s.recv_cnt, s.world))
                check(lib.ngdb_shard_optimizer(self._h, step_no))

    def run(self, step: ShardStep, step_no: Optional[int] = None) -> np.ndarray:
        """All stages + collectives of one step; returns this rank's per-query losses."""
        if step_no is None:
            self.step_count += 1
            step_no = self.step_count
        self._enqueue(step, step_no)
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
        """One step enqueued; returns the ticket of its asynchronous loss
        read-back (ngdb_step_end_async)."""
        self._enqueue(step, step_no)
        ticket = C.c_int64()
        check(lib.ngdb_step_end_async(self._h, C.byref(ticket)))
        return ticket.value

    def train(self, graph, weights, n_steps: int, batch: int, n_neg: int, tag_of,
              producers: int = 8) -> np.ndarray:
        """Pipelined sharded trainer loop (the sharded counterpart of
        ngdb_train_run): host threads sample + plan upcoming batches (the C++
        calls release the GIL), one ordered thread all-gathers each step's
        packed metadata record, the pool builds the owner lists, and the
        calling thread enqueues the step (stages + NCCL collectives + Adam in
        libngdb) and reads step i's losses back while step i+1 runs. Batch of
        step s is Rng(3).fork(tag_of(s)). Returns the per-step loss sums of this
        rank."""
        import concurrent.futures as cf
        cap = self.max_queries

        def prep(s):
            b = Batch.sample(graph, weights, batch, n_neg, seed=3, tag=tag_of(s))
            ps = PlannedStep(b, self.backbone, self.dim, self.b_max,
                             semantic=self.semantic_dim > 0, sharded=True)
            return ps, _local_meta(ps, cap)

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
        # ordered metadata all-gather (one thread: the gloo calls run in step
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

    def train_native(self, graph, weights, n_steps: int, batch: int, n_neg: int, first_tag: int,
                     producers: int = 0, in_flight: int = 0, steady_from: int = 0) -> np.ndarray:
        """The sharded trainer loop in libngdb (ngdb_shard_train_run; NCCL
        transport): producer threads sample + plan + pack, an exchange thread
        all-gathers the packed records over the context's metadata
        communicator and builds the owner lists, the calling thread launches
        each step. Batch of step s: Rng(3).fork((first_tag + s) * world + rank).
        Returns the per-step loss sums of this rank (steady_from: as Engine.train)."""
        from ._native import TrainOpts
        if not self.comm.nccl:
            raise RuntimeError("train_native needs the NCCL transport")
        w = np.ascontiguousarray(weights, dtype=np.float64)
        opts = TrainOpts(_p(w, C.c_double), batch, n_neg, self.b_max, producers, 0, 3, first_tag,
                         in_flight, 0, steady_from)
        sums = np.zeros(n_steps, np.float64)
        timings = (C.c_double * 8)()
        check(lib.ngdb_shard_train_run(self._h, graph._h, C.byref(opts), self.step_count, n_steps,
                                       _p(sums, C.c_double), timings))
        self.step_count += n_steps
        self.last_timings = {"plan_wait_s": timings[0], "submit_s": timings[1],
                             "collect_wait_s": timings[2], "exchange_s": timings[3],
                             "begin_s": timings[4], "producers": int(timings[5]),
                             "steady_s": timings[6], "exec_s": timings[7]}
        return sums

    def capture(self, steps: List[ShardStep]) -> List["ShardGraph"]:
        """Resident copies of `steps`, each captured with its NCCL collectives
        into one CUDA graph by libngdb (ngdb_shard_step_capture). Every resident
        step is created — and the context's buffers sized for all of them —
        before the first capture, so no later growth invalidates a graph."""
        if not self.comm.nccl:
            raise RuntimeError("graph capture of the sharded step needs the NCCL transport")
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
    into one CUDA graph (ngdb_shard_step_capture). replay(step_no) sets the Adam
    step scalars and launches the graph: no host work per stage."""

    def __init__(self, eng: ShardedEngine, handle, n_queries: int):
        self._h = handle  # owned from here on
        self.eng = eng
        self.n_queries = n_queries
        eng.torch.cuda.synchronize()
        check(lib.ngdb_shard_step_capture(eng._h, self._h))

    def replay(self, step_no: int) -> None:
        check(lib.ngdb_shard_step_replay(self.eng._h, self._h, step_no))

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            lib.ngdb_shard_step_destroy(self._h)
            self._h = None


def _host_stages(eng: ShardedEngine, b: ShardBuffers, send_cnt, recv_cnt) -> None:
    """The device stages with host-staged collectives between them (transport
    "host"; the NCCL transport runs the same sequence inside libngdb)."""
    t = {n: _device_view(eng.torch, getattr(b, n), getattr(b, "n_" + n)) for n in SHARD_BUFFERS}
    run = lambda stage: check(lib.ngdb_shard_run(eng._h, FORWARD_STAGES[stage]))  # noqa: E731
    comm = eng.comm
    ew = 2 * eng.dim if eng.backbone == "betae" else eng.dim  # operator entity row width
    run("anchor_pack")
    comm.all_to_all_v(t["anchor_rows"], t["anchor_send"], send_cnt * ew, recv_cnt * ew)
    run("forward")
    run("query_pack")
    comm.all_gather(t["query_all"], t["query_mine"])
    run("score")
    comm.reduce_scatter(t["dq_mine"], t["dq_part"])
    run("score_done")
    run("backward")
    run("grad_pack")
    comm.all_to_all_v(t["grad_all"], t["grad_send"], recv_cnt * ew, send_cnt * ew)
    if eng.semantic_dim:
        run("fuse_bwd")
    comm.all_reduce(t["reduce"])


def gather_entity_table(comm: Comm, local: np.ndarray, n_entities: int) -> Optional[np.ndarray]:
    """Reassemble the full entity table (rank 0 gets it; others None)."""
    parts = [None] * comm.world
    comm.dist.all_gather_object(parts, local, group=comm.meta_group)
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
