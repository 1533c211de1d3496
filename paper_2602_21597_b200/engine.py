"""Python mirror of the reference interface for the training step.

Names follow the reference C++ API (kg.hpp / query.hpp) and the SPEC's trainer,
sampler and scheduler operations; everything computes in the native library
(host C++ planner + sm_100a kernels). numpy arrays are the only currency.
"""
from __future__ import annotations

import ctypes as C
import itertools
import json
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np

from ._native import (ModelDesc, NodeDesc, PoolDesc, StepPlan, TrainFeedback, TrainOpts, check,
                      lib)

# query.hpp:14-29 enum order == index order of π
PATTERNS = ["1p", "2p", "3p", "2i", "3i", "pi", "ip", "2u", "up", "2in", "3in", "pin", "pni", "inp"]
PATTERN_ARITY = {  # (anchors, relations)
    "1p": (1, 1), "2p": (1, 2), "3p": (1, 3), "2i": (2, 2), "3i": (3, 3), "pi": (2, 3),
    "ip": (2, 3), "2u": (2, 2), "up": (2, 3), "2in": (2, 2), "3in": (3, 3), "pin": (2, 3),
    "pni": (2, 3), "inp": (2, 3)}
BACKBONES = {"gqe": 0, "q2b": 1, "betae": 2}
OP_KINDS = ["EmbedAnchor", "FuseSemantic", "Project", "Negate", "Intersect", "Score",
            "UnionScore", "Loss"]


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


def pattern_weights(mix: Sequence[str]) -> np.ndarray:
    """Uniform π over the given patterns (SamplingDistribution::uniform_over)."""
    w = np.zeros(14, dtype=np.float64)
    for p in mix:
        w[PATTERNS.index(p)] += 1.0 / len(mix)
    return w


class DifficultyTracker:
    """DifficultyTracker: per-pattern EMA of the training loss
    plus the adaptive rule's knobs (decay 0.9, temperature η 1.0, floor ε 0.01;
    SPEC.md:244). State lives in numpy arrays the C loop updates in place."""

    def __init__(self, decay: float = 0.9, eta: float = 1.0, floor: float = 0.01):
        self.decay, self.eta, self.floor = decay, eta, floor
        self.ema_loss = np.zeros(14, dtype=np.float64)
        self.observations = np.zeros(14, dtype=np.int64)

    def record(self, pattern: int, loss: float) -> None:
        """record_difficulty; NonFiniteLoss on a bad loss."""
        check(lib.ngdb_record_difficulty(_p(self.ema_loss, C.c_double),
                                         _p(self.observations, C.c_int64), self.decay,
                                         int(pattern), float(loss)))

    def distribution(self, base: Optional[np.ndarray] = None) -> np.ndarray:
        """update_distribution over the support of `base`."""
        out = np.zeros(14, dtype=np.float64)
        b = None if base is None else np.ascontiguousarray(base, dtype=np.float64)
        check(lib.ngdb_update_distribution(_p(self.ema_loss, C.c_double),
                                           _p(self.observations, C.c_int64), self.eta,
                                           self.floor, _p(b, C.c_double) if b is not None else None,
                                           _p(out, C.c_double)))
        return out


class Graph:
    """GraphSplit (kg.hpp:72-77): train graph, valid/test edges, full graph."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def synthetic(cls, shape: str, seed: int = 1) -> "Graph":
        h = C.c_void_p()
        check(lib.ngdb_graph_synthetic(shape.encode(), seed, C.byref(h)))
        return cls(h)

    @classmethod
    def from_triples(cls, n_entities: int, n_relations: int, train: np.ndarray,
                     valid: Optional[np.ndarray] = None, test: Optional[np.ndarray] = None) -> "Graph":
        def arr(x):
            return np.ascontiguousarray(np.zeros((0, 3)) if x is None else x, dtype=np.int32)
        tr, va, te = arr(train), arr(valid), arr(test)
        h = C.c_void_p()
        check(lib.ngdb_graph_from_triples(n_entities, n_relations, _p(tr, C.c_int32), len(tr),
                                          _p(va, C.c_int32), len(va), _p(te, C.c_int32), len(te),
                                          C.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, directory: str) -> "Graph":
        h = C.c_void_p()
        check(lib.ngdb_graph_load(directory.encode(), C.byref(h)))
        return cls(h)

    def info(self) -> Dict[str, int]:
        ne, nr = C.c_int32(), C.c_int32()
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.ngdb_graph_info(self._h, C.byref(ne), C.byref(nr), C.byref(a), C.byref(b),
                                  C.byref(c)))
        return {"n_entities": ne.value, "n_relations": nr.value, "n_train": a.value,
                "n_valid": b.value, "n_test": c.value}

    def triples(self, split: int = 0) -> np.ndarray:
        info = self.info()
        n = [info["n_train"], info["n_valid"], info["n_test"]][split]
        out = np.zeros((n, 3), dtype=np.int32)
        check(lib.ngdb_graph_triples(self._h, split, _p(out, C.c_int32), n))
        return out

    def answer(self, pattern: str, anchors, relations, full: bool = False) -> np.ndarray:
        a = np.array(list(anchors) + [-1] * 3, dtype=np.int32)[:3]
        r = np.array(list(relations) + [-1] * 4, dtype=np.int32)[:4]
        n = C.c_int64()
        cap = self.info()["n_entities"]
        out = np.zeros(cap, dtype=np.int32)
        check(lib.ngdb_graph_answer(self._h, int(full), PATTERNS.index(pattern), _p(a, C.c_int32),
                                    _p(r, C.c_int32), _p(out, C.c_int32), cap, C.byref(n)))
        return out[: n.value].copy()

    def predictive_answers(self, pattern: str, anchors, relations):
        """(obs, miss): answers on the train graph, and the full-graph answers
        missing from it (kg.hpp:87-89)."""
        a = np.array(list(anchors) + [-1] * 3, dtype=np.int32)[:3]
        r = np.array(list(relations) + [-1] * 4, dtype=np.int32)[:4]
        cap = self.info()["n_entities"]
        obs, miss = np.zeros(cap, dtype=np.int32), np.zeros(cap, dtype=np.int32)
        no, nm = C.c_int64(), C.c_int64()
        check(lib.ngdb_graph_predictive_answers(self._h, PATTERNS.index(pattern), _p(a, C.c_int32),
                                                _p(r, C.c_int32), _p(obs, C.c_int32), cap,
                                                C.byref(no), _p(miss, C.c_int32), cap,
                                                C.byref(nm)))
        return obs[: no.value].copy(), miss[: nm.value].copy()

    def __del__(self):
        if getattr(self, "_h", None):
            lib.ngdb_graph_destroy(self._h)
            self._h = None


@dataclass
class BatchArrays:
    patterns: np.ndarray   # [B] int32 (enum index)
    anchors: np.ndarray    # [B,3] int32, -1 padded
    relations: np.ndarray  # [B,4] int32, -1 padded
    positives: np.ndarray  # [B]
    negatives: np.ndarray  # [B,K]


class Batch:
    """A sampled training batch: queries, walked answers (positives), negatives."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def sample(cls, graph: Graph, weights: np.ndarray, b: int, n_neg: int, seed: int = 3,
               tag: int = 0) -> "Batch":
        w = np.ascontiguousarray(weights, dtype=np.float64)
        h = C.c_void_p()
        check(lib.ngdb_batch_sample(graph._h, _p(w, C.c_double), b, n_neg, seed, tag, C.byref(h)))
        return cls(h)

    @classmethod
    def from_arrays(cls, arrs: BatchArrays) -> "Batch":
        b = len(arrs.patterns)
        k = arrs.negatives.shape[1]
        cv = [np.ascontiguousarray(x, dtype=np.int32) for x in
              (arrs.patterns, arrs.anchors, arrs.relations, arrs.positives, arrs.negatives)]
        h = C.c_void_p()
        check(lib.ngdb_batch_from_arrays(b, _p(cv[0], C.c_int32), _p(cv[1], C.c_int32),
                                         _p(cv[2], C.c_int32), _p(cv[3], C.c_int32), k,
                                         _p(cv[4], C.c_int32), C.byref(h)))
        return cls(h)

    def arrays(self) -> BatchArrays:
        b, k = C.c_int32(), C.c_int32()
        check(lib.ngdb_batch_info(self._h, C.byref(b), C.byref(k)))
        B, K = b.value, k.value
        out = BatchArrays(np.zeros(B, np.int32), np.zeros((B, 3), np.int32),
                          np.zeros((B, 4), np.int32), np.zeros(B, np.int32),
                          np.zeros((B, K), np.int32))
        check(lib.ngdb_batch_arrays(self._h, _p(out.patterns, C.c_int32), _p(out.anchors, C.c_int32),
                                    _p(out.relations, C.c_int32), _p(out.positives, C.c_int32),
                                    _p(out.negatives, C.c_int32)))
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            lib.ngdb_batch_destroy(self._h)
            self._h = None


class PlannedStep:
    """A step planned by the host Max-Fillness scheduler (trace + device plan)."""

    def __init__(self, batch: Batch, backbone: str, dim: int, b_max: int = 512,
                 semantic: bool = False, sharded: bool = False, query_level: bool = False,
                 device_reuse: bool = False):
        """query_level: the SPEC's query-level baseline executor.
        device_reuse: device arena slabs reused along the Eq. 7 free list
        (default: private slabs, so independent pools can run concurrently)."""
        h = C.c_void_p()
        check(lib.ngdb_step_build_ex(batch._h, BACKBONES[backbone], dim, b_max,
                                     int(semantic) | (2 if sharded else 0) |
                                     (4 if query_level else 0) | (8 if device_reuse else 0),
                                     C.byref(h)))
        self._h = h

    def trace(self, with_nodes: bool = False) -> dict:
        n = C.c_int64()
        check(lib.ngdb_step_trace_json(self._h, int(with_nodes), None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(lib.ngdb_step_trace_json(self._h, int(with_nodes), buf, n.value + 1, C.byref(n)))
        text = buf.value.decode()
        if with_nodes:
            head, nodes = text.split("\n", 1)
            tr = json.loads(head)
            for rec, nd in zip(tr["records"], json.loads(nodes)):
                rec["nodes"] = nd
            return tr
        return json.loads(text)

    def view(self) -> StepPlan:
        v = StepPlan()
        check(lib.ngdb_step_view(self._h, C.byref(v)))
        return v

    def __del__(self):
        if getattr(self, "_h", None):
            lib.ngdb_step_destroy(self._h)
            self._h = None


def rank_metrics(ranks: Sequence[int]) -> Dict[str, float]:
    """MRR and Hits@{1,3,10} of filtered ranks (SPEC.md:625-630 EvalReport)."""
    r = np.asarray(ranks, dtype=np.float64)
    if r.size == 0:
        return {"mrr": 0.0, "hits@1": 0.0, "hits@3": 0.0, "hits@10": 0.0, "count": 0}
    return {"mrr": float(np.mean(1.0 / r)), "hits@1": float(np.mean(r <= 1)),
            "hits@3": float(np.mean(r <= 3)), "hits@10": float(np.mean(r <= 10)),
            "count": int(r.size)}


def param_specs(backbone: str, n_entities: int, n_relations: int, dim: int,
                semantic_dim: int = 0) -> List[tuple]:
    """(name, rows, cols, sparse) in registry order (trainer.hpp param_specs)."""
    base = _backbone_specs(backbone, n_entities, n_relations, dim)
    if semantic_dim:
        base += [("fus_f", dim, semantic_dim, False), ("fus_wp", dim, 2 * dim, False),
                 ("fus_bp", 1, dim, False)]
        if backbone == "betae":  # Psi_theta (Eq. 3); h is d wide
            base[0] = ("entity", n_entities, dim, True)
            base += [("fus_psi", 2 * dim, dim, False), ("fus_psi_b", 1, 2 * dim, False)]
    return base


def _backbone_specs(backbone, n_entities, n_relations, dim):
    if backbone == "gqe":
        return [("entity", n_entities, dim, True), ("relation", n_relations, dim, True),
                ("int_w1", dim, dim, False), ("int_w2", dim, dim, False)]
    if backbone == "q2b":
        out = [("entity", n_entities, dim, True), ("relation", n_relations, 2 * dim, True)]
        for n in ("att_w1", "att_b1", "att_w2", "att_b2", "off_w1", "off_b1", "off_w2", "off_b2"):
            out.append((n, 1 if "_b" in n else dim, dim, False))
        return out
    if backbone == "betae":
        d = dim
        return [("entity", n_entities, 2 * d, True), ("relation", n_relations, d, True),
                ("prj_w1", 2 * d, 3 * d, False), ("prj_b1", 1, 2 * d, False),
                ("prj_w2", 2 * d, 2 * d, False), ("prj_b2", 1, 2 * d, False),
                ("att_w1", 2 * d, 2 * d, False), ("att_b1", 1, 2 * d, False),
                ("att_w2", d, 2 * d, False), ("att_b2", 1, d, False)]
    raise NotImplementedError(backbone)


def init_params(backbone: str, n_entities: int, n_relations: int, dim: int,
                seed: int = 2, semantic_dim: int = 0) -> Dict[str, np.ndarray]:
    out = {}
    for name, rows, cols, _ in param_specs(backbone, n_entities, n_relations, dim, semantic_dim):
        a = np.zeros((rows, cols), dtype=np.float32)
        check(lib.ngdb_param_init_ex(BACKBONES[backbone], n_entities, n_relations, dim,
                                     semantic_dim, name.encode(), seed, _p(a, C.c_float), a.size))
        out[name] = a
    return out


def semantic_store(n_entities: int, dim: int = 768, seed: int = 5) -> np.ndarray:
    """Synthetic frozen PTE store, N(0,1)/sqrt(dim) rows (host Rng)."""
    out = np.zeros((n_entities, dim), dtype=np.float32)
    check(lib.ngdb_semantic_synth(n_entities, dim, seed, _p(out, C.c_float)))
    return out


def ngse_write(path: str, store: np.ndarray) -> None:
    a = np.ascontiguousarray(store, dtype=np.float32)
    check(lib.ngdb_ngse_write(str(path).encode(), _p(a, C.c_float), a.shape[0], a.shape[1]))


def ngse_read(path: str) -> np.ndarray:
    n, d = C.c_int64(), C.c_int32()
    check(lib.ngdb_ngse_read(str(path).encode(), None, 0, C.byref(n), C.byref(d)))
    out = np.zeros((n.value, d.value), dtype=np.float32)
    check(lib.ngdb_ngse_read(str(path).encode(), _p(out, C.c_float), out.size, C.byref(n),
                             C.byref(d)))
    return out


class Engine:
    """One GPU context (ngdb_ctx): parameters, Adam state, arena, stream."""

    def __init__(self, backbone: str, n_entities: int, n_relations: int, dim: int = 400,
                 n_neg: int = 128, b_max: int = 512, max_queries: int = 512, gamma: float = 12.0,
                 lr: float = 1e-4, alpha_box: float = 0.02, device: int = 0,
                 params: Optional[Dict[str, np.ndarray]] = None, seed: int = 2, debug: bool = False,
                 semantic: Optional[np.ndarray] = None):
        """semantic: frozen store [n_entities][d_l] -> FuseSemantic on anchors and
        candidates."""
        sd = 0 if semantic is None else int(semantic.shape[1])
        d = ModelDesc(BACKBONES[backbone], n_entities, n_relations, dim, n_neg, sd, gamma,
                      alpha_box, lr, 0.9, 0.999, 1e-8, b_max, max_queries, 1, 0)
        self.backbone, self.dim, self.b_max = backbone, dim, b_max
        self.n_entities, self.n_relations, self.semantic_dim = n_entities, n_relations, sd
        self._h = C.c_void_p()
        check(lib.ngdb_ctx_create(C.byref(d), device, C.byref(self._h)))
        self.step_count = 0
        if semantic is not None:
            st = np.ascontiguousarray(semantic, dtype=np.float32)
            check(lib.ngdb_semantic_upload(self._h, _p(st, C.c_float), st.size))
        if params is None:
            params = init_params(backbone, n_entities, n_relations, dim, seed, sd)
        for k, v in params.items():
            self.upload(k, v)
        if debug:
            check(lib.ngdb_set_debug(self._h, 1))

    def upload(self, name: str, value: np.ndarray) -> None:
        a = np.ascontiguousarray(value, dtype=np.float32)
        check(lib.ngdb_param_upload(self._h, name.encode(), _p(a, C.c_float), a.size))

    def download(self, name: str) -> np.ndarray:
        base = name.split(":")[-1]
        spec = {s[0]: s for s in param_specs(self.backbone, self.n_entities, self.n_relations,
                                             self.dim, self.semantic_dim)}[base]
        out = np.zeros((spec[1], spec[2]), dtype=np.float32)
        check(lib.ngdb_param_download(self._h, name.encode(), _p(out, C.c_float), out.size))
        return out

    def train_step(self, batch: Batch) -> np.ndarray:
        """Plan + run one step through the public C ABI; returns per-query losses."""
        arr_b = C.c_int32()
        k = C.c_int32()
        check(lib.ngdb_batch_info(batch._h, C.byref(arr_b), C.byref(k)))
        losses = np.zeros(arr_b.value, dtype=np.float32)
        total = C.c_double()
        self.step_count += 1
        check(lib.ngdb_train_step(self._h, batch._h, self.b_max, self.step_count,
                                  _p(losses, C.c_float), C.byref(total)))
        return losses

    def train(self, graph: Graph, weights: np.ndarray, n_steps: int, batch: int = 512,
              n_neg: int = 128, seed: int = 3, first_tag: int = 0, n_producers: int = 0,
              queue_depth: int = 0, per_query: bool = False, in_flight: int = 0,
              graphs: bool = True, adaptive: bool = False, refresh_every: int = 100,
              tracker: Optional["DifficultyTracker"] = None, metrics_path: Optional[str] = None,
              checkpoint_path: Optional[str] = None, checkpoint_every: int = 0,
              config_hash: int = 0, pi_per_step: bool = False, steady_from: int = 0):
        """The trainer loop: n_steps steps of batches sampled
        from Rng(seed).fork(first_tag + i) by host producer threads, planned,
        uploaded and run back to back (ngdb_train_run_ex), with the trainer's
        feedback paths: the difficulty tracker (always updated; pass `tracker`
        to keep its state across calls), adaptive π refreshed every
        `refresh_every` steps, a JSON-lines metrics log
         and a checkpoint cadence. Returns the
        per-step loss sums (plus [n_steps][batch] per-query losses with
        per_query=True, plus the [n_steps][14] π of each batch with
        pi_per_step=True). steady_from > 0: last_timings['steady_s'] = host
        seconds from the loop reaching step steady_from to the end (the
        steady-state window after warm-up steps of the same call)."""
        w = np.ascontiguousarray(weights, dtype=np.float64)
        opts = TrainOpts(_p(w, C.c_double), batch, n_neg, self.b_max, n_producers, queue_depth,
                         seed, first_tag, in_flight, 0 if graphs else 1, steady_from)
        tr = tracker if tracker is not None else DifficultyTracker()
        pis = np.zeros((n_steps, 14), dtype=np.float64)
        fb = TrainFeedback(1 if adaptive else 0, refresh_every, tr.decay, tr.eta, tr.floor,
                           _p(tr.ema_loss, C.c_double), _p(tr.observations, C.c_int64),
                           _p(pis, C.c_double),
                           str(metrics_path).encode() if metrics_path else None,
                           str(checkpoint_path).encode() if checkpoint_path else None,
                           checkpoint_every, config_hash)
        sums = np.zeros(n_steps, dtype=np.float64)
        pq = np.zeros((n_steps, batch), dtype=np.float32) if per_query else None
        timings = (C.c_double * 7)()
        check(lib.ngdb_train_run_ex(self._h, graph._h, C.byref(opts), C.byref(fb),
                                    self.step_count, n_steps, _p(sums, C.c_double),
                                    _p(pq, C.c_float) if pq is not None else None, timings))
        self.step_count += n_steps
        # host seconds of the calling thread: waiting for plans, submitting, waiting for results
        self.last_timings = {"plan_wait_s": timings[0], "submit_s": timings[1],
                             "collect_wait_s": timings[2], "submit_begin_s": timings[3],
                             "submit_pools_s": timings[4], "submit_optimizer_s": timings[5],
                             "steady_s": timings[6]}
        out = (sums,)
        if per_query:
            out += (pq,)
        if pi_per_step:
            out += (pis,)
        return out if len(out) > 1 else sums

    def save_checkpoint(self, path: str, config_hash: int = 0) -> None:
        """Parameters, Adam moments and the step counter as an NGCK blob."""
        check(lib.ngdb_checkpoint_save(self._h, str(path).encode(), config_hash, self.step_count))

    def load_checkpoint(self, path: str, config_hash: int = 0) -> int:
        """Restore a blob written by save_checkpoint; resumes the step counter."""
        st = C.c_int64()
        check(lib.ngdb_checkpoint_load(self._h, str(path).encode(), config_hash, C.byref(st)))
        self.step_count = st.value
        return st.value

    def query_embeddings(self, step: "PlannedStep"):
        """Forward pools of a planned batch only (no backward, no optimizer:
        parameters unchanged) -> {query index: [n_branches][wq]} embeddings read
        from the score slots (SPEC.md:620-622 `evaluate`: score with the
        backbone's distance). Union queries have one row per DNF branch.
        Returns (embeddings, per-query forward losses)."""
        v = step.view()
        check(lib.ngdb_step_begin(self._h, C.byref(v)))
        for i in range(v.n_pools):
            if v.pools[i].dir == 0:
                check(lib.ngdb_exec_pool(self._h, C.byref(v.pools[i])))
        losses = np.zeros(v.n_queries, dtype=np.float32)
        total, bad = C.c_double(), C.c_int32()
        check(lib.ngdb_step_end(self._h, _p(losses, C.c_float), v.n_queries, C.byref(total),
                                C.byref(bad)))
        wq = self.dim if self.backbone == "gqe" else 2 * self.dim
        emb = np.zeros((max(v.n_score_slots, 1), wq), dtype=np.float32)
        check(lib.ngdb_read_score_queries(self._h, _p(emb, C.c_float), v.n_score_slots))
        slots: Dict[int, List[int]] = {}
        for i in range(v.n_pools):
            p = v.pools[i]
            if p.dir != 0 or p.kind not in (OP_KINDS.index("Score"), OP_KINDS.index("Loss")):
                continue
            for j in range(p.first, p.first + p.count):
                nd = v.nodes[j]
                if nd.aux >= 0:
                    slots.setdefault(int(nd.id), []).append(int(nd.aux))
        return {q: emb[sorted(ss)] for q, ss in slots.items()}, losses

    def eval_ranks_multi(self, embeddings: Sequence[np.ndarray], targets: Sequence[int],
                         filters: Sequence[Sequence[int]]) -> np.ndarray:
        """eval_ranks for queries given as [n_branches][wq] embeddings (union
        patterns: one per DNF branch; an entity's distance is the nearest
        branch's), e.g. the output of query_embeddings (ngdb_eval_ranks_multi)."""
        n = len(targets)
        units = np.ascontiguousarray(np.concatenate([np.atleast_2d(e) for e in embeddings])
                                     if n else np.zeros((1, 1)), dtype=np.float32)
        uo = np.zeros(n + 1, dtype=np.int32)
        np.cumsum([np.atleast_2d(e).shape[0] for e in embeddings], out=uo[1:])
        off = np.zeros(n + 1, dtype=np.int32)
        np.cumsum(np.fromiter(map(len, filters), dtype=np.int64, count=n), out=off[1:])
        ids = np.fromiter(itertools.chain.from_iterable(filters), dtype=np.int32,
                          count=int(off[-1]))
        if ids.size == 0:
            ids = np.zeros(1, dtype=np.int32)
        t = np.ascontiguousarray(targets, dtype=np.int32)
        ranks = np.zeros(n, dtype=np.int32)
        check(lib.ngdb_eval_ranks_multi(self._h, _p(units, C.c_float), n, _p(uo, C.c_int32),
                                        _p(t, C.c_int32), _p(off, C.c_int32), _p(ids, C.c_int32),
                                        _p(ranks, C.c_int32)))
        return ranks

    def eval_entity_table(self):
        """The evaluator's entity side for the current parameters
        (ngdb_eval_entity_table): BetaE (T [n][2d], C [n]) of the linearised
        KL; fusion (fused rows [n][d], None); GQE / Q2B (entity table, None)."""
        n = self.n_entities
        w = 2 * self.dim if self.backbone == "betae" else self.dim
        rows = np.zeros((n, w), dtype=np.float32)
        consts = np.zeros(n, dtype=np.float32) if self.backbone == "betae" else None
        check(lib.ngdb_eval_entity_table(self._h, _p(rows, C.c_float), rows.size,
                                         _p(consts, C.c_float) if consts is not None else None,
                                         n if consts is not None else 0))
        return rows, consts

    def eval_ranks(self, queries: np.ndarray, targets: Sequence[int],
                   filters: Sequence[Sequence[int]]) -> np.ndarray:
        """Filtered ranks of `targets` among all entities (SPEC.md:614-618,
        `filtered_rank`; score = -distance, mean-rank ties) for query embeddings
        [n][wq] (GQE: q; Q2B: centre | offset) against the current entity table
        (ngdb_eval_ranks). filters[i] is query i's filter set (other known answers)."""
        n = len(targets)
        off = np.zeros(n + 1, dtype=np.int32)
        np.cumsum(np.fromiter(map(len, filters), dtype=np.int64, count=n), out=off[1:])
        ids = np.fromiter(itertools.chain.from_iterable(filters), dtype=np.int32,
                          count=int(off[-1]))
        return self.eval_ranks_csr(queries, targets, off, ids)

    def eval_ranks_csr(self, queries: np.ndarray, targets: np.ndarray, filter_offsets: np.ndarray,
                       filter_ids: np.ndarray) -> np.ndarray:
        """eval_ranks with the filter sets as a CSR (offsets [n+1], ids)."""
        q = np.ascontiguousarray(queries, dtype=np.float32)
        n = q.shape[0]
        t = np.ascontiguousarray(targets, dtype=np.int32)
        off = np.ascontiguousarray(filter_offsets, dtype=np.int32)
        ids = np.ascontiguousarray(filter_ids, dtype=np.int32)
        if ids.size == 0:
            ids = np.zeros(1, dtype=np.int32)
        ranks = np.zeros(n, dtype=np.int32)
        check(lib.ngdb_eval_ranks(self._h, _p(q, C.c_float), n, _p(t, C.c_int32),
                                  _p(off, C.c_int32), _p(ids, C.c_int32), _p(ranks, C.c_int32)))
        return ranks

    def run_step(self, step: PlannedStep, n_queries: int) -> np.ndarray:
        losses = np.zeros(n_queries, dtype=np.float32)
        total = C.c_double()
        self.step_count += 1
        check(lib.ngdb_run_step(self._h, step._h, self.step_count, _p(losses, C.c_float),
                                C.byref(total)))
        return losses

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.ngdb_ctx_destroy(self._h)
            self._h = None
