"""ctypes binding of the product library (include/ngdb/ngdb_cuda.h + ngdb_host.h).

The library is built in-tree by ``make lib`` (``__graft_entry__.build()``).
There is no Python or CPU fallback for the compute path: if the library is
missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_lib" / "libngdb_b200.so"

i32, i64, u64, f32, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double
P = C.POINTER


class ModelDesc(C.Structure):
    _fields_ = [
        ("backbone", i32), ("n_entities", i32), ("n_relations", i32), ("dim", i32),
        ("n_neg", i32), ("semantic_dim", i32), ("gamma", f32), ("alpha_box", f32),
        ("lr", f32), ("beta1", f32), ("beta2", f32), ("eps_adam", f32),
        ("max_batch", i32), ("max_queries", i32), ("world", i32), ("rank", i32),
    ]


class NodeDesc(C.Structure):
    _fields_ = [("out", i32), ("in_", i32 * 3), ("grad", i32), ("self_", i32), ("id", i32),
                ("aux", i32)]


class PoolDesc(C.Structure):
    _fields_ = [("kind", i32), ("dir", i32), ("k", i32), ("first", i32), ("count", i32),
                ("cycle", i32)]


class StepPlan(C.Structure):
    _fields_ = [
        ("n_queries", i32), ("n_candidates", i32), ("candidates", P(i32)),
        ("n_pools", i32), ("pools", P(PoolDesc)), ("n_nodes", i32), ("nodes", P(NodeDesc)),
        ("arena_elems", i64), ("n_score_slots", i32), ("n_anchor_slots", i32),
        ("n_project_slots", i32), ("n_entity_rows", i32), ("entity_rows", P(i32)),
        ("entity_seg", P(i32)), ("entity_contrib", P(i32)), ("n_relation_rows", i32),
        ("relation_rows", P(i32)), ("relation_seg", P(i32)), ("relation_contrib", P(i32)),
        ("pool_dep_off", P(i32)), ("pool_deps", P(i32)),
    ]


class ShardPlan(C.Structure):
    _fields_ = [
        ("world", i32), ("rank", i32), ("batch", i32), ("max_anchors", i32), ("max_slots", i32),
        ("n_candidates", i32), ("anchor_ids", P(i32)), ("unit_k", P(i32)),
        ("unit_slots", P(i32)), ("cand", P(i32)), ("unit_off", P(i32)), ("owned", P(i32)),
        ("n_rows", i32), ("rows", P(i32)), ("seg", P(i32)), ("contrib", P(i32)),
        ("send_cnt", P(i32)), ("recv_cnt", P(i32)), ("n_send", i32), ("n_recv", i32),
        ("send_rows", P(i32)), ("recv_slot", P(i32)), ("n_anchor_pos", i32),
        ("anchor_pos", P(i32)),
    ]


class TrainOpts(C.Structure):
    _fields_ = [("pattern_weights", P(f64)), ("batch", i32), ("n_neg", i32), ("b_max", i32),
                ("n_producers", i32), ("queue_depth", i32), ("seed", u64), ("first_tag", u64),
                ("in_flight", i32), ("flags", i32), ("steady_from", i32)]


class TrainFeedback(C.Structure):
    _fields_ = [("adaptive", i32), ("refresh_every", i32), ("decay", f64), ("eta", f64),
                ("floor", f64), ("ema_loss", P(f64)), ("observations", P(i64)),
                ("pi_per_step", P(f64)), ("metrics_path", C.c_char_p),
                ("checkpoint_path", C.c_char_p), ("checkpoint_every", i32), ("config_hash", u64)]


SHARD_BUFFERS = ("anchor_send", "anchor_rows", "query_mine", "query_all", "dq_part", "dq_mine",
                 "grad_send", "grad_all", "reduce")


class ShardBuffers(C.Structure):
    _fields_ = ([(n, C.c_void_p) for n in SHARD_BUFFERS] +
                [("n_" + n, i64) for n in SHARD_BUFFERS])


# (name, restype, argtypes) for every exported entry point of include/ngdb/*.h
SIGNATURES = {
    # ngdb_cuda.h
    "ngdb_last_error": (C.c_char_p, []),
    "ngdb_ctx_create": (C.c_int, [P(ModelDesc), C.c_int, P(C.c_void_p)]),
    "ngdb_ctx_destroy": (C.c_int, [C.c_void_p]),
    "ngdb_ctx_desc": (C.c_int, [C.c_void_p, P(ModelDesc)]),
    "ngdb_param_count": (C.c_int, [C.c_void_p, P(i32)]),
    "ngdb_param_info": (C.c_int, [C.c_void_p, i32, P(C.c_char_p), P(i64), P(i64), P(i32)]),
    "ngdb_param_upload": (C.c_int, [C.c_void_p, C.c_char_p, P(f32), i64]),
    "ngdb_param_download": (C.c_int, [C.c_void_p, C.c_char_p, P(f32), i64]),
    "ngdb_semantic_upload": (C.c_int, [C.c_void_p, P(f32), i64]),
    "ngdb_set_debug": (C.c_int, [C.c_void_p, i32]),
    "ngdb_step_begin": (C.c_int, [C.c_void_p, P(StepPlan)]),
    "ngdb_step_begin_ex": (C.c_int, [C.c_void_p, P(StepPlan), i32]),
    "ngdb_exec_pool": (C.c_int, [C.c_void_p, P(PoolDesc)]),
    "ngdb_optimizer_step": (C.c_int, [C.c_void_p, i64]),
    "ngdb_step_end": (C.c_int, [C.c_void_p, P(f32), i32, P(f64), P(i32)]),
    "ngdb_step_end_async": (C.c_int, [C.c_void_p, P(i64)]),
    "ngdb_step_launch": (C.c_int, [C.c_void_p, i64, i32]),
    "ngdb_step_wait": (C.c_int, [C.c_void_p, i64, P(f32), i32, P(f64), P(i32)]),
    "ngdb_plan_create": (C.c_int, [C.c_void_p, P(StepPlan), P(C.c_void_p)]),
    "ngdb_plan_run": (C.c_int, [C.c_void_p, C.c_void_p, i64]),
    "ngdb_plan_prepare": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ngdb_shard_begin": (C.c_int, [C.c_void_p, P(StepPlan), P(ShardPlan), P(ShardBuffers)]),
    "ngdb_shard_packed_size": (i64, [P(ShardPlan)]),
    "ngdb_shard_pack": (C.c_int, [P(ShardPlan), P(i32), i64]),
    "ngdb_shard_begin_packed": (C.c_int, [C.c_void_p, P(StepPlan), P(i32), i64, P(ShardPlan),
                                          P(i32), i64, P(ShardBuffers)]),
    "ngdb_shard_run": (C.c_int, [C.c_void_p, i32]),
    "ngdb_shard_step_create": (C.c_int, [C.c_void_p, P(StepPlan), P(ShardPlan), P(C.c_void_p)]),
    "ngdb_shard_step_begin": (C.c_int, [C.c_void_p, C.c_void_p, P(ShardBuffers)]),
    "ngdb_shard_step_destroy": (C.c_int, [C.c_void_p]),
    "ngdb_set_step": (C.c_int, [C.c_void_p, i64]),
    "ngdb_shard_optimizer": (C.c_int, [C.c_void_p, i64]),
    "ngdb_exec_flush": (C.c_int, [C.c_void_p]),
    "ngdb_plan_packed_size": (i64, [P(StepPlan)]),
    "ngdb_plan_pack": (C.c_int, [P(StepPlan), P(i32), i64]),
    "ngdb_host_alloc": (C.c_int, [i64, P(C.c_void_p)]),
    "ngdb_host_free": (C.c_int, [C.c_void_p]),
    "ngdb_ctx_pinned_ring": (C.c_int, [C.c_void_p, i64, P(P(i32))]),
    "ngdb_step_begin_packed": (C.c_int, [C.c_void_p, P(StepPlan), P(i32), i64, i32]),
    "ngdb_read_arena": (C.c_int, [C.c_void_p, i64, i64, P(f32)]),
    "ngdb_set_gemm_split": (C.c_int, [i32]),
    "ngdb_comm_unique_id": (C.c_int, [P(C.c_uint8)]),
    "ngdb_comm_init": (C.c_int, [C.c_void_p, P(C.c_uint8)]),
    "ngdb_comm_allgather_i32": (C.c_int, [C.c_void_p, P(i32), i64, P(i32)]),
    "ngdb_shard_step_exec": (C.c_int, [C.c_void_p, i64]),
    "ngdb_shard_step_capture": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ngdb_shard_step_replay": (C.c_int, [C.c_void_p, C.c_void_p, i64]),
    "ngdb_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ngdb_plan_destroy": (C.c_int, [C.c_void_p]),
    "ngdb_sync": (C.c_int, [C.c_void_p]),
    "ngdb_timer_start": (C.c_int, [C.c_void_p]),
    "ngdb_timer_stop": (C.c_int, [C.c_void_p, P(f32)]),
    "ngdb_profile_enable": (C.c_int, [C.c_void_p, i32]),
    "ngdb_profile_read": (C.c_int, [C.c_void_p, i32, P(f64), P(i64), P(f64)]),
    "ngdb_profile_families": (i32, []),
    "ngdb_profile_flops": (C.c_int, [C.c_void_p, i32, P(f64)]),
    "ngdb_profile_family_name": (C.c_char_p, [i32]),
    "ngdb_launch_count": (i64, [C.c_void_p]),
    "ngdb_transfer_bytes": (C.c_int, [C.c_void_p, P(i64), P(i64)]),
    "ngdb_checkpoint_save": (C.c_int, [C.c_void_p, C.c_char_p, u64, i64]),
    "ngdb_checkpoint_load": (C.c_int, [C.c_void_p, C.c_char_p, u64, P(i64)]),
    "ngdb_step_timeline": (C.c_int, [C.c_void_p, P(f64), P(f64), P(i64)]),
    "ngdb_read_score_queries": (C.c_int, [C.c_void_p, P(f32), i64]),
    "ngdb_eval_entity_table": (C.c_int, [C.c_void_p, P(f32), i64, P(f32), i64]),
    "ngdb_eval_ranks_multi": (C.c_int, [C.c_void_p, P(f32), i32, P(i32), P(i32), P(i32), P(i32),
                                        P(i32)]),
    "ngdb_eval_ranks": (C.c_int, [C.c_void_p, P(f32), i32, P(i32), P(i32), P(i32), P(i32)]),
    "ngdb_graph_stats": (C.c_int, [C.c_void_p, P(i64), P(i64)]),
    "ngdb_flush_l2": (C.c_int, [C.c_void_p]),
    # ngdb_host.h
    "ngdb_graph_synthetic": (C.c_int, [C.c_char_p, u64, P(C.c_void_p)]),
    "ngdb_graph_from_triples": (C.c_int, [i32, i32, P(i32), i64, P(i32), i64, P(i32), i64,
                                          P(C.c_void_p)]),
    "ngdb_graph_load": (C.c_int, [C.c_char_p, P(C.c_void_p)]),
    "ngdb_graph_info": (C.c_int, [C.c_void_p, P(i32), P(i32), P(i64), P(i64), P(i64)]),
    "ngdb_graph_triples": (C.c_int, [C.c_void_p, i32, P(i32), i64]),
    "ngdb_graph_answer": (C.c_int, [C.c_void_p, i32, i32, P(i32), P(i32), P(i32), i64, P(i64)]),
    "ngdb_graph_predictive_answers": (C.c_int, [C.c_void_p, i32, P(i32), P(i32), P(i32), i64,
                                                P(i64), P(i32), i64, P(i64)]),
    "ngdb_graph_destroy": (C.c_int, [C.c_void_p]),
    "ngdb_batch_sample": (C.c_int, [C.c_void_p, P(f64), i32, i32, u64, u64, P(C.c_void_p)]),
    "ngdb_batch_from_arrays": (C.c_int, [i32, P(i32), P(i32), P(i32), P(i32), i32, P(i32),
                                         P(C.c_void_p)]),
    "ngdb_batch_info": (C.c_int, [C.c_void_p, P(i32), P(i32)]),
    "ngdb_batch_arrays": (C.c_int, [C.c_void_p, P(i32), P(i32), P(i32), P(i32), P(i32)]),
    "ngdb_batch_destroy": (C.c_int, [C.c_void_p]),
    "ngdb_step_build": (C.c_int, [C.c_void_p, i32, i32, i32, i32, P(C.c_void_p)]),
    "ngdb_step_build_ex": (C.c_int, [C.c_void_p, i32, i32, i32, i32, P(C.c_void_p)]),
    "ngdb_step_view": (C.c_int, [C.c_void_p, P(StepPlan)]),
    "ngdb_step_trace_json": (C.c_int, [C.c_void_p, i32, C.c_char_p, i64, P(i64)]),
    "ngdb_step_destroy": (C.c_int, [C.c_void_p]),
    "ngdb_param_init": (C.c_int, [i32, i32, i32, i32, C.c_char_p, u64, P(f32), i64]),
    "ngdb_param_init_ex": (C.c_int, [i32, i32, i32, i32, i32, C.c_char_p, u64, P(f32), i64]),
    "ngdb_param_init_shard": (C.c_int, [i32, i32, i32, i32, C.c_char_p, u64, i32, i32, P(f32),
                                        i64]),
    "ngdb_step_shard_info": (C.c_int, [C.c_void_p, P(i32), P(i32), P(i32), P(i32)]),
    "ngdb_step_shard_meta": (C.c_int, [C.c_void_p, P(i32), P(i32), P(i32), P(i32)]),
    "ngdb_shard_build": (C.c_int, [i32, i32, i32, i32, i32, i32, P(i32), P(i32), P(i32), P(i32),
                                   P(C.c_void_p)]),
    "ngdb_shard_view": (C.c_int, [C.c_void_p, P(ShardPlan)]),
    "ngdb_shard_meta_stride": (i64, [i32, i32]),
    "ngdb_step_shard_pack": (C.c_int, [C.c_void_p, i32, P(i32), i64]),
    "ngdb_shard_build_packed": (C.c_int, [i32, i32, P(i32), i64, i32, P(C.c_void_p)]),
    "ngdb_shard_destroy": (C.c_int, [C.c_void_p]),
    "ngdb_semantic_synth": (C.c_int, [i32, i32, u64, P(f32)]),
    "ngdb_ngse_write": (C.c_int, [C.c_char_p, P(f32), i64, i32]),
    "ngdb_ngse_read": (C.c_int, [C.c_char_p, P(f32), i64, P(i64), P(i32)]),
    "ngdb_rng_next": (u64, [u64, i64, i32]),
    "ngdb_rng_below": (C.c_int, [u64, P(u64), i32, i32, P(u64)]),
    "ngdb_select_pool": (C.c_int, [P(i64), P(i64), P(i32)]),
    "ngdb_jsonl_roundtrip": (C.c_int, [C.c_char_p, C.c_char_p, i64]),
    "ngdb_train_step": (C.c_int, [C.c_void_p, C.c_void_p, i32, i64, P(f32), P(f64)]),
    "ngdb_train_run_ex": (C.c_int, [C.c_void_p, C.c_void_p, P(TrainOpts), P(TrainFeedback), i64,
                                    i32, P(f64), P(f32), P(f64)]),
    "ngdb_shard_train_run": (C.c_int, [C.c_void_p, C.c_void_p, P(TrainOpts), i64, i32, P(f64),
                                       P(f64)]),
    "ngdb_record_difficulty": (C.c_int, [P(f64), P(i64), f64, i32, f64]),
    "ngdb_update_distribution": (C.c_int, [P(f64), P(i64), f64, f64, P(f64), P(f64)]),
    "ngdb_train_run": (C.c_int, [C.c_void_p, C.c_void_p, P(TrainOpts), i64, i32, P(f64), P(f32),
                                 P(f64)]),
    "ngdb_run_step": (C.c_int, [C.c_void_p, C.c_void_p, i64, P(f32), P(f64)]),
    # test hook (tc_gemm.cu): tcgen05 3xTF32 GEMM on host buffers
    "ngdb_debug_tc_gemm": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     P(f32), C.c_int, P(f32), C.c_int, P(f32), C.c_int, P(f32),
                                     C.c_int]),
}


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make lib` (or __graft_entry__.build()); "
            "the training step has no CPU fallback")
    lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

STATUS = {0: "OK", 1: "ShapeMismatch", 2: "IndexOutOfRange", 3: "ParamOutOfRange",
          4: "DomainError", 5: "MissingKernel", 6: "NonFinite", 7: "ConfigError", 8: "CudaError",
          9: "NoDevice"}


class NgdbError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS.get(code, str(code))


def check(rc: int) -> None:
    if rc != 0:
        raise NgdbError(rc, (lib.ngdb_last_error() or b"").decode(errors="replace"))
