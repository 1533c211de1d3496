"""B200-native operator-level training step of NGDB-Zoo (arxiv 2602.21597).

Host C++ Max-Fillness planner + hand-written sm_100a kernels behind the C ABI in
include/ngdb/ngdb_cuda.h. See DESIGN.md.
"""
from .engine import (BACKBONES, OP_KINDS, PATTERNS, PATTERN_ARITY, Batch, BatchArrays, DifficultyTracker, Engine,
                     Graph, PlannedStep, init_params, ngse_read, ngse_write, param_specs,
                     pattern_weights, rank_metrics, semantic_store)

__all__ = ["BACKBONES", "OP_KINDS", "PATTERNS", "PATTERN_ARITY", "Batch", "BatchArrays", "DifficultyTracker", "Engine",
           "Graph", "PlannedStep", "init_params", "ngse_read", "ngse_write", "param_specs",
           "pattern_weights", "rank_metrics", "semantic_store"]
