"""tcgen05 3xTF32 GEMM timing on the operator-MLP shapes of the benchmark
configs (CUDA events, back-to-back launches): the TMA warp-specialised kernel
and, with NGDB_GEMM_CPASYNC=1, the cp.async kernel. Prints one JSON line per
shape with achieved algorithmic TFLOP/s (2MNK per problem)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_21597_b200._native import lib  # noqa: E402

SHAPES = [  # (label, M, N, K, batch)
    ("c2 intersect fwd (731 rows, d=400)", 731, 400, 400, 1),
    ("c2 intersect level of 4", 731, 400, 400, 4),
    ("c2 weight grad dW = dY^T X (K = rows)", 400, 400, 731, 2),
    ("c3 project L1 (1434 x 1200 -> 800)", 1434, 800, 1200, 1),
    ("c3 project L2 (1434 x 800 -> 800)", 1434, 800, 800, 1),
    ("c3 project dW1 (800 x 1200, K = 1434)", 800, 1200, 1434, 1),
    ("c4 fusion S M^T (14.5k x 768 -> 400)", 14505, 400, 768, 1),
    ("c4 fusion h W_h^T / dh (14.5k x 400 -> 400)", 14505, 400, 400, 1),
    ("c4 fusion dM = dZ^T S (400 x 768, K = 14.5k)", 400, 768, 14505, 1),
    ("c4 fusion dW_h = dZ^T h (400 x 400, K = 14.5k)", 400, 400, 14505, 1),
    ("c3 psi-free project L1 at 4k rows (4096 x 1200 -> 800)", 4096, 800, 1200, 1),
    ("c4 fusion dM^T = S^T dZ (768 x 400, K = 14.5k)", 768, 400, 14505, 1),
]
if os.environ.get("NGDB_GEMM_SPLIT"):  # fixed split-K (ngdb_set_gemm_split; forces the 80-wide tile)
    lib.ngdb_set_gemm_split(int(os.environ["NGDB_GEMM_SPLIT"]))
f = lib.ngdb_debug_tc_gemm_time
f.argtypes = [C.c_int] * 5 + [C.POINTER(C.c_float)]
kind = ("cpasync" if os.environ.get("NGDB_GEMM_CPASYNC") else "tma" + os.environ.get("NGDB_GEMM_BN", "")) + \
    ("_s" + os.environ["NGDB_GEMM_SPLIT"] if os.environ.get("NGDB_GEMM_SPLIT") else "")
for label, M, N, K, b in SHAPES:
    ms = C.c_float()
    rc = f(M, N, K, b, 50, C.byref(ms))
    tf = 2.0 * M * N * K * b / (ms.value * 1e-3) / 1e12 if rc == 0 else 0.0
    print(json.dumps({"kernel": kind, "shape": label, "M": M, "N": N, "K": K, "batch": b,
                      "rc": rc, "us": ms.value * 1e3, "tflops_alg": tf}), flush=True)
