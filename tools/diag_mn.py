import ctypes as C, numpy as np, sys
sys.path.insert(0, '.')
from paper_2602_21597_b200._native import lib
def p(a): return a.ctypes.data_as(C.POINTER(C.c_float))
M, N, K = 128, 160, 128
lib.ngdb_set_gemm_split(1)
for am, bm in [tuple(map(int, sys.argv[1:3]))]:
    A = np.eye(M, K, dtype=np.float32) if bm == 1 else (np.arange(M)[:, None] * 1000 + np.arange(K)[None, :]).astype(np.float32)
    B = (np.arange(N)[:, None] * 1000 + np.arange(K)[None, :]).astype(np.float32) if bm == 1 else np.eye(N, K, dtype=np.float32)
    As = np.ascontiguousarray(A if am == 0 else A.T); Bs = np.ascontiguousarray(B if bm == 0 else B.T)
    Cd = np.zeros((M, N), np.float32)
    rc = lib.ngdb_debug_tc_gemm(M, N, K, am, bm, 0, p(As), As.shape[1], p(Bs), Bs.shape[1], p(Cd), N, None, 0)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    print("am,bm", am, bm, "rc", rc, "maxerr", np.abs(Cd - ref).max())
    np.set_printoptions(linewidth=250, threshold=100000)
    if bm == 1:
        print("C[m][n] should be n*1000+m; rows m=0..9, cols n=0..9 and n=30..35:")
        print(np.round(Cd[:10, :10]).astype(int)); print(np.round(Cd[:10, 30:36]).astype(int))
        print("m=8..12, n=0..4", np.round(Cd[8:13, :5]).astype(int))
        print("m=32..34, n=0..4", np.round(Cd[32:35, :5]).astype(int))
    else:
        print("C[m][n] should be m*1000+n")
        print(np.round(Cd[:10, :10]).astype(int)); print(np.round(Cd[30:36, :6]).astype(int))
        print("m=8..12", np.round(Cd[8:13, :5]).astype(int))
