import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2412_20796_b200 import chg
ctx = chg.Context(0)
rng = np.random.default_rng(0)
for kind in (0, 1):
    for (M, K, N) in [(128, 32, 64), (300, 64, 128), (1000, 192, 128), (777, 256, 256), (64, 64, 64)]:
        A = rng.normal(size=(M, K)).astype(np.float32)
        W = rng.normal(size=(K, N) if kind == 0 else (M, N)).astype(np.float32)
        ref = A.astype(np.float64) @ W if kind == 0 else A.astype(np.float64).T @ W
        for eng in (0, 2):
            try:
                o = ctx.debug_gemm(kind, eng, A, W)
                print(kind, eng, (M, K, N), "rel", np.linalg.norm(o - ref) / np.linalg.norm(ref), "max|o|", np.abs(o).max())
            except chg.ChgError as e:
                print(kind, eng, (M, K, N), "ERR", e)
# bias path through the gated-MLP weight-gradient call sites is covered by the TF32 parity tests
