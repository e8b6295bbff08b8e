"""GEMM timing on C2 shapes and a large square (dev tool)."""
import os
import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tools")
from debug_gemm import G, rel
from paper_2401_11202_b200 import runtime as R
dev = R.Device(0)
rng = np.random.default_rng(0)
print("SPX_GEMM_PIPE", os.environ.get("SPX_GEMM_PIPE"))
SHAPES = [(2048, 4096, 1024, False, False), (2048, 1024, 4096, False, True),
          (1024, 1024, 2048, True, False), (4096, 4096, 4096, False, False),
          (1024, 2048, 1024, False, False), (1024, 1024, 1024, True, False), (2048, 1024, 1024, False, False),
          (1024, 512, 1024, False, False), (1024, 1024, 512, False, False), (1024, 1024, 2048, False, False),
          (1024, 256, 1024, False, False), (1024, 1024, 256, False, False)]
if os.environ.get("SMALL"):
    SHAPES = [(512, 1024, 4096, False, True), (512, 1024, 1024, False, False), (1024, 1024, 512, True, False),
              (512, 4096, 1024, False, False), (1024, 1024, 2048, False, False), (1024, 512, 1024, False, False),
              (1024, 2048, 1024, False, False)]
if os.environ.get("SHAPES"):
    SHAPES = [SHAPES[int(i)] for i in os.environ["SHAPES"].split(",")]
ITERS = int(os.environ.get("ITERS", "10"))
PATHS = [int(x) for x in os.environ.get("GPATHS", "1,3").split(",")]
BNS = os.environ.get("BNS", "").split(",") if os.environ.get("BNS") else [None]
for (M, N, K, at, bt), path, bn in [(s, p, b) for s in SHAPES for p in PATHS for b in BNS]:
    if bn: os.environ["SPX_H3_BN"] = bn
    A = rng.standard_normal((K, M) if at else (M, K)).astype(np.float32)
    B = rng.standard_normal((N, K) if bt else (K, N)).astype(np.float32)
    g = G(dev, A, B, at, bt, path=path)
    C = g.run()
    AA = A.T if at else A
    BB = B.T if bt else B
    err = rel(C, AA.astype(np.float64) @ BB)
    ms = g.time_ms(ITERS)
    g.close()
    print(f"path {path} bn {bn} {M}x{N}x{K} a_mn={int(at)} b_k={int(bt)} {ms*1e3:8.1f} us {2*M*N*K/ms/1e9:6.1f} TF fp32-eq "
          f" rel err {err:.2e}", flush=True)
