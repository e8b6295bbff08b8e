"""Does tcgen05 kind::tf32 truncate or round fp32 operands?  (dev experiment)"""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from debug_gemm import G, rel
from paper_2401_11202_b200 import runtime as R

dev = R.Device(0)
M = N = 128
K = 32
# 1 + 3*2^-12: 0.75 tf32-ulp above 1 -> truncation gives 1, round-to-nearest gives 1 + 2^-10
a = np.full((M, K), 1 + 3 * 2.0 ** -12, np.float32)
b = np.ones((K, N), np.float32)
for flag in (0, 256 | 1):          # keep_raw_hi, promote 1
    # split disabled entirely is not available; use keep_raw_hi: hi slot holds raw x, lo = x - trunc(x)
    g = G(dev, a, b, promote=flag)
    C = g.run()
    g.close()
    print("flag", flag, "C[0,0] =", repr(float(C[0, 0])), "exact K*a =", K * float(a[0, 0]))
rng = np.random.default_rng(0)
A = rng.standard_normal((512, 4096)).astype(np.float32)
B = rng.standard_normal((4096, 512)).astype(np.float32)
ref = A.astype(np.float64) @ B
for flag in (0, 256):
    g = G(dev, A, B, promote=flag)
    print("random K=4096 flag", flag, "rel err", rel(g.run(), ref))
    g.close()
