"""Per-layer latency of a chain of small GEMM + square(+split) layers (the
per-device shapes of C2/C5 at N>=2), CUDA-graph replay with PDL -- how much of
a small GEMM's time is fixed cost (dev tool).

    python tools/gemm_chain.py [M K N LAYERS]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_11202_b200 import runtime as R  # noqa: E402
from paper_2401_11202_b200.evaluator import _Dense  # noqa: E402
from paper_2401_11202_b200.executable import Executable  # noqa: E402
from paper_2401_11202_b200.ir import parse_module  # noqa: E402


def chain(M, K, N, L):
    assert K == N
    t = f"tensor<{M}x{K}xf32>"
    lines = [f"func @main(%x: {t}, %w: tensor<{K}x{N}xf32>) -> {t} {{"]
    prev = "%x"
    for i in range(L):
        lines.append(f"  %m{i} = matmul {prev}, %w : {t}")
        lines.append(f"  %s{i} = mul %m{i}, %m{i} : {t}")
        prev = f"%s{i}"
    lines += [f"  return {prev}", "}", ""]
    return parse_module("\n".join(lines))


def main():
    M, K, N, L = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (1024, 512, 512, 64)))
    dev = R.Device(0)
    m = chain(M, K, N, L)
    ex = Executable(_Dense(m), devices=[0], device=dev)
    rng = np.random.default_rng(0)
    ex.upload_args([{"x": (0.05 * rng.standard_normal((M, K))).astype(np.float32),
                     "w": (0.05 * rng.standard_normal((K, N))).astype(np.float32)}])
    ex.run()
    dev.sync()
    ex.plan.capture()
    for _ in range(3):
        ex.plan.replay()
    dev.sync()
    e0, e1 = dev.event(), dev.event()
    it = 20
    dev.record(e0)
    for _ in range(it):
        ex.plan.replay()
    dev.record(e1)
    dev.sync()
    ms = dev.elapsed_ms(e0, e1) / it
    prof = ex.plan.profile()
    kinds = [k for k, _ in ex.records()]
    g = [t for k, t in zip(kinds, prof) if k == R.K_GEMM]
    e = [t for k, t in zip(kinds, prof) if k == R.K_EW]
    fl = 2.0 * M * K * N * 3
    print(f"{M}x{N}x{K} x{L} layers: graph {ms * 1e3 / L:.2f} us/layer; eager per record: gemm {np.median(g) * 1e3:.2f} us "
          f"({fl / (np.median(g) * 1e-3) / 1e12:.0f} TF/s tensor), square+split {np.median(e) * 1e3:.2f} us; "
          f"launches/step {ex.plan.launch_count()}", flush=True)
    ex.close()


if __name__ == "__main__":
    main()
