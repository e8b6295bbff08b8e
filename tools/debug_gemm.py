"""GEMM diagnostics and microbenchmark on the GPU (development tool)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2401_11202_b200 import runtime as R  # noqa: E402


def pad(n):
    return (n + 63) // 64 * 64


class G:
    def __init__(self, dev, A, B, at=False, bt=False, promote=0, path=1):
        self.dev = dev
        M, K = (A.shape[1], A.shape[0]) if at else A.shape
        N = B.shape[0] if bt else B.shape[1]
        self.M, self.N, self.K = M, N, K
        na, nb, nc = A.size, B.size, M * N
        import os
        nc = nc * max(1, int(os.environ.get("SPLITS", "1")))
        self.base = dev.malloc(4 * (pad(na) + pad(nb) + pad(nc)))
        dev.h2d(self.base, A.astype(np.float32))
        dev.h2d(self.base + 4 * pad(na), B.astype(np.float32))
        self.coff = self.base + 4 * (pad(na) + pad(nb))
        dev.memset(self.coff, 4 * nc, 0)
        p = R.GemmParams()
        p.base, p.dev_stride, p.ndev = self.base, 0, 1
        p.M, p.N, p.K = M, N, K
        p.a_off, p.b_off, p.c_off = 0, pad(na), pad(na) + pad(nb)
        p.lda, p.ldb, p.ldc = A.shape[1], B.shape[1], N
        p.a_mn_major, p.b_k_major = int(at), int(bt)
        p.path, p.promote = path, promote
        import os
        p.splits = int(os.environ.get("SPLITS", "1"))
        self.plan = R.NativePlan(dev)
        self.plan.add(R.K_GEMM, p)
        self.plan.finalize()

    def run(self):
        self.plan.run()
        self.dev.sync()
        C = np.empty((self.M, self.N), np.float32)
        self.dev.d2h(C, self.coff)
        self.dev.sync()
        return C

    def time_ms(self, iters=20):
        self.plan.run()
        self.dev.sync()
        e0, e1 = self.dev.event(), self.dev.event()
        self.dev.record(e0)
        for _ in range(iters):
            self.plan.run()
        self.dev.record(e1)
        return self.dev.elapsed_ms(e0, e1) / iters

    def close(self):
        self.plan.destroy()
        self.dev.free(self.base)


def rel(a, b):
    return float(np.max(np.abs(a.astype(np.float64) - b)) / (np.max(np.abs(b)) + 1e-12))


def main():
    dev = R.Device(0)
    rng = np.random.default_rng(0)
    for K in (512, 2048, 8192):
        A = rng.standard_normal((256, K)).astype(np.float32)
        B = rng.standard_normal((K, 256)).astype(np.float32)
        ref = A.astype(np.float64) @ B
        line = f"K={K}: numpy-f32 {rel(A @ B, ref):.2e}"
        for pr in (1, 2, 4, 8, 100000):
            g = G(dev, A, B, promote=pr)
            line += f" | P={pr} {rel(g.run(), ref):.2e}"
            g.close()
        print(line, flush=True)
    for at in (False, True):
        for bt in (False, True):
            M, N, K = 256, 384, 4096
            A = rng.standard_normal((K, M) if at else (M, K)).astype(np.float32)
            B = rng.standard_normal((N, K) if bt else (K, N)).astype(np.float32)
            AA = A.T if at else A
            BB = B.T if bt else B
            g = G(dev, A, B, at, bt)
            print(f"layout at={at} bt={bt} K=4096: rel {rel(g.run(), AA.astype(np.float64) @ BB):.2e}", flush=True)
            g.close()
    # throughput on the C2 shapes (b=2048, d=1024, d_ff=4096)
    shapes = [(2048, 1024, 1024, False, False), (2048, 4096, 1024, False, False),
              (2048, 1024, 4096, False, False), (1024, 1024, 2048, True, False),
              (4096, 1024, 2048, True, False), (2048, 4096, 1024, False, True),
              (8192, 8192, 8192, False, False)]
    for M, N, K, at, bt in shapes:
        A = rng.standard_normal((K, M) if at else (M, K)).astype(np.float32)
        B = rng.standard_normal((N, K) if bt else (K, N)).astype(np.float32)
        for pr in (4,):
            g = G(dev, A, B, at, bt, promote=pr)
            ms = g.time_ms(10)
            tf = 2.0 * M * N * K / ms / 1e9
            print(f"gemm {M}x{N}x{K} at={at} bt={bt} P={pr}: {ms*1e3:.1f} us  {tf:.1f} TFLOP/s (fp32-equiv)", flush=True)
            g.close()


if __name__ == "__main__":
    main()
