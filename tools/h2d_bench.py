"""Host<->device transfer options for the drop-in call (the plugin e2e copies
every input in and every result out): pageable vs pinned vs registered
(cudaHostRegister) copies, and the host-side staging memcpy."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_11202_b200 import runtime as R  # noqa: E402

GB = 1 << 30


def t(fn, n=3):
    fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def main():
    dev = R.Device(0)
    lib = dev.lib
    nb = int(float(os.environ.get("GBYTES", "1")) * GB)
    d = dev.malloc(nb)
    a = np.random.default_rng(0).standard_normal(nb // 4).astype(np.float32)
    out = {}
    out["h2d_pageable"] = nb / t(lambda: (dev.h2d(d, a), dev.sync())) / 1e9
    b = np.empty_like(a)
    b[...] = 0
    out["d2h_pageable_touched"] = nb / t(lambda: (dev.d2h(b, d), dev.sync())) / 1e9

    def fresh():
        c = np.empty_like(a)
        dev.d2h(c, d)
        dev.sync()
    out["d2h_pageable_fresh"] = nb / t(fresh) / 1e9
    p = dev.pinned(a.shape)
    p[...] = a
    out["h2d_pinned"] = nb / t(lambda: (R.call(lib.spx_memcpy_h2d, d, p.ctypes.data, nb, dev.stream), dev.sync())) / 1e9
    out["d2h_pinned"] = nb / t(lambda: (R.call(lib.spx_memcpy_d2h, p.ctypes.data, d, nb, dev.stream), dev.sync())) / 1e9

    def reg():
        R.call(lib.spx_host_register, C.c_void_p(a.ctypes.data), nb)
        R.call(lib.spx_host_unregister, C.c_void_p(a.ctypes.data))
    out["register_unregister_GBps"] = nb / t(reg) / 1e9

    def reg_copy():
        R.call(lib.spx_host_register, C.c_void_p(a.ctypes.data), nb)
        R.call(lib.spx_memcpy_h2d, d, a.ctypes.data, nb, dev.stream)
        dev.sync()
        R.call(lib.spx_host_unregister, C.c_void_p(a.ctypes.data))
    out["h2d_register_copy"] = nb / t(reg_copy) / 1e9
    for th in (1, 4, 8, 16, 32):
        out[f"host_memcpy_{th}t"] = nb / t(lambda: R.call(lib.spx_host_copy, C.c_void_p(p.ctypes.data),
                                                          C.c_void_p(a.ctypes.data), nb, th)) / 1e9
    out["cpu_threads"] = len(os.sched_getaffinity(0))
    for k, v in out.items():
        print(f"{k:28s} {v:8.2f}")


if __name__ == "__main__":
    main()
