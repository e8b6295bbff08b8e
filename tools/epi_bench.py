"""Fused GEMM epilogue vs GEMM + elementwise kernel (dev tool).

    python tools/epi_bench.py [M N K]
"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")


def run(text, epi, iters=50):
    os.environ["SPX_EPILOGUE"] = epi
    from paper_2401_11202_b200.ir import parse_module
    from paper_2401_11202_b200.session import Session
    m = parse_module(text)
    sess = Session(m)
    rng = np.random.default_rng(0)
    sess.load({n: rng.standard_normal(t.dims).astype(np.float32) for n, t in m.func("main").args})
    sess.run()
    sess.capture()
    for _ in range(3):
        sess.step()
    sess.sync()
    dev = sess.device
    e0, e1 = dev.event(), dev.event()
    dev.record(e0)
    for _ in range(iters):
        sess.step()
    dev.record(e1)
    dev.sync()
    graph_us = dev.elapsed_ms(e0, e1) / iters * 1e3
    prof = [t * 1e3 for t in sess.ex.plan.profile()]
    sess.close()
    return graph_us, prof


def main():
    M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (2048, 1024, 1024)
    t = f"tensor<{M}x{N}xf32>"
    progs = {
        "add": f"""func @main(%a: tensor<{M}x{K}xf32>, %b: tensor<{K}x{N}xf32>, %x: {t}) -> {t} {{
  %c = matmul %a, %b : {t}
  %o = add %x, %c : {t}
  return %o
}}
""",
        "none": f"""func @main(%a: tensor<{M}x{K}xf32>, %b: tensor<{K}x{N}xf32>) -> {t} {{
  %c = matmul %a, %b : {t}
  return %c
}}
""",
    }
    for name, text in progs.items():
        for epi in ("0", "1"):
            g, prof = run(text, epi)
            print(f"{name:5s} epilogue={epi} {M}x{N}x{K}: graph {g:7.1f} us  records {[round(x, 1) for x in prof]}")


if __name__ == "__main__":
    main()
