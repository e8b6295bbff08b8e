"""Per-GEMM time of a dependent GEMM chain replayed as a CUDA graph (dev tool):
the Megatron MP pattern at N=4, x(1024x1024) @ W1(1024x512) @ W2(512x1024) ...

    python tools/chain_bench.py [M D F] [--links 16]
"""
import sys

import numpy as np

sys.path.insert(0, ".")


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    M, D, F = (int(x) for x in args[:3]) if len(args) >= 3 else (1024, 1024, 512)
    links = 16
    from paper_2401_11202_b200.ir import parse_module
    from paper_2401_11202_b200.session import Session
    lines = [f"func @main(%x: tensor<{M}x{D}xf32>, %w1: tensor<{D}x{F}xf32>, %w2: tensor<{F}x{D}xf32>) -> tensor<{M}x{D}xf32> {{"]
    prev = "%x"
    for i in range(links):
        lines.append(f"  %h{i} = matmul {prev}, %w1 : tensor<{M}x{F}xf32>")
        lines.append(f"  %y{i} = matmul %h{i}, %w2 : tensor<{M}x{D}xf32>")
        prev = f"%y{i}"
    lines += [f"  return {prev}", "}", ""]
    m = parse_module("\n".join(lines))
    rng = np.random.default_rng(0)
    sess = Session(m)
    sess.load({"x": rng.standard_normal((M, D)).astype(np.float32) * 0.03,
               "w1": rng.standard_normal((D, F)).astype(np.float32) * 0.03,
               "w2": rng.standard_normal((F, D)).astype(np.float32) * 0.03})
    sess.run()
    sess.capture()
    for _ in range(3):
        sess.step()
    sess.sync()
    dev = sess.device
    e0, e1 = dev.event(), dev.event()
    iters = 20
    dev.record(e0)
    for _ in range(iters):
        sess.step()
    dev.record(e1)
    dev.sync()
    us = dev.elapsed_ms(e0, e1) / iters * 1e3
    flops = 2.0 * M * D * F * 2 * links
    print(f"chain {M}x{D}x{F}: {us / (2 * links):.1f} us per GEMM in the graph "
          f"({3 * flops / (us * 1e-6) / 1e12:.0f} TF/s tf32 work)")
    sess.close()


if __name__ == "__main__":
    main()
