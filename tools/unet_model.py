"""U-Net analog training step (BASELINE.json config 4), built ONLY from the
reference's IR and builder (`spindle.ir.FuncBuilder`, ir.py:525-567) so the
reference's unchanged tactic API partitions it.

The reference IR has no convolution (ir.py:18-21), so this is a
1x1-convolution U-Net over NHWC activations:
  * channel mixing  = rank-2 matmul on reshape(N*H*W, C)
  * down-sampling   = reshape (N, H/2, 2, W/2, 2, C) + sum-reduce dims [2, 4]
  * up-sampling     = broadcast dims [0, 1, 3, 5] + reshape (nearest neighbour)
  * skip connection = add
  * activation      = square (like the model zoo, models.py:73-77)
with the backward pass written by hand (as models.py does; no autodiff) and
the momentum-SGD update of models._Grad.momentum_update (models.py:79-85).
Gradients are validated against central finite differences in float64 by
tests/test_unet_model.py (the method of the reference's
`grads_by_finite_difference`, conftest.py:99-139, at unit input scale and
per-tensor relative error -- see that test for why).

Needs the reference importable (PYTHONPATH=/root/reference/pkg/src).
"""
from __future__ import annotations

from spindle.ir import FuncBuilder
from spindle.models import LEARNING_RATE, MOMENTUM


def unet_train(batch: int = 4, height: int = 4, width: int = 4, c0: int = 4, c1: int = 8,
               c2: int = 8):
    N, H, W = batch, height, width
    assert H % 2 == 0 and W % 2 == 0
    P = N * H * W
    Q = N * (H // 2) * (W // 2)
    b = FuncBuilder()

    def emit(kind, ops, attrs=None, name=None):
        return b.emit(kind, ops, attrs or {}, name=name)

    def sq(z):
        return emit("mul", [z, z])

    def scaled(c, v, dims):
        return emit("mul", [b.constant(c, dims), v])

    def tr(v):
        return emit("transpose", [v], {"perm": [1, 0]})

    x = b.arg("x", (N, H, W, c0))
    y = b.arg("y", (N, H, W, c0))
    shapes = {"w1": (c0, c1), "w2": (c1, c2), "w3": (c2, c1), "w4": (c1, c0)}
    for n, s in shapes.items():
        b.arg(n, s)
    for n, s in shapes.items():
        b.arg("m_" + n, s)

    # ---- forward
    x2 = emit("reshape", [x], {"dims": [P, c0]})
    z1 = emit("matmul", [x2, "w1"])                                   # (P, c1)
    h1 = sq(z1)
    h1r = emit("reshape", [h1], {"dims": [N, H // 2, 2, W // 2, 2, c1]})
    pool = emit("reduce", [h1r], {"dims": [2, 4]})                     # (N, H/2, W/2, c1)
    p2 = emit("reshape", [pool], {"dims": [Q, c1]})
    z2 = emit("matmul", [p2, "w2"])                                   # (Q, c2)
    h2 = sq(z2)
    h2r = emit("reshape", [h2], {"dims": [N, H // 2, W // 2, c2]})
    u6 = emit("broadcast", [h2r], {"dims": [0, 1, 3, 5], "shape": [N, H // 2, 2, W // 2, 2, c2]})
    u = emit("reshape", [u6], {"dims": [P, c2]})
    z3 = emit("matmul", [u, "w3"])                                    # (P, c1)
    h3 = sq(z3)
    s = emit("add", [h3, h1])                                         # skip
    out = emit("matmul", [s, "w4"])                                   # (P, c0)
    out4 = emit("reshape", [out], {"dims": [N, H, W, c0]})
    d = emit("add", [out4, emit("neg", [y])])
    loss = emit("reduce", [emit("mul", [d, d])], {"dims": [0, 1, 2, 3]}, name="loss")
    dout4 = scaled(2.0, d, (N, H, W, c0))
    dout = emit("reshape", [dout4], {"dims": [P, c0]})

    # ---- backward
    g = {}
    g["w4"] = emit("matmul", [tr(s), dout])                            # (c1, c0)
    ds = emit("matmul", [dout, tr("w4")])                              # (P, c1)
    dz3 = emit("mul", [ds, scaled(2.0, z3, (P, c1))])
    g["w3"] = emit("matmul", [tr(u), dz3])                             # (c2, c1)
    du = emit("matmul", [dz3, tr("w3")])                               # (P, c2)
    du6 = emit("reshape", [du], {"dims": [N, H // 2, 2, W // 2, 2, c2]})
    dh2r = emit("reduce", [du6], {"dims": [2, 4]})                     # grad of the broadcast
    dh2 = emit("reshape", [dh2r], {"dims": [Q, c2]})
    dz2 = emit("mul", [dh2, scaled(2.0, z2, (Q, c2))])
    g["w2"] = emit("matmul", [tr(p2), dz2])                            # (c1, c2)
    dp2 = emit("matmul", [dz2, tr("w2")])                              # (Q, c1)
    dp = emit("reshape", [dp2], {"dims": [N, H // 2, W // 2, c1]})
    dh1r = emit("broadcast", [dp], {"dims": [0, 1, 3, 5], "shape": [N, H // 2, 2, W // 2, 2, c1]})
    dh1p = emit("reshape", [dh1r], {"dims": [P, c1]})                   # grad of the sum-pool
    dh1 = emit("add", [dh1p, ds])                                      # + skip branch
    dz1 = emit("mul", [dh1, scaled(2.0, z1, (P, c1))])
    g["w1"] = emit("matmul", [tr(x2), dz1])                            # (c0, c1)
    dx2 = emit("matmul", [dz1, tr("w1")])
    dx = emit("reshape", [dx2], {"dims": [N, H, W, c0]}, name="dx")

    # ---- momentum updates (models.py:79-85)
    outs, new_ms = [loss, dx], []
    for n, sh in shapes.items():
        m2 = emit("add", [scaled(MOMENTUM, "m_" + n, sh), g[n]], name="new_m_" + n)
        step = scaled(LEARNING_RATE, m2, sh)
        p2_ = emit("add", [n, emit("neg", [step])], name="new_" + n)
        outs.append(p2_)
        new_ms.append(m2)
    b.ret(*(outs + new_ms))
    return b.build()


def unet_schedule(names, module):
    """BP and Z2 tactics for the U-Net analog, mirroring the transformer
    cookbook entries (schedule.py:327-330)."""
    from spindle.schedule import FIRST_DIVISIBLE_DIM, REPLICATED, ManualPartition
    book = {
        "bp": lambda: ManualPartition("B", {"x": 0}),
        "z2": lambda: ManualPartition("B", {"m_w*": FIRST_DIVISIBLE_DIM, "w*": REPLICATED}),
        "z3": lambda: ManualPartition("B", {"w*": FIRST_DIVISIBLE_DIM, "m_w*": FIRST_DIVISIBLE_DIM}),
    }
    return [book[n]() for n in names]
