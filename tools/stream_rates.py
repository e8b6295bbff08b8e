"""Algorithmic HBM rates of the streaming kernels of one step, from an ncu
launch list (tools/profile_step.py under `ncu --metrics gpu__time_duration.sum
...`) matched record by record against the plan's own records.

    python tools/stream_rates.py profiles/r01_ncu_launches_c2_n1.csv [program] [steps]

Bytes per record are algorithmic: every input once (broadcast operands at their
own size), every output, and the fp16 pieces (4 B per element) a split writes
-- standalone splits also read their fp32 source.  A batched split launch
(split_h16_batch_kernel) carries the bytes of every record it runs.  ncu serialises kernels and
flushes caches between them (cold L2), so these are DRAM-bound rates.
"""
import collections
import csv
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, mi, vi, ui, ii = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                          hdr.index("Metric Unit"), hdr.index("ID"))
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        v = v / 1e3 if r[ui] in ("nsecond", "ns") else (v * 1e3 if r[ui] in ("msecond", "ms") else v)
        per[int(r[ii])] = (r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", ""), v)
    return list(per.values())


def ew_bytes(q):
    tot = 4 * q.numel * q.n_out
    for j in range(q.n_in):
        cnt = 1
        for k in range(q.rank):
            if q.inp[j].stride[k] != 0:
                cnt *= q.dims[k]
        tot += 4 * cnt
    return tot


def main(path, program="c2_tf8_dense", steps=2):
    from paper_2401_11202_b200 import runtime as R
    from paper_2401_11202_b200.executable import Executable
    from paper_2401_11202_b200.programs import load_program
    p = load_program(program)
    ex = Executable(p.dense if p.local is None else p.local, devices=[0], dry=True)
    recs = ex.records()
    # the runtime fuses a SPLIT into the elementwise record right before it on the same stream
    st = {i: s for i, s, _ in ex.sched}
    fused = set()
    for i in range(len(recs) - 1):
        (ka, a), (kb, b) = recs[i], recs[i + 1]
        if (ka == R.K_EW and kb == R.K_SPLIT and st.get(i, 0) == st.get(i + 1, 0) and a.vec
                and b.ld == b.cols and b.rows * b.cols == a.numel and b.cols % 4 == 0
                and any(a.out_off[j] == b.src_off for j in range(a.n_out))):
            fused.add(i + 1)
    # ... and runs consecutive standalone SPLITs of one stream as one batched launch
    wt = {i: w for i, _, w in ex.sched}
    batched = {}                      # member -> leader
    i = 0
    while i < len(recs):
        if recs[i][0] == R.K_SPLIT and i not in fused:
            j = i + 1
            while (j < len(recs) and recs[j][0] == R.K_SPLIT and j not in fused and st.get(j, 0) == st.get(i, 0)
                   and not wt.get(j) and j - i < 48):
                batched[j] = i
                j += 1
            i = j
        else:
            i += 1
    L = launches(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    pos = 0
    for _ in range(steps):
        for i, (k, q) in enumerate(recs):
            if k == R.K_SPLIT and i in fused:
                continue
            if k == R.K_SPLIT and i in batched:
                agg[last_split][2] += 8 * q.rows * q.cols
                continue
            if k == R.K_REDUCE:
                while pos < len(L) and L[pos][0].startswith("reduce"):
                    pos += 1
                continue
            name, us = L[pos]
            pos += 1
            if k == R.K_EW:
                b = ew_bytes(q)
                if i + 1 in fused:
                    b += 4 * recs[i + 1][1].rows * recs[i + 1][1].cols
                a = agg[name]
                a[0] += 1; a[1] += us; a[2] += b
            elif k == R.K_SPLIT:
                last_split = name
                a = agg[name]
                a[0] += 1; a[1] += us; a[2] += 8 * q.rows * q.cols
    tb = tt = 0.0
    print(f"{'kernel':70s} {'launches':>8s} {'us/step':>9s} {'GB/step':>8s} {'GB/s':>7s}")
    for name, (n, us, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{name[:70]:70s} {n / steps:8.0f} {us / steps:9.1f} {b / steps / 1e9:8.3f} {b / (us * 1e-6) / 1e9:7.0f}")
        tb += b
        tt += us
    print(f"{'all streaming kernels':70s} {'':8s} {tt / steps:9.1f} {tb / steps / 1e9:8.3f} {tb / (tt * 1e-6) / 1e9:7.0f}"
          f"  ({tb / (tt * 1e-6) / 1e9 / 6481.1:.2f} of 6481 GB/s)")


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3] or []), *([int(sys.argv[3])] if len(sys.argv) > 3 else []))
