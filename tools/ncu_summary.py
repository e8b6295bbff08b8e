"""Summarise an ncu launch-list CSV (gpu__time_duration [+ dram bytes]) per kernel."""
import collections
import csv
import sys


def main(path, steps=1):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui, ii = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                          hdr.index("Metric Unit"), hdr.index("ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in data:
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        if r[mi] == "gpu__time_duration.sum":
            v = v / 1e3 if u == "nsecond" or u == "ns" else (v * 1e3 if u in ("msecond", "ms") else v)
        elif "bytes" in r[mi]:
            v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        per[r[ii]][r[mi]] = v
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    tot = 0.0
    for i, m in per.items():
        t = m.get("gpu__time_duration.sum", 0.0)
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a = agg[names[i]]
        a[0] += 1
        a[1] += t
        a[2] += b
        tot += t
    print(f"{'kernel':40s} {'launches/step':>13s} {'us/step':>10s} {'share':>6s} {'DRAM GB/s':>10s}")
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        gbs = b / (t * 1e-6) / 1e9 if t else 0
        print(f"{k:40s} {n / steps:13.0f} {t / steps:10.1f} {100 * t / tot:5.1f}% {gbs:10.0f}")
    print(f"total us/step {tot / steps:.1f} (serialised, cold-ish caches: compare shares)")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
