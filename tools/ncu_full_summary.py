"""Key metrics (+ top stall reasons) of every kernel in an `ncu --set full`
report, as JSON (dev tool): python tools/ncu_full_summary.py report.ncu-rep"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic"]


def main(path):
    raw = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        d = {"kernel": v[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{v[i]} {units[i]}".strip()
        stalls = {}
        for i, n in enumerate(hdr):
            if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("_not_issued"):
                try:
                    stalls[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["top_stalls_pct"] = {k: round(100 * s / tot, 1) for k, s in
                               sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
        out.append(d)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
