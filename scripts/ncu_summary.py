#!/usr/bin/env python
"""Summarize ncu output for profiles/: key metrics of a --set full report, and kernel shares of
a launch list (gpu__time_duration.sum CSV).

    python scripts/ncu_summary.py report <file.ncu-rep> [name]   -> text summary on stdout
    python scripts/ncu_summary.py launches <launches.csv>         -> per-kernel totals and shares
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "SM_A.TriageCompute.sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__inst_executed_pipe_alu_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def report(path, name=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary: {name or path}")
    for r in rows[2:]:
        kname = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"kernel: {kname[:120]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k} = {r[i]} {units[i]}")
        # stall reasons (warp state) if present
        stalls = [(h, r[i]) for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warp_latency_issue_stalled") and h.endswith(".ratio")]
        for h, v in sorted(stalls, key=lambda x: -float(x[1] or 0))[:8]:
            print(f"  {h} = {v}")


def launches(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        k = r["Kernel Name"].split("(")[0][:90]
        tot[k] += v * scale
        cnt[k] += 1
    allt = sum(tot.values())
    print("# kernel launch list summary (ncu gpu__time_duration.sum, cold-cache, serialised)")
    print(f"{'kernel':92s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
    for k, t in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:92s} {cnt[k]:8d} {t:10.1f} {t / cnt[k]:9.2f} {100 * t / allt:5.1f}%")


if __name__ == "__main__":
    if sys.argv[1] == "report":
        report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        launches(sys.argv[2])
