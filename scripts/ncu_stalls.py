#!/usr/bin/env python
"""Stall-reason breakdown per SASS region from an ncu --set full report (source page, SASS).

    python scripts/ncu_stalls.py report.ncu-rep [--top N]
Prints the instructions with the most warp-stall samples and a per-opcode-class summary, plus
the totals per stall reason over the whole kernel (first kernel in the report)."""
import collections
import csv
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
insts = []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    try:
        samp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    st = {k: int(r[ix[k]] or 0) for k in reasons}
    insts.append((r[ix["Address"]], r[ix["Source"]].strip(), samp, st))
tot = collections.Counter()
for _, _, _, st in insts:
    tot.update(st)
all_s = sum(tot.values())
print(f"total stall samples {all_s}")
for k, v in tot.most_common():
    if v:
        print(f"  {k:24s} {v:8d}  {100 * v / all_s:5.1f}%")
print(f"\ntop {top} instructions by samples:")
for i, (a, s, n, st) in enumerate(sorted(insts, key=lambda x: -x[2])[:top]):
    main = ", ".join(f"{k[6:]}={v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3] if v)
    print(f"{a[-6:]} {n:7d}  {s[:60]:60s} {main}")
op = collections.Counter()
for _, s, n, _ in insts:
    o = s.split()[0] if s else "?"
    if o.startswith("@"):
        o = s.split()[1]
    op[o.split(".")[0]] += n
print("\nsamples by opcode:")
for k, v in op.most_common(20):
    print(f"  {k:12s} {v:8d}  {100 * v / max(1, all_s):5.1f}%")
