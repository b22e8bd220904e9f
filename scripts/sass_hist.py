#!/usr/bin/env python
"""Histogram of SASS opcodes in the address range from the first instruction of source line
first_line to the next instruction of last_line (nvdisasm line info, outermost file lines).
usage: scripts/sass_hist.py file.cu kernel_substring first_line last_line [file_filter] [nvcc flags]"""
import collections
import os
import re
import subprocess
import sys

src, pat, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
ffilt = sys.argv[5] if len(sys.argv) > 5 else os.path.basename(src)
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.makedirs("/tmp/spills", exist_ok=True)
cub = "/tmp/spills/h.cubin"
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                       "--expt-relaxed-constexpr", "-lineinfo", "-I", os.path.join(root, "include"), "-cubin", src,
                       "-o", cub] + sys.argv[6:])
sass = subprocess.run(["/usr/local/cuda/bin/nvdisasm", "--print-line-info", cub], capture_output=True,
                      text=True).stdout.split("\n")
fn, cur = None, None
hist = collections.Counter()
state = 0
for line in sass:
    m = re.match(r"\s*\.text\.(\S+):", line)
    if m:
        fn = m.group(1)
    if "//##" in line:
        # outermost location: the last "line N" of the comment (inlined-at chain ends at the caller)
        locs = re.findall(r'"([^"]+)", line (\d+)', line)
        if locs:
            cur = [(f.split("/")[-1], int(n)) for f, n in locs]
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if m and pat in (fn or "") and cur:
        here = [n for f, n in cur if f == ffilt]
        if state == 0 and lo in here:
            state = 1
        if state == 1:
            hist[m.group(2).split(".")[0]] += 1
            if hi in here:
                state = 2
tot = sum(hist.values())
print("total", tot)
for k, v in hist.most_common(40):
    print(f"{k:12s} {v}")
