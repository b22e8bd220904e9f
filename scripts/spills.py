#!/usr/bin/env python
"""List local-memory spill instructions (STL/LDL) of a kernel with their source lines.
usage: scripts/spills.py file.cu kernel_substring"""
import os
import re
import subprocess
import sys

src, pat = sys.argv[1], sys.argv[2]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.makedirs("/tmp/spills", exist_ok=True)
cub = "/tmp/spills/k.cubin"
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                       "--expt-relaxed-constexpr", "-lineinfo", "-I", os.path.join(root, "include"), "-cubin", src,
                       "-o", cub])
sass = subprocess.run(["/usr/local/cuda/bin/nvdisasm", "--print-line-info", cub], capture_output=True,
                      text=True).stdout.split("\n")
fn, cur = None, None
for line in sass:
    m = re.match(r"\s*\.text\.(\S+):", line)
    if m:
        fn = m.group(1)
    m = re.search(r"line (\d+)", line)
    if m and "//##" in line:
        f = re.search(r'"([^"]+)"', line)
        cur = (f.group(1).split("/")[-1] if f else "", int(m.group(1)))
    if ("STL" in line or "LDL" in line) and pat in (fn or ""):
        print(cur, line.strip()[:80])
