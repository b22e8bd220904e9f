"""Build variants/lib_<name>.so with extra nvcc defines (A/B experiments; load with VISTA_LIB).
usage: python scripts/build_variant.py name [-DFOO=1 ...]"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as g  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
src = sorted(glob.glob(os.path.join(ROOT, "paper_2510_22049_b200/csrc/*.cu")))
out = os.path.join(ROOT, "variants", f"lib_{name}.so")
r = subprocess.run([g._nvcc(), *g.NVCC_FLAGS, *defs, "-I", os.path.join(ROOT, "include"), "-o", out, *src, "-lcudart"],
                   capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr[-3000:])
print(out)
