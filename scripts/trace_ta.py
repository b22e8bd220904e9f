"""Timeline of CTA 0 of the stage-2 target-attention kernel (VISTA_TRACE build, libvista_trace.so):
clock64 per event and tile.   python scripts/trace_ta.py [candidates per user]"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["VISTA_LIB"] = os.path.join(ROOT, "paper_2510_22049_b200", os.environ.get("TRACE_LIB", "libvista_trace.so"))
import torch  # noqa: E402

import paper_2510_22049_b200 as vista  # noqa: E402

cpu = int(sys.argv[1]) if len(sys.argv) > 1 else 256
B, S, H, d = 64, 256, 4, 128
dev = "cuda"
g = torch.Generator(device=dev)
g.manual_seed(1)
codes = torch.randint(-127, 128, (B, S, H, d), device=dev, generator=g, dtype=torch.int8)
tsc = torch.rand((B, S, H), device=dev, generator=g) / 64 + 1e-3
tzp = torch.rand((B, S, H), device=dev, generator=g) - 0.5
R = B * cpu
grid = lambda: (torch.randint(-128, 128, (R, H, d), device=dev, generator=g).float() / 64).to(torch.bfloat16)  # noqa
q, k, v = grid(), grid(), grid()
roff = torch.arange(B + 1, device=dev, dtype=torch.int64) * cpu
for _ in range(3):
    vista.target_attend(codes, tsc, tzp, q, k, v, roff, R)
torch.cuda.synchronize()
lib = vista.load()
buf = np.zeros((16, 64), dtype=np.uint64)
lib.vista_debug_ta_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.vista_debug_ta_trace(buf.ctypes.data, buf.nbytes) == 0
t0 = int(buf[14, 0])
rel = buf.astype(np.int64) - t0
print("kernel start -> end (clk):", int(rel[15, 0]))
names = ["prod_qk", "mma_qk", "mma_S", "mma_p", "mma_PV", "smx_qk", "smx_S", "smx_max", "smx_done", "epi_ml",
         "epi_O", "epi_done"]
ntiles = int(((rel[0] > 0) | (np.arange(64) == 0)).sum())
print("g  " + " ".join(f"{n:>9s}" for n in names))
for t in range(min(ntiles, 12)):
    print(f"{t:2d} " + " ".join(f"{rel[e, t]:9d}" for e in range(12)))
print("items (dequant start, end):", [(int(rel[12, kk]), int(rel[13, kk])) for kk in range(4)])
print("items (loads landed, VISTA_TRACE):", [int(rel[13, 32 + kk]) for kk in range(4)])

cb = np.zeros((160, 3), dtype=np.uint64)
lib.vista_debug_ta_cta.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.vista_debug_ta_cta(cb.ctypes.data, cb.nbytes) == 0
n = 148
c = cb[:n].astype(np.int64)
g0 = c[:, 0].min()
st, wt, en = (c[:, 0] - g0) / 1e3, (c[:, 1] - g0) / 1e3, (c[:, 2] - g0) / 1e3
print("per-CTA (us from the first CTA start): start max %.2f, PDL wait done min/med/max %.2f/%.2f/%.2f, "
      "end min/med/max %.2f/%.2f/%.2f" % (st.max(), wt.min(), np.median(wt), wt.max(), en.min(), np.median(en), en.max()))
print("end percentiles 10/50/90/100:", [round(float(np.percentile(en, p)), 2) for p in (10, 50, 90, 100)])
