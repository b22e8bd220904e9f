"""Per-CTA timeline of the QLA target-rows kernel (VISTA_TRACE build, libvista_trace.so) on the c2
target-rows-from-state workload (64 users x 256 target rows, H = 4, d = 128, Delta term):
globaltimer at start, after the PDL wait, first W_u ready, first tile's MMA issued, first tile
stored, end, first q/k tile landed (transform), first tile transformed.   python scripts/trace_rows.py [rows per user]"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["VISTA_LIB"] = os.path.join(ROOT, "paper_2510_22049_b200", os.environ.get("TRACE_LIB", "libvista_trace.so"))
import torch  # noqa: E402

import paper_2510_22049_b200 as vista  # noqa: E402

rpu = int(sys.argv[1]) if len(sys.argv) > 1 else 256
B, S, H, d = 64, 256, 4, 128
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1)
grid = lambda shape: (torch.randint(-128, 128, shape, device=dev, generator=g).float() / 64).to(torch.bfloat16)  # noqa
desc = vista.make_desc(B, S, H, d, in_dtype=vista.BF16, out_dtype=vista.BF16, attn=vista.QLA)
z = torch.randn((B, H, d, d), device=dev, generator=g) * 100
ulen = torch.full((B,), 10000, dtype=torch.int64, device=dev)
n = B * rpu
roff = torch.arange(B + 1, dtype=torch.int64, device=dev) * rpu
COLD = os.environ.get("COLD", "0") == "1"  # rotate over 6 input copies (> L2) as bench.py does
sets = [(grid((n, H, d)), grid((n, H, d)), grid((n, H, d))) for _ in range(6 if COLD else 1)]
q, k, v = sets[0]
out = torch.empty((n, H, d), dtype=torch.bfloat16, device=dev)
wsb = vista.vista_qla_rows_from_state_workspace_size(desc, n)
ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)
for i in range(7):
    q, k, v = sets[i % len(sets)]
    vista.vista_qla_rows_from_state(desc, z, ulen, q, roff, n, k, v, out, ws, wsb, None)
torch.cuda.synchronize()
lib = vista.load()
cb = np.zeros((160, 8), dtype=np.uint64)
lib.vista_debug_rows_cta.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.vista_debug_rows_cta(cb.ctypes.data, cb.nbytes) == 0
c = cb[:148].astype(np.int64)
lib.vista_debug_scan_end.restype = ctypes.c_ulonglong
scan_end = int(lib.vista_debug_scan_end())
print(f"tile scan end -> first rows CTA start: {(c[:, 0].min() - scan_end) / 1e3:.2f} us "
      "(negative: the rows kernel started before the scan ended, PDL)")
g0 = c[:, 0].min()
rel = (c - g0) / 1e3
names = ["start", "pdl_wait_done", "first_W_ready", "first_mma", "first_tile_stored", "end", "xform_q_full", "xform_done"]
for i, nm in enumerate(names):
    col = rel[:, i]
    print(f"{nm:18s} min {col.min():7.2f}  p50 {np.median(col):7.2f}  p90 {np.percentile(col, 90):7.2f}  max {col.max():7.2f} us")
span = (c[:, 5].max() - c[:, 0].min()) / 1e3
# the same call timed by the library's main-kernel events (as bench.py does), eager
ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ca, cb2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ea.record()
eb.record()  # materialize the handles (the library records them through the raw cudaEvent_t)
ks = []
for _ in range(20):
    vista.vista_time_next_main_kernel(ea, eb)
    ca.record()
    vista.vista_qla_rows_from_state(desc, z, ulen, q, roff, n, k, v, out, ws, wsb, None)
    cb2.record()
    torch.cuda.synchronize()
    ks.append((ea.elapsed_time(eb), ca.elapsed_time(cb2)))
ks = np.asarray(ks[5:])
print(f"CTA span {span:.2f} us; main-kernel events {1e3 * np.median(ks[:, 0]):.2f} us; whole call {1e3 * np.median(ks[:, 1]):.2f} us")
