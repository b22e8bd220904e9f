#!/usr/bin/env python
"""Per-item timeline of CTA 0 of the softmax kernel (debug build -DVISTA_TRACE via VISTA_LIB).

Workload: B users of exactly L items (env L, S, H, TOTAL).  Columns (clock64 relative to the
first MMA item start): MMA item start / q_full / k_full / last PV issued; softmax WG0 item
start / first S / O ready / epilogue done; producer pre-q_empty / q_empty acquired / first K.
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_22049_b200 as vista  # noqa: E402
import synth  # noqa: E402

L = int(os.environ.get("L", 128))
S = int(os.environ.get("S", 256))
H = int(os.environ.get("H", 4))
TOTAL = int(os.environ.get("TOTAL", 2_560_000))
B = max(1, TOTAL // (L * H))
q, K, V, off = synth.make_batch([L] * B, S, H, 128, backend="torch", device="cuda")
ot = torch.from_numpy(off).cuda()
for _ in range(3):
    vista.summarize(q, K, V, ot, int(off[-1]))
torch.cuda.synchronize()
lib = vista.load()
buf = np.zeros((16, 64), dtype=np.uint64)
lib.vista_debug_itrace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.vista_debug_itrace(buf.ctypes.data, buf.nbytes) == 0
t0 = int(buf[0, 0])
ev = buf.astype(np.int64) - t0
names = ["mma_start", "mma_q", "mma_k", "mma_lastPV", "sm_start", "sm_S0", "sm_O", "sm_epi_done",
         "pr_pre_qe", "pr_qe", "pr_K0", "mma_end", "sch_pub", "sch_pre_e", "sch_got_e"]
print(f"L={L} S={S} H={H} B={B}")
print("item " + " ".join(f"{n:>11s}" for n in names))
for i in range(40):
    if buf[0, i] == 0:
        break
    print(f"{i:4d} " + " ".join(f"{int(ev[e, i]):11d}" for e in range(15)))
n = 30
if buf[0, n] != 0:
    per = np.diff(ev[0, 5:n]).mean()
    print("mean item period (clk): %.0f" % per)
    for a, b, what in [(0, 1, "mma start->q_full"), (1, 2, "q_full->k_full"), (2, 3, "k_full->lastPV"),
                       (3, 6, "lastPV->O ready"), (6, 7, "epilogue"), (4, 5, "sm start->S0"),
                       (9, 1, "pr q_empty->mma q_full"), (3, 9, "lastPV(i)->q_empty(i+1)")]:
        if what.startswith("lastPV(i)"):
            x = ev[9, 6:n + 1] - ev[3, 5:n]
        else:
            x = ev[b, 5:n] - ev[a, 5:n]
        print(f"{what:>26s}: mean {x.mean():8.0f}  min {x.min():8d}  max {x.max():8d}")
