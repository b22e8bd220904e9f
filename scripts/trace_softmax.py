#!/usr/bin/env python
"""Timeline of CTA 0 of the softmax kernel (debug build with -DVISTA_TRACE, loaded via VISTA_LIB).

Events (clock64, per tile t of the first item, per Q tile q):
  0 MMA wait p_full start   1 MMA p_full acquired   2 MMA PV+S issued
  3 softmax wait s_full      4 s_full acquired       5 S loaded from TMEM
  6 exp done                 7 P arrive              8 K TMA issue   9 V TMA issue
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

cfg = synth.CONFIGS["c2"]
lens = synth.user_lengths("c2")
q, K, V, off = synth.make_batch(lens, cfg["S"], cfg["H"], cfg["d"], backend="torch", device="cuda")
ot = torch.from_numpy(off).cuda()
for _ in range(3):
    vista.summarize(q, K, V, ot, int(off[-1]))
torch.cuda.synchronize()
lib = vista.load()
buf = np.zeros((12, 64, 2), dtype=np.uint64)
lib.vista_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
rc = lib.vista_debug_trace(buf.ctypes.data, buf.nbytes)
assert rc == 0, rc
t0 = int(buf[8, 0, 0])
ev = buf.astype(np.int64) - t0
names = ["mma_wait_p", "mma_got_p", "mma_issued", "sm_wait_s", "sm_got_s", "sm_loaded", "sm_exp_done",
         "sm_arrive", "k_issue", "v_issue"]
print("tile  " + " ".join(f"{n:>11s}" for n in names))
for t in range(40):
    for qq in range(2):
        row = [ev[e, t, qq] if (e < 8 or qq == 0) else 0 for e in range(10)]
        print(f"{t:3d}/{qq} " + " ".join(f"{x:11d}" for x in row))
# per-tile deltas (steady state)
d = np.diff(ev[1, 5:35, 0])
print("period (clk) of PV_0 issue: mean %.0f" % d.mean())
for qq in range(2):
    print(f"q{qq}: s-wait->got %.0f, got->loaded %.0f, loaded->exp %.0f, exp->arrive %.0f, arrive->mma_got %.0f"
          % tuple(np.mean(x) for x in [ev[4, 5:35, qq] - ev[3, 5:35, qq], ev[5, 5:35, qq] - ev[4, 5:35, qq],
                                         ev[6, 5:35, qq] - ev[5, 5:35, qq], ev[7, 5:35, qq] - ev[6, 5:35, qq],
                                         ev[1, 5:35, qq] - ev[7, 5:35, qq]]))
    print(f"q{qq}: mma got p -> issued %.0f; issued(t) -> softmax got S(t+1) %.0f"
          % (np.mean(ev[2, 5:35, qq] - ev[1, 5:35, qq]), np.mean(ev[4, 6:36, qq] - ev[2, 5:35, qq])))
# items of CTA 0 (clock64, globaltimer) and end times of CTAs 0..31
print("items of CTA 0: (clock64, ns, ntiles)")
for i in range(32):
    if buf[10, i, 1] == 0:
        break
    print(i, int(buf[10, i, 0]) - t0, int(buf[10, i, 1]) - int(buf[10, 0, 1]), int(buf[11, i, 0]))
ends_ns = [int(buf[11, 32 + c, 1]) - int(buf[10, 0, 1]) for c in range(32)]
print("CTA end (ns after CTA0 first item):", ends_ns)
print("CTA0 end clock64:", int(buf[11, 32, 0]) - t0, "ns:", ends_ns[0])
