#!/usr/bin/env python
"""Timeline of CTA pair 0 of the 2-CTA softmax kernel (debug build -DVISTA_TRACE via VISTA_LIB).
Events: 0 MMA wait p(t)  1 MMA got p  2 MMA issued PV(t)+S(t+2)  3 softmax wait S  4 got S
        5 S loaded  6 exp done  7 P arrived  8 producer stage issue.  Slot = rank*2 + warpgroup."""
import ctypes, os, sys
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
buf = np.zeros((16, 64, 4), dtype=np.uint64)
lib.vista_debug_trace2.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.vista_debug_trace2(buf.ctypes.data, buf.nbytes) == 0
t0 = int(buf[0, 0, 0])
ev = buf.astype(np.int64) - t0
print("t  | mma: wait_p got_p issued | slot: wait_s got_s loaded exp_done arrived (r0A r0B r1A r1B)")
for t in range(24):
    s = f"{t:2d} | {ev[0,t,0]:8d} {ev[1,t,0]:8d} {ev[2,t,0]:8d} |"
    for slot in range(4):
        if (slot % 2) != (t % 2):
            continue
        s += f" [{slot}] " + " ".join(f"{ev[e,t,slot]:7d}" for e in (3, 4, 5, 6, 7))
    print(s)
d = np.diff(ev[1, 4:40, 0])
print("period per tile (MMA got p): %.0f" % d.mean())
for slot in range(4):
    ts = np.arange(4 + (slot % 2), 40, 2)
    print(f"slot {slot}: wait_s->got %.0f, got->loaded %.0f, loaded->exp %.0f, exp->arrive %.0f" % (
        np.mean(ev[4, ts, slot] - ev[3, ts, slot]), np.mean(ev[5, ts, slot] - ev[4, ts, slot]),
        np.mean(ev[6, ts, slot] - ev[5, ts, slot]), np.mean(ev[7, ts, slot] - ev[6, ts, slot])))
print("mma got_p->issued %.0f, wait_p->got_p %.0f" % (np.mean(ev[2, 4:40, 0] - ev[1, 4:40, 0]),
                                                     np.mean(ev[1, 4:40, 0] - ev[0, 4:40, 0])))
print("mma: got_p->PV issued %.0f, PV issued->stage ready %.0f, stage ready->S issued %.0f" % (
    np.mean(ev[9, 4:40, 0] - ev[1, 4:40, 0]), np.mean(ev[10, 4:40, 0] - ev[9, 4:40, 0]),
    np.mean(ev[2, 4:40, 0] - ev[10, 4:40, 0])))
print("producer stage issue deltas r0:", np.diff(ev[8, 4:24, 0]).tolist())
