"""Timeline of cluster 0 / CTA rank 0 of the softmax kernel (VISTA_TRACE build): per global tile g,
S issue (MMA), P half 0 seen by MMA, PV issued, softmax got S, softmax done.  Usage (GPU box):
    python scripts/trace_mc.py [L] [S] [H]      (needs paper_2510_22049_b200/libvista_trace.so)"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["VISTA_LIB"] = os.path.join(ROOT, "paper_2510_22049_b200", os.environ.get("TRACE_LIB", "libvista_trace.so"))
import torch  # noqa: E402

import paper_2510_22049_b200 as vista  # noqa: E402
import synth  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
S = int(sys.argv[2]) if len(sys.argv) > 2 else 256
H = int(sys.argv[3]) if len(sys.argv) > 3 else 4
B = int(sys.argv[4]) if len(sys.argv) > 4 else 64
lib = vista.load()
q, k, v, off = synth.make_batch([L] * B, S, H, 128, backend="torch", device="cuda")
ot = torch.from_numpy(off).cuda()
for _ in range(3):
    out, lse = vista.summarize(q, k, v, ot, int(off[-1]))
torch.cuda.synchronize()
buf = np.zeros((28, 64), dtype=np.uint64)
lib.vista_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
assert lib.vista_debug_trace(buf.ctypes.data, buf.nbytes) == 0
t0 = int(buf[0, 0])
rel = buf.astype(np.int64) - t0
names = ["S_issued", "P0_seen", "PV_issued", "smx_got_S", "smx_done", "K_req", "V_req", "S_wK", "S_gotK",
         "PV_wV", "PV_gotV", "PV_top"]
print("g   " + " ".join(f"{n:>9s}" for n in names) + "   period(P0_seen)")
for g in range(48):
    row = " ".join(f"{rel[e, g]:9d}" for e in range(12))
    per = rel[1, g] - rel[1, g - 1] if g else 0
    print(f"{g:3d} {row}   {per}")
d = np.diff(rel[1, 8:48])
print("median period per tile (P0_seen):", int(np.median(d)))
print("median softmax busy (got_S -> done):", int(np.median(rel[4, 8:48] - rel[3, 8:48])))
print("median S wait (done(g-1) -> got_S(g)):", int(np.median(rel[3, 9:48] - rel[4, 8:47])))
print("median MMA: P0 seen -> PV issued:", int(np.median(rel[2, 8:48] - rel[1, 8:48])))
print("median S(g+2) issue after PV(g) issued:", int(np.median(rel[0, 10:48] - rel[2, 8:46])))
print("median S issued -> softmax got S:", int(np.median(rel[3, 8:48] - rel[0, 8:48])))
print("median K wait in S issue:", int(np.median(rel[8, 8:48] - rel[7, 8:48])))
print("median V wait in PV:", int(np.median(rel[10, 8:48] - rel[9, 8:48])))
print("median K request -> S got K:", int(np.median(rel[8, 8:48] - rel[5, 8:48])))
print("median V request -> PV got V:", int(np.median(rel[10, 8:48] - rel[6, 8:48])))
print("softmax phases: got_S->loaded", int(np.median(rel[12, 8:48] - rel[3, 8:48])), " loaded->max exchanged",
      int(np.median(rel[13, 8:48] - rel[12, 8:48])), " ->p_free", int(np.median(rel[14, 8:48] - rel[13, 8:48])),
      " ->exps done", int(np.median(rel[15, 8:48] - rel[14, 8:48])), " ->arrived", int(np.median(rel[4, 8:48] - rel[15, 8:48])))
pr = np.zeros((2, 64), dtype=np.int32)
if hasattr(lib, "vista_debug_probe"):
    lib.vista_debug_probe.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    lib.vista_debug_probe(pr.ctypes.data, pr.nbytes)
    ws = rel[3, 8:48] - rel[26, 8:48]
    wp = rel[14, 8:48] - rel[27, 8:48]
    print("s_full: ready at first probe", int(pr[0, 8:48].sum()), "/ 40; wait (probe -> passed) median",
          int(np.median(ws)), "ready-only median", int(np.median(ws[pr[0, 8:48] == 1])) if pr[0, 8:48].any() else None)
    print("p_free: ready at first probe", int(pr[1, 8:48].sum()), "/ 40; wait median", int(np.median(wp)),
          "ready-only median", int(np.median(wp[pr[1, 8:48] == 1])) if pr[1, 8:48].any() else None)
    print("arrive(g-1) -> s_full probe(g):", int(np.median(rel[26, 9:48] - rel[4, 8:47])))
print("items (k: producer Q issued, S got Q, PV got O free, epi got ml, epi got O, epi done):")
for k in range(6):
    print(k, [int(rel[e, k]) for e in (17, 16, 18, 20, 21, 19)])
print("S issue times g=0..", [int(x) for x in rel[0, :64:8]])
lib.vista_debug_softmax_clusters.restype = ctypes.c_int
print("clusters:", lib.vista_debug_softmax_clusters(256))
ct = np.zeros((256, 4), dtype=np.uint64)
lib.vista_debug_cta_times.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
lib.vista_debug_cta_times(ct.ctypes.data, ct.nbytes)
n = 148
st = ct[:n, 0].astype(np.int64); en = ct[:n, 1].astype(np.int64)
dur = en - st
clk = (ct[:n, 3].astype(np.int64) - ct[:n, 2].astype(np.int64)) / np.maximum(dur, 1)
t0g = st.min()
print("CTA start skew (us): max", (st.max() - t0g) / 1e3, " end: min", (en.min() - t0g) / 1e3, "max", (en.max() - t0g) / 1e3)
print("CTA durations (us): min", dur.min() / 1e3, "median", np.median(dur) / 1e3, "max", dur.max() / 1e3)
print("SM clock during kernel (GHz): min", clk.min(), "median", np.median(clk), "max", clk.max())
order = np.argsort(dur)
print("slowest CTAs:", [(int(i), round(dur[i] / 1e3, 1)) for i in order[-6:]])
print("exp body A:", int(np.median(rel[23, 8:48] - rel[22, 8:48])), " B:", int(np.median(rel[25, 8:48] - rel[24, 8:48])),
      " A(g) end -> B(g) start:", int(np.median(rel[24, 8:48] - rel[23, 8:48])), " B(g) end -> A(g+1) start:",
      int(np.median(rel[22, 9:48] - rel[25, 8:47])))
for g in range(20, 26):
    print(g, "A", int(rel[22, g]), int(rel[23, g]), "B", int(rel[24, g]), int(rel[25, g]))
