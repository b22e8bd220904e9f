"""Every tcgen05 / TMA kernel of libvista once on small shapes (for compute-sanitizer memcheck,
racecheck and synccheck, one tool per run): softmax forward (clusters of 1, 2 and 4 CTAs, split
units, the fused int8 export), the split-L merge, QLA state + finalize, QLA rows (history / target,
from a saved state), softmax and QLA backward, stage-2 target attention and two summarizer layers.
Exits 0 when every call returned; parity is the tests' job."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_22049_b200 as vista  # noqa: E402
import synth  # noqa: E402

vista.load()
dev = torch.device("cuda:0")
bf = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev, torch.bfloat16)  # noqa: E731
lens = [300, 0, 129, 1000, 5]
for S, H in ((128, 1), (256, 2), (512, 1)):
    q, k, v, off = synth.make_batch(lens, S, H, 128, seed=1)
    qt, kt, vt, ot = bf(q), bf(k), bf(v), torch.from_numpy(off).to(dev)
    out, lse = vista.summarize(qt, kt, vt, ot, int(off[-1]), out_dtype=vista.BF16)
    po, pl = vista.summarize_partial(qt, kt, vt, ot, int(off[-1]))
    vista.summarize_merge(torch.stack([po, po]), torch.stack([pl, pl]), q=qt)
    if S == 256:
        g = bf(np.random.default_rng(2).integers(-128, 128, size=out.shape) / 64.0)
        vista.summarize_bwd(qt, kt, vt, ot, int(off[-1]), g, attn=vista.SOFTMAX, out=out, lse=lse)
        vista.summarize_bwd(qt, kt, vt, ot, int(off[-1]), g, attn=vista.QLA)
        z, _ = vista.summarize_partial(qt, kt, vt, ot, int(off[-1]), attn=vista.QLA)
        vista.summarize(qt, kt, vt, ot, int(off[-1]), attn=vista.QLA)
        rows = np.array([5, 0, 130, 2, 1])
        roff = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
        R = int(roff[-1])
        qr, ks, vs = [bf(np.random.default_rng(i).integers(-128, 128, size=(R, H, 128)) / 64.0) for i in range(3)]
        rt = torch.from_numpy(roff).to(dev)
        vista.qla_rows(kt, vt, ot, int(off[-1]), qr, rt, R, k_self=ks, v_self=vs)
        vista.qla_rows(kt, vt, ot, int(off[-1]), qr, rt, R)
        vista.qla_rows_from_state(z, torch.from_numpy(np.diff(off)).to(dev), qr, rt, R, k_self=ks, v_self=vs)
        # int8 export fused into the epilogue, then stage 2 over it
        B = len(lens)
        desc = vista.make_desc(B, S, H, 128, in_dtype=vista.BF16, out_dtype=vista.BF16)
        need = vista.vista_summarize_workspace_size(desc, int(off[-1]))
        ws = torch.empty(max(need, 16), dtype=torch.uint8, device=dev)
        codes = torch.empty((B, S, H, 128), dtype=torch.int8, device=dev)
        sc = torch.empty((B, S, H), dtype=torch.float32, device=dev)
        zp = torch.empty((B, S, H), dtype=torch.float32, device=dev)
        vista.vista_summarize_fwd_int8(desc, qt, kt, vt, ot, int(off[-1]), out, lse, codes, sc, zp, ws, need)
        vista.target_attend(codes, sc, zp, qr, ks, vs, rt)
# two summarizer layers
S, H, D = 128, 1, 128
seg = [S + 200, S, S + 70]
xoff = np.concatenate([[0], np.cumsum(seg)]).astype(np.int64)
rng = np.random.default_rng(3)
x = bf(rng.integers(-128, 128, size=(int(xoff[-1]), D)) / 64.0)
W = bf(rng.integers(-128, 128, size=(2, 5, D, D)) / (128.0 * np.sqrt(D)))
vista.summarize_layers(x, torch.from_numpy(xoff).to(dev), W, S, H)
torch.cuda.synchronize()
print("sanitize_small: all calls returned")
