#!/usr/bin/env python
"""Softmax kernel frac for c5's length mix under variations (S, rounding of L to 128, order)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_22049_b200 as vista  # noqa: E402
import synth  # noqa: E402

tf = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
dev = torch.device("cuda")
stream = torch.cuda.current_stream()
base = np.asarray(synth.user_lengths("c5"), dtype=np.int64)
cases = [("c5 S=512", base, 512), ("c5 S=256", base, 256), ("c5 round128 S=512", (base + 127) // 128 * 128, 512),
         ("c5 sorted S=512", np.sort(base), 512), ("c5 no>100k S=512", np.minimum(base, 100000), 512)]
for name, lens, S in cases:
    H, d = 1, 128
    q, K, V, off = synth.make_batch([int(x) for x in lens], S, H, d, seed=0, backend="torch", device=dev)
    total = int(off[-1])
    B = len(lens)
    off_t = torch.from_numpy(off).to(dev)
    desc = vista.make_desc(B, S, H, d, in_dtype=vista.BF16, out_dtype=vista.BF16, attn=vista.SOFTMAX)
    wsb = vista.vista_summarize_workspace_size(desc, total)
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)
    out = torch.empty((B, S, H, d), dtype=torch.bfloat16, device=dev)
    lse = torch.empty((B, H, S), dtype=torch.float32, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for a, b in evs:
        a.record(stream)
        b.record(stream)
    for _ in range(3):
        vista.vista_summarize_fwd(desc, q, K, V, off_t, total, out, lse, ws, wsb, stream.cuda_stream)
    torch.cuda.synchronize()
    for a, b in evs:
        vista.vista_time_next_main_kernel(a, b)
        vista.vista_summarize_fwd(desc, q, K, V, off_t, total, out, lse, ws, wsb, stream.cuda_stream)
    torch.cuda.synchronize()
    km = sum(a.elapsed_time(b) for a, b in evs) / len(evs)
    flops = 4.0 * total * H * S * d
    tiles = int(((lens + 127) // 128).sum()) * (S // 256)
    print(f"{name:22s} total={total} kernel_ms={km:.4f} frac={flops / km / 1e9 / tf:.4f} "
          f"ns_per_tile_per_sm={km * 1e6 * 148 / tiles:.1f}", flush=True)
    del q, K, V, out, lse, ws
    torch.cuda.empty_cache()
