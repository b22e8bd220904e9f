#!/usr/bin/env python
"""Per-unit overhead probe: softmax kernel time vs user length at a fixed total history.

For each L, B = TOTAL // L users of exactly L items (S, H from argv).  Prints kernel ms and the
fraction of the measured bf16 peak, so the cost of a unit boundary (epilogue + pipeline restart)
and of the ragged tail can be read off the trend.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_22049_b200 as vista  # noqa: E402
import synth  # noqa: E402

S = int(os.environ.get("S", 256))
H = int(os.environ.get("H", 4))
TOTAL = int(os.environ.get("TOTAL", 2_560_000))
ATTN = os.environ.get("ATTN", "softmax")
LENS = [int(x) for x in os.environ.get("LENS", "128,256,512,1024,2048,4096,10000,40000,160000").split(",")]
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
tf = peak["bf16_tflops"]
d = 128
dev = torch.device("cuda")
stream = torch.cuda.current_stream()
attn = vista.SOFTMAX if ATTN == "softmax" else vista.QLA
for L in LENS:
    B = max(1, TOTAL // (L * H)) if H > 1 else max(1, TOTAL // L)
    lens = [L] * B
    q, K, V, off = synth.make_batch(lens, S, H, d, seed=0, backend="torch", device=dev)
    total = int(off[-1])
    off_t = torch.from_numpy(off).to(dev)
    desc = vista.make_desc(B, S, H, d, in_dtype=vista.BF16, out_dtype=vista.BF16, attn=attn)
    wsb = vista.vista_summarize_workspace_size(desc, total)
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)
    out = torch.empty((B, S, H, d), dtype=torch.bfloat16, device=dev)
    lse = torch.empty((B, H, S), dtype=torch.float32, device=dev) if attn == vista.SOFTMAX else None
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for a, b in evs:  # materialize the event handles
        a.record(stream)
        b.record(stream)
    for _ in range(5):
        vista.vista_summarize_fwd(desc, q, K, V, off_t, total, out, lse, ws, wsb, stream.cuda_stream)
    torch.cuda.synchronize()
    s0.record(stream)
    for a, b in evs:
        vista.vista_time_next_main_kernel(a, b)
        vista.vista_summarize_fwd(desc, q, K, V, off_t, total, out, lse, ws, wsb, stream.cuda_stream)
    s1.record(stream)
    torch.cuda.synchronize()
    km = sum(a.elapsed_time(b) for a, b in evs) / len(evs)
    sm = s0.elapsed_time(s1) / len(evs)
    flops = 4.0 * total * H * S * d
    print(f"L={L:7d} B={B:6d} items={total*H:9d} kernel_ms={km:.4f} step_ms={sm:.4f} "
          f"frac={flops / km / 1e9 / tf:.4f} ns_per_tile_per_sm={km * 1e6 * 148 / (B * H * ((L + 127) // 128) * max(1, S // 256)):.1f}",
          flush=True)
