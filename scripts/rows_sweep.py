"""QLA target rows (Delta term) from saved states: rows-kernel time vs rows per user, read from the
library's own per-launch CUDA events (vista_time_next_main_kernel).  GPU box only.
    python scripts/rows_sweep.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2510_22049_b200 as vista  # noqa: E402

B, H, d = 64, 4, 128
dev = "cuda"
g = torch.Generator(device=dev)
g.manual_seed(1)
z = (torch.randn((B, H, d, d), device=dev, generator=g) * 0.05).float()
ulen = torch.full((B,), 10000, dtype=torch.int64, device=dev)
for rpu in [128, 256, 512, 1024, 2048, 4096]:
    R = B * rpu
    grid = lambda: (torch.randint(-128, 128, (R, H, d), device=dev, generator=g).float() / 64).to(torch.bfloat16)  # noqa
    q, k, v = grid(), grid(), grid()
    roff = torch.arange(B + 1, device=dev, dtype=torch.int64) * rpu
    out = vista.qla_rows_from_state(z, ulen, q, roff, R, k_self=k, v_self=v)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        b.record()  # materialize the handles (recorded again by the library around the rows kernel)
        vista.vista_time_next_main_kernel(a, b)
        vista.qla_rows_from_state(z, ulen, q, roff, R, k_self=k, v_self=v)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    ms = ts[len(ts) // 2]
    tiles = B * H * ((rpu + 127) // 128)
    gb = R * H * d * 2 * 4 / 1e9 + B * H * d * d * 2 / 1e9
    print(f"rows/user {rpu:5d} tiles/SM {tiles / 148:6.2f}  rows kernel ms {ms:.4f}  {gb / (ms / 1e3):7.1f} GB/s")
