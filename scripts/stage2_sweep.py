"""Stage-2 target attention: kernel time vs candidates per user (per-tile cost and fixed cost of the
launch).  Random int8 tokens; GPU box only.   python scripts/stage2_sweep.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2510_22049_b200 as vista  # noqa: E402

B, S, H, d = 64, 256, 4, 128
dev = "cuda"
g = torch.Generator(device=dev)
g.manual_seed(1)
codes = torch.randint(-127, 128, (B, S, H, d), device=dev, generator=g, dtype=torch.int8)
tsc = torch.rand((B, S, H), device=dev, generator=g) / 64 + 1e-3
tzp = torch.rand((B, S, H), device=dev, generator=g) - 0.5
for cpu in [16, 64, 128, 256, 512, 1024, 2048]:
    R = B * cpu
    grid = lambda: (torch.randint(-128, 128, (R, H, d), device=dev, generator=g).float() / 64).to(torch.bfloat16)  # noqa
    q, k, v = grid(), grid(), grid()
    roff = torch.arange(B + 1, device=dev, dtype=torch.int64) * cpu
    for _ in range(3):
        vista.target_attend(codes, tsc, tzp, q, k, v, roff, R)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        vista.target_attend(codes, tsc, tzp, q, k, v, roff, R)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    tiles = B * H * ((cpu + 127) // 128)
    print(f"cand/user {cpu:5d} tiles {tiles:6d} tiles/SM {tiles / 148:6.2f}  ms {ts[len(ts) // 2]:.4f}  "
          f"(incl. allocation of out / lse / workspace)")
