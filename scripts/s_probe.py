"""Forward kernel time at the c5 length mix for S = 256 vs 512 (same K/V): does S = 512 (two
256-row units per user, each streaming the user's K/V) lose efficiency per unit of work?"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2510_22049_b200 as vista  # noqa: E402
import synth  # noqa: E402
from bench import workload  # noqa: E402

cfg, lens, S0, H, d, _ = workload("c5", "softmax")
dev = torch.device("cuda:0")
_, K, V, off = synth.make_batch(lens, 1, H, d, seed=0, backend="torch", device=dev)
total = int(off[-1])
off_t = torch.from_numpy(off).to(dev)
for S in (256, 512, 1024):
    q = synth.make_q(S, H, d, seed=0, backend="torch", device=dev)
    desc = vista.make_desc(len(lens), S, H, d, in_dtype=vista.BF16, out_dtype=vista.BF16)
    n = vista.vista_summarize_workspace_size(desc, total)
    ws = torch.empty(n, dtype=torch.uint8, device=dev)
    out = torch.empty((len(lens), S, H, d), dtype=torch.bfloat16, device=dev)
    lse = torch.empty((len(lens), H, S), dtype=torch.float32, device=dev)
    for _ in range(3):
        vista.vista_summarize_fwd(desc, q, K, V, off_t, total, out, lse, ws, n, 0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    b.record()  # materialize the event handles
    ms = []
    for _ in range(20):
        vista.vista_time_next_main_kernel(a, b)
        vista.vista_summarize_fwd(desc, q, K, V, off_t, total, out, lse, ws, n, 0)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    ms.sort()
    k_ms = ms[len(ms) // 2]
    tf = 4.0 * S * d * H * total / (k_ms / 1e3) / 1e12
    print(f"S={S} kernel {k_ms:.4f} ms  {tf:.0f} TF/s  frac {tf / 1674.3:.3f}")
