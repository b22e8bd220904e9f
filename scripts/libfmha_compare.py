"""Context measurement: a library Blackwell FMHA on the c2 shape, beside this repo's softmax kernel.

Not part of the product path or of bench.py.  It answers one question for DESIGN.md §4.1: what does
NVIDIA's own sm100 attention kernel (flashinfer's trtllm-gen cubins, shipped precompiled in
flashinfer_cubin) reach on the same workload -- 64 users x 10,000 items, H = 4, S = 256 seed rows per
user, d = 128, bf16, no mask -- on the same box and clocks.  The seed rows are replicated per user
(the library has no shared-query mode), so it moves 64x more Q bytes (42 MB, ~3% of the traffic).

Usage (GPU box): python scripts/libfmha_compare.py [--iters 100] [--page 64]
The two arms alternate, 5 repetitions of --iters back-to-back launches each (median reported).
"""
import argparse
import json
import math
import sys

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--page", type=int, default=64)  # page 128 has no bf16 context cubin
    ap.add_argument("--users", type=int, default=64)
    ap.add_argument("--items", type=int, default=10000)
    ap.add_argument("--seeds", type=int, default=256)
    ap.add_argument("--heads", type=int, default=4)
    a = ap.parse_args()
    import flashinfer.prefill as fp

    dev = torch.device("cuda", 0)
    B, L, S, H, d, P = a.users, a.items, a.seeds, a.heads, 128, a.page
    g = torch.Generator(device=dev).manual_seed(0)
    pages_per = (L + P - 1) // P
    n_pages = B * pages_per
    k = torch.randn(n_pages, H, P, d, device=dev, dtype=torch.bfloat16, generator=g)
    v = torch.randn(n_pages, H, P, d, device=dev, dtype=torch.bfloat16, generator=g)
    q = torch.randn(B * S, H, d, device=dev, dtype=torch.bfloat16, generator=g)
    block_tables = torch.arange(n_pages, device=dev, dtype=torch.int32).view(B, pages_per)
    seq_lens = torch.full((B,), L, device=dev, dtype=torch.int32)
    cu_q = torch.arange(0, (B + 1) * S, S, device=dev, dtype=torch.int32)
    cu_kv = torch.arange(0, (B + 1) * L, L, device=dev, dtype=torch.int32)
    ws = torch.zeros(256 << 20, device=dev, dtype=torch.uint8)
    out = torch.empty_like(q)
    scale = 1.0 / math.sqrt(d)

    def run():
        fp.trtllm_batch_context_with_kv_cache(
            q, (k, v), ws, block_tables, seq_lens, S, L, scale, 1.0, B, cu_q, cu_kv,
            out=out, kv_layout="HND", causal=False)

    run()
    torch.cuda.synchronize()
    # correctness spot check on user 0, head 0 (fp32 reference of the same op)
    kk = k[:pages_per, 0].reshape(-1, d)[:L].float()
    vv = v[:pages_per, 0].reshape(-1, d)[:L].float()
    ref = torch.softmax(q[:S, 0].float() @ kk.T * scale, dim=-1) @ vv
    err = (out[:S, 0].float() - ref).abs().max().item()
    # this repo's path on the same shape (shared seed rows [S, H, d], K/V [B*L, H, d]), same loop
    sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    import paper_2510_22049_b200 as vista
    vista.load()
    qs = q[:S].contiguous()
    K2 = torch.randn(B * L, H, d, device=dev, dtype=torch.bfloat16, generator=g)
    V2 = torch.randn(B * L, H, d, device=dev, dtype=torch.bfloat16, generator=g)
    off = cu_kv.to(torch.int64)
    desc = vista.make_desc(B, S, H, d, in_dtype=vista.BF16, out_dtype=vista.BF16, attn=vista.SOFTMAX)
    wsb = vista.vista_summarize_workspace_size(desc, B * L)
    ws2 = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)
    out2 = torch.empty((B, S, H, d), dtype=torch.bfloat16, device=dev)
    lse2 = torch.empty((B, H, S), dtype=torch.float32, device=dev)
    sh = torch.cuda.current_stream(dev).cuda_stream

    def ours():
        vista.vista_summarize_fwd(desc, qs, K2, V2, off, B * L, out2, lse2, ws2, wsb, sh)

    for _ in range(5):
        run()
        ours()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = {"lib": [], "ours": []}
    for rep in range(5):  # alternate the two arms so both see the same clocks and power state
        for name, fn in (("lib", run), ("ours", ours)):
            torch.cuda.synchronize()
            st.record()
            for _ in range(a.iters):
                fn()
            en.record()
            torch.cuda.synchronize()
            times[name].append(st.elapsed_time(en) / a.iters)
    flop = 4.0 * S * d * H * B * L
    res = {"users": B, "items": L, "seeds": S, "heads": H, "d": d, "iters_per_rep": a.iters,
           "lib": "flashinfer trtllm-gen fmha (sm100 cubin, paged KV, page %d, per-user Q)" % P,
           "lib_max_abs_err_u0h0": err}
    for name, ts in times.items():
        ms = sorted(ts)[len(ts) // 2]
        res[name] = {"ms_median_of_5": round(ms, 5), "times_ms": [round(t, 5) for t in ts],
                     "tflops": round(flop / ms / 1e9, 1)}
    print(json.dumps(res))


if __name__ == "__main__":
    sys.exit(main())
