#!/usr/bin/env python
"""bench.py -- VISTA stage-1 user-history summarization throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--attn softmax|qla]
                    [--impl own|reference]

A step = one pass of the whole hot path (vista_summarize_fwd: tile scan, TMA/tcgen05 summarize
kernel, split-L merge) over one batch of synthetic histories already resident in HBM.  Default
workload = BASELINE.json configs[1] (c2: 64 users x 10,000 items, S=256, d=128, H=4, bf16).
Multi-GPU (torchrun, one process per GPU): every rank summarizes its own batch of users (by-user
sharding, weak scaling, no data-path collective); timing is max over ranks of CUDA-event time.

Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement" for every field.
``--impl reference`` times the float64 CPU oracle (the reference arm of this tier) on a bounded
sample of the same workload, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "history items summarized/sec (S=256,d=128) + % bf16 tensor peak, 1/2/4/8 GPU"
METRIC_STAGE2 = "stage-2 candidates scored/sec over the cached int8 summary tokens (NEXT-4; not the headline metric)"
L2_BYTES = 126 * 1024 * 1024  # B200 L2 (the timing rule: inputs larger than L2, or rotated copies)
TARGETS_PER_USER = 256  # --qla-rows target: candidate rows per user (NEXT-4)
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--attn", default="softmax", choices=["softmax", "qla"])
    ap.add_argument("--impl", default="own", choices=["own", "reference"])
    ap.add_argument("--mode", default=None, choices=["by_user", "by_length", "flat"],
                    help="multi-GPU partitioner (default per config: c2/c3 by_user, c4 by_length, c5 flat)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--qla-rows", choices=["history", "target"], default=None,
                    help="NEXT-3/4 (QLA): the step is vista_qla_rows -- every history item as a query row of its "
                         "own user (history), or 256 target rows per user with the Delta self term (target)")
    ap.add_argument("--layers", type=int, default=0,
                    help="NEXT-3: the step is an N-layer summarizer (vista_summarize_layers: projections, QLA over "
                         "[seeds; history], SGLU, output projection, residual) over the batch")
    ap.add_argument("--stage2", action="store_true",
                    help="NEXT-4: the step is stage-2 target-aware attention (vista_target_attend) of "
                         f"{TARGETS_PER_USER} candidates per user over the int8 export of the batch's summary tokens")
    ap.add_argument("--backward", action="store_true",
                    help="NEXT-2: the step is the QLA backward (vista_summarize_bwd: Z recompute, dQ, dK, dV)")
    ap.add_argument("--export-int8", action="store_true",
                    help="NEXT-1: the step also exports the summary tokens as int8 (vista_quantize_rows_int8)")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="run the K timed steps eagerly instead of as one captured CUDA graph")
    ap.add_argument("--no-sustained", dest="sustained", action="store_false",
                    help="skip the SURVEY 8(d) protocol block (>= 200 ms graph replays, median of 5)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process group for N > 1 (gloo: host-staged exchange; a dry run of the multi-rank "
                         "path when fewer GPUs than ranks are visible)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p", "p2p-push"],
                    help="by_length split-L exchange: NCCL all_gather (default) or peer-memory stores over NVLink "
                         "(dist.PeerExchange, CUDA IPC; one node) -- p2p: made by the partial's own kernels "
                         "(vista_summarize_partial_peers), p2p-push: by a push kernel after the partial")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle time for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return dict(FALLBACK_PEAKS), "fallback"


def workload(config, attn):
    import synth
    cfg = synth.CONFIGS[config]
    lens = synth.user_lengths(config, seed=0)
    S, H, d = cfg["S"], cfg["H"], cfg["d"]
    desc = {
        "c2": "c2: 64 users x 10,000 items, S=256, d=128, H=4, bf16",
        "c3": "c3: 32 users x U[10k,100k] items, S=256, d=128, H=1, bf16",
        "c4": "c4: 8 users x 1,000,000 items, S=256, d=128, H=1, bf16",
        "c5": "c5: 1,024 users x power-law[1k,1M] items, S=512, d=128, H=1, bf16",
    }[config]
    return cfg, lens, S, H, d, desc + f", {attn}"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms; keep samples in [t0, t1]."""
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.lines = []
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self, t0, t1):
        if self.p is None:
            return None
        time.sleep(0.12)
        self.p.terminate()
        try:
            self.p.wait(timeout=2)
        except Exception:
            self.p.kill()
        rows = [l for (ts, l) in self.lines if t0 - 0.06 <= ts <= t1 + 0.06]
        if not rows:  # timed region shorter than one sample period: nearest sample after it
            after = [l for (ts, l) in self.lines if ts >= t0]
            rows = after[:1]
        mhz, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            f = [x.strip() for x in r.split(",")]
            if len(f) < 7:
                continue
            try:
                mhz.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not mhz:
            return None
        mhz.sort()
        return {"sm_mhz": mhz[len(mhz) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(mhz)}


# ----------------------------------------------------------------------------- own arm
def run_own(args, rank, world, local_rank):
    phase_fns = None  # by_length: (partial, all_gather, merge) callables for the per-phase breakdown
    import numpy as np
    import torch

    import paper_2510_22049_b200 as vista
    import synth

    vista.load()
    from paper_2510_22049_b200 import dist as vdist
    dev = torch.device("cuda", local_rank % max(torch.cuda.device_count(), 1))
    torch.cuda.set_device(dev)
    cfg, lens, S, H, d, wdesc = workload(args.config, args.attn)
    if args.backward:
        wdesc += " backward (NEXT-2, from the forward's saved " + ("out, lse)" if args.attn == "softmax" else "state Z)")
    if args.layers:
        wdesc += (f" {args.layers}-layer summarizer (NEXT-3: X = [S seeds; history] per user, D = H d; per layer the "
                  "QKVG projection GEMM, QLA state + rows over all rows, SGLU-gated output GEMM + residual)")
    if args.stage2:
        wdesc += (f" stage-2 target-aware attention (NEXT-4: {TARGETS_PER_USER} candidates per user over the "
                  f"{S} int8 summary tokens of the user + itself)")
    if args.qla_rows:
        wdesc += (" QLA history rows from the saved state (NEXT-3: every item a query row of its user)"
                  if args.qla_rows == "history"
                  else f" QLA target rows from the saved state (NEXT-4: {TARGETS_PER_USER} targets per user, Delta self term)")
    attn = vista.SOFTMAX if args.attn == "softmax" else vista.QLA
    mode = args.mode or {"c2": "by_user", "c3": "by_user", "c4": "by_length", "c5": "flat"}[args.config]
    if (world == 1 or args.qla_rows) and mode != "by_user":
        mode = "by_user"  # one shard: the split-L paths degenerate to the plain forward; rows: per-user batches
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream
    B_all = len(lens)
    off_all = synth.offsets_from_lengths(lens)
    if mode == "by_user":
        # weak scaling: rank r summarizes its own batch of the configured shape (seed r)
        q, K, V, off = synth.make_batch(lens, S, H, d, seed=rank, backend="torch", device=dev)
        total = int(off[-1])
        off_t = torch.from_numpy(off).to(dev)
        B = len(lens)
        desc = vista.make_desc(B, S, H, d, in_dtype=vista.BF16, out_dtype=vista.BF16, attn=attn)
        ws_bytes = vista.vista_summarize_workspace_size(desc, total)
        ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=dev)
        out = torch.empty((B, S, H, d), dtype=torch.bfloat16, device=dev)
        lse = torch.empty((B, H, S), dtype=torch.float32, device=dev) if attn == vista.SOFTMAX else None
        inputs = [q, K, V, off_t]
        nrows = B * S * H
        codes = torch.empty((nrows, d), dtype=torch.int8, device=dev) if args.export_int8 else None
        qscale = torch.empty(nrows, dtype=torch.float32, device=dev) if args.export_int8 else None
        qzp = torch.empty(nrows, dtype=torch.float32, device=dev) if args.export_int8 else None

        def export():
            vista.vista_quantize_rows_int8(nrows, d, vista.BF16, out, codes, qscale, qzp, None)

        def step(ins=inputs):
            if args.export_int8:  # NEXT-1: the export fused into the summarization's epilogues
                vista.vista_summarize_fwd_int8(desc, ins[0], ins[1], ins[2], ins[3], total, out, lse, codes, qscale,
                                               qzp, ws, ws_bytes, None)
                return [codes, qscale, qzp] + ([lse] if lse is not None else [])
            vista.vista_summarize_fwd(desc, ins[0], ins[1], ins[2], ins[3], total, out, lse, ws, ws_bytes, None)
            return [out] + ([lse] if lse is not None else [])
        if args.backward:
            gen = torch.Generator(device=dev)
            gen.manual_seed(1234 + rank)
            dout = (torch.randint(-128, 128, (B, S, H, d), device=dev, generator=gen).float() / 64).to(torch.bfloat16)
            dq = torch.empty((S, H, d), dtype=torch.float32, device=dev)
            dk = torch.empty_like(K)
            dv = torch.empty_like(V)
            bws_bytes = vista.vista_summarize_bwd_workspace_size(desc, total)
            bws = torch.empty(max(bws_bytes, 16), dtype=torch.uint8, device=dev)
            inputs = [q, K, V, off_t, dout]

            fwd_out, fwd_lse, fwd_z = (None, None, None)
            if attn == vista.SOFTMAX:  # the forward's out / lse (computed once, outside the timed region)
                vista.vista_summarize_fwd(desc, q, K, V, off_t, total, out, lse, ws, ws_bytes, sh)
                fwd_out, fwd_lse = out.clone(), lse.clone()
            else:  # the forward's saved state Z (partial mode; computed once, outside the timed region)
                fwd_z = torch.empty((B, H, d, d), dtype=torch.float32, device=dev)
                vista.vista_summarize_partial(desc, q, K, V, off_t, total, fwd_z, None, ws, ws_bytes, sh)

            def step(ins=inputs):
                if fwd_z is not None:
                    vista.vista_summarize_bwd_qla_saved(desc, ins[0], ins[1], ins[2], ins[3], total, fwd_z, ins[4],
                                                        dq, dk, dv, bws, bws_bytes, None)
                else:
                    vista.vista_summarize_bwd(desc, ins[0], ins[1], ins[2], ins[3], total, fwd_out, fwd_lse, ins[4],
                                              dq, dk, dv, bws, bws_bytes, None)
                if world > 1:  # data parallel: the shared seeds' gradient is summed over the ranks (NCCL)
                    torch.distributed.all_reduce(dq)
                return [dq, dk, dv]
        if args.qla_rows:
            gen = torch.Generator(device=dev)
            gen.manual_seed(4321 + rank)
            grid = lambda shape: (torch.randint(-128, 128, shape, device=dev, generator=gen).float() / 64  # noqa: E731
                                  ).to(torch.bfloat16)
            if args.qla_rows == "history":
                roff_t, n_rows = off_t, total
                q_rows, k_self, v_self = grid((total, H, d)), None, None
            else:
                n_rows = TARGETS_PER_USER * B
                roff_t = torch.arange(B + 1, dtype=torch.int64, device=dev) * TARGETS_PER_USER
                q_rows, k_self, v_self = grid((n_rows, H, d)), grid((n_rows, H, d)), grid((n_rows, H, d))
            rows_out = torch.empty((n_rows, H, d), dtype=torch.bfloat16, device=dev)
            # the layer's state is computed once (the summarization pass, outside the timed step) and
            # reused by the rows: "can be computed first, then multiplied with Q[S]_l, Q[T]_l"
            z_state = torch.empty((B, H, d, d), dtype=torch.float32, device=dev)
            vista.vista_summarize_partial(desc, q, K, V, off_t, total, z_state, None, ws, ws_bytes, None)
            ulen_t = torch.from_numpy(np.asarray(lens, dtype=np.int64)).to(dev)
            rws_bytes = vista.vista_qla_rows_from_state_workspace_size(desc, n_rows)
            rws = torch.empty(max(rws_bytes, 16), dtype=torch.uint8, device=dev)
            inputs = [z_state, ulen_t, q_rows, roff_t] + ([k_self, v_self] if k_self is not None else [])

            def step(ins=inputs):
                ks, vs = (ins[4], ins[5]) if len(ins) > 4 else (None, None)
                vista.vista_qla_rows_from_state(desc, ins[0], ins[1], ins[2], ins[3], n_rows, ks, vs, rows_out,
                                                rws, rws_bytes, None)
                return [rows_out]
        if args.stage2:
            # the batch's summary tokens as the int8 export (vista_summarize_fwd_int8, outside the step)
            codes = torch.empty((B, S, H, d), dtype=torch.int8, device=dev)
            tsc = torch.empty((B, S, H), dtype=torch.float32, device=dev)
            tzp = torch.empty((B, S, H), dtype=torch.float32, device=dev)
            vista.vista_summarize_fwd_int8(desc, q, K, V, off_t, total, out, lse, codes, tsc, tzp, ws, ws_bytes, None)
            gen = torch.Generator(device=dev)
            gen.manual_seed(5678 + rank)
            grid = lambda shape: (torch.randint(-128, 128, shape, device=dev, generator=gen).float() / 64  # noqa: E731
                                  ).to(torch.bfloat16)
            n_rows = TARGETS_PER_USER * B
            roff_t = torch.arange(B + 1, dtype=torch.int64, device=dev) * TARGETS_PER_USER
            cq, ck, cv = grid((n_rows, H, d)), grid((n_rows, H, d)), grid((n_rows, H, d))
            sdesc = vista.make_desc(B, S, H, d, in_dtype=vista.BF16, out_dtype=vista.BF16, attn=vista.SOFTMAX)
            s2_out = torch.empty((n_rows, H, d), dtype=torch.bfloat16, device=dev)
            s2_lse = torch.empty((n_rows, H), dtype=torch.float32, device=dev)
            s2_bytes = vista.vista_target_attend_workspace_size(sdesc, n_rows)
            s2_ws = torch.empty(max(s2_bytes, 16), dtype=torch.uint8, device=dev)
            inputs = [codes, tsc, tzp, cq, ck, cv, roff_t]

            def step(ins=inputs):
                vista.vista_target_attend(sdesc, ins[0], ins[1], ins[2], ins[3], ins[4], ins[5], None, ins[6], n_rows,
                                          s2_out, s2_lse, s2_ws, s2_bytes, None)
                return [s2_out, s2_lse]
        if args.layers:
            D = H * d
            seg = np.asarray([S + int(L) for L in lens], dtype=np.int64)
            x_off = synth.offsets_from_lengths(seg)
            R_rows = int(x_off[-1])
            gen = torch.Generator(device=dev)
            gen.manual_seed(999 + rank)
            x0 = (torch.randint(-128, 128, (R_rows, D), device=dev, generator=gen).float() / 64).to(torch.bfloat16)
            wl = (torch.randint(-128, 128, (args.layers, 5, D, D), device=dev, generator=gen).float()
                  / (128.0 * math.sqrt(D))).to(torch.bfloat16)
            xw = torch.empty_like(x0)
            xoff_t = torch.from_numpy(x_off).to(dev)
            ldesc = vista.make_desc(B, S, H, d, in_dtype=vista.BF16, out_dtype=vista.BF16, attn=vista.QLA)
            l_bytes = vista.vista_summarize_layers_workspace_size(ldesc, args.layers, R_rows)
            l_ws = torch.empty(max(l_bytes, 16), dtype=torch.uint8, device=dev)
            tokens = torch.empty((B, S, H, d), dtype=torch.bfloat16, device=dev)
            inputs = [x0, wl, xoff_t]

            def step(ins=inputs):
                xw.copy_(ins[0])  # the layers update X in place: every step starts from the embeddings
                vista.vista_summarize_layers(ldesc, args.layers, ins[1], xw, ins[2], R_rows, tokens, l_ws, l_bytes,
                                             None)
                return [tokens]
        items_per_step = world * (n_rows if args.stage2 else total)
        scaling = "weak"
        parallel = f"by_user x{world} (weak: a {args.config} batch per GPU, no data-path collective)"
        if args.backward:
            parallel = f"by_user x{world} (weak: a {args.config} batch per GPU; NCCL all_reduce of the seed gradient)"
    else:
        # strong scaling: one batch of the configured shape split across the ranks
        q = synth.make_q(S, H, d, seed=0, backend="torch", device=dev)
        if mode == "by_length":
            cuts = vdist.partition_by_length(lens, world)
            seg = [(u, int(cuts[rank, u]), int(cuts[rank + 1, u])) for u in range(B_all)]
        else:
            seg = [(s.user, s.start, s.end) for s in vdist.partition_flat(lens, world)[rank]]
            all_segs = vdist.partition_flat(lens, world)
        seg_len = np.array([e - a for _, a, e in seg], dtype=np.int64)
        soff = synth.offsets_from_lengths(seg_len)
        total = int(soff[-1])
        tdt = torch.bfloat16
        K = torch.empty((total, H, d), dtype=tdt, device=dev)
        V = torch.empty((total, H, d), dtype=tdt, device=dev)
        off_dev = torch.from_numpy(off_all).to(dev)
        for n, (u, a0, e0) in enumerate(seg):  # generate this rank's rows (global row ids)
            for r0 in range(a0, e0, 1 << 18):
                r1 = min(e0, r0 + (1 << 18))
                rows = torch.arange(int(off_all[u]) + r0, int(off_all[u]) + r1, dtype=torch.int64, device=dev)
                users = torch.full_like(rows, u)
                k, v = synth.make_kv(rows, users, H, d, seed=0, backend="torch", device=dev)
                K[int(soff[n]) + r0 - a0:int(soff[n]) + r1 - a0] = k
                V[int(soff[n]) + r0 - a0:int(soff[n]) + r1 - a0] = v
        soff_t = torch.from_numpy(soff).to(dev)
        ulen = torch.from_numpy(np.asarray(lens, dtype=np.int64)).to(dev)
        inputs = [q, K, V, soff_t]
        if mode == "by_length":
            acode = 0 if args.attn == "softmax" else 1
            xchg = None
            fused = args.exchange == "p2p"
            if args.exchange in ("p2p", "p2p-push"):  # peer-memory exchange (CUDA IPC buffers, NVLink stores)
                part_shape = (B_all, H, S, d) if acode == 0 else (B_all, H, d, d)
                xchg = vdist.PeerExchange(part_shape, (B_all, H, S) if acode == 0 else None)

            def step(ins=inputs):
                out, lse = vdist.summarize_by_length(ins[0], ins[1], ins[2], ins[3], ulen, attn=args.attn,
                                                     total_len=total, exchange=xchg, fused=fused)
                return [out] + ([lse] if lse is not None else [])

            # the same three phases, separately callable for the breakdown (summarize_by_length's body)
            be = vdist.CudaBackend()
            if xchg is None:
                phase_fns = (lambda: be.partial(q, K, V, soff_t, total, acode),
                             lambda pp: (vdist._all_gather(pp[0], None),
                                         vdist._all_gather(pp[1], None) if acode == 0 else None),
                             lambda gg: be.merge(gg[0], gg[1], q, acode, ulen))
            else:
                def _merge_release(gg):
                    res = be.merge(gg[0], gg[1] if acode == 0 else None, q, acode, ulen)
                    xchg.release()
                    return res
                if fused:  # partial + stores into every receive buffer | signal + wait | merge
                    phase_fns = (lambda: be.partial_peers(q, K, V, soff_t, total, xchg, acode),
                                 lambda pp: xchg.signal_wait(),
                                 _merge_release)
                else:
                    phase_fns = (lambda: be.partial(q, K, V, soff_t, total, acode),
                                 lambda pp: xchg.gather(pp[0], pp[1] if acode == 0 else None),
                                 _merge_release)
        else:
            segs_obj = [vdist.Segment(u, a0, e0) for u, a0, e0 in seg]
            fplan = vdist.FlatPlan(all_segs, lens, rank, dev)

            def step(ins=inputs):
                res = vdist.summarize_flat(ins[0], ins[1], ins[2], segs_obj, all_segs, lens, attn=args.attn,
                                           plan=fplan)
                return [o for o, _ in res.values()][:1] or [ins[0]]
        items_per_step = int(off_all[-1])
        scaling = "strong"
        parallel = (f"{mode} x{world} (strong: one {args.config} batch split; all_gather of partials over "
                    + (("peer memory (CUDA IPC, NVLink stores"
                        + (", fused into the partial's kernels)" if args.exchange == "p2p" else ", push kernel)"))
                       if (mode == "by_length" and args.exchange != "nccl") else "NCCL") + ")")
        B = B_all
    path = vista.vista_dispatch_name(vista.make_desc(B, S, H, d, in_dtype=vista.BF16, attn=attn))

    # Timing rule: no step may find its inputs in L2 from the previous step.  Workloads whose inputs
    # fit in L2 (stage 2, target rows: ~70 MB) rotate over R device copies, R x inputs > 3 x L2.
    in_bytes = sum(x.numel() * x.element_size() for x in inputs if isinstance(x, torch.Tensor))
    l2_note = f"inputs {in_bytes / 1e9:.2f} GB/GPU > 126 MB L2, no flush"
    if mode == "by_user" and 0 < in_bytes < 2 * L2_BYTES:
        n_rot = min(16, -(-3 * L2_BYTES // in_bytes))
        rot = [inputs] + [[x.clone() if isinstance(x, torch.Tensor) else x for x in inputs] for _ in range(n_rot - 1)]
        rot_ctr = [0]
        base_step = step

        def step(ins=None):
            if ins is None:
                ins = rot[rot_ctr[0] % n_rot]
                rot_ctr[0] += 1
            return base_step(ins)
        l2_note = (f"inputs {in_bytes / 1e6:.1f} MB/GPU < L2: the steps rotate over {n_rot} device copies "
                   f"({n_rot * in_bytes / 1e6:.0f} MB > 126 MB L2), no flush")

    # warm-up (eager: also initializes NCCL communicators and the library's per-device state)
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    K_steps = args.steps
    ev_k = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K_steps)]
    for a, b in ev_k:  # materialize the handles (the library records them through the raw cudaEvent_t)
        a.record(stream)
        b.record(stream)
    t_start, t_stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def run_steps(n, evs=None):
        for i in range(n):
            if evs is not None:
                vista.vista_time_next_main_kernel(evs[i][0], evs[i][1])
            step()

    # The K timed steps are captured once into a CUDA graph (one launch per replay: no host gaps
    # between the steps' kernels); eager if capture is unavailable (gloo host staging) or fails.
    # Two captures of the same K steps: `graph` (the timed region) without instrumentation, and
    # `graph_ev` with CUDA events around each step's dominant kernel, replayed right after the timed
    # region for the kernel time -- an event node between two kernels breaks their programmatic
    # (PDL) overlap and costs ~8 us per step (scripts/microbench/gtimer_check.cu), which must not
    # land in the timed steps.
    graph, graph_ev, graph_note = None, None, None
    if args.graph and args.dist_backend != "gloo":
        try:
            graph, graph_ev = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            cs.wait_stream(stream)
            with torch.cuda.stream(cs):
                run_steps(1)  # warm the capture stream
                graph.capture_begin()
                c0 = vista.vista_launch_counter()
                run_steps(K_steps)
                captured_launches = vista.vista_launch_counter() - c0
                graph.capture_end()
                graph_ev.capture_begin()
                run_steps(K_steps, ev_k)
                graph_ev.capture_end()
            stream.wait_stream(cs)
            torch.cuda.synchronize()
            graph.replay()  # first replays upload the graphs: outside the timed region
            graph_ev.replay()
            torch.cuda.synchronize()
        except Exception as exc:  # noqa: BLE001 -- recorded in the JSON line
            graph, graph_ev = None, None
            graph_note = f"eager (capture failed: {type(exc).__name__}: {str(exc)[:120]})"
            torch.cuda.synchronize()
    elif not args.graph:
        graph_note = "eager (--no-graph)"
    else:
        graph_note = "eager (gloo exchange is host-staged, not capturable)"
    gpu_index = os.environ.get("CUDA_VISIBLE_DEVICES", str(dev.index)).split(",")[dev.index] \
        if "CUDA_VISIBLE_DEVICES" in os.environ else str(dev.index)
    sampler = ClockSampler(gpu_index)
    time.sleep(0.3)  # let nvidia-smi start sampling
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = vista.vista_launch_counter()
    w0 = time.time()
    t_start.record(stream)
    if graph is not None:
        graph.replay()
    else:
        run_steps(K_steps, ev_k)
    t_stop.record(stream)
    torch.cuda.synchronize()
    w1 = time.time()
    if world > 1:
        torch.distributed.barrier()
    # library launches inside the timed region: counted at capture time for a graph (one replay
    # runs exactly the captured launches), live otherwise
    launches = (captured_launches if graph is not None else vista.vista_launch_counter() - launches0)
    clocks = sampler.stop(w0, w1)
    elapsed_ms = t_start.elapsed_time(t_stop)
    if graph_ev is not None:  # the instrumented replay of the same K steps, right after the timed one
        graph_ev.replay()
        torch.cuda.synchronize()
    try:
        kern_ms = sum(a.elapsed_time(b) for a, b in ev_k) / K_steps
    except Exception as exc:  # noqa: BLE001 -- graph-recorded events not timeable: time the kernel eagerly
        torch.cuda.synchronize()
        ev_k = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K_steps)]
        for a, b in ev_k:
            a.record(stream)
            b.record(stream)
        run_steps(K_steps, ev_k)
        torch.cuda.synchronize()
        kern_ms = sum(a.elapsed_time(b) for a, b in ev_k) / K_steps
        graph_note = (graph_note or "graph") + f"; kernel events re-timed over K eager steps ({type(exc).__name__})"

    phases = None
    if world > 1 and mode == "by_length" and phase_fns is not None:
        # per-phase breakdown of the split-L step (eager, after the timed region):
        # partial kernel(s), the all_gather of the partials, the merge; CUDA events, max over ranks
        pf, xf, mf = phase_fns
        acc = [0.0, 0.0, 0.0]
        nrep = 5
        for _ in range(nrep):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e[0].record(stream)
            parts = pf()
            e[1].record(stream)
            gathered = xf(parts)
            e[2].record(stream)
            mf(gathered)
            e[3].record(stream)
            torch.cuda.synchronize()
            for i in range(3):
                acc[i] += e[i].elapsed_time(e[i + 1]) / nrep
        t = torch.tensor(acc, device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        phases = {"partial_ms": round(float(t[0]), 5), "all_gather_ms": round(float(t[1]), 5),
                  "merge_ms": round(float(t[2]), 5),
                  "note": "eager, 5 repetitions after the timed region, each phase max over ranks"}
    if world > 1:
        t = torch.tensor([elapsed_ms, kern_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        elapsed_ms, kern_ms = float(t[0]), float(t[1])
    value = items_per_step * K_steps / (elapsed_ms / 1e3)

    # ---- SURVEY 8(d) protocol, beside the K-step number: R graph-replayed steps with R * t >= 200 ms,
    # median of 5 runs, with the clocks of those runs (the sustained, power-capped regime)
    sustained = None
    if args.sustained and world == 1 and graph is not None:
        R = max(1, int(math.ceil(200.0 / max(elapsed_ms / K_steps, 1e-3))))
        reps = max(1, int(math.ceil(R / K_steps)))
        sampler2 = ClockSampler(gpu_index)
        time.sleep(0.3)
        runs = []
        w2 = time.time()
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                graph.replay()
            b.record(stream)
            torch.cuda.synchronize()
            runs.append(a.elapsed_time(b) / (reps * K_steps))
        w3 = time.time()
        graph_ev.replay()  # per-step kernel events in the sustained regime
        torch.cuda.synchronize()
        try:
            kern_sus = sum(a.elapsed_time(b) for a, b in ev_k) / K_steps
        except Exception:  # noqa: BLE001
            kern_sus = kern_ms  # graph-recorded events not timeable: the K-step figure
        runs.sort()
        sustained = {"ms_per_step_median": runs[2], "ms_per_step_runs": [round(x, 5) for x in runs],
                     "steps_per_run": reps * K_steps, "value": items_per_step / (runs[2] / 1e3),
                     "kernel_ms": round(kern_sus, 5), "clocks": sampler2.stop(w2, w3)}

    # ---- end to end through the C ABI with host buffers (pinned), copies inside the timed region
    e2e = None
    if args.e2e_steps > 0:
        host_in = [x.cpu().pin_memory() for x in inputs]
        dev_in = [torch.empty_like(x) for x in inputs]
        outs0 = step()
        host_out = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in outs0]

        def e2e_step():
            for hx, dx in zip(host_in, dev_in):
                dx.copy_(hx, non_blocking=True)
            outs = step(dev_in)
            for ho, o in zip(host_out, outs):
                ho.copy_(o, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e_ms = float(t[0])
        h2d = sum(x.numel() * x.element_size() for x in host_in)
        d2h = sum(x.numel() * x.element_size() for x in host_out)
        e2e = {"value": items_per_step * args.e2e_steps / (e_ms / 1e3), "unit": "candidates/s" if args.stage2 else "items/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
               "note": "per rank: pinned host inputs -> H2D -> the step through the C ABI -> D2H of outputs; "
                       "CUDA events, max over ranks"}

    export_info = None
    if args.export_int8 and mode == "by_user":
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(20):
            export()
        b.record(stream)
        torch.cuda.synchronize()
        xms = a.elapsed_time(b) / 20
        xbytes = nrows * d * 2 + nrows * d + nrows * 8
        export_info = {"fused": "the step runs vista_summarize_fwd_int8 (export inside the epilogues)",
                       "separate_kernel": "quantize_rows_kernel", "separate_kernel_ms": round(xms, 5),
                       "separate_bytes_per_launch": xbytes,
                       "separate_achieved_gbs": round(xbytes / (xms / 1e3) / 1e9, 1), "rows": nrows,
                       "scheme": "per-row affine int8, SPEC.md:339-347 (NEXT-1)"}
    if rank != 0:
        return None
    pk, pk_kind = peaks()
    # algorithmic work of ONE launch of the dominant kernel on this rank (its `total` items)
    flops = 4.0 * S * d * H * total if attn == vista.SOFTMAX else 2.0 * d * d * H * total
    kv_bytes = 4.0 * d * H * total  # bf16 K + V, read once
    io_bytes = kv_bytes + S * H * d * 2 + B * S * H * d * 2 + (B * H * S * 4 if attn == vista.SOFTMAX else 0)
    if args.backward and attn == vista.QLA:  # dK / dV kernel: K, V read, dK, dV written (bf16)
        flops = 4.0 * d * d * H * total
        io_bytes = 2 * kv_bytes + B * H * d * d * 2
    elif args.backward:  # softmax dK / dV kernel: S^T, dP^T, dV, dK GEMMs = 8 S d flop per item-head
        flops = 8.0 * S * d * H * total
        io_bytes = 2 * kv_bytes + 2 * B * S * H * d * 2
    if args.qla_rows:  # rows kernel: q read, out written (bf16) [+ k_self, v_self read], W_u per unit
        flops = 2.0 * d * d * H * n_rows
        io_bytes = 4.0 * d * H * n_rows * (2 if args.qla_rows == "target" else 1) + B * H * d * d * 2
    if args.layers:  # projection GEMM of the first layer: X [R, D] x [Wq|Wk|Wv|Wg]^T [4D, D]
        flops = 2.0 * R_rows * D * 4 * D
        io_bytes = 2.0 * R_rows * D * 5 + 4 * D * D * 2
    if args.stage2:  # target attention: q, k_c, v_c read, out written (bf16), lse; int8 tokens + scales
        flops = 4.0 * S * d * H * n_rows
        io_bytes = 4.0 * 2 * d * H * n_rows + 4.0 * H * n_rows + B * S * H * (d + 8)
    # The per-kernel events carry a fixed cost (~8 us: the event nodes serialize the kernels they
    # bracket); a kernel cannot take longer than the whole step that contains it, so for the short
    # kernels (stage 2, target rows) the achieved rate uses the step time when it is the smaller.
    kern_events_ms = kern_ms
    kern_ms = min(kern_ms, elapsed_ms / K_steps)
    tflops = flops / (kern_ms / 1e3) / 1e12
    gbs = io_bytes / (kern_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        tkey = f"{args.config}_{args.attn}" + ("_bwd" if args.backward else "") + \
            (f"_rows_{args.qla_rows}" if args.qla_rows else "") + ("_stage2" if args.stage2 else "") + \
            (f"_layers{args.layers}" if args.layers else "")
        traffic = json.load(open(tpath)).get(tkey)
    if args.layers:
        roof = {"bound": "tensor", "achieved": round(tflops, 2), "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                "frac": round(tflops / pk["bf16_tflops"], 4), "traffic": traffic,
                "peak_kind": f"{pk_kind} bf16 burst", "kernel": "sm100_gemm_kernel (QKVG projection)",
                "kernel_ms": round(kern_ms, 5), "algorithmic_flop_per_launch": flops,
                "hbm": {"achieved": round(gbs, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": round(gbs / pk["hbm_gbs"], 4), "algorithmic_bytes_per_launch": io_bytes}}
    elif args.stage2:
        roof = {"bound": "hbm", "achieved": round(gbs, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(gbs / pk["hbm_gbs"], 4), "traffic": traffic, "peak_kind": f"{pk_kind} HBM copy",
                "kernel": "sm100_target_attend_kernel", "kernel_ms": round(kern_ms, 5),
                "algorithmic_bytes_per_launch": io_bytes,
                "tensor": {"achieved": round(tflops, 2), "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                           "frac": round(tflops / pk["bf16_tflops"], 4)}}
    elif attn == vista.SOFTMAX:
        roof = {"bound": "tensor", "achieved": round(tflops, 2), "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                "frac": round(tflops / pk["bf16_tflops"], 4), "traffic": traffic,
                "peak_kind": f"{pk_kind} bf16 burst (kernel timed alone per launch)",
                "kernel": "sm100_softmax_bwd_kv_kernel" if args.backward else "sm100_softmax_kernel",
                "kernel_ms": round(kern_ms, 5),
                # context: the same against the power-capped sustained GEMM figure, the denominator for
                # a kernel inside a long run (this run's clocks say whether sw_power_cap was active)
                "sustained": ({"peak": pk["bf16_tflops_sustained"],
                               "frac": round(tflops / pk["bf16_tflops_sustained"], 4)}
                              if pk.get("bf16_tflops_sustained") else None),
                "algorithmic_flop_per_launch": flops,
                "hbm": {"achieved": round(gbs, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": round(gbs / pk["hbm_gbs"], 4), "algorithmic_bytes_per_launch": io_bytes}}
    else:
        roof = {"bound": "hbm", "achieved": round(gbs, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": round(gbs / pk["hbm_gbs"], 4), "traffic": traffic, "peak_kind": f"{pk_kind} HBM copy",
                "kernel": ("sm100_qla_rows_kernel" if args.qla_rows else
                           "sm100_qla_bwd_kv_kernel" if args.backward else "sm100_qla_state_kernel"),
                "kernel_ms": round(kern_ms, 5),
                "algorithmic_bytes_per_launch": io_bytes,
                "tensor": {"achieved": round(tflops, 2), "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                           "frac": round(tflops / pk["bf16_tflops"], 4)}}
    res = {
        "metric": METRIC_STAGE2 if args.stage2 else METRIC, "value": value,
        "unit": "candidates/s" if args.stage2 else "items/s", "n_gpus": world, "steps": K_steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / K_steps, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded counter-based generator, bf16-exact grid values; synth/)",
        "config": {"workload": wdesc, "users_per_gpu": B, "items_per_gpu": total, "S": S, "d": d, "H": H,
                   "attn": args.attn, "parallelism": parallel, "mode": mode,
                   "path": path, "l2": l2_note,
                   "pct_bf16_tensor_peak": round(100 * tflops / pk["bf16_tflops"], 2)},
        "roofline": roof,
        "clocks": clocks,
        "e2e": e2e,
        "gpu_launches": launches,
        "timing": {"steps": graph_note or f"the {K_steps} timed steps replayed as one captured CUDA graph",
                   "kernel_events": ("per-step CUDA events around the dominant kernel (vista_time_next_main_kernel), "
                                     "on the launching stream" +
                                     ("; in a second capture of the same K steps replayed right after the timed "
                                      "one (event nodes break the PDL overlap of the kernels they separate: "
                                      "~8 us per step)" if graph_ev is not None else ", inside the timed steps"))},
    }
    if kern_events_ms > kern_ms:
        roof["kernel_ms_events"] = round(kern_events_ms, 5)
        roof["kernel_ms_note"] = ("the per-kernel events (kernel_ms_events) exceed the whole step: kernel_ms is the "
                                  "step time, an upper bound of the kernel's duration")
    if sustained is not None:
        sustained["kernel_ms"] = round(min(sustained["kernel_ms"], sustained["ms_per_step_median"]), 5)
        # same bound and unit as the burst roofline above, against the sustained denominator
        tensor_bound = roof["bound"] == "tensor"
        sp = pk.get("bf16_tflops_sustained") if tensor_bound else pk["hbm_gbs"]
        if tensor_bound:
            ach = flops / (sustained["kernel_ms"] / 1e3) / 1e12
        else:
            ach = io_bytes / (sustained["kernel_ms"] / 1e3) / 1e9
        sustained["roofline"] = {"bound": roof["bound"], "achieved": round(ach, 2), "unit": roof["unit"],
                                 "peak": sp, "frac": round(ach / sp, 4) if sp else None,
                                 "peak_kind": ("measured bf16 sustained (power-capped GEMM)" if tensor_bound
                                               else "measured HBM copy")}
        sustained["note"] = ("SURVEY 8(d) protocol: R graph-replayed steps per run (>= 200 ms), median of 5 runs; "
                             "the sustained regime the K-step burst number sits above")
        res["sustained"] = sustained
    if phases is not None:
        res["phases"] = phases
    if world > 1 and args.dist_backend == "gloo":
        res["dry_run"] = ("gloo process group: the exchange is staged through host memory and the ranks may share "
                          "one GPU -- a functional run of the multi-rank path, not a scaling measurement")
    if export_info is not None:
        res["export_int8"] = export_info
    return res


# ----------------------------------------------------------------------------- oracle timing
def oracle_sample(config, attn, seconds, rows=None, backward=False, qla_rows=None, stage2=False, layers=0):
    """Time the float64 oracle on whole users (all rows, all heads) of the rank-0 batch until
    ~`seconds` of CPU work; returns (items/s, cores, sample description, equivalent items, s)."""
    import numpy as np

    import oracle
    import synth
    cfg, lens, S, H, d, _ = workload(config, attn)
    off = synth.offsets_from_lengths(lens)
    cores = len(os.sched_getaffinity(0))
    q = synth.make_q(S, H, d, seed=0)
    done_items, done_t, users = 0.0, 0.0, 0
    rsel = None if rows is None else np.arange(rows, dtype=np.int64)
    frac = 1.0 if rows is None else rows / S
    for u in range(len(lens)):
        a, b = int(off[u]), int(off[u + 1])
        rr = np.arange(a, b, dtype=np.int64)
        k, v = synth.make_kv(rr, np.full(b - a, u), H, d, seed=0)
        t0 = time.perf_counter()
        if layers:  # NEXT-3: the multi-layer summarizer over [seeds; history] of one user
            rng = np.random.default_rng(u)
            D = H * d
            xu = (rng.integers(-128, 128, size=(S + b - a, D)) / 64.0).astype(np.float32)
            wl = (rng.integers(-128, 128, size=(layers, 5, D, D)) / (128.0 * np.sqrt(D))).astype(np.float32)
            t0 = time.perf_counter()
            oracle.summarize_layers(xu, [0, S + b - a], wl, S, H, threads=cores)
        elif stage2:  # NEXT-4: target attention of the user's candidates over its int8 tokens
            rng = np.random.default_rng(u)
            n = TARGETS_PER_USER
            cds = rng.integers(-127, 128, size=(1, S, H, d)).astype(np.int8)
            tsc = (rng.integers(1, 64, size=(1, S, H)) / 1024.0).astype(np.float32)
            tzp = (rng.integers(-64, 64, size=(1, S, H)) / 128.0).astype(np.float32)
            cq, ck, cv = [(rng.integers(-128, 128, size=(n, H, d)) / 64.0).astype(np.float32) for _ in range(3)]
            t0 = time.perf_counter()
            oracle.target_attend(cds, tsc, tzp, cq, ck, cv, [0, n], threads=cores)
        elif qla_rows:  # NEXT-3/4: QLA at per-user query rows
            rng = np.random.default_rng(u)
            n = (b - a) if qla_rows == "history" else TARGETS_PER_USER
            qr = (rng.integers(-128, 128, size=(n, H, d)) / 64.0).astype(np.float32)
            ks = vs = None
            if qla_rows == "target":
                ks = (rng.integers(-128, 128, size=(n, H, d)) / 64.0).astype(np.float32)
                vs = (rng.integers(-128, 128, size=(n, H, d)) / 64.0).astype(np.float32)
            oracle.qla_rows(qr, [0, n], k, v, [0, b - a], k_self=ks, v_self=vs, threads=cores)
        elif backward:  # backward (NEXT-2), dout grid values
            g = (np.random.default_rng(u).integers(-128, 128, size=(1, S, H, d)) / 64.0).astype(np.float32)
            if attn == "softmax":
                oracle.softmax_backward(q, k, v, [0, b - a], g, threads=cores)
            else:
                oracle.qla_backward(q, k, v, [0, b - a], g, threads=cores)
        elif attn == "softmax":
            oracle.softmax_summarize(q, k, v, [0, b - a], rows=rsel, threads=cores)
        else:
            oracle.qla_summarize(q, k, v, [0, b - a], threads=cores)
        done_t += time.perf_counter() - t0
        done_items += TARGETS_PER_USER if stage2 else (b - a) * frac
        users += 1
        if done_t >= seconds:
            break
    rdesc = "all S rows" if rows is None else f"{rows} of {S} rows (items counted x {rows}/{S})"
    sample = f"{users} whole user(s) of {config} ({rdesc}, all {H} heads, full histories), float64 C oracle, OpenMP"
    if backward:
        sample += f", {attn} backward (oracle.{attn}_backward)"
    if qla_rows:
        sample += f", QLA {qla_rows} rows (oracle.qla_rows)"
    if layers:
        sample += f", {layers}-layer summarizer (oracle.summarize_layers)"
    if stage2:
        sample = (f"{users} user(s) x {TARGETS_PER_USER} candidates over {S} int8 tokens, all {H} heads, "
                  "float64 C oracle (oracle.target_attend), OpenMP; unit candidates/s")
    return done_items / done_t, cores, sample, done_items, done_t


def run_reference(args, rank, world):
    """Reference arm: the float64 oracle on the host cores (rank 0 only)."""
    if rank != 0:
        return None
    import numpy as np

    import oracle
    import synth
    cfg, lens, S, H, d, wdesc = workload(args.config, args.attn)
    oracle.build()
    cores = len(os.sched_getaffinity(0))
    off = synth.offsets_from_lengths(lens)
    q = synth.make_q(S, H, d, seed=0)
    # per-step sample: user (i mod B), all heads, R query rows; R sized so the run takes ~90 s
    total_steps = args.steps + args.warmup
    u0 = 0
    a, b = int(off[u0]), int(off[u0 + 1])
    k, v = synth.make_kv(np.arange(a, b, dtype=np.int64), np.full(b - a, u0), H, d, seed=0)
    t0 = time.perf_counter()
    if args.attn == "softmax":
        oracle.softmax_summarize(q, k, v, [0, b - a], rows=np.arange(1), threads=cores)
    else:
        oracle.qla_state(k[: max(1, (b - a) // 16)], v[: max(1, (b - a) // 16)], [0, max(1, (b - a) // 16)],
                         threads=cores)
    t_unit = max(time.perf_counter() - t0, 1e-4)
    budget = 90.0 / max(total_steps, 1)
    R = int(max(1, min(S, budget / t_unit)))
    cache = {}

    def kv_of(u):
        if u not in cache:
            a, b = int(off[u]), int(off[u + 1])
            cache.clear()
            cache[u] = synth.make_kv(np.arange(a, b, dtype=np.int64), np.full(b - a, u), H, d, seed=0)
        return cache[u]

    items, tt = 0.0, 0.0
    for i in range(total_steps):
        u = i % len(lens)
        k, v = kv_of(u)
        L = k.shape[0]
        t0 = time.perf_counter()
        if args.attn == "softmax":
            oracle.softmax_summarize(q, k, v, [0, L], rows=np.arange(R), threads=cores)
            eq = L * R / S
        else:
            n = max(1, min(L, int(L * R / S)))
            oracle.qla_state(k[:n], v[:n], [0, n], threads=cores)
            eq = n
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            items += eq
            tt += dt
    value = items / tt
    sample = (f"per step: 1 user of {args.config} (cycling), all {H} heads, "
              + (f"{R} of {S} query rows over the full history (items counted x {R}/{S})" if args.attn == "softmax"
                 else f"QLA state over the first {R}/{S} of the history"))
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "items/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tt / max(args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (same generator and seed as the own arm)",
        "config": {"workload": wdesc, "S": S, "d": d, "H": H, "attn": args.attn},
        "cpu_baseline": {"value": value, "unit": "items/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "items/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
    if args.layers:
        args.attn = "qla"  # the summarizer layers are QLA layers
        if args.backward or args.export_int8 or args.qla_rows or args.stage2:
            raise SystemExit("--layers excludes --backward / --export-int8 / --qla-rows / --stage2")
    if args.stage2:
        args.attn = "softmax"  # stage 2 reads the softmax summary's int8 export
        if args.backward or args.export_int8 or args.qla_rows:
            raise SystemExit("--stage2 excludes --backward / --export-int8 / --qla-rows")
    if args.qla_rows:
        args.attn = "qla"  # the rows path is QLA's
        if args.backward or args.export_int8:
            raise SystemExit("--qla-rows excludes --backward / --export-int8")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # --gpus N without a launcher: start N ranks (one process per GPU) under torch.distributed.run
        if args.dist_backend == "nccl" and args.impl == "own":
            import torch
            have = torch.cuda.device_count()
            if have < args.gpus:
                raise SystemExit(f"--gpus {args.gpus}: only {have} CUDA device(s) visible; NCCL needs one GPU per "
                                 f"rank (use --dist-backend gloo for a functional dry run)")
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus and args.impl == "own":
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        res = run_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    if world > 1:
        import torch
        if args.dist_backend == "gloo":  # dry run: ranks may share the visible GPU(s)
            torch.cuda.set_device(local_rank % max(torch.cuda.device_count(), 1))
            torch.distributed.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res = run_own(args, rank, world, local_rank)
    if res is not None and world == 1 and not args.no_cpu_baseline:
        v, cores, sample, _, t = oracle_sample(args.config, args.attn, args.cpu_seconds, rows=None,
                                               backward=args.backward, qla_rows=args.qla_rows, stage2=args.stage2,
                                               layers=args.layers)
        res["cpu_baseline"] = {"value": v, "unit": "candidates/s" if args.stage2 else "items/s", "cores": cores,
                               "kind": "oracle",
                               "sample": sample, "seconds": round(t, 2)}
    elif res is not None:
        res["cpu_baseline"] = None
    if res is not None:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
