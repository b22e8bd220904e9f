"""The multi-GPU sharding layer (paper_2510_22049_b200/dist.py) with the CUDA backend: two ranks
(gloo process group, collectives staged through host memory) each computing their shard through
the C ABI on the one visible GPU, against the float64 oracle of the unsplit batch.  The kernels of
the two ranks never wait on each other (the exchange is a host-side gloo all_gather), so this
exercises partition -> vista_summarize_partial -> exchange -> vista_summarize_merge exactly as
the NCCL run does, without standing in for a second GPU's timing."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

pytestmark = pytest.mark.gpu


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, attn, lens, S, H, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_22049_b200 as vista
        from paper_2510_22049_b200 import dist as vdist
        vista.load()
        dev = torch.device("cuda", 0)
        d = 128
        lens = np.asarray(lens, dtype=np.int64)
        off = synth.offsets_from_lengths(lens)
        q = synth.make_q(S, H, d, seed=3, tau=2, backend="torch", device=dev)
        if mode == "by_length":
            cuts = vdist.partition_by_length(lens, world)
            segs = [(u, int(cuts[rank, u]), int(cuts[rank + 1, u])) for u in range(len(lens))]
        else:
            all_segs = vdist.partition_flat(lens, world)
            segs = [(s.user, s.start, s.end) for s in all_segs[rank]]
        rows = np.concatenate([np.arange(off[u] + a, off[u] + e) for u, a, e in segs] or [np.zeros(0, np.int64)])
        users = synth.row_users(off, rows)
        k, v = synth.make_kv(torch.as_tensor(rows, device=dev), torch.as_tensor(users, device=dev), H, d, seed=3,
                             backend="torch", device=dev)
        soff = torch.as_tensor(synth.offsets_from_lengths(np.array([e - a for _, a, e in segs], np.int64)), device=dev)
        if mode == "by_length":
            out, lse = vdist.summarize_by_length(q, k, v, soff, torch.as_tensor(lens, device=dev), attn=attn,
                                                 total_len=int(rows.size))
            res = {u: (out[u].float().cpu().numpy(), None if lse is None else lse[u].cpu().numpy())
                   for u in range(len(lens))}
        else:
            plan = vdist.FlatPlan(all_segs, lens, rank, dev)
            got = vdist.summarize_flat(q, k, v, all_segs[rank], all_segs, lens, attn=attn, plan=plan)
            res = {u: (o.float().cpu().numpy(), None if l is None else l.cpu().numpy()) for u, (o, l) in got.items()}
        torch.cuda.synchronize()
        result_q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _run(world, mode, attn, lens, S, H):
    ctx = mp.get_context("spawn")
    rq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, attn, lens, S, H, rq)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(rq.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("mode", ["by_length", "flat"])
@pytest.mark.parametrize("attn", ["softmax", "qla"])
def test_dist_cuda_backend_world2(mode, attn):
    lens = [5000, 0, 129, 20_000, 1, 3000]
    S, H = 256, 2
    res = _run(2, mode, attn, lens, S, H)
    q, k, v, off = synth.make_batch(lens, S, H, 128, seed=3, tau=2)
    if attn == "softmax":
        ref, ref_lse = oracle.softmax_summarize(q, k, v, off)
    else:
        ref, ref_lse = oracle.qla_summarize(q, k, v, off), None
    if mode == "by_length":
        owned = res[0]
        for u in range(len(lens)):  # every rank holds every user, bitwise identical
            assert np.array_equal(res[0][u][0], res[1][u][0])
    else:
        owned = {}
        for r in range(2):
            for u, val in res[r].items():
                assert u not in owned
                owned[u] = val
        assert sorted(owned) == [u for u in range(len(lens)) if lens[u] > 0]
    for u, (o, l) in owned.items():
        for h in range(H):
            den = max(np.abs(ref[u, :, h]).max(), 1e-30)
            if lens[u] == 0 and attn == "softmax":
                assert np.all(o[:, h] == 0) and np.all(l[h] == -np.inf)
                continue
            assert np.abs(o[:, h] - ref[u, :, h]).max() / den <= 2e-2, (mode, attn, u, h)
            if attn == "softmax":
                assert np.abs(l[h] - ref_lse[u, h]).max() <= 1e-3
