"""Multi-process (world_size 2 and 3, gloo, CPU) tests of the sharding layer
(paper_2510_22049_b200/dist.py): partitioners, the all_gather exchange and the merge order, with
the per-shard compute injected as the float64 oracle (tests only).  The same code runs with the
CUDA backend and NCCL on GPUs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2510_22049_b200 import dist as vdist


class OracleBackend:
    """CPU float64 stand-in for CudaBackend with the same tensor contract."""

    def partial(self, q, k, v, offsets, total_len, attn):
        qn, kn, vn = q.numpy(), k.numpy(), v.numpy()
        off = offsets.numpy()
        if attn == 0:
            out, lse = oracle.softmax_summarize(qn, kn, vn, off, q_per_user=q.dim() == 4)
            return torch.from_numpy(out.transpose(0, 2, 1, 3).copy()), torch.from_numpy(lse)
        return torch.from_numpy(oracle.qla_state(kn, vn, off)), None

    def merge(self, part_o, part_lse, q, attn, user_len):
        po = part_o.numpy()
        if attn == 0:
            out, lse = oracle.merge_lse(po, part_lse.numpy())    # [B,H,S,d], [B,H,S]
            return torch.from_numpy(out.transpose(0, 2, 1, 3).copy()), torch.from_numpy(lse)
        z = oracle.merge_sum(po)
        return torch.from_numpy(oracle.qla_finalize(q.numpy(), z, user_len.numpy(), q_per_user=q.dim() == 4)), None


    def bwd(self, q, k, v, offsets, total_len, dout, attn, **kw):
        qn, kn, vn, gn, off = q.numpy(), k.numpy(), v.numpy(), dout.numpy(), offsets.numpy()
        if attn == 0:
            g = oracle.softmax_backward(qn, kn, vn, off, gn)
        else:
            g = oracle.qla_backward(qn, kn, vn, off, gn)
        return tuple(torch.from_numpy(np.ascontiguousarray(x)) for x in g)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _per_user_q(B, S, H, d):
    return (np.random.default_rng(77).integers(-128, 128, size=(B, S, H, d)) / 64.0).astype(np.float32)


def _worker(rank, world, port, mode, attn, lens, result_q, per_user=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        S, H, d = 6, 2, 8
        lens = np.asarray(lens, dtype=np.int64)
        off = synth.offsets_from_lengths(lens)
        q = torch.from_numpy(synth.make_q(S, H, d, seed=3, tau=2)).double()
        if per_user:
            q = torch.from_numpy(_per_user_q(len(lens), S, H, d)).double()
        be = OracleBackend()
        if mode == "by_length":
            cuts = vdist.partition_by_length(lens, world)
            rows = np.concatenate([np.arange(off[u] + cuts[rank, u], off[u] + cuts[rank + 1, u]) for u in range(len(lens))])
            users = synth.row_users(off, rows)
            k, v = synth.make_kv(rows.astype(np.int64), users, H, d, seed=3)
            soff = synth.offsets_from_lengths(cuts[rank + 1] - cuts[rank])
            out, lse = vdist.summarize_by_length(q, torch.from_numpy(k).double(), torch.from_numpy(v).double(),
                                                 torch.from_numpy(soff), torch.from_numpy(lens), attn=attn,
                                                 backend=be)
            res = {u: (out[u].numpy(), None if lse is None else lse[u].numpy()) for u in range(len(lens))}
        else:
            segs = vdist.partition_flat(lens, world)
            mine = segs[rank]
            rows = np.concatenate([np.arange(off[s.user] + s.start, off[s.user] + s.end) for s in mine]) \
                if mine else np.zeros(0, np.int64)
            users = synth.row_users(off, rows)
            k, v = synth.make_kv(rows.astype(np.int64), users, H, d, seed=3)
            got = vdist.summarize_flat(q, torch.from_numpy(k).double(), torch.from_numpy(v).double(), mine, segs,
                                       lens, attn=attn, backend=be)
            res = {u: (o.numpy(), None if l is None else l.numpy()) for u, (o, l) in got.items()}
        result_q.put((rank, res))
    finally:
        dist.destroy_process_group()


def run_world(world, mode, attn, lens, per_user=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, attn, lens, q, per_user)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return dict(out)


def reference(lens, attn):
    S, H, d = 6, 2, 8
    q, k, v, off = synth.make_batch(lens, S, H, d, seed=3, tau=2)
    if attn == "softmax":
        return oracle.softmax_summarize(q, k, v, off)
    return oracle.qla_summarize(q, k, v, off), None


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("attn", ["softmax", "qla"])
def test_by_length_matches_unsplit(world, attn):
    lens = [50, 0, 7, 129, 1]
    res = run_world(world, "by_length", attn, lens)
    ref, ref_lse = reference(lens, attn)
    for r in range(world):  # every rank holds the merged result of every user
        for u in range(len(lens)):
            o, l = res[r][u]
            np.testing.assert_allclose(o, ref[u], rtol=1e-11, atol=1e-12)
            if attn == "softmax":
                np.testing.assert_allclose(l, ref_lse[u], rtol=1e-12)
    for u in range(len(lens)):  # identical on every rank (fixed merge order)
        assert all(np.array_equal(res[0][u][0], res[r][u][0]) for r in range(world))


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("attn", ["softmax", "qla"])
def test_flat_matches_unsplit(world, attn):
    lens = [40, 3, 0, 90, 17, 5, 61]
    res = run_world(world, "flat", attn, lens)
    ref, ref_lse = reference(lens, attn)
    owned = {}
    for r in range(world):
        for u, v in res[r].items():
            assert u not in owned, "a user is owned by exactly one rank"
            owned[u] = v
    assert sorted(owned) == [u for u in range(len(lens)) if lens[u] > 0]
    for u, (o, l) in owned.items():
        np.testing.assert_allclose(o, ref[u], rtol=1e-11, atol=1e-12)
        if attn == "softmax":
            np.testing.assert_allclose(l, ref_lse[u], rtol=1e-12)


@pytest.mark.parametrize("attn", ["softmax", "qla"])
def test_flat_per_user_seeds(attn):
    """Flat sharding with per-user seeds q [B,S,H,d]: every segment (and every straddling user's
    merge) uses its own user's seeds; 3 ranks so a user can straddle two boundaries."""
    lens = [40, 3, 0, 90, 17, 5, 61]
    res = run_world(3, "flat", attn, lens, per_user=True)
    S, H, d = 6, 2, 8
    _, k, v, off = synth.make_batch(lens, S, H, d, seed=3, tau=2)
    q = _per_user_q(len(lens), S, H, d)
    if attn == "softmax":
        ref, ref_lse = oracle.softmax_summarize(q, k, v, off, q_per_user=True)
    else:
        ref, ref_lse = oracle.qla_summarize(q, k, v, off, q_per_user=True), None
    owned = {u: v_ for r in range(3) for u, v_ in res[r].items()}
    assert sorted(owned) == [u for u in range(len(lens)) if lens[u] > 0]
    for u, (o, l) in owned.items():
        np.testing.assert_allclose(o, ref[u], rtol=1e-11, atol=1e-12)
        if attn == "softmax":
            np.testing.assert_allclose(l, ref_lse[u], rtol=1e-12)


def test_partitioners():
    lens = np.array([5, 100, 0, 30, 30, 70])
    parts = vdist.partition_by_user(lens, 3)
    assert sorted(u for p in parts for u in p) == list(range(6))
    loads = [int(lens[p].sum()) for p in parts]
    assert max(loads) - min(loads) <= 100 and loads[0] == 100  # LPT: the 100-item user alone on rank 0
    cuts = vdist.partition_by_length(lens, 4)
    assert np.array_equal(cuts[0], np.zeros(6)) and np.array_equal(cuts[-1], lens)
    assert np.all(np.diff(cuts, axis=0) >= 0) and np.all(np.diff(cuts, axis=0).max(0) - np.diff(cuts, axis=0).min(0) <= 1)
    segs = vdist.partition_flat(lens, 4)
    covered = {}
    for rank in segs:
        for s in rank:
            covered.setdefault(s.user, []).append((s.start, s.end))
    for u, ranges in covered.items():
        ranges.sort()
        assert ranges[0][0] == 0 and ranges[-1][1] == lens[u]
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    sizes = [sum(s.end - s.start for s in r) for r in segs]
    assert max(sizes) - min(sizes) <= 1


def _bwd_worker(rank, world, port, attn, lens, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        S, H, d = 6, 2, 8
        q, k, v, off = synth.make_batch(lens, S, H, d, seed=5, tau=1)
        mine = vdist.partition_by_user(lens, world)[rank]
        rng = np.random.default_rng(9)
        g = (rng.integers(-128, 128, size=(len(lens), S, H, d)) / 64.0).astype(np.float32)
        kk = np.concatenate([k[off[u]:off[u + 1]] for u in mine]) if mine else np.zeros((0, H, d), np.float32)
        vv = np.concatenate([v[off[u]:off[u + 1]] for u in mine]) if mine else np.zeros((0, H, d), np.float32)
        soff = synth.offsets_from_lengths(np.asarray([lens[u] for u in mine], dtype=np.int64))
        dq, dk, dv = vdist.summarize_bwd_by_user(torch.from_numpy(q), torch.from_numpy(kk), torch.from_numpy(vv),
                                                 torch.from_numpy(soff), int(soff[-1]), torch.from_numpy(g[mine]),
                                                 attn=attn, backend=OracleBackend())
        result_q.put((rank, (dq.numpy(), mine, dk.numpy(), soff)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("attn", ["softmax", "qla"])
def test_backward_by_user_all_reduces_seed_gradient(attn):
    """Data-parallel backward over 2 ranks (gloo): the seed gradient after the all_reduce equals the
    unsplit one on every rank; each rank's dK covers exactly its own users."""
    lens = [30, 0, 12, 45, 7]
    ctx = mp.get_context("spawn")
    rq = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_bwd_worker, args=(r, 2, port, attn, lens, rq)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(rq.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    S, H, d = 6, 2, 8
    q, k, v, off = synth.make_batch(lens, S, H, d, seed=5, tau=1)
    g = (np.random.default_rng(9).integers(-128, 128, size=(len(lens), S, H, d)) / 64.0).astype(np.float32)
    ref = (oracle.softmax_backward if attn == "softmax" else oracle.qla_backward)(q, k, v, off, g)
    for r in range(2):
        dq, mine, dk, soff = res[r]
        np.testing.assert_allclose(dq, ref[0], rtol=0, atol=1e-12 * max(1.0, np.abs(ref[0]).max()))
        for n, u in enumerate(mine):
            np.testing.assert_allclose(dk[soff[n]:soff[n + 1]], ref[1][off[u]:off[u + 1]], rtol=0, atol=1e-12)


def _peer_worker(rank, world, port, result_q):
    """Host logic of dist.PeerExchange at world size 2: the CUDA IPC calls are replaced by a fake
    handle / pointer scheme (CPU tensors), so the handle all_gather, the per-rank pointer tables and
    the rank ordering are checked without GPUs."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2510_22049_b200 as vista
        vista.vista_ipc_get_handle = lambda t: (b"R%d:%d" % (rank, t.data_ptr() % 1000003)).ljust(64, b"\0")
        opened = []

        def fake_open(h):
            opened.append(bytes(h).rstrip(b"\0"))
            return 10**12 + len(opened)
        vista.vista_ipc_open_handle = fake_open
        ex = vdist.PeerExchange((3, 2, 4, 8), (3, 2, 4), device="cpu")
        own = [ex.recv_o.data_ptr(), ex.recv_lse.data_ptr(), ex.flags.data_ptr(), ex.acks.data_ptr()]
        result_q.put((rank, (ex.world, ex.rank, ex.o_ptrs, ex.lse_ptrs, ex.flag_ptrs, ex.ack_ptrs, own, opened)))
    finally:
        dist.destroy_process_group()


def test_peer_exchange_host_logic_world2():
    ctx = mp.get_context("spawn")
    rq = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port, rq)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(rq.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        world, rank, o, l, f, a, own, opened = res[r]
        assert (world, rank) == (2, r)
        # own arrays at index rank, the peer's (opened from its 4 handles, in order) at the other index
        assert [o[r], l[r], f[r], a[r]] == own
        peer = 1 - r
        assert [o[peer], l[peer], f[peer], a[peer]] == [10**12 + i for i in range(1, 5)]
        assert all(h.startswith(b"R%d:" % peer) for h in opened) and len(opened) == 4


def test_by_length_fused_exchange_call_order():
    """summarize_by_length with a peer exchange and fused=True (softmax): the backend's partial_peers
    stores the partial (no separate partial / push), then signal_wait hands the receive buffers to the
    merge, then release -- in that order (softmax and QLA); fused=False takes the push path."""
    calls = []

    class Ex:
        recv = (torch.ones(1, 2), torch.zeros(1, 2))

        def signal_wait(self, stream=None):
            calls.append("signal_wait")
            return self.recv

        def gather(self, po, pl=None, stream=None):
            calls.append("gather")
            return self.recv

        def release(self, stream=None):
            calls.append("release")

    class Be:
        def partial_peers(self, q, k, v, off, total, ex, attn=0):
            calls.append("partial_peers")

        def partial(self, q, k, v, off, total, attn):
            calls.append("partial")
            return torch.ones(2), (torch.zeros(2) if attn == 0 else None)

        def merge(self, go, gl, q, attn, ulen):
            calls.append("merge")
            return go, gl

    ex, be = Ex(), Be()
    out = vdist.summarize_by_length(None, None, None, None, None, attn="softmax", backend=be, total_len=0,
                                    exchange=ex)
    assert calls == ["partial_peers", "signal_wait", "merge", "release"] and out[0] is Ex.recv[0]
    calls.clear()
    vdist.summarize_by_length(None, None, None, None, None, attn="softmax", backend=be, total_len=0, exchange=ex,
                              fused=False)
    assert calls == ["partial", "gather", "merge", "release"]
    calls.clear()
    vdist.summarize_by_length(None, None, None, None, None, attn="qla", backend=be, total_len=0, exchange=ex)
    assert calls == ["partial_peers", "signal_wait", "merge", "release"]
