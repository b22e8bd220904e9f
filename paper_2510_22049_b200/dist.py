"""Multi-GPU sharding of VISTA stage-1 summarization (one process per GPU, torch.distributed).

SURVEY.md §8(e).  Users are independent, and within a user the history splits with one exchange
of O(B*H*S*d) partials whatever L is (the flash-decoding identity for softmax; the sum of states
for QLA, "sum_j K[S]_j^T V[S]_j").  Three partitioners over the jagged histories:

  by_user    whole users to ranks, longest-processing-time greedy on L_u (C3).  No collective on the
             data path: every rank summarizes its own users.
  by_length  each user's [0, L_u) cut into `world` equal contiguous ranges; rank g gets range g of
             every user (C4, 1M-item histories).  Each rank computes partials with
             vista_summarize_partial, one all_gather (NCCL over NVLink) exchanges them, and every
             rank merges them in rank order with vista_summarize_merge (bitwise identical results on
             all ranks; deterministic for a fixed world size).
  flat       the concatenated item stream cut into `world` equal ranges (C5 power-law mix): at most
             world - 1 users straddle ranks; only their boundary partials are exchanged.

The per-shard compute is a `backend` object (default: CudaBackend, the C-ABI library); tests inject
a CPU backend so the partition / exchange / merge logic runs under gloo without a GPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["partition_by_user", "partition_by_length", "partition_flat", "CudaBackend",
           "summarize_by_length", "summarize_flat", "summarize_bwd_by_user", "FlatPlan", "Segment",
           "PeerExchange"]


# ----------------------------------------------------------------------------- partitioners (host)
def partition_by_user(lengths, world: int) -> list[list[int]]:
    """LPT greedy: users by decreasing L_u (ties: lower index first) onto the least-loaded rank
    (ties: lower rank).  Returns each rank's users in increasing user order."""
    lengths = np.asarray(lengths, dtype=np.int64)
    order = sorted(range(len(lengths)), key=lambda u: (-int(lengths[u]), u))
    load = [0] * world
    out: list[list[int]] = [[] for _ in range(world)]
    for u in order:
        r = min(range(world), key=lambda g: (load[g], g))
        out[r].append(u)
        load[r] += int(lengths[u])
    return [sorted(x) for x in out]


def partition_by_length(lengths, world: int) -> np.ndarray:
    """Cut points: returns int64 [world + 1, B]; rank g owns items [cuts[g, u], cuts[g + 1, u]) of
    user u (equal contiguous ranges, the first ranges one item shorter when L_u % world != 0)."""
    lengths = np.asarray(lengths, dtype=np.int64)
    g = np.arange(world + 1, dtype=np.int64)[:, None]
    return (lengths[None, :] * g) // world


@dataclass(frozen=True)
class Segment:
    user: int
    start: int  # item offset within the user's history
    end: int


def partition_flat(lengths, world: int) -> list[list[Segment]]:
    """Cut the concatenated item stream [0, sum L) into `world` equal ranges; each rank gets the
    user segments overlapping its range (in user order).  Empty users belong to no segment."""
    lengths = np.asarray(lengths, dtype=np.int64)
    off = np.zeros(len(lengths) + 1, dtype=np.int64)
    np.cumsum(lengths, out=off[1:])
    total = int(off[-1])
    out: list[list[Segment]] = []
    for g in range(world):
        a, b = total * g // world, total * (g + 1) // world
        segs = []
        u = int(np.searchsorted(off, a, side="right") - 1) if a < total else len(lengths)
        while u < len(lengths) and off[u] < b:
            s, e = max(a, int(off[u])), min(b, int(off[u + 1]))
            if e > s:
                segs.append(Segment(u, s - int(off[u]), e - int(off[u])))
            u += 1
        out.append(segs)
    return out


# ----------------------------------------------------------------------------- compute backends
class CudaBackend:
    """Per-shard compute through the C ABI (paper_2510_22049_b200)."""

    def __init__(self, **kw):
        import paper_2510_22049_b200 as vista
        self.v = vista
        self.kw = kw

    def partial(self, q, k, v, offsets, total_len, attn):
        return self.v.summarize_partial(q, k, v, offsets, total_len, attn=attn, **self.kw)

    def partial_peers(self, q, k, v, offsets, total_len, exchange, attn=0):
        """Partial whose kernels store straight into every rank's receive buffer (softmax or QLA)."""
        self.v.summarize_partial_peers(q, k, v, offsets, total_len, exchange, attn=attn, **self.kw)

    def merge(self, part_o, part_lse, q, attn, user_len):
        return self.v.summarize_merge(part_o, part_lse, q=q, attn=attn, user_len=user_len, **self.kw)

    def bwd(self, q, k, v, offsets, total_len, dout, attn, **kw):
        return self.v.summarize_bwd(q, k, v, offsets, total_len, dout, attn=attn, **self.kw, **kw)


def summarize_bwd_by_user(q, k, v, offsets, total_len, dout, *, attn="softmax", group=None, backend=None, **kw):
    """Data-parallel backward (NEXT-2) of a by_user shard: the local gradients from the backend, then
    the one exchange the path has -- the shared seeds' gradient dq [S,H,d] summed over the ranks
    (all_reduce; per-user seeds have no exchange).  dk, dv stay local (the rank's own items).
    kw: forwarded to the backend's bwd (out / lse for softmax, z for QLA)."""
    import torch.distributed as dist
    be = backend or CudaBackend()
    dq, dk, dv = be.bwd(q, k, v, offsets, total_len, dout, _attn_code(attn), **kw)
    if q.dim() == 3 and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(dq, group=group)
    return dq, dk, dv


def _attn_code(attn):
    return 0 if attn in (0, "softmax") else 1


# ----------------------------------------------------------------------------- split-L paths
def _all_gather(t, group):
    """[*shape] on every rank -> [world, *shape] in rank order (one all_gather_into_tensor).

    NCCL gathers device tensors directly (NVLink / NVSwitch).  Under gloo (CPU tests, or a
    single-GPU dry run of several ranks) a device tensor is staged through host memory."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = t.contiguous()
    staged = t.is_cuda and dist.get_backend(group) == "gloo"
    src = t.cpu() if staged else t
    out = torch.empty((world * src.shape[0],) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    dist.all_gather_into_tensor(out, src, group=group)
    out = out.view((world,) + tuple(src.shape))
    return out.to(t.device, non_blocking=True) if staged else out


class PeerExchange:
    """The split-L exchange over peer memory (SURVEY.md 8(e) phase 2; vista_exchange_* in
    include/vista.h): every rank of the node owns a receive buffer for all ranks' partials, shared
    through CUDA IPC, and the partial of a rank is stored straight into every rank's buffer (NVLink /
    NVSwitch peer stores), then published with a system-scope flag; the merge reads the local buffer.
    No NCCL call and no host synchronization on the step (the epoch is a device counter, so the step
    can be captured in a CUDA graph).  Built once per (shape, group); world <= 8.

    part_shape: the partial's shape (softmax O_p [B,H,S,d]; QLA Z_p [B,H,d,d]); lse_shape: the
    softmax lse_p shape [B,H,S] or None (QLA)."""

    def __init__(self, part_shape, lse_shape=None, group=None, device=None):
        import torch
        import torch.distributed as dist
        from . import vista_ipc_get_handle, vista_ipc_open_handle
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if self.world > 8:
            raise ValueError("PeerExchange: at most 8 ranks (one node)")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.part_shape, self.lse_shape = tuple(part_shape), (tuple(lse_shape) if lse_shape else None)
        self.recv_o = torch.zeros((self.world,) + self.part_shape, dtype=torch.float32, device=dev)
        self.recv_lse = (torch.zeros((self.world,) + self.lse_shape, dtype=torch.float32, device=dev)
                         if self.lse_shape else None)
        self.flags = torch.zeros(self.world, dtype=torch.int32, device=dev)
        self.acks = torch.zeros(self.world, dtype=torch.int32, device=dev)
        self.epoch = torch.zeros(1, dtype=torch.int32, device=dev)
        if dev.type == "cuda":
            torch.cuda.synchronize(dev)  # the zeroed arrays exist before any peer writes into them
        mine = [self.recv_o] + ([self.recv_lse] if self.recv_lse is not None else []) + [self.flags, self.acks]
        handles = [vista_ipc_get_handle(t) for t in mine] if self.world > 1 else None
        if self.world > 1:
            allh = [None] * self.world
            dist.all_gather_object(allh, handles, group=group)
        self._opened = []
        cols = []
        for r in range(self.world):
            if r == self.rank:
                cols.append([t.data_ptr() for t in mine])
            else:
                ptrs = [vista_ipc_open_handle(h) for h in allh[r]]
                self._opened += ptrs
                cols.append(ptrs)
        k = 0
        self.o_ptrs = [c[k] for c in cols]
        k += 1
        self.lse_ptrs = [c[k] for c in cols] if self.recv_lse is not None else None
        k += 1 if self.recv_lse is not None else 0
        self.flag_ptrs = [c[k] for c in cols]
        self.ack_ptrs = [c[k + 1] for c in cols]
        if self.world > 1:
            dist.barrier(group=group)  # every rank mapped every buffer before the first push

    def gather(self, part_o, part_lse=None, stream=None):
        """push + signal + wait: returns the local receive buffers [world, ...] holding every rank's
        partial (stream-ordered after this call)."""
        from . import vista_exchange_push, vista_exchange_signal, vista_exchange_wait
        n_o = part_o.numel()
        n_l = part_lse.numel() if (part_lse is not None and self.recv_lse is not None) else 0
        vista_exchange_push(self.world, self.rank, part_o, n_o, part_lse if n_l else None, n_l, self.o_ptrs,
                            self.lse_ptrs if n_l else None, self.acks, self.epoch, stream)
        vista_exchange_signal(self.world, self.rank, self.flag_ptrs, self.epoch, stream)
        vista_exchange_wait(self.world, self.flags, self.epoch, stream)
        return self.recv_o, self.recv_lse

    def signal_wait(self, stream=None):
        """signal + wait after a fused partial (vista_summarize_partial_peers already stored this rank's
        rows into every receive buffer): returns the local receive buffers [world, ...]."""
        from . import vista_exchange_signal, vista_exchange_wait
        vista_exchange_signal(self.world, self.rank, self.flag_ptrs, self.epoch, stream)
        vista_exchange_wait(self.world, self.flags, self.epoch, stream)
        return self.recv_o, self.recv_lse

    def release(self, stream=None):
        """ack: this rank has consumed the current epoch (after the merge read the receive buffer)."""
        from . import vista_exchange_ack
        vista_exchange_ack(self.world, self.rank, self.ack_ptrs, self.epoch, stream)

    def close(self):
        from . import vista_ipc_close
        for p in self._opened:
            vista_ipc_close(p)
        self._opened = []


def summarize_by_length(q, k_shard, v_shard, shard_offsets, user_len, *, attn="softmax", group=None,
                        backend=None, total_len=None, exchange=None, fused=True):
    """Rank-local shard (this rank's range of every user) -> merged summary of every user on every
    rank.  shard_offsets: int64 [B+1] (device), user_len: int64 [B] total L_u (device, QLA 1/N).
    One all_gather of the partials (softmax: O_p [B,H,S,d] + lse_p [B,H,S]; QLA: Z_p [B,H,d,d]):
    NCCL (or gloo), or, with exchange = a PeerExchange, peer-memory stores over NVLink -- made by the
    partial's own kernels (fused=True), else by a push kernel after it.
    No host synchronization: the step is capturable in a CUDA graph."""
    backend = backend or CudaBackend()
    a = _attn_code(attn)
    if total_len is None:
        total_len = k_shard.shape[0]
    if exchange is not None and fused and hasattr(backend, "partial_peers"):
        # the exchange fused into the partial's stores (SURVEY 8(e) phase 2): no push, no collective
        backend.partial_peers(q, k_shard, v_shard, shard_offsets, total_len, exchange, a)
        go, gl = exchange.signal_wait()
        res = backend.merge(go, gl if a == 0 else None, q, a, user_len)
        exchange.release()
        return res
    po, pl = backend.partial(q, k_shard, v_shard, shard_offsets, total_len, a)
    if exchange is not None:
        go, gl = exchange.gather(po, pl if a == 0 else None)
        res = backend.merge(go, gl if a == 0 else None, q, a, user_len)
        exchange.release()
        return res
    go = _all_gather(po, group)
    gl = _all_gather(pl, group) if a == 0 else None
    return backend.merge(go, gl, q, a, user_len)


class FlatPlan:
    """Host-side plan of the flat (item-stream) exchange for one rank, built once per partition.

    Every rank knows the whole partition, so it knows -- without communicating -- which boundary
    slot of which rank carries which straddling user: rank g sends its first segment in slot 0 and
    its last in slot 1 when they are incomplete.  The plan holds the device index tensors that
    (1) gather the rank's complete segments for one merge call and (2) gather each owned
    straddling user's parts from the all_gathered slots, padded to the largest part count with a
    null slot (lse = -inf / Z = 0, the identity of either merge), for a second merge call.  No
    step ever reads a device value on the host."""

    def __init__(self, all_segments: list[list[Segment]], lengths, rank: int, device, q_per_user: bool = False):
        import torch
        lengths = np.asarray(lengths, dtype=np.int64)
        world = len(all_segments)
        self.world, self.rank = world, rank
        self.segments = segs = all_segments[rank]
        seg_len = np.array([s.end - s.start for s in segs], dtype=np.int64)
        off = np.zeros(len(segs) + 1, dtype=np.int64)
        np.cumsum(seg_len, out=off[1:])
        self.total_len = int(off[-1])
        self.offsets = torch.as_tensor(off, device=device)
        self.seg_users = torch.as_tensor([s.user for s in segs], dtype=torch.int64, device=device)
        self.q_per_user = q_per_user

        def complete(s):
            return s.start == 0 and s.end == int(lengths[s.user])

        def slots_of(g):  # [(slot, local segment index)] rank g sends
            sg = all_segments[g]
            ends = [0] if len(sg) == 1 else ([0, len(sg) - 1] if sg else [])
            return [(sl, j) for sl, j in enumerate(ends) if not complete(sg[j])]

        self.send = slots_of(rank)
        owner = {}
        for g in range(world):
            for s in all_segments[g]:
                owner.setdefault(s.user, g)
        comp = [j for j, s in enumerate(segs) if complete(s)]
        self.comp_users = [segs[j].user for j in comp]
        self.comp_idx = torch.as_tensor(comp, dtype=torch.int64, device=device)
        self.comp_len = torch.as_tensor([int(lengths[u]) for u in self.comp_users], dtype=torch.int64, device=device)
        parts: dict[int, list[int]] = {}
        for g in range(world):
            for sl, j in slots_of(g):
                u = all_segments[g][j].user
                if owner[u] == rank:
                    parts.setdefault(u, []).append(2 * g + sl)  # ascending rank order
        self.str_users = sorted(parts)
        pmax = max((len(v) for v in parts.values()), default=0)
        null = 2 * world
        gidx = np.full((pmax, len(self.str_users)), null, dtype=np.int64)
        for n, u in enumerate(self.str_users):
            gidx[:len(parts[u]), n] = parts[u]
        self.str_gidx = torch.as_tensor(gidx, device=device)
        self.str_users_t = torch.as_tensor(self.str_users, dtype=torch.int64, device=device)
        self.str_len = torch.as_tensor([int(lengths[u]) for u in self.str_users], dtype=torch.int64, device=device)


def summarize_flat(q, k_local, v_local, segments: list[Segment], all_segments: list[list[Segment]], lengths, *,
                   attn="softmax", group=None, backend=None, plan: FlatPlan | None = None):
    """Flat (item-stream) sharding.  k_local / v_local hold this rank's segments back to back.
    Returns {user: (out [S,H,d], lse [H,S] or None)} for the users this rank OWNS (a straddling user
    is owned by the lowest rank holding part of it).  Only straddling users' partials are exchanged
    (one all_gather of two fixed-size boundary slots per rank).  q: shared seeds [S,H,d] or
    per-user seeds [B,S,H,d] (each segment then uses its own user's seeds).  Pass a prebuilt
    `plan` (FlatPlan) on the hot path; the step then does no host-side work beyond launches."""
    import torch
    import torch.distributed as dist
    backend = backend or CudaBackend()
    a = _attn_code(attn)
    rank = dist.get_rank(group)
    per_user = q.dim() == 4
    if plan is None:
        plan = FlatPlan(all_segments, lengths, rank, k_local.device, per_user)
    q_seg = q.index_select(0, plan.seg_users.to(q.device)) if per_user else q
    po, pl = backend.partial(q_seg, k_local, v_local, plan.offsets.to(k_local.device), plan.total_len, a)
    dev = po.device
    slot_shape = tuple(po.shape[1:])
    send_o = torch.zeros((2,) + slot_shape, dtype=po.dtype, device=dev)
    send_l = torch.full((2,) + tuple(pl.shape[1:]), float("-inf"), dtype=pl.dtype, device=dev) if a == 0 else None
    for slot, j in plan.send:
        send_o[slot] = po[j]
        if a == 0:
            send_l[slot] = pl[j]
    recv_o = _all_gather(send_o, group).reshape((-1,) + slot_shape)
    recv_l = _all_gather(send_l, group).reshape((-1,) + tuple(pl.shape[1:])) if a == 0 else None
    results = {}
    if plan.comp_users:
        ci = plan.comp_idx.to(dev)
        qc = q_seg.index_select(0, ci) if per_user else q
        out, lse = backend.merge(po.index_select(0, ci)[None], None if a else pl.index_select(0, ci)[None], qc, a,
                                 plan.comp_len.to(dev))
        for n, u in enumerate(plan.comp_users):
            results[u] = (out[n], None if lse is None else lse[n])
    if plan.str_users:
        # null slot (index 2 * world): the identity of the merge (lse -inf / Z = 0)
        flat_o = torch.cat([recv_o, torch.zeros((1,) + slot_shape, dtype=recv_o.dtype, device=dev)])
        gidx = plan.str_gidx.to(dev)
        parts_o = flat_o[gidx]
        parts_l = None
        if a == 0:
            flat_l = torch.cat([recv_l, torch.full((1,) + tuple(recv_l.shape[1:]), float("-inf"), dtype=recv_l.dtype,
                                                   device=dev)])
            parts_l = flat_l[gidx]
        qs = q.index_select(0, plan.str_users_t.to(q.device)) if per_user else q
        out, lse = backend.merge(parts_o, parts_l, qs, a, plan.str_len.to(dev))
        for n, u in enumerate(plan.str_users):
            results[u] = (out[n], None if lse is None else lse[n])
    return results
