"""Seeded synthetic inputs for VISTA stage-1 summarization (shared by oracle tests and the CUDA path).

This module holds NONE of the method's arithmetic: it only draws numbers. Both sides of every
parity check (the float64 oracle in ``oracle/`` and the CUDA library in
``paper_2510_22049_b200``) receive their inputs from here, so neither side ever produces the
other's inputs.

Generator (counter based, so any shard or any row range regenerates identical values):

    h     = splitmix64(block ^ (seed << 32) ^ (tensor_id << 56)),   block = index // 8
    level = byte (index % 8) of h                                   -> uint8 in [0, 256)

Every value is an integer numerator over a power of two, chosen so that it is EXACTLY
representable in bfloat16 (|numerator| <= 256, 8 significant bits) and in float32; the oracle
converts the same bits to float64 without rounding and the GPU reads the same bits.

    bf16 grid: x = (level - 128) / 64                         in [-2, 2), step 1/64
    f32  grid: x = (level16 - 32768) / 16384                  (two bytes per element)

Tensors (SURVEY.md §8(d) "Synthetic inputs", with the bf16-exact grid replacing the
uniform-then-round recipe so that no rounding step exists on either side):
    Q [S, H, d]          tensor 1, times tau (power of two: 1 for the bench, 4 for the peaky set)
    K [sum L, H, d]      tensor 2 (optional "category persistent" structure, SPEC.md:428 idea:
                         K_j += 2 * centroid[c_j], c_j a sticky chain over 64 centroids)
    V [sum L, H, d]      tensor 3, (level >> 1) + mu[u, h, c] with mu = tensor 4 level >> 1,
                         so each (user, head, channel) has its own mean and |O| = O(1).

User lengths (numpy PCG64, seed 0 unless stated), SURVEY.md §8(d):
    C3: L = 10,000 + floor(U * 90,001)
    C5: truncated power law alpha = 2 on [1e3, 1e6]: L = floor(1 / (1e-3 - U (1e-3 - 1e-6)))
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "CONFIGS", "user_lengths", "offsets_from_lengths", "make_q", "make_kv",
    "row_users", "levels",
]

_M64 = (1 << 64) - 1
_GOLD = 0x9E3779B97F4A7C15
_MUL1 = 0xBF58476D1CE4E5B9
_MUL2 = 0x94D049BB133111EB

TID_Q, TID_K, TID_V, TID_VMU, TID_CENT, TID_CHAIN = 1, 2, 3, 4, 5, 6

# Workload configurations of BASELINE.json "configs" (index 0..4 -> c1..c5).
CONFIGS = {
    "c1": dict(B=1, S=16, H=1, d=32, dtype="f32", lengths="fixed", L=1024),
    "c2": dict(B=64, S=256, H=4, d=128, dtype="bf16", lengths="fixed", L=10_000),
    "c3": dict(B=32, S=256, H=1, d=128, dtype="bf16", lengths="uniform", lo=10_000, hi=100_000),
    "c4": dict(B=8, S=256, H=1, d=128, dtype="bf16", lengths="fixed", L=1_000_000),
    "c5": dict(B=1024, S=512, H=1, d=128, dtype="bf16", lengths="powerlaw", lo=1_000, hi=1_000_000),
}


# ----------------------------------------------------------------------------- hashing
def _splitmix64_np(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (x + np.uint64(_GOLD)).astype(np.uint64)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_MUL1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_MUL2)
        return z ^ (z >> np.uint64(31))


def _s64(c: int) -> int:
    """Unsigned 64-bit constant -> the int64 with the same bits (torch has no uint64 math)."""
    return c - (1 << 64) if c >= (1 << 63) else c


def _srl_t(z, s: int):
    """Logical right shift of an int64 torch tensor."""
    return (z >> s) & ((1 << (64 - s)) - 1)


def _splitmix64_torch(x):
    z = x + _s64(_GOLD)
    z = (z ^ _srl_t(z, 30)) * _s64(_MUL1)
    z = (z ^ _srl_t(z, 27)) * _s64(_MUL2)
    return z ^ _srl_t(z, 31)


def _key(seed: int, tid: int) -> int:
    assert 0 <= seed < (1 << 24) and 0 < tid < 256
    return (seed << 32) ^ (tid << 56)


def levels(seed: int, tid: int, index, backend: str = "numpy"):
    """uint8 level in [0,256) for each flat element index (int64 array / tensor)."""
    if backend == "numpy":
        idx = np.asarray(index, dtype=np.int64).astype(np.uint64)
        h = _splitmix64_np((idx >> np.uint64(3)) ^ np.uint64(_key(seed, tid)))
        return ((h >> ((idx & np.uint64(7)) * np.uint64(8))) & np.uint64(255)).astype(np.int32)
    import torch
    idx = index.to(torch.int64)
    h = _splitmix64_torch((idx >> 3) ^ _s64(_key(seed, tid)))
    return (_srl_t_var(h, (idx & 7) * 8) & 255).to(torch.int32)


def _srl_t_var(z, s):
    """Logical right shift by a per-element amount s in [0, 56] (int64 tensors)."""
    import torch
    one = torch.ones((), dtype=torch.int64, device=z.device)
    mask = torch.where(s == 0, torch.full_like(s, -1), (one << (64 - s)) - 1)
    return (z >> s) & mask


def _levels16(seed, tid, index, backend):
    lo = levels(seed, tid, index * 2, backend)
    hi = levels(seed, tid, index * 2 + 1, backend)
    return lo + hi * 256


# ----------------------------------------------------------------------------- lengths
def user_lengths(config: str, seed: int = 0) -> np.ndarray:
    cfg = CONFIGS[config]
    B = cfg["B"]
    if cfg["lengths"] == "fixed":
        return np.full(B, cfg["L"], dtype=np.int64)
    u = np.random.default_rng(seed).random(B)
    if cfg["lengths"] == "uniform":
        return (cfg["lo"] + np.floor(u * (cfg["hi"] - cfg["lo"] + 1))).astype(np.int64)
    a, b = 1.0 / cfg["lo"], 1.0 / cfg["hi"]
    return np.floor(1.0 / (a - u * (a - b))).astype(np.int64)


def offsets_from_lengths(lengths) -> np.ndarray:
    lengths = np.asarray(lengths, dtype=np.int64)
    off = np.zeros(len(lengths) + 1, dtype=np.int64)
    np.cumsum(lengths, out=off[1:])
    return off


def row_users(offsets, rows, backend="numpy"):
    """User index of each global history row, given the user offsets [B+1]."""
    if backend == "numpy":
        return np.searchsorted(np.asarray(offsets), np.asarray(rows), side="right") - 1
    import torch
    return torch.searchsorted(offsets, rows, right=True) - 1


# ----------------------------------------------------------------------------- tensors
def _to_values(n, dtype, backend, device, denom):
    if backend == "numpy":
        return (n.astype(np.float32) / np.float32(denom))
    import torch
    x = n.to(torch.float32) / denom
    return x.to(torch.bfloat16 if dtype == "bf16" else torch.float32)


def make_q(S: int, H: int, d: int, *, seed: int = 0, dtype: str = "bf16", tau: int = 1,
           users: int | None = None, backend: str = "numpy", device=None):
    """Seed (query) tokens Q[S,H,d] shared across users, or Q[users,S,H,d] if ``users`` given."""
    assert tau in (1, 2, 4)
    shape = (S, H, d) if users is None else (users, S, H, d)
    count = int(np.prod(shape))
    if backend == "numpy":
        idx = np.arange(count, dtype=np.int64)
    else:
        import torch
        idx = torch.arange(count, dtype=torch.int64, device=device)
    if dtype == "bf16":
        n = (levels(seed, TID_Q, idx, backend) - 128) * tau
        x = _to_values(n, dtype, backend, device, 64.0)
    else:
        n = (_levels16(seed, TID_Q, idx, backend) - 32768) * tau
        x = _to_values(n, dtype, backend, device, 16384.0)
    return x.reshape(shape)


def make_kv(rows, users, H: int, d: int, *, seed: int = 0, dtype: str = "bf16",
            category: bool = False, backend: str = "numpy", device=None, chain_start=None):
    """K and V rows for the given global history rows (1-D int64) owned by ``users`` (same length).

    Returns (K, V) with shape [len(rows), H, d].  Values depend only on (seed, global row, h, c,
    user), never on how the rows are sharded.  ``chain_start`` (category mode) is, per row, the
    first global row of its user (the chain restarts at every user boundary).
    """
    if backend == "numpy":
        rows = np.asarray(rows, dtype=np.int64)
        users = np.asarray(users, dtype=np.int64)
        hc = np.arange(H * d, dtype=np.int64)
        flat = rows[:, None] * (H * d) + hc[None, :]
        mu_idx = users[:, None] * (H * d) + hc[None, :]
    else:
        import torch
        hc = torch.arange(H * d, dtype=torch.int64, device=device)
        flat = rows[:, None] * (H * d) + hc[None, :]
        mu_idx = users[:, None] * (H * d) + hc[None, :]
    if dtype == "bf16":
        kn = levels(seed, TID_K, flat, backend) - 128
        if category:
            kn = kn + 2 * (_centroid_level(seed, rows, chain_start, H, d, backend, device) - 32)
        vn = (levels(seed, TID_V, flat, backend) >> 1) + (levels(seed, TID_VMU, mu_idx, backend) >> 1) - 128
        K = _to_values(kn, dtype, backend, device, 64.0)
        V = _to_values(vn, dtype, backend, device, 64.0)
    else:
        assert not category
        kn = _levels16(seed, TID_K, flat, backend) - 32768
        vn = (_levels16(seed, TID_V, flat, backend) >> 1) + (_levels16(seed, TID_VMU, mu_idx, backend) >> 1) - 32768
        K = _to_values(kn, dtype, backend, device, 16384.0)
        V = _to_values(vn, dtype, backend, device, 16384.0)
    return K.reshape(-1, H, d), V.reshape(-1, H, d)


def _centroid_level(seed, rows, chain_start, H, d, backend, device):
    """Centroid level (0..63) per (row, h, c): a sticky chain over 64 centroids per user.

    Row j switches category with probability 26/256 (~0.1) or at its user's first row; the
    category is then a hashed byte mod 64.  c_j = category of the last switch point <= j.
    The switch rule is counter based so any row range reproduces the same chain: we scan back
    from the row to the nearest switch point (bounded, since switches are frequent; rows whose
    scan passes the user start use the user start).
    """
    assert chain_start is not None
    if backend == "numpy":
        rows_a = np.asarray(rows, dtype=np.int64)
        start = np.asarray(chain_start, dtype=np.int64)
        sw_row = rows_a.copy()
        done = (levels(seed, TID_CHAIN, 2 * sw_row, backend) < 26) | (sw_row <= start)
        for _ in range(4096):
            if done.all():
                break
            sw_row = np.where(done, sw_row, sw_row - 1)
            done = done | (levels(seed, TID_CHAIN, 2 * sw_row, backend) < 26) | (sw_row <= start)
        sw_row = np.maximum(sw_row, start)
        cat = levels(seed, TID_CHAIN, 2 * sw_row + 1, backend) % 64
        cidx = cat[:, None] * (H * d) + np.arange(H * d, dtype=np.int64)[None, :]
        return levels(seed, TID_CENT, cidx, backend) >> 2
    import torch
    start = chain_start
    sw_row = rows.clone()
    done = (levels(seed, TID_CHAIN, 2 * sw_row, backend) < 26) | (sw_row <= start)
    for _ in range(4096):
        if bool(done.all()):
            break
        sw_row = torch.where(done, sw_row, sw_row - 1)
        done = done | (levels(seed, TID_CHAIN, 2 * sw_row, backend) < 26) | (sw_row <= start)
    sw_row = torch.maximum(sw_row, start)
    cat = (levels(seed, TID_CHAIN, 2 * sw_row + 1, backend) % 64).to(torch.int64)
    cidx = cat[:, None] * (H * d) + torch.arange(H * d, dtype=torch.int64, device=device)[None, :]
    return levels(seed, TID_CENT, cidx, backend) >> 2


def make_batch(lengths, S: int, H: int, d: int, *, seed: int = 0, dtype: str = "bf16",
               tau: int = 1, category: bool = False, backend: str = "numpy", device=None,
               chunk_rows: int = 1 << 18):
    """Full batch: (Q[S,H,d], K[sumL,H,d], V[sumL,H,d], offsets[B+1]) for the given lengths."""
    off = offsets_from_lengths(lengths)
    total = int(off[-1])
    q = make_q(S, H, d, seed=seed, dtype=dtype, tau=tau, backend=backend, device=device)
    if backend == "numpy":
        ks, vs = [], []
        for r0 in range(0, max(total, 1), chunk_rows):
            rows = np.arange(r0, min(total, r0 + chunk_rows), dtype=np.int64)
            if len(rows) == 0:
                break
            us = row_users(off, rows)
            k, v = make_kv(rows, us, H, d, seed=seed, dtype=dtype, category=category,
                           chain_start=off[us] if category else None)
            ks.append(k)
            vs.append(v)
        if not ks:
            z = np.zeros((0, H, d), np.float32)
            return q, z, z.copy(), off
        return q, np.concatenate(ks), np.concatenate(vs), off
    import torch
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    K = torch.empty((total, H, d), dtype=tdt, device=device)
    V = torch.empty((total, H, d), dtype=tdt, device=device)
    off_t = torch.as_tensor(off, device=device)
    for r0 in range(0, total, chunk_rows):
        rows = torch.arange(r0, min(total, r0 + chunk_rows), dtype=torch.int64, device=device)
        us = row_users(off_t, rows, backend="torch")
        k, v = make_kv(rows, us, H, d, seed=seed, dtype=dtype, category=category, backend="torch",
                       device=device, chain_start=off_t[us] if category else None)
        K[r0:r0 + len(rows)] = k
        V[r0:r0 + len(rows)] = v
    return q, K, V, off
