"""float64 CPU oracle for VISTA stage-1 summarization -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` leg may import this package.  The product package ``paper_2510_22049_b200`` never
imports it and shares no code with it.

The arithmetic lives in ``vista_oracle.c`` (plain C, float64, OpenMP over (user, head, row));
this file only marshals numpy arrays.  Every function cites the passage it implements in the C
source.  Parity pins: tests/test_oracle_pins.py.  Readings where the paper is silent are listed
in DESIGN.md ("Readings"); the softmax scale (R4), the 1/N-before-phi2 order (R10) and the
empty-history convention (R6) have no paper value to match -> "parity unpinned" for those
choices specifically (their arithmetic is pinned by the closed forms below).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "vista_oracle.c")
_LIB = os.path.join(_HERE, "libvista_oracle.so")

ACT = {"identity": 0, "silu": 1, "shifted_elu": 2}

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2 -fopenmp, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i64, f64, i32 = ctypes.c_int64, ctypes.c_double, ctypes.c_int
        P = ctypes.c_void_p
        lib.vo_softmax.argtypes = [i64, i64, i64, i64, P, i64, P, P, P, f64, P, i64, P, P, i32]
        lib.vo_qla_state.argtypes = [i64, i64, i64, P, P, P, i32, P, i32]
        lib.vo_qla_finalize.argtypes = [i64, i64, i64, i64, P, i64, P, P, i32, i32, i32, P, i32]
        lib.vo_qla_rows.argtypes = [i64, i64, i64, P, P, P, P, P, P, i32, i32, i32, P, i32]
        lib.vo_merge_lse.argtypes = [i64, i64, i64, P, P, P, P]
        lib.vo_merge_sum.argtypes = [i64, i64, P, P]
        lib.vo_quantize_rows_f32.argtypes = [i64, i64, P, P, P, P]
        lib.vo_act.argtypes = [i32, f64]
        lib.vo_act.restype = f64
        lib.vo_act_prime.argtypes = [i32, f64]
        lib.vo_act_prime.restype = f64
        lib.vo_softmax_backward.argtypes = [i64, i64, i64, i64, P, i64, P, P, P, f64, P, P, P, P, i32]
        lib.vo_qla_backward.argtypes = [i64, i64, i64, i64, P, i64, P, P, P, P, i32, i32, i32, P, P, P, i32]
        lib.vo_num_threads.restype = i32
        lib.vo_target_attend.argtypes = [i64, i64, i64, i64, P, P, P, P, P, P, P, P, f64, P, P, i32]
        lib.vo_summarize_layers.argtypes = [i64, i64, i64, i64, i64, P, P, P, i32, i32, i32, P, i32]
        _lib = lib
    return _lib


def num_threads() -> int:
    return int(_load().vo_num_threads())


def _f32(x):
    x = np.ascontiguousarray(x)
    if x.dtype != np.float32:
        # the inputs are grid values exact in float32 (synth/); float64 inputs are accepted
        # only when they are exactly representable in float32
        y = x.astype(np.float32)
        if not np.array_equal(y.astype(x.dtype), x):
            raise ValueError("oracle inputs must be exactly representable in float32")
        x = y
    return x


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def act(kind: str, x: float) -> float:
    """phi(x) in float64."""
    return float(_load().vo_act(ACT[kind], float(x)))


def _with_prefix(k, v, offsets, k_prefix, v_prefix):
    """Histories with a shared key prefix prepended to every user: the key set of user u is
    [prefix; history of u] (reading R18; self-attention over [seeds; UIH]).
    Returns (k', v', offsets') of the concatenated per-user histories."""
    offsets = np.asarray(offsets, dtype=np.int64)
    kp = np.asarray(k_prefix)
    vp = np.asarray(v_prefix)
    P = kp.shape[0]
    B = len(offsets) - 1
    ks, vs = [], []
    for u in range(B):
        ks += [kp, np.asarray(k[offsets[u]:offsets[u + 1]])]
        vs += [vp, np.asarray(v[offsets[u]:offsets[u + 1]])]
    lens = np.diff(offsets) + P
    off2 = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    H, d = kp.shape[1:]
    k2 = np.concatenate(ks) if ks else np.zeros((0, H, d), kp.dtype)
    v2 = np.concatenate(vs) if vs else np.zeros((0, H, d), vp.dtype)
    return k2, v2, off2


def softmax_summarize(q, k, v, offsets, scale=None, rows=None, q_per_user=False, threads=0,
                      k_prefix=None, v_prefix=None):
    """Seed-row softmax attention over each user's history.

    q: [S,H,d] (shared seeds) or [B,S,H,d] with q_per_user=True; k, v: [sumL,H,d];
    offsets: [B+1] int64.  rows: optional subset of query rows.
    Returns out [B, R, H, d] float64 and lse [B, H, R] float64 (natural log).
    k_prefix, v_prefix: optional shared keys [P,H,d] attended by every user (see _with_prefix).
    """
    if k_prefix is not None:
        k, v, offsets = _with_prefix(k, v, offsets, k_prefix, v_prefix)
    q, k, v = _f32(q), _f32(k), _f32(v)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    B = len(offsets) - 1
    S, H, d = q.shape[-3:]
    if k.shape[1:] != (H, d) or v.shape != k.shape or offsets[-1] != k.shape[0]:
        raise ValueError("shape mismatch")
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    rows = np.arange(S, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
    R = len(rows)
    out = np.empty((B, R, H, d), np.float64)
    lse = np.empty((B, H, R), np.float64)
    stride = S * H * d if q_per_user else 0
    if k.shape[0] == 0:
        k = np.zeros((1, H, d), np.float32)
        v = k
    rc = _load().vo_softmax(B, S, H, d, _ptr(q), stride, _ptr(k), _ptr(v), _ptr(offsets),
                            float(scale), _ptr(rows), R, _ptr(out), _ptr(lse), int(threads))
    if rc != 0:
        raise ValueError("vo_softmax failed")
    return out, lse


def qla_state(k, v, offsets, phi1="silu", threads=0):
    """Z[u,h] = sum_j phi1(k_j)^T v_j.  Returns [B,H,d,d] float64."""
    k, v = _f32(k), _f32(v)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    B = len(offsets) - 1
    _, H, d = k.shape
    z = np.empty((B, H, d, d), np.float64)
    if k.shape[0] == 0:
        k = np.zeros((1, H, d), np.float32)
        v = k
    _load().vo_qla_state(B, H, d, _ptr(k), _ptr(v), _ptr(offsets), ACT[phi1], _ptr(z), int(threads))
    return z


def qla_finalize(q, z, n_items, phi1="silu", phi2="silu", normalize=True, q_per_user=False,
                 threads=0):
    """O = phi1(Q) phi2(Z / N_u).  Returns [B,S,H,d]."""
    q = _f32(q)
    z = np.ascontiguousarray(z, dtype=np.float64)
    n_items = np.ascontiguousarray(n_items, dtype=np.int64)
    B, H, d, _ = z.shape
    S = q.shape[-3]
    out = np.empty((B, S, H, d), np.float64)
    stride = S * H * d if q_per_user else 0
    _load().vo_qla_finalize(B, S, H, d, _ptr(q), stride, _ptr(z), _ptr(n_items), ACT[phi1],
                            ACT[phi2], int(bool(normalize)), _ptr(out), int(threads))
    return out


def qla_summarize(q, k, v, offsets, phi1="silu", phi2="silu", normalize=True, q_per_user=False,
                  threads=0, k_prefix=None, v_prefix=None):
    """QLA source part at the seed rows: state then finalize.  Returns out [B,S,H,d].
    With a shared key prefix the state and N_u run over [prefix; history] (_with_prefix)."""
    if k_prefix is not None:
        k, v, offsets = _with_prefix(k, v, offsets, k_prefix, v_prefix)
    offsets = np.asarray(offsets, dtype=np.int64)
    z = qla_state(k, v, offsets, phi1, threads)
    return qla_finalize(q, z, np.diff(offsets), phi1, phi2, normalize, q_per_user, threads)


def qla_rows(q_rows, row_offsets, k, v, offsets, phi1="silu", phi2="silu", normalize=True,
             k_self=None, v_self=None, threads=0):
    """QLA at per-user query rows (NEXT-3 history rows; NEXT-4 target rows with
    the Delta self term): out[r] = phi1(q_r) phi2(Zbar_u) [+ (phi1(q_r) .
    phi1(k_self_r)) v_self_r] for r in [row_offsets[u], row_offsets[u+1]).  Returns [R,H,d]."""
    q_rows = _f32(q_rows)
    row_offsets = np.ascontiguousarray(row_offsets, dtype=np.int64)
    offsets = np.asarray(offsets, dtype=np.int64)
    z = qla_state(k, v, offsets, phi1, threads)
    B, H, d, _ = z.shape
    R = q_rows.shape[0]
    out = np.empty((R, H, d), np.float64)
    if R == 0:
        return out
    ks = vs = None
    if k_self is not None:
        ks, vs = _f32(k_self), _f32(v_self)
    n_items = np.ascontiguousarray(np.diff(offsets), dtype=np.int64)
    rc = _load().vo_qla_rows(B, H, d, _ptr(z), _ptr(n_items), _ptr(q_rows), _ptr(row_offsets),
                             _ptr(ks) if ks is not None else None, _ptr(vs) if vs is not None else None,
                             ACT[phi1], ACT[phi2], int(bool(normalize)), _ptr(out), int(threads))
    if rc != 0:
        raise ValueError("vo_qla_rows failed")
    return out


def act_prime(kind: str, x: float) -> float:
    """phi'(x) in float64 (shifted ELU PAPER.md:795-809)."""
    return float(_load().vo_act_prime(ACT[kind], float(x)))


def qla_backward(q, k, v, offsets, dout, phi1="silu", phi2="silu", normalize=True, q_per_user=False,
                 threads=0, sum_users=None):
    """QLA backward (NEXT-2; chain rule, vo_qla_backward).  dout [B,S,H,d].
    Returns dq, dk [sumL,H,d], dv [sumL,H,d] (float64).  dq is [B,S,H,d] per user; with shared
    seeds (q_per_user False) it is summed over users to [S,H,d] unless sum_users=False."""
    q, k, v, dout = _f32(q), _f32(k), _f32(v), _f32(dout)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    B = len(offsets) - 1
    S, H, d = q.shape[-3:]
    T = k.shape[0]
    dq = np.empty((B, S, H, d), np.float64)
    dk = np.empty((T, H, d), np.float64)
    dv = np.empty((T, H, d), np.float64)
    kk, vv = (k, v) if T > 0 else (np.zeros((1, H, d), np.float32),) * 2
    dkk, dvv = (dk, dv) if T > 0 else (np.zeros((1, H, d)), np.zeros((1, H, d)))
    stride = S * H * d if q_per_user else 0
    rc = _load().vo_qla_backward(B, S, H, d, _ptr(q), stride, _ptr(kk), _ptr(vv), _ptr(offsets), _ptr(dout),
                                 ACT[phi1], ACT[phi2], int(bool(normalize)), _ptr(dq), _ptr(dkk), _ptr(dvv),
                                 int(threads))
    if rc != 0:
        raise ValueError("vo_qla_backward failed")
    if (sum_users if sum_users is not None else not q_per_user):
        dq = dq.sum(axis=0)
    return dq, dk, dv


def softmax_backward(q, k, v, offsets, dout, scale=None, q_per_user=False, threads=0, sum_users=None):
    """Softmax backward (NEXT-2; vo_softmax_backward).  dout [B,S,H,d].  Returns dq (summed over
    users for shared seeds unless sum_users=False; else [B,S,H,d]), dk, dv [sumL,H,d], float64."""
    q, k, v, dout = _f32(q), _f32(k), _f32(v), _f32(dout)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    B = len(offsets) - 1
    S, H, d = q.shape[-3:]
    T = k.shape[0]
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    dq = np.empty((B, S, H, d), np.float64)
    dk = np.empty((max(T, 1), H, d), np.float64)
    dv = np.empty((max(T, 1), H, d), np.float64)
    kk, vv = (k, v) if T > 0 else (np.zeros((1, H, d), np.float32),) * 2
    stride = S * H * d if q_per_user else 0
    rc = _load().vo_softmax_backward(B, S, H, d, _ptr(q), stride, _ptr(kk), _ptr(vv), _ptr(offsets), float(scale),
                                     _ptr(dout), _ptr(dq), _ptr(dk), _ptr(dv), int(threads))
    if rc != 0:
        raise ValueError("vo_softmax_backward failed")
    if (sum_users if sum_users is not None else not q_per_user):
        dq = dq.sum(axis=0)
    return dq, dk[:T], dv[:T]


def merge_lse(part_o, part_lse):
    """LSE merge of P partials. part_o [P, ..., d], part_lse [P, ...] -> (out, lse)."""
    part_o = np.ascontiguousarray(part_o, dtype=np.float64)
    part_lse = np.ascontiguousarray(part_lse, dtype=np.float64)
    P = part_o.shape[0]
    d = part_o.shape[-1]
    n = int(np.prod(part_o.shape[1:-1]))
    assert part_lse.shape == part_o.shape[:-1]
    out = np.empty(part_o.shape[1:], np.float64)
    lse = np.empty(part_lse.shape[1:], np.float64)
    _load().vo_merge_lse(P, n, d, _ptr(part_o), _ptr(part_lse), _ptr(out), _ptr(lse))
    return out, lse


def merge_sum(parts):
    parts = np.ascontiguousarray(parts, dtype=np.float64)
    out = np.empty(parts.shape[1:], np.float64)
    _load().vo_merge_sum(parts.shape[0], int(np.prod(parts.shape[1:])), _ptr(parts), _ptr(out))
    return out


def quantize_rows_int8(x):
    """Int8 export of token rows (scheme SPEC.md:339-347), float32 arithmetic.
    x: [..., d] float32 -> (codes int8 [..., d], scale float32 [...], zero_point float32 [...])."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    d = x.shape[-1]
    n = int(np.prod(x.shape[:-1]))
    codes = np.empty(x.shape, np.int8)
    scale = np.empty(x.shape[:-1], np.float32)
    zp = np.empty(x.shape[:-1], np.float32)
    _load().vo_quantize_rows_f32(n, d, _ptr(x), _ptr(codes), _ptr(scale), _ptr(zp))
    return codes, scale, zp


def dequantize_rows_int8(codes, scale, zp):
    """x^ = code * scale + zero_point, float64."""
    return codes.astype(np.float64) * scale[..., None].astype(np.float64) + zp[..., None].astype(np.float64)


def target_attend(codes, tscale, tzp, q, k_self, v_self, row_offsets, scale=None, resid=None, threads=0):
    """Stage-2 target-aware attention (NEXT-4, vo_target_attend): every candidate row attends to the
    dequantized summary tokens of its user and to itself.  codes [B,S,H,d] int8, tscale / tzp
    [B,S,H]; q, k_self, v_self (, resid) [R,H,d].  Returns out [R,H,d], lse [R,H] (float64)."""
    codes = np.ascontiguousarray(codes, dtype=np.int8)
    tscale, tzp = _f32(tscale), _f32(tzp)
    q, k_self, v_self = _f32(q), _f32(k_self), _f32(v_self)
    rz = None if resid is None else _f32(resid)
    row_offsets = np.ascontiguousarray(row_offsets, dtype=np.int64)
    B, S, H, d = codes.shape
    R = q.shape[0]
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    out = np.empty((R, H, d), np.float64)
    lse = np.empty((R, H), np.float64)
    if R == 0:
        return out, lse
    rc = _load().vo_target_attend(B, S, H, d, _ptr(codes), _ptr(tscale), _ptr(tzp), _ptr(q), _ptr(k_self),
                                  _ptr(v_self), _ptr(rz) if rz is not None else None, _ptr(row_offsets), float(scale),
                                  _ptr(out), _ptr(lse), int(threads))
    if rc != 0:
        raise ValueError("vo_target_attend failed")
    return out, lse


def summarize_layers(x, offsets, weights, S, H, phi1="silu", phi2="silu", normalize=True, threads=0):
    """Multi-layer summarizer (NEXT-3, vo_summarize_layers): x [R, D] (user u = rows [offsets[u],
    offsets[u+1]), its first S rows the seed rows), weights [L, 5, D, D] (q, k, v, g, o; row = output).
    Returns x after the layers [R, D] float64; the summary tokens are each user's first S rows."""
    x = _f32(x)
    weights = _f32(weights)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    R, D = x.shape
    L = weights.shape[0]
    assert weights.shape[1:] == (5, D, D) and D % H == 0
    out = np.empty((R, D), np.float64)
    rc = _load().vo_summarize_layers(len(offsets) - 1, S, H, D // H, L, _ptr(weights), _ptr(x), _ptr(offsets),
                                     ACT[phi1], ACT[phi2], int(bool(normalize)), _ptr(out), int(threads))
    if rc != 0:
        raise ValueError("vo_summarize_layers failed")
    return out
