"""Pins of the oracle's QLA at per-user query rows (NEXT-3 history rows; NEXT-4
target rows with the Delta self term), CPU only.

  R1 associativity: phi = Id, no 1/N -> o_r = sum_j (q_r . k_j) v_j, dense brute force
  R2 Delta as attention to the target itself: phi = Id -> o_t = sum_{j in S_u + {t}} (q_t . k_j) v_j
  R3 worked scalars (tests/golden/worked_values.json "qla_target_scalar")
  R4 rows = the seeds of every user reproduces the seed-row summary (qla_summarize)
  R5 empty history: Z = 0, W = phi2(0) (0 for SiLU; e^-1 for shifted ELU, a closed form)
  R6 invariants: permutation of a user's history; linearity of the Delta term in v_self
  R7 App. B's dense mixed form: phi = Id, 1/N -> source and target rows together equal
     (Q K^T (.) M) V / N with M = [[1,0],[1,I_m]], one N for both kinds of row
A dropped Delta term, a Delta without phi1 on either side, a transposed state or rows assigned to
the wrong user fails at least one of them.
"""
import json
import math
import os

import numpy as np

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")


def grid(rng, shape, den=64.0):
    return (rng.integers(-128, 128, size=shape) / den).astype(np.float32)


def _case(rng, lens, rows, H=2, d=8):
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    roff = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
    k, v = grid(rng, (off[-1], H, d)), grid(rng, (off[-1], H, d))
    q = grid(rng, (roff[-1], H, d))
    ks, vs = grid(rng, (roff[-1], H, d)), grid(rng, (roff[-1], H, d))
    return q, roff, k, v, off, ks, vs


def test_r1_identity_associativity():
    rng = np.random.default_rng(1)
    q, roff, k, v, off, _, _ = _case(rng, [5, 0, 9], [3, 2, 4])
    got = oracle.qla_rows(q, roff, k, v, off, "identity", "identity", False)
    for u in range(3):
        for r in range(roff[u], roff[u + 1]):
            for h in range(q.shape[1]):
                kk = k[off[u]:off[u + 1], h].astype(np.float64)
                vv = v[off[u]:off[u + 1], h].astype(np.float64)
                want = ((kk @ q[r, h].astype(np.float64))[:, None] * vv).sum(0)
                np.testing.assert_allclose(got[r, h], want, rtol=0, atol=1e-12)


def test_r2_delta_is_attention_to_itself():
    rng = np.random.default_rng(2)
    q, roff, k, v, off, ks, vs = _case(rng, [4, 7, 0], [2, 3, 2])
    got = oracle.qla_rows(q, roff, k, v, off, "identity", "identity", False, k_self=ks, v_self=vs)
    for u in range(3):
        for r in range(roff[u], roff[u + 1]):
            for h in range(q.shape[1]):
                kk = np.concatenate([k[off[u]:off[u + 1], h], ks[r:r + 1, h]]).astype(np.float64)
                vv = np.concatenate([v[off[u]:off[u + 1], h], vs[r:r + 1, h]]).astype(np.float64)
                want = ((kk @ q[r, h].astype(np.float64))[:, None] * vv).sum(0)
                np.testing.assert_allclose(got[r, h], want, rtol=0, atol=1e-12)


def test_r3_worked_scalars():
    for e in json.load(open(GOLDEN))["qla_target_scalar"]:
        one = lambda x: np.array([[[x]]], np.float32)  # noqa: E731
        if "k_hist" in e:  # several source items, App. B's 1/N
            col = lambda xs: np.array(xs, np.float32).reshape(-1, 1, 1)  # noqa: E731
            n = len(e["k_hist"])
            got = oracle.qla_rows(one(e["q_t"]), [0, 1], col(e["k_hist"]), col(e["v_hist"]), [0, n], e["phi1"],
                                  e["phi2"], e["normalize"], k_self=one(e["k_t"]), v_self=one(e["v_t"]))
            assert abs(got[0, 0, 0] - e["value"]) <= 1e-12, (e, got)
            continue
        got = oracle.qla_rows(one(e["q_t"]), [0, 1], one(e["k"]), one(e["v"]), [0, 1], e["phi1"], e["phi2"],
                              e["normalize"], k_self=one(e["k_t"]), v_self=one(e["v_t"]))
        assert abs(got[0, 0, 0] - e["value"]) <= 1e-12, (e, got)
        # the history-row form (no Delta) is the seed-row scalar example
        got_h = oracle.qla_rows(one(e["q_hist"]), [0, 1], one(e["k"]), one(e["v"]), [0, 1], e["phi1"], e["phi2"],
                                e["normalize"])
        assert abs(got_h[0, 0, 0] - 30.0) <= 1e-12


def test_r3_silu_scalar_closed_form():
    silu = lambda x: x / (1.0 + math.exp(-x))  # noqa: E731
    one = lambda x: np.array([[[x]]], np.float32)  # noqa: E731
    got = oracle.qla_rows(one(2.0), [0, 1], one(3.0), one(5.0), [0, 1], "silu", "silu", True,
                          k_self=one(3.0), v_self=one(5.0))
    want = silu(2.0) * silu(silu(3.0) * 5.0 / 1.0) + silu(2.0) * silu(3.0) * 5.0 / 1.0
    assert abs(got[0, 0, 0] - want) <= 1e-12 * abs(want)
    # two source items (N = 2): the Delta term is halved with the state (App. B)
    k2, v2 = np.array([3.0, -1.0], np.float32).reshape(2, 1, 1), np.array([5.0, 2.0], np.float32).reshape(2, 1, 1)
    got = oracle.qla_rows(one(2.0), [0, 1], k2, v2, [0, 2], "silu", "silu", True, k_self=one(3.0), v_self=one(5.0))
    z = (silu(3.0) * 5.0 + silu(-1.0) * 2.0) / 2.0
    want = silu(2.0) * silu(z) + silu(2.0) * silu(3.0) * 5.0 / 2.0
    assert abs(got[0, 0, 0] - want) <= 1e-12 * abs(want)


def test_r4_rows_equal_seed_summary():
    rng = np.random.default_rng(4)
    lens, S, H, d = [6, 0, 3, 11], 5, 2, 8
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    k, v = grid(rng, (off[-1], H, d)), grid(rng, (off[-1], H, d))
    seeds = grid(rng, (S, H, d))
    for phi1, phi2, norm in [("silu", "silu", True), ("shifted_elu", "identity", False)]:
        want = oracle.qla_summarize(seeds, k, v, off, phi1, phi2, norm)  # [B,S,H,d]
        q = np.tile(seeds, (len(lens), 1, 1))
        roff = np.arange(len(lens) + 1, dtype=np.int64) * S
        got = oracle.qla_rows(q, roff, k, v, off, phi1, phi2, norm)
        np.testing.assert_allclose(got.reshape(want.shape), want, rtol=0, atol=1e-12)


def test_r5_empty_history():
    rng = np.random.default_rng(5)
    H, d = 2, 8
    q, ks, vs = grid(rng, (3, H, d)), grid(rng, (3, H, d)), grid(rng, (3, H, d))
    k = np.zeros((0, H, d), np.float32)
    off, roff = np.array([0, 0], np.int64), np.array([0, 3], np.int64)
    got = oracle.qla_rows(q, roff, k, k, off, "silu", "silu", True)
    assert np.all(got == 0.0)
    # shifted ELU outer: W = phi2(0) = e^-1 everywhere -> o_r[c2] = e^-1 sum_c1 phi1(q_r)[c1]
    got = oracle.qla_rows(q, roff, k, k, off, "identity", "shifted_elu", True)
    want = math.exp(-1.0) * q.astype(np.float64).sum(-1, keepdims=True) * np.ones((1, 1, d))
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)
    # with the Delta term only the self term remains (SiLU outer)
    got = oracle.qla_rows(q, roff, k, k, off, "identity", "silu", True, k_self=ks, v_self=vs)
    want = (q.astype(np.float64) * ks).sum(-1, keepdims=True) * vs
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)


def test_r6_invariants():
    rng = np.random.default_rng(6)
    q, roff, k, v, off, ks, vs = _case(rng, [9, 4], [3, 3])
    base = oracle.qla_rows(q, roff, k, v, off, "silu", "silu", True, k_self=ks, v_self=vs)
    perm = np.concatenate([rng.permutation(np.arange(0, 9)), 9 + rng.permutation(np.arange(0, 4))])
    np.testing.assert_allclose(oracle.qla_rows(q, roff, k[perm], v[perm], off, "silu", "silu", True,
                                               k_self=ks, v_self=vs), base, rtol=0, atol=1e-12)
    no_delta = oracle.qla_rows(q, roff, k, v, off, "silu", "silu", True)
    twice = oracle.qla_rows(q, roff, k, v, off, "silu", "silu", True, k_self=ks, v_self=2 * vs)
    np.testing.assert_allclose(twice - no_delta, 2 * (base - no_delta), rtol=0, atol=1e-12)


def test_r7_appendix_b_dense_mixed_form():
    """SPEC.md:186's kernel equivalence: phi = Id with 1/N, every user's source rows (no Delta) and
    target rows (Delta) equal the dense (Q K^T (.) M) V / N of App. B, M = [[1_nn, 0], [1_mn, I_m]],
    N = n = the user's source length (one scalar for the whole product)."""
    rng = np.random.default_rng(7)
    lens, ntgt, H, d = [6, 3, 11], [4, 1, 5], 2, 8
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    toff = np.concatenate([[0], np.cumsum(ntgt)]).astype(np.int64)
    ks, vs, qs = grid(rng, (off[-1], H, d)), grid(rng, (off[-1], H, d)), grid(rng, (off[-1], H, d))
    qt, kt, vt = grid(rng, (toff[-1], H, d)), grid(rng, (toff[-1], H, d)), grid(rng, (toff[-1], H, d))
    src = oracle.qla_rows(qs, off, ks, vs, off, "identity", "identity", True)
    tgt = oracle.qla_rows(qt, toff, ks, vs, off, "identity", "identity", True, k_self=kt, v_self=vt)
    for u in range(len(lens)):
        n, m = lens[u], ntgt[u]
        M = np.zeros((n + m, n + m))
        M[:, :n] = 1.0
        M[n:, n:] = np.eye(m)
        for h in range(H):
            Q = np.concatenate([qs[off[u]:off[u + 1], h], qt[toff[u]:toff[u + 1], h]]).astype(np.float64)
            K = np.concatenate([ks[off[u]:off[u + 1], h], kt[toff[u]:toff[u + 1], h]]).astype(np.float64)
            V = np.concatenate([vs[off[u]:off[u + 1], h], vt[toff[u]:toff[u + 1], h]]).astype(np.float64)
            O = ((Q @ K.T) * M) @ V / n
            np.testing.assert_allclose(src[off[u]:off[u + 1], h], O[:n], rtol=0, atol=1e-12)
            np.testing.assert_allclose(tgt[toff[u]:toff[u + 1], h], O[n:], rtol=0, atol=1e-12)
