"""Pins of the oracle's stage-2 target-aware attention (NEXT-4; Sec. 3.3 over the
cached, dequantized summary tokens PAPER.md:125-126; SPEC.md:264-272 target_attend), CPU only.

  T1 SPEC.md:270: tokens all zero and the value zero -> output = the candidate's residual, exactly
  T2 SPEC.md:269 / PAPER.md:156: a candidate alone == the same candidate inside a batch of 100 (bitwise)
  T3 the definition through a library routine: torch SDPA (float64) over K = [tokens; k_c], V = [tokens; v_c]
  T4 a hand-evaluated scalar case (dequantization code * scale + zero point, then a two-key softmax)
  T5 invariants: permuting a user's tokens, shifting every logit by a constant (q . c) leaves out unchanged
A wrong dequantization, a dropped self key, a softmax over the wrong axis or candidates leaking into
each other fails at least one of them.
"""
import math

import numpy as np
import torch

import oracle


def _case(rng, B, S, H, d, rows):
    codes = rng.integers(-127, 128, size=(B, S, H, d)).astype(np.int8)
    tscale = (rng.integers(1, 64, size=(B, S, H)) / 1024.0).astype(np.float32)
    tzp = (rng.integers(-64, 64, size=(B, S, H)) / 128.0).astype(np.float32)
    roff = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
    R = int(roff[-1])
    g = lambda: (rng.integers(-128, 128, size=(R, H, d)) / 64.0).astype(np.float32)  # noqa: E731
    return codes, tscale, tzp, g(), g(), g(), roff


def test_t1_zero_tokens_zero_value_is_the_residual():
    rng = np.random.default_rng(1)
    codes, ts, tz, q, k, v, roff = _case(rng, 2, 4, 2, 8, [3, 2])
    codes[:] = 0
    tz[:] = 0.0
    resid = (rng.integers(-128, 128, size=q.shape) / 64.0).astype(np.float32)
    out, _ = oracle.target_attend(codes, ts, tz, q, k, np.zeros_like(v), roff, resid=resid)
    assert np.array_equal(out, resid.astype(np.float64))


def test_t2_candidate_independence_bitwise():
    rng = np.random.default_rng(2)
    codes, ts, tz, q, k, v, roff = _case(rng, 1, 6, 2, 8, [100])
    full, lse_full = oracle.target_attend(codes, ts, tz, q, k, v, roff)
    for c in (0, 37, 99):
        one, lse_one = oracle.target_attend(codes, ts, tz, q[c:c + 1], k[c:c + 1], v[c:c + 1], [0, 1])
        assert np.array_equal(one[0], full[c]) and np.array_equal(lse_one[0], lse_full[c])


def test_t3_equals_sdpa_over_tokens_and_self():
    rng = np.random.default_rng(3)
    B, S, H, d = 3, 7, 2, 16
    codes, ts, tz, q, k, v, roff = _case(rng, B, S, H, d, [4, 0, 5])
    out, lse = oracle.target_attend(codes, ts, tz, q, k, v, roff, scale=0.3)
    t = codes.astype(np.float64) * ts[..., None].astype(np.float64) + tz[..., None].astype(np.float64)
    for u in range(B):
        for c in range(roff[u], roff[u + 1]):
            for h in range(H):
                K = torch.from_numpy(np.concatenate([t[u, :, h], k[c:c + 1, h].astype(np.float64)]))
                V = torch.from_numpy(np.concatenate([t[u, :, h], v[c:c + 1, h].astype(np.float64)]))
                Q = torch.from_numpy(q[c:c + 1, h].astype(np.float64))
                want = torch.nn.functional.scaled_dot_product_attention(Q[None], K[None], V[None], scale=0.3)[0, 0]
                np.testing.assert_allclose(out[c, h], want.numpy(), rtol=1e-12, atol=1e-13)
                logits = 0.3 * (K @ Q[0])
                np.testing.assert_allclose(lse[c, h], torch.logsumexp(logits, 0).item(), rtol=1e-13)


def test_t4_scalar_hand_evaluated():
    # one token, d = 1: code 2, scale 0.5, zero point 1 -> t = 2; q = 1, k_c = 0, v_c = 4, scale 1:
    # logits (2, 0) -> out = (e^2 * 2 + 1 * 4) / (e^2 + 1)
    codes = np.array([[[[2]]]], np.int8)
    out, lse = oracle.target_attend(codes, np.array([[[0.5]]], np.float32), np.array([[[1.0]]], np.float32),
                                    np.ones((1, 1, 1), np.float32), np.zeros((1, 1, 1), np.float32),
                                    np.full((1, 1, 1), 4.0, np.float32), [0, 1], scale=1.0)
    e2 = math.exp(2.0)
    assert abs(out[0, 0, 0] - (2 * e2 + 4) / (e2 + 1)) <= 1e-15
    assert abs(lse[0, 0] - math.log(e2 + 1)) <= 1e-15


def test_t5_invariants():
    rng = np.random.default_rng(5)
    codes, ts, tz, q, k, v, roff = _case(rng, 1, 9, 1, 8, [6])
    base, lse = oracle.target_attend(codes, ts, tz, q, k, v, roff)
    perm = rng.permutation(9)
    pout, plse = oracle.target_attend(codes[:, perm], ts[:, perm], tz[:, perm], q, k, v, roff)
    np.testing.assert_allclose(pout, base, rtol=0, atol=1e-12)
    np.testing.assert_allclose(plse, lse, rtol=0, atol=1e-12)
    # shift: add a constant 1/8 to every token channel through the zero point and to k_c: each logit of
    # a candidate moves by scale * q . (1/8 ...) -> out moves by the same constant, lse by the shift
    shift = 0.125
    tz2 = tz + np.float32(shift)
    out2, lse2 = oracle.target_attend(codes, ts, tz2, q, k + np.float32(shift), v + np.float32(shift), roff)
    np.testing.assert_allclose(out2, base + shift, rtol=0, atol=1e-12)
    delta = q.astype(np.float64).sum(-1) * shift / math.sqrt(8)
    np.testing.assert_allclose(lse2, lse + delta, rtol=0, atol=1e-12)
