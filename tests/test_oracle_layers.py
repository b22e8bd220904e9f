"""Pins of the oracle's multi-layer summarizer (NEXT-3; reading R23,
SPEC.md:237-254), CPU only.

  L1 SPEC.md:243: no history, one layer, identity projections, phi = Id, no 1/N: tokens =
     seeds + g * seeds (seeds^T seeds) with the gate g = sigmoid(0) = 1/2 (W_g = 0)
  L2 the layer written densely: per head (Q K^T) V / N (associativity, phi = Id), the SGLU gate and
     the residual composed with numpy
  L3 two layers = the one-layer oracle applied twice
  L4 purity and shape: two users with the same [seeds; history] get bitwise the same tokens; the token
     block is S x D whatever M in {0, 10, 1000}
  L5 full attention without positions: permuting a user's history rows leaves its tokens unchanged
A dropped residual, gate or 1/N, a per-user state that mixes users, or heads mixed up fails one of them.
"""
import numpy as np
import pytest

import oracle


def grid(rng, shape, den=64.0):
    return (rng.integers(-128, 128, size=shape) / den).astype(np.float32)


def weights(rng, L, D, den=None):
    den = den or 64.0 * np.sqrt(D)
    return (rng.integers(-128, 128, size=(L, 5, D, D)) / den).astype(np.float32)


def test_l1_spec_no_history_closed_form():
    rng = np.random.default_rng(1)
    S, D = 3, 4
    seeds = grid(rng, (S, D))
    W = np.zeros((1, 5, D, D), np.float32)
    for t in (0, 1, 2, 4):
        W[0, t] = np.eye(D, dtype=np.float32)
    out = oracle.summarize_layers(seeds, [0, S], W, S, 1, "identity", "identity", False)
    s = seeds.astype(np.float64)
    np.testing.assert_allclose(out, s + 0.5 * s @ (s.T @ s), rtol=0, atol=1e-12)


def _dense_layer(x, off, W, H, normalize):
    D = x.shape[1]
    d = D // H
    q, k, v, g = (x @ W[t].astype(np.float64).T for t in range(4))
    o = np.zeros_like(x)
    for u in range(len(off) - 1):
        a, b = off[u], off[u + 1]
        N = b - a
        for h in range(H):
            c = slice(h * d, (h + 1) * d)
            o[a:b, c] = (q[a:b, c] @ k[a:b, c].T) @ v[a:b, c] / (N if normalize else 1.0)
    return x + (o / (1.0 + np.exp(-g))) @ W[4].astype(np.float64).T


@pytest.mark.parametrize("normalize", [True, False])
def test_l2_dense_associativity(normalize):
    rng = np.random.default_rng(2)
    S, H, d = 3, 2, 4
    lens = [5, 0, 9]
    off = np.concatenate([[0], np.cumsum([S + L for L in lens])]).astype(np.int64)
    x = grid(rng, (off[-1], H * d))
    W = weights(rng, 1, H * d)
    got = oracle.summarize_layers(x, off, W, S, H, "identity", "identity", normalize)
    np.testing.assert_allclose(got, _dense_layer(x.astype(np.float64), off, W[0], H, normalize), rtol=1e-12, atol=1e-12)


def test_l3_two_layers_compose():
    rng = np.random.default_rng(3)
    S, H, d = 2, 2, 8
    off = np.array([0, S + 7, 2 * S + 10], np.int64)
    x = grid(rng, (off[-1], H * d))
    W = weights(rng, 2, H * d)
    two = oracle.summarize_layers(x, off, W, S, H)
    one = oracle.summarize_layers(x, off, W[:1], S, H)
    # the one-layer output is not float32-exact: run layer 2 with the float64 input through the
    # dense reference of the same definition instead (phi = SiLU, 1/N)
    import torch
    xx = torch.from_numpy(one)
    Wt = torch.from_numpy(W[1].astype(np.float64))
    q, k, v, g = (xx @ Wt[t].T for t in range(4))
    o = torch.zeros_like(xx)
    silu = torch.nn.functional.silu
    for u in range(2):
        a, b = int(off[u]), int(off[u + 1])
        for h in range(H):
            c = slice(h * d, (h + 1) * d)
            z = silu(silu(k[a:b, c]).T @ v[a:b, c] / (b - a))
            o[a:b, c] = silu(q[a:b, c]) @ z
    ref = xx + (o * torch.sigmoid(g)) @ Wt[4].T
    np.testing.assert_allclose(two, ref.numpy(), rtol=1e-11, atol=1e-11)


def test_l4_purity_and_shape():
    rng = np.random.default_rng(4)
    S, H, d = 3, 1, 8
    seeds = grid(rng, (S, H * d))
    W = weights(rng, 2, H * d)
    uih = grid(rng, (12, H * d))
    x = np.concatenate([seeds, uih, seeds, uih])
    off = np.array([0, S + 12, 2 * S + 24], np.int64)
    out = oracle.summarize_layers(x, off, W, S, H)
    assert np.array_equal(out[0:S], out[S + 12:2 * S + 12])
    for M in (0, 10, 1000):
        xm = np.concatenate([seeds, grid(rng, (M, H * d))])
        o = oracle.summarize_layers(xm, [0, S + M], W[:1], S, H)
        assert o[:S].shape == (S, H * d) and np.all(np.isfinite(o))


def test_l5_history_permutation():
    rng = np.random.default_rng(5)
    S, H, d, M = 4, 2, 8, 30
    x = grid(rng, (S + M, H * d))
    W = weights(rng, 2, H * d)
    base = oracle.summarize_layers(x, [0, S + M], W, S, H)
    perm = np.concatenate([np.arange(S), S + rng.permutation(M)])
    got = oracle.summarize_layers(x[perm], [0, S + M], W, S, H)
    np.testing.assert_allclose(got[:S], base[:S], rtol=0, atol=1e-11)
    np.testing.assert_allclose(got, base[perm], rtol=0, atol=1e-11)
