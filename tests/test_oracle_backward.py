"""Pins of the float64 oracle's QLA backward (NEXT-2, oracle.qla_backward), independent of it:
  B1  torch autograd (float64) through the forward definition O = phi1(Q) phi2(phi1(K)^T V / N)
  B2  central finite differences of a random linear functional of O (numpy float64 forward)
  B3  the worked scalar example of SPEC.md:161 (tests/golden/worked_values.json)
  B4  structure: dO = 0 -> zero gradients; gradients linear in dO; user independence
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")
PHIS = ["identity", "silu", "shifted_elu"]


def grid(rng, shape, lo=-128, hi=128, den=32.0):
    return (rng.integers(lo, hi, size=shape).astype(np.float32) / np.float32(den))


def _case(seed, lens, S=3, H=2, d=4, q_per_user=False):
    rng = np.random.default_rng(seed)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    B = len(lens)
    q = grid(rng, (B, S, H, d) if q_per_user else (S, H, d))
    k = grid(rng, (off[-1], H, d))
    v = grid(rng, (off[-1], H, d))
    g = grid(rng, (B, S, H, d))
    return q, k, v, off, g


def _t_act(kind, x):
    if kind == "identity":
        return x
    if kind == "silu":
        return torch.nn.functional.silu(x)
    return torch.where(x >= 1.0, x, torch.exp(x - 1.0))


def _torch_grads(q, k, v, off, g, phi1, phi2, normalize, q_per_user):
    qt = torch.tensor(q, dtype=torch.float64, requires_grad=True)
    kt = torch.tensor(k, dtype=torch.float64, requires_grad=True)
    vt = torch.tensor(v, dtype=torch.float64, requires_grad=True)
    gt = torch.tensor(g, dtype=torch.float64)
    loss = 0.0
    B = len(off) - 1
    H = k.shape[1]
    for u in range(B):
        a, b = int(off[u]), int(off[u + 1])
        n = b - a
        qu = qt[u] if q_per_user else qt
        for h in range(H):
            z = _t_act(phi1, kt[a:b, h]).T @ vt[a:b, h]
            if normalize and n > 0:
                z = z / n
            o = _t_act(phi1, qu[:, h]) @ _t_act(phi2, z)
            loss = loss + (o * gt[u, :, h]).sum()
    loss.backward()
    return qt.grad.numpy(), kt.grad.numpy(), vt.grad.numpy()


@pytest.mark.parametrize("phi1", PHIS)
@pytest.mark.parametrize("phi2", PHIS)
@pytest.mark.parametrize("normalize", [True, False])
def test_b1_qla_backward_vs_torch_autograd(phi1, phi2, normalize):
    q, k, v, off, g = _case(hash((phi1, phi2, normalize)) % 1000, [5, 0, 3, 1])
    dq, dk, dv = oracle.qla_backward(q, k, v, off, g, phi1, phi2, normalize)
    tq, tk, tv = _torch_grads(q, k, v, off, g, phi1, phi2, normalize, False)
    np.testing.assert_allclose(dq, tq, rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(dk, tk, rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(dv, tv, rtol=1e-11, atol=1e-12)


def test_b1_per_user_seeds_vs_torch_autograd():
    q, k, v, off, g = _case(7, [4, 2], q_per_user=True)
    dq, dk, dv = oracle.qla_backward(q, k, v, off, g, "silu", "shifted_elu", True, q_per_user=True)
    tq, tk, tv = _torch_grads(q, k, v, off, g, "silu", "shifted_elu", True, True)
    np.testing.assert_allclose(dq, tq, rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(dk, tk, rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(dv, tv, rtol=1e-11, atol=1e-12)


def _np_act(kind, x):
    if kind == "identity":
        return x
    if kind == "silu":
        return x / (1.0 + np.exp(-x))
    return np.where(x >= 1.0, x, np.exp(x - 1.0))


def _np_loss(q, k, v, off, g, phi1, phi2, normalize):
    tot = 0.0
    for u in range(len(off) - 1):
        a, b = off[u], off[u + 1]
        for h in range(k.shape[1]):
            z = _np_act(phi1, k[a:b, h]).T @ v[a:b, h]
            if normalize and b > a:
                z = z / (b - a)
            tot += np.sum((_np_act(phi1, q[:, h]) @ _np_act(phi2, z)) * g[u, :, h])
    return tot


@pytest.mark.parametrize("phi1,phi2,normalize", [("silu", "silu", True), ("shifted_elu", "identity", False),
                                                 ("silu", "shifted_elu", True)])
def test_b2_qla_backward_vs_finite_differences(phi1, phi2, normalize):
    q, k, v, off, g = _case(11, [3, 2], S=2, H=1, d=3)
    dq, dk, dv = oracle.qla_backward(q, k, v, off, g, phi1, phi2, normalize)
    args = [q.astype(np.float64), k.astype(np.float64), v.astype(np.float64)]
    eps = 1e-6
    for which, ana in zip(range(3), (dq, dk, dv)):
        num = np.zeros_like(args[which])
        it = np.nditer(args[which], flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            plus = [a.copy() for a in args]
            minus = [a.copy() for a in args]
            plus[which][idx] += eps
            minus[which][idx] -= eps
            num[idx] = (_np_loss(*plus[:3], off, g, phi1, phi2, normalize) -
                        _np_loss(*minus[:3], off, g, phi1, phi2, normalize)) / (2 * eps)
        np.testing.assert_allclose(ana, num, rtol=1e-6, atol=1e-7)


def test_b3_golden_scalar_backward():
    for e in json.load(open(GOLDEN))["qla_backward_scalar"]:
        q = np.array([[[e["q"]]]], np.float32)
        k = np.array([[[e["k"]]]], np.float32)
        v = np.array([[[e["v"]]]], np.float32)
        g = np.array([[[[e["dout"]]]]], np.float32)
        dq, dk, dv = oracle.qla_backward(q, k, v, [0, 1], g, e["phi1"], e["phi2"], e["normalize"])
        assert dq.item() == e["dq"] and dk.item() == e["dk"] and dv.item() == e["dv"], e["cite"]


def test_b4_zero_and_linear_in_dout():
    q, k, v, off, g = _case(3, [4, 3])
    z = oracle.qla_backward(q, k, v, off, np.zeros_like(g), "silu", "silu", True)
    assert all(np.all(x == 0) for x in z)
    a = oracle.qla_backward(q, k, v, off, g, "silu", "silu", True)
    b = oracle.qla_backward(q, k, v, off, 2 * g, "silu", "silu", True)
    for x, y in zip(a, b):
        np.testing.assert_allclose(y, 2 * x, rtol=1e-13, atol=1e-14)


def test_b4_user_independence():
    q, k, v, off, g = _case(5, [4, 3])
    _, dk, dv = oracle.qla_backward(q, k, v, off, g, "silu", "silu", True)
    _, dk1, dv1 = oracle.qla_backward(q, k[4:], v[4:], [0, 3], g[1:], "silu", "silu", True)
    np.testing.assert_array_equal(dk[4:], dk1)
    np.testing.assert_array_equal(dv[4:], dv1)


# ----------------------------------------------------------------------------- softmax backward
def _torch_softmax_grads(q, k, v, off, g, scale, q_per_user):
    qt = torch.tensor(q, dtype=torch.float64, requires_grad=True)
    kt = torch.tensor(k, dtype=torch.float64, requires_grad=True)
    vt = torch.tensor(v, dtype=torch.float64, requires_grad=True)
    gt = torch.tensor(g, dtype=torch.float64)
    loss = 0.0
    for u in range(len(off) - 1):
        a, b = int(off[u]), int(off[u + 1])
        if b == a:
            continue
        qu = qt[u] if q_per_user else qt
        for h in range(k.shape[1]):
            att = torch.softmax(scale * qu[:, h] @ kt[a:b, h].T, dim=-1)
            loss = loss + ((att @ vt[a:b, h]) * gt[u, :, h]).sum()
    loss.backward()
    z = lambda t: t.grad.numpy() if t.grad is not None else np.zeros(t.shape)
    return z(qt), z(kt), z(vt)


@pytest.mark.parametrize("q_per_user", [False, True])
def test_b1_softmax_backward_vs_torch_autograd(q_per_user):
    q, k, v, off, g = _case(31, [6, 0, 3, 1], q_per_user=q_per_user)
    dq, dk, dv = oracle.softmax_backward(q, k, v, off, g, scale=0.7, q_per_user=q_per_user)
    tq, tk, tv = _torch_softmax_grads(q, k, v, off, g, 0.7, q_per_user)
    np.testing.assert_allclose(dq, tq, rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(dk, tk, rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(dv, tv, rtol=1e-11, atol=1e-12)


def test_b2_softmax_backward_vs_finite_differences():
    q, k, v, off, g = _case(32, [3, 2], S=2, H=1, d=3)
    dq, dk, dv = oracle.softmax_backward(q, k, v, off, g, scale=0.5)
    args = [q.astype(np.float64), k.astype(np.float64), v.astype(np.float64)]

    def loss(qq, kk, vv):
        tot = 0.0
        for u in range(len(off) - 1):
            a, b = off[u], off[u + 1]
            s = 0.5 * qq[:, 0] @ kk[a:b, 0].T
            p = np.exp(s - s.max(axis=1, keepdims=True))
            p /= p.sum(axis=1, keepdims=True)
            tot += np.sum((p @ vv[a:b, 0]) * g[u, :, 0])
        return tot
    eps = 1e-6
    for which, ana in zip(range(3), (dq, dk, dv)):
        num = np.zeros_like(args[which])
        it = np.nditer(args[which], flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            pl = [a.copy() for a in args]
            mi = [a.copy() for a in args]
            pl[which][idx] += eps
            mi[which][idx] -= eps
            num[idx] = (loss(*pl) - loss(*mi)) / (2 * eps)
        np.testing.assert_allclose(ana, num, rtol=1e-6, atol=1e-8)


def test_b4_softmax_backward_single_key_and_zero():
    """One key: softmax = 1 so dV = sum_i dO_i, dK = dQ = 0 (dS = p (dP - D) = 0); dO = 0 -> 0."""
    q, k, v, off, g = _case(33, [1], S=3, H=1, d=4)
    dq, dk, dv = oracle.softmax_backward(q, k, v, off, g, scale=1.0)
    np.testing.assert_allclose(dv[0, 0], g[0, :, 0].astype(np.float64).sum(axis=0), rtol=1e-14, atol=1e-14)
    assert np.all(np.abs(dk) < 1e-15) and np.all(np.abs(dq) < 1e-15)
    z = oracle.softmax_backward(q, k, v, off, np.zeros_like(g))
    assert all(np.all(x == 0) for x in z)
