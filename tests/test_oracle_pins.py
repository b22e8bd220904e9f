"""Pins of the float64 oracle against things other than itself (CPU only).

Pins:
  P1 brute force: mpmath at 50 digits on tiny instances, logit gaps up to ~80, empty users
  P2 library routine: torch scaled_dot_product_attention (float64, CPU)
  P3 closed forms: L=1, two keys (sigmoid), constant V, logit gap 50
  P4 invariants: permutation, duplication (lse + ln 2), key shift, user/row independence
  P5 split == unsplit through the oracle's own LSE merge / state sum
  Q1 QLA associativity vs the dense App. B form (QK^T)V/N
  Q2 worked values (tests/golden/worked_values.json)
  Q3 QLA invariants: linearity in V, V=0, split = sum of states, duplication with 1/N, permutation
Each pin is chosen so that a dropped term, a wrong sign/index or a transposed operand in the oracle
fails at least one of them (see test docstrings).
"""
import json
import math
import os

import mpmath
import numpy as np
import pytest
import torch

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")
mpmath.mp.dps = 50


def grid(rng, shape, lo=-128, hi=128, den=64.0):
    """Random values on the bf16-exact grid (integers / 64)."""
    return (rng.integers(lo, hi, size=shape) / den).astype(np.float32)


def mp_softmax(q, k, v, scale):
    """mpmath brute force of RowSoftmax(q K^T) V for one row."""
    s = [mpmath.mpf(scale) * mpmath.fsum(mpmath.mpf(float(a)) * mpmath.mpf(float(b)) for a, b in zip(q, kj))
         for kj in k]
    m = max(s)
    w = [mpmath.exp(x - m) for x in s]
    l = mpmath.fsum(w)
    o = [mpmath.fsum(w[j] * mpmath.mpf(float(v[j][c])) for j in range(len(k))) / l for c in range(len(q))]
    return [float(x) for x in o], float(m + mpmath.log(l))


def mp_act(kind, x):
    x = mpmath.mpf(float(x)) if not isinstance(x, mpmath.mpf) else x
    if kind == "identity":
        return x
    if kind == "silu":
        return x / (1 + mpmath.exp(-x))
    return x if x >= 1 else mpmath.exp(x - 1)


# ----------------------------------------------------------------------------- P1
@pytest.mark.parametrize("seed", range(40))
def test_p1_softmax_vs_mpmath(seed):
    """Catches: wrong max subtraction, missing 1/l, lse off by m, transposed q/k, wrong scale."""
    rng = np.random.default_rng(seed)
    B, S, H, d = 3, int(rng.integers(1, 5)), int(rng.integers(1, 3)), int(rng.integers(1, 9))
    lens = rng.integers(0, 17, size=B)
    lens[rng.integers(0, B)] = 0 if seed % 3 == 0 else lens[0]
    off = synth.offsets_from_lengths(lens)
    tau = [1, 4, 16][seed % 3]           # logit gaps up to ~80 at tau=16
    q = grid(rng, (S, H, d)) * tau
    k = grid(rng, (off[-1], H, d))
    v = grid(rng, (off[-1], H, d))
    scale = [None, 0.5, 1.0][seed % 3]
    out, lse = oracle.softmax_summarize(q, k, v, off, scale=scale)
    sc = 1.0 / math.sqrt(d) if scale is None else scale
    for u in range(B):
        for h in range(H):
            for i in range(S):
                if lens[u] == 0:
                    assert np.all(out[u, i, h] == 0) and lse[u, h, i] == -np.inf
                    continue
                kk = k[off[u]:off[u + 1], h]
                vv = v[off[u]:off[u + 1], h]
                o_ref, l_ref = mp_softmax(q[i, h], kk, vv, sc)
                np.testing.assert_allclose(out[u, i, h], o_ref, rtol=1e-13, atol=1e-13)
                assert abs(lse[u, h, i] - l_ref) <= 1e-13 * max(1.0, abs(l_ref))


# ----------------------------------------------------------------------------- P2
@pytest.mark.parametrize("L", [1, 7, 128, 129, 1000, 4096])
def test_p2_softmax_vs_torch_sdpa(L):
    """Library routine: torch SDPA in float64 on the same exact inputs."""
    rng = np.random.default_rng(L)
    S, H, d = 32, 2, 64
    q = grid(rng, (S, H, d)) * 4
    lens = np.array([L, L // 2 + 1])
    off = synth.offsets_from_lengths(lens)
    k = grid(rng, (off[-1], H, d))
    v = grid(rng, (off[-1], H, d))
    out, _ = oracle.softmax_summarize(q, k, v, off)
    for u in range(2):
        qt = torch.from_numpy(q.astype(np.float64)).permute(1, 0, 2)[None]
        kt = torch.from_numpy(k[off[u]:off[u + 1]].astype(np.float64)).permute(1, 0, 2)[None]
        vt = torch.from_numpy(v[off[u]:off[u + 1]].astype(np.float64)).permute(1, 0, 2)[None]
        ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt)[0].permute(1, 0, 2).numpy()
        np.testing.assert_allclose(out[u], ref, rtol=1e-12, atol=1e-12)


# ----------------------------------------------------------------------------- P3
def test_p3_single_key():
    """one key -> output = v and lse = scale*q.k exactly."""
    rng = np.random.default_rng(1)
    q = grid(rng, (4, 1, 8))
    k = grid(rng, (1, 1, 8))
    v = grid(rng, (1, 1, 8))
    out, lse = oracle.softmax_summarize(q, k, v, [0, 1])
    for i in range(4):
        np.testing.assert_allclose(out[0, i, 0], v[0, 0], rtol=0, atol=1e-15)
        assert abs(lse[0, 0, i] - float(np.dot(q[i, 0].astype(np.float64), k[0, 0])) / math.sqrt(8)) < 1e-14


def test_p3_two_keys_sigmoid():
    """Two keys: o = sigma(s1-s2) v1 + sigma(s2-s1) v2 (closed form of a 2-way softmax)."""
    rng = np.random.default_rng(2)
    q = grid(rng, (3, 1, 16)) * 4
    k = grid(rng, (2, 1, 16))
    v = grid(rng, (2, 1, 16))
    out, lse = oracle.softmax_summarize(q, k, v, [0, 2], scale=0.25)
    for i in range(3):
        s1 = 0.25 * float(np.dot(q[i, 0].astype(np.float64), k[0, 0]))
        s2 = 0.25 * float(np.dot(q[i, 0].astype(np.float64), k[1, 0]))
        sig = 1.0 / (1.0 + math.exp(-(s1 - s2)))
        v64 = v.astype(np.float64)
        np.testing.assert_allclose(out[0, i, 0], sig * v64[0, 0] + (1 - sig) * v64[1, 0], rtol=0, atol=1e-14)
        assert abs(lse[0, 0, i] - (max(s1, s2) + math.log1p(math.exp(-abs(s1 - s2))))) < 1e-13


def test_p3_constant_v():
    """Constant V -> output equals that constant whatever the logits (north_star invariant)."""
    rng = np.random.default_rng(3)
    q = grid(rng, (8, 2, 32)) * 4
    k = grid(rng, (500, 2, 32))
    c = grid(rng, (1, 2, 32))
    v = np.repeat(c, 500, axis=0)
    out, _ = oracle.softmax_summarize(q, k, v, [0, 123, 500])
    for u in range(2):
        for i in range(8):
            np.testing.assert_allclose(out[u, i], c[0], rtol=0, atol=1e-14)


def test_p3_logit_gap_50():
    """a logit gap of 50 selects the argmax key's v within 1e-6."""
    d = 4
    q = np.array([[[1, 0, 0, 0]]], np.float32)
    k = np.array([[[100, 0, 0, 0]], [[50, 0, 0, 0]], [[0, 1, 0, 0]]], np.float32)
    v = np.array([[[1, 2, 3, 4]], [[9, 9, 9, 9]], [[-5, 5, -5, 5]]], np.float32)
    out, _ = oracle.softmax_summarize(q, k, v, [0, 3], scale=1.0)
    assert np.max(np.abs(out[0, 0, 0] - v[0, 0])) < 1e-6


def test_p3_golden_softmax_rules_cited():
    g = json.load(open(GOLDEN))
    assert {c["case"] for c in g["softmax"]} == {"single key", "logit gap 50"}


# ----------------------------------------------------------------------------- P4
def _batch(seed, lens, S=6, H=2, d=16, tau=4):
    rng = np.random.default_rng(seed)
    off = synth.offsets_from_lengths(lens)
    return grid(rng, (S, H, d)) * tau, grid(rng, (off[-1], H, d)), grid(rng, (off[-1], H, d)), off


def test_p4_permutation_invariance():
    """No positional term (reading R5): permuting a user's items leaves O, lse."""
    q, k, v, off = _batch(4, [300])
    perm = np.random.default_rng(0).permutation(300)
    o1, l1 = oracle.softmax_summarize(q, k, v, off)
    o2, l2 = oracle.softmax_summarize(q, k[perm], v[perm], off)
    np.testing.assert_allclose(o1, o2, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(l1, l2, rtol=1e-13)


def test_p4_duplication():
    """Every item twice -> same O, lse + ln 2 (catches a missing max/normalizer pairing)."""
    q, k, v, off = _batch(5, [77])
    o1, l1 = oracle.softmax_summarize(q, k, v, off)
    o2, l2 = oracle.softmax_summarize(q, np.concatenate([k, k]), np.concatenate([v, v]), [0, 154])
    np.testing.assert_allclose(o1, o2, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(l2, l1 + math.log(2.0), rtol=0, atol=1e-12)


def test_p4_key_shift():
    """K + 1 c^T shifts every logit of row i by scale*q_i.c: O unchanged, lse + scale*q.c.
    Values chosen so the shift is exact in float32; +1000-ish logits exercise the max shift."""
    q, k, v, off = _batch(6, [50], S=4, H=1, d=8, tau=4)
    c = np.full((1, 1, 8), 8.0, np.float32)
    o1, l1 = oracle.softmax_summarize(q, k, v, off, scale=1.0)
    o2, l2 = oracle.softmax_summarize(q, k + c, v, off, scale=1.0)
    np.testing.assert_allclose(o1, o2, rtol=1e-11, atol=1e-12)
    shift = (q[:, 0].astype(np.float64) @ c[0, 0].astype(np.float64))
    np.testing.assert_allclose(l2[0, 0], l1[0, 0] + shift, rtol=1e-13)


def test_p4_user_and_row_independence():
    """A user's result does not depend on other users or on which rows are computed (bitwise)."""
    q, k, v, off = _batch(7, [40, 0, 90, 13])
    o_all, l_all = oracle.softmax_summarize(q, k, v, off)
    o_2, l_2 = oracle.softmax_summarize(q, k[40:130], v[40:130], [0, 90])
    assert np.array_equal(o_all[2], o_2[0]) and np.array_equal(l_all[2], l_2[0])
    rows = np.array([5, 1])
    o_r, l_r = oracle.softmax_summarize(q, k, v, off, rows=rows)
    assert np.array_equal(o_r, o_all[:, rows]) and np.array_equal(l_r, l_all[:, :, rows])


# ----------------------------------------------------------------------------- P5
@pytest.mark.parametrize("cuts", [[0, 0, 1, 257], [128], [1, 2, 3], [256, 256, 257], [10, 130, 200]])
def test_p5_split_equals_unsplit(cuts):
    """Split-L: partials over disjoint contiguous key ranges merged by LSE equal the unsplit
    result (the identity behind the flash-decoding merge; template SPEC.md:169-170)."""
    q, k, v, off = _batch(8, [257], S=5, H=2, d=16)
    o, l = oracle.softmax_summarize(q, k, v, off)
    bounds = [0] + list(cuts) + [257]
    po, pl = [], []
    for a, b in zip(bounds[:-1], bounds[1:]):
        oo, ll = oracle.softmax_summarize(q, k[a:b], v[a:b], [0, b - a])
        po.append(oo[0].transpose(1, 0, 2))   # [H,S,d]
        pl.append(ll[0])                      # [H,S]
    mo, ml = oracle.merge_lse(np.stack(po), np.stack(pl))
    np.testing.assert_allclose(mo.transpose(1, 0, 2), o[0], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(ml, l[0], rtol=1e-13)


def test_p5_merge_all_empty():
    mo, ml = oracle.merge_lse(np.zeros((3, 2, 4)), np.full((3, 2), -np.inf))
    assert np.all(mo == 0) and np.all(ml == -np.inf)


# ----------------------------------------------------------------------------- Q1
@pytest.mark.parametrize("normalize", [False, True])
def test_q1_qla_identity_equals_dense_appendix_form(normalize):
    """phi1=phi2=Id: O = Q (K^T V) [/N] must equal the dense App. B form (Q K^T ⊙ M) V / N with
    the all-ones source mask M (m = 0 targets), computed by numpy matmul.
    Catches a transposed state (V^T K instead of K^T V) and a missing/extra 1/N."""
    rng = np.random.default_rng(11)
    S, H, d = 7, 2, 12
    lens = [33, 1, 0, 64]
    off = synth.offsets_from_lengths(lens)
    q = grid(rng, (S, H, d))
    k = grid(rng, (off[-1], H, d))
    v = grid(rng, (off[-1], H, d))
    out = oracle.qla_summarize(q, k, v, off, "identity", "identity", normalize)
    for u in range(len(lens)):
        for h in range(H):
            Q = q[:, h].astype(np.float64)
            K = k[off[u]:off[u + 1], h].astype(np.float64)
            V = v[off[u]:off[u + 1], h].astype(np.float64)
            dense = (Q @ K.T) @ V
            if normalize and lens[u] > 0:
                dense = dense / lens[u]
            np.testing.assert_allclose(out[u, :, h], dense, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("phi1,phi2", [("silu", "silu"), ("shifted_elu", "identity"),
                                       ("silu", "identity"), ("shifted_elu", "silu"),
                                       ("identity", "silu")])
@pytest.mark.parametrize("normalize", [False, True])
def test_q1_qla_vs_mpmath(phi1, phi2, normalize):
    """Brute force of phi1(Q) phi2(phi1(K)^T V / N) at 50 digits.
    Catches phi1 applied to V (or not to K/Q), phi2 applied before summation, wrong N."""
    rng = np.random.default_rng(hash((phi1, phi2, normalize)) % 1000)
    S, d = 3, 4
    lens = [5, 2]
    off = synth.offsets_from_lengths(lens)
    q = grid(rng, (S, 1, d)) * 2
    k = grid(rng, (off[-1], 1, d)) * 2
    v = grid(rng, (off[-1], 1, d))
    out = oracle.qla_summarize(q, k, v, off, phi1, phi2, normalize)
    for u in range(2):
        K = k[off[u]:off[u + 1], 0]
        V = v[off[u]:off[u + 1], 0]
        Z = [[mpmath.fsum(mp_act(phi1, K[j, a]) * mpmath.mpf(float(V[j, b])) for j in range(lens[u]))
              for b in range(d)] for a in range(d)]
        N = lens[u] if normalize else 1
        W = [[mp_act(phi2, Z[a][b] / N) for b in range(d)] for a in range(d)]
        for i in range(S):
            ref = [float(mpmath.fsum(mp_act(phi1, q[i, 0, a]) * W[a][b] for a in range(d))) for b in range(d)]
            np.testing.assert_allclose(out[u, i, 0], ref, rtol=1e-13, atol=1e-13)


# ----------------------------------------------------------------------------- Q2
def test_q2_golden_activations():
    g = json.load(open(GOLDEN))
    for e in g["activations"]:
        assert abs(oracle.act(e["phi"], e["x"]) - e["value"]) <= e.get("tol", 0.0), e["cite"]


def test_q2_shifted_elu_continuity_at_one():
    """continuous at x = 1 from both sides."""
    for eps in (1e-9, 1e-12):
        assert abs(oracle.act("shifted_elu", 1 - eps) - 1) <= 2 * eps
        assert abs(oracle.act("shifted_elu", 1 + eps) - 1) <= 2 * eps


def test_q2_golden_qla_scalar():
    g = json.load(open(GOLDEN))
    for e in g["qla_scalar"]:
        q = np.array([[[e["q"]]]], np.float32)
        k = np.array([[[e["k"]]]], np.float32)
        v = np.array([[[e["v"]]]], np.float32)
        out = oracle.qla_summarize(q, k, v, [0, 1], e["phi1"], e["phi2"], e["normalize"])
        assert abs(out[0, 0, 0, 0] - e["value"]) <= 1e-13, e["cite"]


def test_q2_silu_scalar_brute_force():
    """SiLU scalar: silu(2) * silu(3) * 5 with phi2 = Id (25.17073522387596)."""
    q = np.array([[[2.0]]], np.float32)
    k = np.array([[[3.0]]], np.float32)
    v = np.array([[[5.0]]], np.float32)
    out = oracle.qla_summarize(q, k, v, [0, 1], "silu", "identity", False)
    ref = float(mp_act("silu", 2) * mp_act("silu", 3) * 5)
    assert abs(ref - 25.17073522387596) < 1e-14
    assert abs(out[0, 0, 0, 0] - ref) < 1e-13


# ----------------------------------------------------------------------------- Q3
def test_q3_linear_in_v_and_zero_v():
    rng = np.random.default_rng(21)
    S, H, d = 4, 1, 8
    off = np.array([0, 40])
    q = grid(rng, (S, H, d))
    k = grid(rng, (40, H, d))
    v1, v2 = grid(rng, (40, H, d)), grid(rng, (40, H, d))
    o1 = oracle.qla_summarize(q, k, v1, off, "silu", "identity")
    o2 = oracle.qla_summarize(q, k, v2, off, "silu", "identity")
    o12 = oracle.qla_summarize(q, k, v1 + v2, off, "silu", "identity")
    np.testing.assert_allclose(o12, o1 + o2, rtol=1e-12, atol=1e-13)
    for phi2 in ("identity", "silu"):
        oz = oracle.qla_summarize(q, k, np.zeros_like(v1), off, "silu", phi2)
        assert np.all(oz == 0)


def test_q3_split_is_sum_of_states_and_dup_and_perm():
    rng = np.random.default_rng(22)
    S, H, d = 4, 2, 8
    q = grid(rng, (S, H, d))
    k = grid(rng, (100, H, d))
    v = grid(rng, (100, H, d))
    z = oracle.qla_state(k, v, [0, 100], "shifted_elu")
    parts = np.stack([oracle.qla_state(k[a:b], v[a:b], [0, b - a], "shifted_elu")
                      for a, b in [(0, 0), (0, 1), (1, 60), (60, 100)]])
    np.testing.assert_allclose(oracle.merge_sum(parts), z, rtol=1e-13, atol=1e-12)
    o = oracle.qla_summarize(q, k, v, [0, 100], "shifted_elu", "silu", True)
    od = oracle.qla_summarize(q, np.concatenate([k, k]), np.concatenate([v, v]), [0, 200],
                              "shifted_elu", "silu", True)
    np.testing.assert_allclose(od, o, rtol=1e-12, atol=1e-13)
    perm = rng.permutation(100)
    op = oracle.qla_summarize(q, k[perm], v[perm], [0, 100], "shifted_elu", "silu", True)
    np.testing.assert_allclose(op, o, rtol=1e-12, atol=1e-13)


# ----------------------------------------------------------------------------- generator
def test_synth_numpy_torch_identical_and_recipe():
    for dt in ("bf16", "f32"):
        q, k, v, off = synth.make_batch([3, 0, 70], 5, 2, 16, dtype=dt, seed=9)
        qt, kt, vt, _ = synth.make_batch([3, 0, 70], 5, 2, 16, dtype=dt, seed=9, backend="torch")
        assert np.array_equal(q, qt.float().numpy())
        assert np.array_equal(k, kt.float().numpy()) and np.array_equal(v, vt.float().numpy())
    # bf16 grid values survive a bf16 round trip (exactness claim of synth/)
    q, k, v, off = synth.make_batch([3, 0, 70], 5, 2, 16, dtype="bf16", seed=9, tau=4, category=True)
    assert torch.equal(torch.from_numpy(v).bfloat16().float(), torch.from_numpy(v))
    assert torch.equal(torch.from_numpy(k).bfloat16().float(), torch.from_numpy(k))
    # seed-0 realized sizes quoted in SURVEY.md §8(d)
    assert int(synth.user_lengths("c3").sum()) == 1_859_714
    L5 = synth.user_lengths("c5")
    assert int(L5.sum()) == 6_906_453 and int(L5.max()) == 667_490


# ----------------------------------------------------------------------------- NEXT-1 int8 export
def test_quantize_error_bound_and_special_rows():
    """|dequant - x| <= scale/2 per entry (+ float32 rounding slack); all-zero row
    -> scale at the floor and codes 0; a row on the 255-point grid round-trips exactly; codes stay in
    [-127, 127] and the extremes map to -127 / +127."""
    rng = np.random.default_rng(5)
    x = rng.uniform(-3, 3, size=(64, 128)).astype(np.float32)
    x[0] = 0.0
    kk = rng.integers(-127, 128, size=128)
    kk[0], kk[1] = -127, 127
    x[1] = (kk * 0.5 + 1.0).astype(np.float32)  # zero point 1, scale 0.5: on the 255-point grid
    codes, scale, zp = oracle.quantize_rows_int8(x)
    assert codes.min() >= -127 and codes.max() <= 127
    deq = oracle.dequantize_rows_int8(codes, scale, zp)
    err = np.abs(deq - x.astype(np.float64))
    assert np.all(err <= scale[:, None] * (0.5 + 1e-5) + 1e-6)
    assert scale[0] == np.float32(1e-12) and np.all(codes[0] == 0) and np.all(deq[0] == 0)
    # grid row: max - min = 127 * 0.5 * 2 -> scale 0.5, exact round trip
    assert scale[1] == np.float32(0.5) and zp[1] == np.float32(1.0)
    assert np.array_equal(codes[1], kk) and np.array_equal(deq[1], x[1].astype(np.float64))
    r = 5
    assert codes[r, np.argmax(x[r])] == 127 and codes[r, np.argmin(x[r])] == -127


def _tie_row(d=128):
    """A row with min -127, max +127 -> stored scale exactly 1.0 and zero point exactly 0.0, so
    t = (x - zp) / s = x: the half-integers below are exact ties in float32 (R21)."""
    x = np.zeros(d, np.float32)
    x[:2] = [-127.0, 127.0]
    ties = np.array([0.5, 1.5, 2.5, 3.5, -0.5, -1.5, -2.5, -3.5, 126.5, -126.5], np.float32)
    x[2:2 + len(ties)] = ties
    want = np.zeros(d, np.int64)
    want[:2] = [-127, 127]
    want[2:2 + len(ties)] = [0, 2, 2, 4, 0, -2, -2, -4, 126, -126]  # half to even
    return x, want


def test_quantize_exact_ties_round_half_to_even():
    """R21 tie rule: an exact .5 goes to the even code (SPEC.md:342 says only "round"); values
    exact in bf16 and f32, and the stored scale / zero point are exactly 1 and 0."""
    x, want = _tie_row()
    codes, scale, zp = oracle.quantize_rows_int8(x[None])
    assert scale[0] == np.float32(1.0) and zp[0] == np.float32(0.0)
    assert np.array_equal(codes[0].astype(np.int64), want)
    # the bound with the STORED scale holds with equality at a tie (|2 - 2.5| = s/2)
    deq = oracle.dequantize_rows_int8(codes, scale, zp)
    assert np.max(np.abs(deq[0] - x)) == 0.5


def test_quantize_bound_with_stored_scale():
    """R21: the codes are decided from the stored float32 scale / zero point, so the SPEC.md:346
    bound |code s + zp - x| <= s/2 holds for the values a consumer actually dequantizes with (up to
    one float32 rounding of the dequantization itself), on rows with awkward ranges."""
    rng = np.random.default_rng(9)
    x = (rng.standard_normal((256, 128)) * rng.uniform(1e-3, 1e3, size=(256, 1))).astype(np.float32)
    codes, scale, zp = oracle.quantize_rows_int8(x)
    deq = codes.astype(np.float64) * scale.astype(np.float64)[:, None] + zp.astype(np.float64)[:, None]
    slack = np.abs(x).max(1, keepdims=True) * 2.0 ** -23
    assert np.all(np.abs(deq - x) <= scale[:, None] * 0.5 + slack)


# ----------------------------------------------------------------------------- prefix (R18)
def _prefix_case(seed, lens, P, S=5, H=2, d=8):
    rng = np.random.default_rng(seed)
    q, k, v, off = _batch(seed, lens, S=S, H=H, d=d, tau=2)
    kp = grid(rng, (P, H, d))
    vp = grid(rng, (P, H, d))
    return q, k, v, off, kp, vp


def test_prefix_softmax_is_lse_merge_of_history_and_prefix():
    """Attention over [prefix; history] == LSE merge of the history-only and prefix-only results
    (the merge is pinned separately by P5).  Covers an empty user (= prefix-only result)."""
    q, k, v, off, kp, vp = _prefix_case(21, [40, 0, 7], P=9)
    o, l = oracle.softmax_summarize(q, k, v, off, k_prefix=kp, v_prefix=vp)
    oh, lh = oracle.softmax_summarize(q, k, v, off)
    op, lp = oracle.softmax_summarize(q, kp, vp, [0, 9])
    B = len(off) - 1
    for u in range(B):
        po = np.stack([oh[u].transpose(1, 0, 2), op[0].transpose(1, 0, 2)])  # [2, H, S, d]
        pl = np.stack([lh[u], lp[0]])                                        # [2, H, S]
        mo, ml = oracle.merge_lse(po, pl)
        np.testing.assert_allclose(o[u].transpose(1, 0, 2), mo, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(l[u], ml, rtol=1e-13, atol=1e-13)


def test_prefix_softmax_single_prefix_key_empty_user_closed_form():
    """One prefix key, empty history: O = v_prefix, lse = scale q.k_prefix (P3(i) on the prefix)."""
    q, k, v, off, kp, vp = _prefix_case(22, [0], P=1, S=3, H=1, d=8)
    o, l = oracle.softmax_summarize(q, k, v, off, k_prefix=kp, v_prefix=vp, scale=0.5)
    np.testing.assert_allclose(o[0, :, 0], np.broadcast_to(vp[0, 0].astype(np.float64), (3, 8)), rtol=0, atol=1e-15)
    np.testing.assert_allclose(l[0, 0], 0.5 * (q[:, 0].astype(np.float64) @ kp[0, 0].astype(np.float64)),
                               rtol=1e-14, atol=1e-14)


@pytest.mark.parametrize("phi1,phi2,normalize", [("silu", "silu", True), ("shifted_elu", "identity", False)])
def test_prefix_qla_state_is_additive(phi1, phi2, normalize):
    """QLA over [prefix; history]: Z = Z_prefix + Z_u, N_u = P + L_u, then the finalize."""
    q, k, v, off, kp, vp = _prefix_case(23, [30, 0, 4], P=6)
    o = oracle.qla_summarize(q, k, v, off, phi1, phi2, normalize, k_prefix=kp, v_prefix=vp)
    zh = oracle.qla_state(k, v, off, phi1)
    zp = oracle.qla_state(kp, vp, [0, 6], phi1)
    o2 = oracle.qla_finalize(q, zh + zp[0][None], np.diff(off) + 6, phi1, phi2, normalize)
    np.testing.assert_allclose(o, o2, rtol=1e-12, atol=1e-12)
