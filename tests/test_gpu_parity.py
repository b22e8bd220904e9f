"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle on the same seeded
inputs.  Gate (reading R14): per (user, head) block
    max|gpu - oracle| / max|oracle| <= 2e-2 (bf16 inputs) or 1e-4 (f32 inputs)
and |lse_gpu - lse_oracle| <= 1e-3 (bf16) / 1e-5 (f32), natural log.
"""
import os

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = {"bf16": (2e-2, 1e-3), "f32": (1e-4, 1e-5)}


def to_dev(x, dtype):
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return t.to(torch.bfloat16) if dtype == "bf16" else t.float()


def block_err(g, o):
    den = np.abs(o).max()
    return np.abs(g - o).max() / den if den > 0 else np.abs(g).max()


def check_softmax(out, lse, ref, ref_lse, lens, dtype, rows=None):
    tol, ltol = TOL[dtype]
    g = out.float().cpu().numpy().astype(np.float64)
    gl = lse.cpu().numpy().astype(np.float64)
    if rows is not None:
        g = g[:, rows]
        gl = gl[:, :, rows]
    B, _, H, _ = ref.shape
    worst = 0.0
    for u in range(B):
        for h in range(H):
            if lens[u] == 0:
                assert np.all(g[u, :, h] == 0) and np.all(gl[u, h] == -np.inf)
                continue
            e = block_err(g[u, :, h], ref[u, :, h])
            worst = max(worst, e)
            assert e <= tol, f"user {u} head {h}: rel err {e:.3g} > {tol}"
            le = np.abs(gl[u, h] - ref_lse[u, h]).max()
            assert le <= ltol, f"user {u} head {h}: lse err {le:.3g}"
    return worst


def run_case(vista, lens, S, H, d, dtype="bf16", tau=1, category=False, seed=0, attn=None, **kw):
    q, k, v, off = synth.make_batch(lens, S, H, d, dtype=dtype, seed=seed, tau=tau, category=category)
    qt, kt, vt = to_dev(q, dtype), to_dev(k, dtype), to_dev(v, dtype)
    ot = torch.from_numpy(off).cuda()
    res = vista.summarize(qt, kt, vt, ot, int(off[-1]), attn=vista.SOFTMAX if attn is None else attn,
                          out_dtype=vista.F32, **kw)
    torch.cuda.synchronize()
    return (q, k, v, off), res


EDGE_LENS = [0, 1, 127, 128, 129, 300, 1000, 0, 2049, 5]


@pytest.mark.parametrize("S", [128, 256, 384, 512])
def test_softmax_tcgen05_jagged_edges(cuda_lib, S):
    vista = cuda_lib
    assert vista.vista_dispatch_name(vista.make_desc(1, S, 2, 128)) == "sm100_softmax"
    (q, k, v, off), (out, lse) = run_case(vista, EDGE_LENS, S, 2, 128, tau=2, seed=S)
    ref, ref_lse = oracle.softmax_summarize(q, k, v, off)
    check_softmax(out, lse, ref, ref_lse, EDGE_LENS, "bf16")


@pytest.mark.parametrize("tau,category", [(4, False), (1, True), (4, True)])
def test_softmax_tcgen05_peaky_and_category(cuda_lib, tau, category):
    lens = [10_000, 3000, 129]
    (q, k, v, off), (out, lse) = run_case(cuda_lib, lens, 256, 1, 128, tau=tau, category=category, seed=7)
    ref, ref_lse = oracle.softmax_summarize(q, k, v, off)
    check_softmax(out, lse, ref, ref_lse, lens, "bf16")


def test_softmax_many_users_split_across_ctas(cuda_lib):
    """More users than SMs with power-law lengths: exercises stream-K splits and the slot merge."""
    rng = np.random.default_rng(3)
    lens = np.minimum((1.0 / (1e-3 - rng.random(300) * (1e-3 - 1e-5))).astype(np.int64), 40_000)
    lens[::37] = 0
    S, H = 256, 1
    (q, k, v, off), (out, lse) = run_case(cuda_lib, lens, S, H, 128, seed=11)
    rows = np.array([0, 77, 128, 255])
    ref, ref_lse = oracle.softmax_summarize(q, k, v, off, rows=rows)
    check_softmax(out, lse, ref, ref_lse, lens, "bf16", rows=rows)


def test_softmax_c1_fp32_simt(cuda_lib):
    vista = cuda_lib
    cfg = synth.CONFIGS["c1"]
    lens = synth.user_lengths("c1")
    assert vista.vista_dispatch_name(vista.make_desc(1, 16, 1, 32, in_dtype=vista.F32)) == "simt_softmax"
    (q, k, v, off), (out, lse) = run_case(vista, lens, cfg["S"], cfg["H"], cfg["d"], dtype="f32", seed=0)
    ref, ref_lse = oracle.softmax_summarize(q, k, v, off)
    check_softmax(out, lse, ref, ref_lse, lens, "f32")


@pytest.mark.parametrize("d,dtype,S", [(64, "bf16", 256), (128, "bf16", 100), (32, "f32", 33), (128, "f32", 64)])
def test_softmax_simt_shapes(cuda_lib, d, dtype, S):
    lens = [0, 1, 33, 500]
    (q, k, v, off), (out, lse) = run_case(cuda_lib, lens, S, 2, d, dtype=dtype, tau=2, seed=d + S)
    ref, ref_lse = oracle.softmax_summarize(q, k, v, off)
    check_softmax(out, lse, ref, ref_lse, lens, dtype)


def test_softmax_c2_full_size_sampled_rows(cuda_lib):
    """BASELINE config 2 at full size (64 users x 10k items, S=256, H=4) in the bench's launch
    configuration; sampled rows of sampled users checked one by one against the oracle."""
    vista = cuda_lib
    cfg = synth.CONFIGS["c2"]
    lens = synth.user_lengths("c2")
    S, H, d = cfg["S"], cfg["H"], cfg["d"]
    q, K, V, off = synth.make_batch(lens, S, H, d, backend="torch", device="cuda")
    ot = torch.from_numpy(off).cuda()
    out, lse = vista.summarize(q, K, V, ot, int(off[-1]), out_dtype=vista.BF16)
    torch.cuda.synchronize()
    users = [0, 31, 63]
    rows = np.array([0, 1, 127, 128, 200, 255])
    qn = q.float().cpu().numpy()
    for u in users:
        a, b = int(off[u]), int(off[u + 1])
        kn = K[a:b].float().cpu().numpy()
        vn = V[a:b].float().cpu().numpy()
        ref, ref_lse = oracle.softmax_summarize(qn, kn, vn, [0, b - a], rows=rows)
        check_softmax(out[u:u + 1], lse[u:u + 1], ref, ref_lse, [b - a], "bf16", rows=rows)


@pytest.mark.parametrize("phi1,phi2,normalize", [("silu", "silu", True), ("shifted_elu", "identity", False),
                                                 ("identity", "identity", True), ("shifted_elu", "shifted_elu", True),
                                                 ("silu", "identity", False)])
def test_qla_tcgen05(cuda_lib, phi1, phi2, normalize):
    vista = cuda_lib
    assert vista.vista_dispatch_name(vista.make_desc(1, 256, 2, 128, attn=vista.QLA)) == "sm100_qla"
    lens = EDGE_LENS
    (q, k, v, off), (out, _) = run_case(vista, lens, 256, 2, 128, seed=5, attn=vista.QLA, phi1=phi1, phi2=phi2,
                                        normalize=normalize)
    ref = oracle.qla_summarize(q, k, v, off, phi1, phi2, normalize)
    g = out.cpu().numpy()
    for u in range(len(lens)):
        for h in range(2):
            e = block_err(g[u, :, h], ref[u, :, h])
            assert e <= 2e-2, f"user {u} head {h} ({phi1},{phi2},{normalize}): {e:.3g}"


@pytest.mark.parametrize("phi1,phi2", [("silu", "silu"), ("shifted_elu", "identity")])
def test_qla_simt_fp32(cuda_lib, phi1, phi2):
    vista = cuda_lib
    lens = [1024, 0, 7]
    (q, k, v, off), (out, _) = run_case(vista, lens, 16, 1, 32, dtype="f32", seed=2, attn=vista.QLA, phi1=phi1,
                                        phi2=phi2)
    ref = oracle.qla_summarize(q, k, v, off, phi1, phi2, True)
    g = out.cpu().numpy()
    for u in range(3):
        assert block_err(g[u, :, 0], ref[u, :, 0]) <= 1e-4


def test_qla_state_split_across_ctas(cuda_lib):
    vista = cuda_lib
    lens = [200_000, 128, 70_001]
    (q, k, v, off), (out, _) = run_case(vista, lens, 256, 1, 128, seed=9, attn=vista.QLA)
    ref = oracle.qla_summarize(q, k, v, off, "silu", "silu", True)
    g = out.cpu().numpy()
    for u in range(3):
        assert block_err(g[u, :, 0], ref[u, :, 0]) <= 2e-2


@pytest.mark.parametrize("attn", ["softmax", "qla"])
def test_partial_merge_equals_oracle(cuda_lib, attn):
    """History-length shards (the multi-GPU split-L path, run here shard by shard on one GPU):
    partial on each shard, stack, merge -> oracle of the unsplit history."""
    vista = cuda_lib
    a = vista.SOFTMAX if attn == "softmax" else vista.QLA
    lens = np.array([3000, 0, 129, 1001])
    S, H, d = 256, 2, 128
    q, k, v, off = synth.make_batch(lens, S, H, d, seed=21, tau=2)
    P = 3
    parts_o, parts_l = [], []
    qt = to_dev(q, "bf16")
    for p in range(P):
        # shard p = p-th contiguous third of every user's history
        sl = [(int(off[u] + lens[u] * p // P), int(off[u] + lens[u] * (p + 1) // P)) for u in range(len(lens))]
        ks = np.concatenate([k[x:y] for x, y in sl]) if sum(y - x for x, y in sl) else np.zeros((0, H, d), np.float32)
        vs = np.concatenate([v[x:y] for x, y in sl]) if sum(y - x for x, y in sl) else np.zeros((0, H, d), np.float32)
        soff = synth.offsets_from_lengths([y - x for x, y in sl])
        po, pl = vista.summarize_partial(qt, to_dev(ks, "bf16"), to_dev(vs, "bf16"), torch.from_numpy(soff).cuda(),
                                         int(soff[-1]), attn=a)
        parts_o.append(po)
        parts_l.append(pl)
    po = torch.stack(parts_o)
    pl = torch.stack(parts_l) if a == vista.SOFTMAX else None
    ulen = torch.from_numpy(lens).cuda()
    out, lse = vista.summarize_merge(po, pl, q=qt, attn=a, user_len=ulen, out_dtype=vista.F32)
    torch.cuda.synchronize()
    if a == vista.SOFTMAX:
        ref, ref_lse = oracle.softmax_summarize(q, k, v, off)
        check_softmax(out, lse, ref, ref_lse, lens, "bf16")
    else:
        ref = oracle.qla_summarize(q, k, v, off)
        g = out.cpu().numpy()
        for u in range(len(lens)):
            for h in range(H):
                assert block_err(g[u, :, h], ref[u, :, h]) <= 2e-2


def test_determinism_and_invariants(cuda_lib):
    vista = cuda_lib
    lens = [5000, 777, 0, 12_000]
    q, k, v, off = synth.make_batch(lens, 256, 2, 128, seed=31)
    qt, kt, vt = to_dev(q, "bf16"), to_dev(k, "bf16"), to_dev(v, "bf16")
    ot = torch.from_numpy(off).cuda()
    o1, l1 = vista.summarize(qt, kt, vt, ot, int(off[-1]), out_dtype=vista.F32)
    o2, l2 = vista.summarize(qt, kt, vt, ot, int(off[-1]), out_dtype=vista.F32)
    assert torch.equal(o1, o2) and torch.equal(l1, l2)          # bitwise deterministic
    # item permutation within each user (no positional term): same result within tolerance
    perm = np.concatenate([off[u] + np.random.default_rng(u).permutation(lens[u]) for u in range(len(lens))])
    o3, l3 = vista.summarize(qt, kt[perm], vt[perm], ot, int(off[-1]), out_dtype=vista.F32)
    # constant V -> output equals that constant
    vc = torch.zeros_like(vt) + vt[:1]
    o4, _ = vista.summarize(qt, kt, vc, ot, int(off[-1]), out_dtype=vista.F32)
    torch.cuda.synchronize()
    for u in (0, 1, 3):
        assert block_err(o3[u].cpu().numpy(), o1[u].cpu().numpy()) <= 2e-2
        assert (l3[u] - l1[u]).abs().max().item() <= 1e-3
        np.testing.assert_allclose(o4[u].cpu().numpy(), np.broadcast_to(vc[0].float().cpu().numpy(), o4[u].shape),
                                   rtol=2e-2, atol=2e-2)


def test_gpu_generator_matches_numpy(cuda_lib):
    q, k, v, off = synth.make_batch([100, 0, 300], 8, 2, 128, seed=4, category=True)
    qt, kt, vt, _ = synth.make_batch([100, 0, 300], 8, 2, 128, seed=4, category=True, backend="torch", device="cuda")
    assert np.array_equal(k, kt.float().cpu().numpy()) and np.array_equal(v, vt.float().cpu().numpy())
    assert np.array_equal(q, qt.float().cpu().numpy())


@pytest.mark.parametrize("attn", ["softmax", "qla"])
def test_per_user_seeds_and_bf16_out(cuda_lib, attn):
    """q_user_stride != 0 (personalized seeds, reading R12) and bf16 output."""
    vista = cuda_lib
    lens = [700, 0, 129]
    S, H, d = 256, 2, 128
    B = len(lens)
    q = synth.make_q(S, H, d, seed=13, users=B, tau=2)
    _, k, v, off = synth.make_batch(lens, S, H, d, seed=13)
    qt, kt, vt = to_dev(q, "bf16"), to_dev(k, "bf16"), to_dev(v, "bf16")
    a = vista.SOFTMAX if attn == "softmax" else vista.QLA
    out, lse = vista.summarize(qt, kt, vt, torch.from_numpy(off).cuda(), int(off[-1]), attn=a, out_dtype=vista.BF16)
    torch.cuda.synchronize()
    if attn == "softmax":
        ref, ref_lse = oracle.softmax_summarize(q, k, v, off, q_per_user=True)
        check_softmax(out, lse, ref, ref_lse, lens, "bf16")
    else:
        ref = oracle.qla_summarize(q, k, v, off, q_per_user=True)
        g = out.float().cpu().numpy()
        for u in range(B):
            for h in range(H):
                assert block_err(g[u, :, h], ref[u, :, h]) <= 2e-2


def test_qla_c2_full_size_sampled_users(cuda_lib):
    """QLA at BASELINE config 2 size (bench launch configuration), three users checked."""
    vista = cuda_lib
    cfg = synth.CONFIGS["c2"]
    lens = synth.user_lengths("c2")
    S, H, d = cfg["S"], cfg["H"], cfg["d"]
    q, K, V, off = synth.make_batch(lens, S, H, d, backend="torch", device="cuda")
    out, _ = vista.summarize(q, K, V, torch.from_numpy(off).cuda(), int(off[-1]), attn=vista.QLA, out_dtype=vista.BF16)
    torch.cuda.synchronize()
    qn = q.float().cpu().numpy()
    for u in (0, 40, 63):
        a, b = int(off[u]), int(off[u + 1])
        ref = oracle.qla_summarize(qn, K[a:b].float().cpu().numpy(), V[a:b].float().cpu().numpy(), [0, b - a])
        g = out[u].float().cpu().numpy()
        for h in range(H):
            assert block_err(g[:, h], ref[0, :, h]) <= 2e-2


def test_c5_full_size_sampled(cuda_lib):
    """BASELINE config 5 (1,024 power-law users, S=512) at full size: the longest user, a median
    one and the shortest, sampled rows of both 256-row groups, against the oracle."""
    vista = cuda_lib
    cfg = synth.CONFIGS["c5"]
    lens = synth.user_lengths("c5")
    S, H, d = cfg["S"], cfg["H"], cfg["d"]
    q, K, V, off = synth.make_batch(lens, S, H, d, backend="torch", device="cuda")
    out, lse = vista.summarize(q, K, V, torch.from_numpy(off).cuda(), int(off[-1]), out_dtype=vista.BF16)
    torch.cuda.synchronize()
    rows = np.array([0, 255, 256, 511])
    qn = q.float().cpu().numpy()
    order = np.argsort(lens)
    for u in (int(order[-1]), int(order[len(order) // 2]), int(order[0])):
        a, b = int(off[u]), int(off[u + 1])
        ref, ref_lse = oracle.softmax_summarize(qn, K[a:b].float().cpu().numpy(), V[a:b].float().cpu().numpy(),
                                                [0, b - a], rows=rows)
        check_softmax(out[u:u + 1], lse[u:u + 1], ref, ref_lse, [b - a], "bf16", rows=rows)


def test_c4_partial_shards_full_size(cuda_lib):
    """BASELINE config 4 (8 users x 1M items): by_length split into 8 shards run on this GPU one
    after another (the multi-GPU split-L data flow without NCCL), merged, sampled rows checked."""
    vista = cuda_lib
    cfg = synth.CONFIGS["c4"]
    lens = synth.user_lengths("c4")
    S, H, d = cfg["S"], cfg["H"], cfg["d"]
    from paper_2510_22049_b200 import dist as vdist
    world = 8
    cuts = vdist.partition_by_length(lens, world)
    off_all = synth.offsets_from_lengths(lens)
    q = synth.make_q(S, H, d, backend="torch", device="cuda")
    parts_o, parts_l = [], []
    for g in range(world):
        seg_len = cuts[g + 1] - cuts[g]
        soff = synth.offsets_from_lengths(seg_len)
        rows = torch.cat([torch.arange(int(off_all[u] + cuts[g, u]), int(off_all[u] + cuts[g + 1, u]), device="cuda")
                          for u in range(len(lens))])
        users = synth.row_users(torch.from_numpy(off_all).cuda(), rows, backend="torch")
        k, v = synth.make_kv(rows, users, H, d, backend="torch", device="cuda")
        po, pl = vista.summarize_partial(q, k.contiguous(), v.contiguous(), torch.from_numpy(soff).cuda(), int(soff[-1]))
        parts_o.append(po)
        parts_l.append(pl)
        del k, v
    out, lse = vista.summarize_merge(torch.stack(parts_o), torch.stack(parts_l), q=q, out_dtype=vista.F32)
    torch.cuda.synchronize()
    u = 3
    a, b = int(off_all[u]), int(off_all[u + 1])
    rows_u = torch.arange(a, b, device="cuda")
    k, v = synth.make_kv(rows_u, torch.full_like(rows_u, u), H, d, backend="torch", device="cuda")
    sel = np.array([0, 200])
    ref, ref_lse = oracle.softmax_summarize(q.float().cpu().numpy(), k.float().cpu().numpy(), v.float().cpu().numpy(),
                                            [0, b - a], rows=sel)
    check_softmax(out[u:u + 1], lse[u:u + 1], ref, ref_lse, [b - a], "bf16", rows=sel)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_int8_export_bit_exact(cuda_lib, dtype):
    """NEXT-1: the CUDA quantizer takes the same float32 decisions as the oracle -> identical codes,
    scales and zero points (bit-exact) on seeded rows, incl. a constant row and a zero row."""
    vista = cuda_lib
    q, k, v, off = synth.make_batch([1000], 8, 1, 128, dtype=dtype, seed=17)
    x = np.concatenate([k[:, 0, :], v[:, 0, :]]).astype(np.float32)
    x[3] = 0.0
    x[4] = x[4, 0]
    codes, scale, zp = oracle.quantize_rows_int8(x)
    gc, gs, gz = vista.quantize_int8(to_dev(x, dtype))
    torch.cuda.synchronize()
    assert np.array_equal(gc.cpu().numpy(), codes)
    assert np.array_equal(gs.cpu().numpy(), scale) and np.array_equal(gz.cpu().numpy(), zp)


def test_int8_export_of_summary_tokens(cuda_lib):
    """Summarize -> export: dequantized tokens stay within scale/2 of the exported bf16 tokens and
    within the bf16 parity gate of the oracle summary."""
    vista = cuda_lib
    lens = [3000, 129]
    (q, k, v, off), (out, lse) = run_case(vista, lens, 256, 2, 128, seed=19)
    codes, scale, zp = vista.quantize_int8(out)
    torch.cuda.synchronize()
    deq = codes.float() * scale[..., None] + zp[..., None]
    assert torch.all((deq - out).abs() <= scale[..., None] * 0.5 * (1 + 1e-5) + 1e-6)
    ref, _ = oracle.softmax_summarize(q, k, v, off)
    g = deq.cpu().numpy().astype(np.float64)
    for u in range(len(lens)):
        for h in range(2):
            assert block_err(g[u, :, h], ref[u, :, h]) <= 2e-2


# ----------------------------------------------------------------------------- shared key prefix (R18)
def _prefix_inputs(lens, P, S, H, d, dtype="bf16", seed=0):
    q, k, v, off = synth.make_batch(lens, S, H, d, dtype=dtype, seed=seed, tau=2)
    _, kp, vp, _ = synth.make_batch([P], S, H, d, dtype=dtype, seed=seed + 1000)
    return q, k, v, off, kp, vp


@pytest.mark.parametrize("S,H,d,dtype,P", [(256, 2, 128, "bf16", 300), (256, 1, 128, "bf16", 1),
                                          (33, 2, 64, "f32", 17)])
def test_softmax_prefix(cuda_lib, S, H, d, dtype, P):
    vista = cuda_lib
    lens = [0, 129, 2049, 5]
    q, k, v, off, kp, vp = _prefix_inputs(lens, P, S, H, d, dtype, seed=S + P)
    out, lse = vista.summarize(to_dev(q, dtype), to_dev(k, dtype), to_dev(v, dtype), torch.from_numpy(off).cuda(),
                               int(off[-1]), out_dtype=vista.F32, k_prefix=to_dev(kp, dtype),
                               v_prefix=to_dev(vp, dtype))
    torch.cuda.synchronize()
    ref, ref_lse = oracle.softmax_summarize(q, k, v, off, k_prefix=kp, v_prefix=vp)
    check_softmax(out, lse, ref, ref_lse, [n + P for n in lens], dtype)


@pytest.mark.parametrize("phi1,phi2,normalize", [("silu", "silu", True), ("shifted_elu", "identity", False)])
def test_qla_prefix(cuda_lib, phi1, phi2, normalize):
    vista = cuda_lib
    lens = [0, 129, 2049, 5]
    P, S, H, d = 200, 256, 2, 128
    q, k, v, off, kp, vp = _prefix_inputs(lens, P, S, H, d, seed=3)
    out, _ = vista.summarize(to_dev(q, "bf16"), to_dev(k, "bf16"), to_dev(v, "bf16"), torch.from_numpy(off).cuda(),
                             int(off[-1]), attn=vista.QLA, phi1=phi1, phi2=phi2, normalize=normalize,
                             out_dtype=vista.F32, k_prefix=to_dev(kp, "bf16"), v_prefix=to_dev(vp, "bf16"))
    torch.cuda.synchronize()
    ref = oracle.qla_summarize(q, k, v, off, phi1, phi2, normalize, k_prefix=kp, v_prefix=vp)
    g = out.cpu().numpy()
    for u in range(len(lens)):
        for h in range(H):
            assert block_err(g[u, :, h], ref[u, :, h]) <= 2e-2, (u, h)


@pytest.mark.parametrize("attn", ["softmax", "qla"])
def test_prefix_partial_then_merge(cuda_lib, attn):
    """Split-L with a prefix: the prefix goes to exactly one shard's partial call."""
    vista = cuda_lib
    lens = [3000, 0, 700]
    P, S, H, d = 64, 256, 1, 128
    q, k, v, off, kp, vp = _prefix_inputs(lens, P, S, H, d, seed=8)
    a = vista.SOFTMAX if attn == "softmax" else vista.QLA
    cut = [n // 2 for n in lens]
    shards = []
    for si, (lo_f, hi_f) in enumerate([(lambda u: 0, lambda u: cut[u]), (lambda u: cut[u], lambda u: lens[u])]):
        rows = np.concatenate([np.arange(off[u] + lo_f(u), off[u] + hi_f(u)) for u in range(len(lens))]).astype(np.int64)
        soff = synth.offsets_from_lengths([hi_f(u) - lo_f(u) for u in range(len(lens))])
        kw = dict(k_prefix=to_dev(kp, "bf16"), v_prefix=to_dev(vp, "bf16")) if si == 0 else {}
        po, pl = vista.summarize_partial(to_dev(q, "bf16"), to_dev(k[rows], "bf16"), to_dev(v[rows], "bf16"),
                                         torch.from_numpy(soff).cuda(), int(soff[-1]), attn=a, **kw)
        shards.append((po, pl))
    po = torch.stack([s[0] for s in shards])
    pl = torch.stack([s[1] for s in shards]) if attn == "softmax" else None
    ulen = torch.tensor([n + P for n in lens], dtype=torch.int64, device="cuda")
    out, lse = vista.summarize_merge(po, pl, q=to_dev(q, "bf16"), attn=a, user_len=ulen, out_dtype=vista.F32)
    torch.cuda.synchronize()
    if attn == "softmax":
        ref, ref_lse = oracle.softmax_summarize(q, k, v, off, k_prefix=kp, v_prefix=vp)
        check_softmax(out, lse, ref, ref_lse, [n + P for n in lens], "bf16")
    else:
        ref = oracle.qla_summarize(q, k, v, off, k_prefix=kp, v_prefix=vp)
        g = out.cpu().numpy()
        for u in range(len(lens)):
            assert block_err(g[u, :, 0], ref[u, :, 0]) <= 2e-2


def test_prefix_requires_shared_seeds(cuda_lib):
    vista = cuda_lib
    d = vista.make_desc(2, 256, 1, 128, q_user_stride=256 * 128)
    P = 4
    n = 1 << 20
    buf = torch.empty(n, dtype=torch.uint8, device="cuda")
    with pytest.raises(vista.VistaError) as e:
        vista.vista_summarize_fwd_prefix(d, buf, buf, buf, buf, 0, buf, buf, P, buf, None, buf, n)
    assert "UNSUPPORTED" in str(e.value)


# ----------------------------------------------------------------------------- QLA backward (NEXT-2)
def _bwd_check(g, ref, tol, what):
    g = g.float().cpu().numpy().astype(np.float64) if hasattr(g, "cpu") else g
    den = np.abs(ref).max()
    e = np.abs(g - ref).max() / (den if den > 0 else 1.0)
    assert e <= tol, f"{what}: rel err {e:.3g} > {tol}"


@pytest.mark.parametrize("phi1,phi2,normalize", [("silu", "silu", True), ("shifted_elu", "identity", False),
                                                 ("identity", "shifted_elu", True)])
def test_qla_backward_tcgen05(cuda_lib, phi1, phi2, normalize):
    vista = cuda_lib
    lens = [0, 129, 2049, 5, 300]
    S, H, d = 256, 2, 128
    q, k, v, off = synth.make_batch(lens, S, H, d, seed=21, tau=1)
    rng = np.random.default_rng(4)
    g = ((rng.integers(-128, 128, size=(len(lens), S, H, d)) / 64.0)).astype(np.float32)
    dq, dk, dv = vista.summarize_bwd(to_dev(q, "bf16"), to_dev(k, "bf16"), to_dev(v, "bf16"),
                                     torch.from_numpy(off).cuda(), int(off[-1]), to_dev(g, "bf16"),
                                     phi1=phi1, phi2=phi2, normalize=normalize)
    torch.cuda.synchronize()
    rq, rk, rv = oracle.qla_backward(q, k, v, off, g, phi1, phi2, normalize)
    _bwd_check(dq, rq, 2e-2, "dq")
    # dk / dv per user block (users' gradient scales differ by 1/N)
    dkn = dk.float().cpu().numpy()
    dvn = dv.float().cpu().numpy()
    for u in range(len(lens)):
        a, b = off[u], off[u + 1]
        if b > a:
            _bwd_check(dkn[a:b], rk[a:b], 2e-2, f"dk user {u}")
            _bwd_check(dvn[a:b], rv[a:b], 2e-2, f"dv user {u}")


@pytest.mark.parametrize("d,dtype", [(128, "bf16"), (64, "f32")])
def test_qla_backward_from_saved_state(cuda_lib, d, dtype):
    """vista_summarize_bwd_qla_saved with the forward's partial state Z == the recomputing backward,
    bit for bit (same kernels after the state), and both match the oracle."""
    vista = cuda_lib
    lens = [0, 129, 2049, 5, 300]
    S, H = 256, 2
    q, k, v, off = synth.make_batch(lens, S, H, d, seed=22, tau=1)
    rng = np.random.default_rng(7)
    g = ((rng.integers(-128, 128, size=(len(lens), S, H, d)) / 64.0)).astype(np.float32)
    qt, kt, vt, gt = to_dev(q, dtype), to_dev(k, dtype), to_dev(v, dtype), to_dev(g, dtype)
    ot = torch.from_numpy(off).cuda()
    z, _ = vista.summarize_partial(qt, kt, vt, ot, int(off[-1]), attn=vista.QLA)
    a = vista.summarize_bwd(qt, kt, vt, ot, int(off[-1]), gt, z=z)
    b = vista.summarize_bwd(qt, kt, vt, ot, int(off[-1]), gt)
    torch.cuda.synchronize()
    for x, y, what in zip(a, b, ("dq", "dk", "dv")):
        assert torch.equal(x, y), what
    rq, rk, rv = oracle.qla_backward(q, k, v, off, g, "silu", "silu", True)
    tol = 1e-4 if dtype == "f32" else 2e-2
    _bwd_check(a[0], rq, tol, "dq")
    dkn = a[1].float().cpu().numpy()
    for u in range(len(lens)):
        lo, hi = off[u], off[u + 1]
        if hi > lo:
            _bwd_check(dkn[lo:hi], rk[lo:hi], tol, f"dk user {u}")


@pytest.mark.parametrize("d,dtype", [(32, "f32"), (64, "bf16"), (128, "f32")])
def test_qla_backward_simt(cuda_lib, d, dtype):
    vista = cuda_lib
    lens = [100, 0, 33]
    S, H = 16, 2
    q, k, v, off = synth.make_batch(lens, S, H, d, dtype=dtype, seed=d, tau=1)
    rng = np.random.default_rng(5)
    g = ((rng.integers(-128, 128, size=(len(lens), S, H, d)) / 64.0)).astype(np.float32)
    dq, dk, dv = vista.summarize_bwd(to_dev(q, dtype), to_dev(k, dtype), to_dev(v, dtype),
                                     torch.from_numpy(off).cuda(), int(off[-1]), to_dev(g, dtype),
                                     phi1="silu", phi2="silu", normalize=True)
    torch.cuda.synchronize()
    rq, rk, rv = oracle.qla_backward(q, k, v, off, g, "silu", "silu", True)
    tol = 1e-4 if dtype == "f32" else 2e-2
    _bwd_check(dq, rq, tol, "dq")
    dkn, dvn = dk.float().cpu().numpy(), dv.float().cpu().numpy()
    for u in range(len(lens)):
        a, b = off[u], off[u + 1]
        if b > a:
            _bwd_check(dkn[a:b], rk[a:b], tol, f"dk user {u}")
            _bwd_check(dvn[a:b], rv[a:b], tol, f"dv user {u}")


def test_qla_backward_per_user_seeds(cuda_lib):
    vista = cuda_lib
    lens = [700, 3]
    S, H, d = 128, 1, 128
    rng = np.random.default_rng(6)
    q = ((rng.integers(-128, 128, size=(len(lens), S, H, d)) / 64.0)).astype(np.float32)
    _, k, v, off = synth.make_batch(lens, S, H, d, seed=6)
    g = ((rng.integers(-128, 128, size=(len(lens), S, H, d)) / 64.0)).astype(np.float32)
    dq, dk, dv = vista.summarize_bwd(to_dev(q, "bf16"), to_dev(k, "bf16"), to_dev(v, "bf16"),
                                     torch.from_numpy(off).cuda(), int(off[-1]), to_dev(g, "bf16"))
    torch.cuda.synchronize()
    rq, rk, rv = oracle.qla_backward(q, k, v, off, g, "silu", "silu", True, q_per_user=True)
    for u in range(len(lens)):
        _bwd_check(dq[u], rq[u], 2e-2, f"dq user {u}")


# ----------------------------------------------------------------------------- softmax backward (NEXT-2)
@pytest.mark.parametrize("S,H,lens,per_user", [(256, 2, [0, 1, 127, 129, 300, 2049, 5], False),
                                               (128, 1, [10_000, 3, 640], False),
                                               (256, 1, [700, 129], True),
                                               (512, 1, [0, 1500, 129, 3], False),
                                               (384, 2, [260, 1], True),
                                               (128, 2, [50, 0, 131, 7, 256, 1, 90, 3, 129, 64, 1], False)])
def test_softmax_backward_tcgen05(cuda_lib, S, H, lens, per_user):
    vista = cuda_lib
    d = 128
    rng = np.random.default_rng(S + len(lens))
    q, k, v, off = synth.make_batch(lens, S, H, d, seed=41, tau=1)
    if per_user:
        q = ((rng.integers(-128, 128, size=(len(lens), S, H, d)) / 64.0)).astype(np.float32)
    g = ((rng.integers(-128, 128, size=(len(lens), S, H, d)) / 64.0)).astype(np.float32)
    qt, kt, vt = to_dev(q, "bf16"), to_dev(k, "bf16"), to_dev(v, "bf16")
    ot = torch.from_numpy(off).cuda()
    out, lse = vista.summarize(qt, kt, vt, ot, int(off[-1]), out_dtype=vista.BF16)
    dq, dk, dv = vista.summarize_bwd(qt, kt, vt, ot, int(off[-1]), to_dev(g, "bf16"), attn=vista.SOFTMAX,
                                     out=out, lse=lse)
    torch.cuda.synchronize()
    rq, rk, rv = oracle.softmax_backward(q, k, v, off, g, q_per_user=per_user)
    if per_user:
        for u in range(len(lens)):
            if lens[u]:
                _bwd_check(dq[u], rq[u], 2e-2, f"dq user {u}")
    else:
        _bwd_check(dq, rq, 2e-2, "dq")
    dkn, dvn = dk.float().cpu().numpy(), dv.float().cpu().numpy()
    for u in range(len(lens)):
        a, b = off[u], off[u + 1]
        if b > a:
            _bwd_check(dkn[a:b], rk[a:b], 2e-2, f"dk user {u}")
            _bwd_check(dvn[a:b], rv[a:b], 2e-2, f"dv user {u}")


@pytest.mark.parametrize("S,H,d,dtype,out_dtype,per_user", [(200, 1, 128, "bf16", "bf16", False),
                                                             (16, 2, 32, "f32", "f32", False),
                                                             (64, 1, 64, "bf16", "f32", True),
                                                             (1100, 1, 128, "bf16", "bf16", False)])
def test_softmax_backward_simt(cuda_lib, S, H, d, dtype, out_dtype, per_user):
    """Shapes outside the tcgen05 backward (S % 128 != 0, f32, d < 128, f32 dout, S > 1024): the
    CUDA-core path, against the oracle."""
    vista = cuda_lib
    lens = [300, 0, 17, 129]
    rng = np.random.default_rng(S + d)
    q, k, v, off = synth.make_batch(lens, S, H, d, seed=43, tau=1)
    if per_user:
        q = ((rng.integers(-128, 128, size=(len(lens), S, H, d)) / 64.0)).astype(np.float32)
    g = ((rng.integers(-128, 128, size=(len(lens), S, H, d)) / 64.0)).astype(np.float32)
    qt, kt, vt = to_dev(q, dtype), to_dev(k, dtype), to_dev(v, dtype)
    ot = torch.from_numpy(off).cuda()
    odt = vista.BF16 if out_dtype == "bf16" else vista.F32
    out, lse = vista.summarize(qt, kt, vt, ot, int(off[-1]), out_dtype=odt)
    dq, dk, dv = vista.summarize_bwd(qt, kt, vt, ot, int(off[-1]), to_dev(g, out_dtype), attn=vista.SOFTMAX,
                                     out=out, lse=lse)
    torch.cuda.synchronize()
    rq, rk, rv = oracle.softmax_backward(q, k, v, off, g, q_per_user=per_user)
    tol = 1e-4 if (dtype == "f32" and out_dtype == "f32") else 2e-2
    if per_user:
        for u in range(len(lens)):
            if lens[u]:
                _bwd_check(dq[u], rq[u], tol, f"dq user {u}")
    else:
        _bwd_check(dq, rq, tol, "dq")
    dkn, dvn = dk.float().cpu().numpy(), dv.float().cpu().numpy()
    for u in range(len(lens)):
        a, b = off[u], off[u + 1]
        if b > a:
            _bwd_check(dkn[a:b], rk[a:b], tol, f"dk user {u}")
            _bwd_check(dvn[a:b], rv[a:b], tol, f"dv user {u}")


# ----------------------------------------------------------------------------- NEXT-1 fused export
@pytest.mark.parametrize("S,H,out_bf16,attn", [(256, 2, True, "softmax"), (512, 1, True, "softmax"),
                                               (256, 1, False, "softmax"), (256, 2, True, "qla")])
def test_int8_export_fused_equals_separate(cuda_lib, S, H, out_bf16, attn):
    """vista_summarize_fwd_int8 (fused into the softmax epilogue / slot merge / empty-user fill on
    the tcgen05 path, a separate pass otherwise) == vista_quantize_rows_int8 of the output == the
    oracle's quantizer applied to that output, bit for bit; many users force stream-K splits."""
    vista = cuda_lib
    rng = np.random.default_rng(S + H)
    lens = [int(x) for x in rng.integers(0, 3000, size=160)]
    lens[3] = 0
    lens[10] = 129
    d = 128
    q, k, v, off = synth.make_batch(lens, S, H, d, seed=23)
    qt, kt, vt = to_dev(q, "bf16"), to_dev(k, "bf16"), to_dev(v, "bf16")
    ot = torch.from_numpy(off).cuda()
    a = vista.SOFTMAX if attn == "softmax" else vista.QLA
    desc = vista.make_desc(len(lens), S, H, d, in_dtype=vista.BF16, out_dtype=vista.BF16 if out_bf16 else vista.F32,
                           attn=a)
    total = int(off[-1])
    need = vista.vista_summarize_workspace_size(desc, total)
    ws = torch.empty(max(need, 16), dtype=torch.uint8, device="cuda")
    B = len(lens)
    out = torch.empty((B, S, H, d), dtype=torch.bfloat16 if out_bf16 else torch.float32, device="cuda")
    lse = torch.empty((B, H, S), dtype=torch.float32, device="cuda") if attn == "softmax" else None
    codes = torch.empty((B, S, H, d), dtype=torch.int8, device="cuda")
    sc = torch.empty((B, S, H), dtype=torch.float32, device="cuda")
    zp = torch.empty((B, S, H), dtype=torch.float32, device="cuda")
    vista.vista_summarize_fwd_int8(desc, qt, kt, vt, ot, total, out, lse, codes, sc, zp, ws, need)
    c2, s2, z2 = vista.quantize_int8(out)
    torch.cuda.synchronize()
    assert torch.equal(codes, c2.view(codes.shape)), "codes"
    assert torch.equal(sc, s2.view(sc.shape)) and torch.equal(zp, z2.view(zp.shape)), "scale / zero point"
    rc, rs, rz = oracle.quantize_rows_int8(out.float().cpu().numpy().reshape(-1, d))
    assert np.array_equal(codes.cpu().numpy().reshape(-1, d), rc)
    assert np.array_equal(sc.cpu().numpy().reshape(-1), rs) and np.array_equal(zp.cpu().numpy().reshape(-1), rz)


# ----------------------------------------------------------------------------- QLA at per-user rows (NEXT-3/4)
def _rows_case(lens, rows, H, d, dtype, seed, delta):
    rng = np.random.default_rng(seed)
    _, k, v, off = synth.make_batch(lens, 1, H, d, seed=seed)
    roff = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
    R = int(roff[-1])
    q = ((rng.integers(-128, 128, size=(R, H, d)) / 64.0)).astype(np.float32)
    ks = vs = None
    if delta:
        ks = ((rng.integers(-128, 128, size=(R, H, d)) / 64.0)).astype(np.float32)
        vs = ((rng.integers(-128, 128, size=(R, H, d)) / 64.0)).astype(np.float32)
    return q, roff, k, v, off, ks, vs


def _rows_check(vista, lens, rows, H, d, dtype, seed, delta, phi1, phi2, normalize, out_dtype, tol):
    q, roff, k, v, off, ks, vs = _rows_case(lens, rows, H, d, dtype, seed, delta)
    dev = lambda x: None if x is None else to_dev(x, dtype)  # noqa: E731
    out = vista.qla_rows(dev(k), dev(v), torch.from_numpy(off).cuda(), int(off[-1]), dev(q),
                         torch.from_numpy(roff).cuda(), int(roff[-1]), k_self=dev(ks), v_self=dev(vs), phi1=phi1,
                         phi2=phi2, normalize=normalize, out_dtype=out_dtype)
    torch.cuda.synchronize()
    ref = oracle.qla_rows(q, roff, k, v, off, phi1, phi2, normalize, k_self=ks, v_self=vs)
    g = out.float().cpu().numpy()
    for u in range(len(lens)):
        a, b = roff[u], roff[u + 1]
        for h in range(H):
            if b > a:
                e = block_err(g[a:b, h], ref[a:b, h])
                assert e <= tol, f"user {u} head {h} ({phi1},{phi2},{normalize},delta={delta}): {e:.3g}"


@pytest.mark.parametrize("phi1,phi2,normalize,delta", [("silu", "silu", True, False), ("silu", "silu", True, True),
                                                       ("shifted_elu", "identity", False, True),
                                                       ("identity", "shifted_elu", True, False)])
def test_qla_rows_tcgen05(cuda_lib, phi1, phi2, normalize, delta):
    """History rows (no Delta) and target rows (Delta) against the oracle: ragged rows per user
    (empty, 1, tile tails, several tiles), users without history, bf16 and f32 out."""
    vista = cuda_lib
    lens = [300, 0, 129, 2049, 5, 1]
    rows = [130, 3, 0, 257, 1, 128]
    for out_dtype in (vista.BF16, vista.F32):
        _rows_check(vista, lens, rows, 2, 128, "bf16", 61, delta, phi1, phi2, normalize, out_dtype, 2e-2)


def test_qla_rows_history_rows_are_the_histories(cuda_lib):
    """NEXT-3 form: every history item as a query row of its own user (rows = offsets), many units
    per CTA so the stream-K ranges split users."""
    vista = cuda_lib
    lens = [5000, 1, 0, 777, 12_000]
    _rows_check(vista, lens, lens, 1, 128, "bf16", 62, False, "silu", "silu", True, vista.BF16, 2e-2)


@pytest.mark.parametrize("d,dtype", [(32, "f32"), (64, "bf16"), (128, "f32")])
def test_qla_rows_simt(cuda_lib, d, dtype):
    vista = cuda_lib
    tol = 1e-4 if dtype == "f32" else 2e-2
    _rows_check(vista, [40, 0, 3], [5, 2, 7], 2, d, dtype, 63, True, "silu", "silu", True, None, tol)


# ----------------------------------------------------------------------------- full-size sampled (NEXT-2..4)
def _c2_full():
    cfg = synth.CONFIGS["c2"]
    lens = synth.user_lengths("c2")
    S, H, d = cfg["S"], cfg["H"], cfg["d"]
    q, K, V, off = synth.make_batch(lens, S, H, d, backend="torch", device="cuda")
    return lens, S, H, d, q, K, V, off


@pytest.mark.parametrize("attn", ["softmax", "qla"])
def test_backward_c2_full_size_sampled_users(cuda_lib, attn):
    """The backward at BASELINE config 2 size in the bench's launch configuration (softmax from the
    forward's out / lse, QLA from the forward's saved state); dK, dV of three users against the
    oracle run on those users alone (their gradients depend on their own history only)."""
    vista = cuda_lib
    lens, S, H, d, q, K, V, off = _c2_full()
    ot = torch.from_numpy(off).cuda()
    rng = np.random.default_rng(11)
    g = ((rng.integers(-128, 128, size=(len(lens), S, H, d)) / 64.0)).astype(np.float32)
    gt = torch.from_numpy(g).cuda().to(torch.bfloat16)
    if attn == "softmax":
        out, lse = vista.summarize(q, K, V, ot, int(off[-1]), out_dtype=vista.BF16)
        dq, dk, dv = vista.summarize_bwd(q, K, V, ot, int(off[-1]), gt, attn=vista.SOFTMAX, out=out, lse=lse)
    else:
        z, _ = vista.summarize_partial(q, K, V, ot, int(off[-1]), attn=vista.QLA)
        dq, dk, dv = vista.summarize_bwd(q, K, V, ot, int(off[-1]), gt, z=z)
    torch.cuda.synchronize()
    qn = q.float().cpu().numpy()
    for u in (0, 40, 63):
        a, b = int(off[u]), int(off[u + 1])
        kn, vn = K[a:b].float().cpu().numpy(), V[a:b].float().cpu().numpy()
        if attn == "softmax":
            _, rk, rv = oracle.softmax_backward(qn, kn, vn, [0, b - a], g[u:u + 1])
        else:
            _, rk, rv = oracle.qla_backward(qn, kn, vn, [0, b - a], g[u:u + 1])
        _bwd_check(dk[a:b], rk, 2e-2, f"{attn} dk user {u}")
        _bwd_check(dv[a:b], rv, 2e-2, f"{attn} dv user {u}")


def test_qla_rows_c2_full_size_sampled_users(cuda_lib):
    """QLA history rows (NEXT-3) at config 2 size, bench launch configuration; three users' rows."""
    vista = cuda_lib
    lens, S, H, d, q, K, V, off = _c2_full()
    ot = torch.from_numpy(off).cuda()
    rng = np.random.default_rng(12)
    qr = ((rng.integers(-128, 128, size=(int(off[-1]), H, d)) / 64.0)).astype(np.float32)
    out = vista.qla_rows(K, V, ot, int(off[-1]), torch.from_numpy(qr).cuda().to(torch.bfloat16), ot, int(off[-1]),
                         out_dtype=vista.BF16)
    torch.cuda.synchronize()
    for u in (0, 40, 63):
        a, b = int(off[u]), int(off[u + 1])
        ref = oracle.qla_rows(qr[a:b], [0, b - a], K[a:b].float().cpu().numpy(), V[a:b].float().cpu().numpy(),
                              [0, b - a])
        gq = out[a:b].float().cpu().numpy()
        for h in range(H):
            assert block_err(gq[:, h], ref[:, h]) <= 2e-2, f"user {u} head {h}"


def test_qla_rows_edge_cases(cuda_lib):
    """No history at all (Z = 0 for every user: out = phi1(q) phi2(0) + Delta), no rows at all, and
    a single row."""
    vista = cuda_lib
    for phi2 in ("silu", "shifted_elu"):
        _rows_check(vista, [0, 0, 0], [3, 0, 129], 2, 128, "bf16", 64, True, "silu", phi2, True, vista.F32, 2e-2)
    _rows_check(vista, [70, 2], [0, 1], 1, 128, "bf16", 65, False, "silu", "silu", True, vista.BF16, 2e-2)
    k = torch.zeros((5, 1, 128), dtype=torch.bfloat16, device="cuda")
    off = torch.tensor([0, 5], dtype=torch.int64, device="cuda")
    q = torch.zeros((0, 1, 128), dtype=torch.bfloat16, device="cuda")
    out = vista.qla_rows(k, k, off, 5, q, torch.tensor([0, 0], dtype=torch.int64, device="cuda"), 0)
    assert out.shape == (0, 1, 128)


# ----------------------------------------------------------------------------- invariants / robustness (SURVEY §4 tier 3)
def test_int8_exact_ties_bit_exact(cuda_lib):
    """DESIGN.md R21 on the GPU: exact .5 ties (stored scale 1, zero point 0) round half to even, the
    same codes as the oracle, through the separate quantizer and the bf16 path."""
    vista = cuda_lib
    x = np.zeros((4, 128), np.float32)
    x[:, :2] = [-127.0, 127.0]
    x[:, 2:12] = [0.5, 1.5, 2.5, 3.5, -0.5, -1.5, -2.5, -3.5, 126.5, -126.5]
    want = np.zeros(128, np.int8)
    want[:12] = [-127, 127, 0, 2, 2, 4, 0, -2, -2, -4, 126, -126]
    rc, rs, rz = oracle.quantize_rows_int8(x)
    for dtype in ("bf16", "f32"):
        gc, gs, gz = vista.quantize_int8(to_dev(x, dtype))
        torch.cuda.synchronize()
        assert np.array_equal(gc.cpu().numpy(), rc) and np.all(rc == want[None])
        assert np.all(gs.cpu().numpy() == 1.0) and np.all(gz.cpu().numpy() == 0.0)


def _grid8(rng, shape, lo=-8, hi=9):
    return (rng.integers(lo, hi, size=shape) / 8.0).astype(np.float32)


def test_softmax_key_shift_large_logits(cuda_lib):
    """Key shift K + 1 c^T (c = 8 in every channel, values exact in bf16): every row's logits move by
    the constant scale q.c (~ +1000 with scale 1 and positive seeds), so O is unchanged and
    lse moves by scale q.c.  Exercises the first-tile rescale of the online softmax with huge
    logits; checked against the oracle on the shifted inputs and against the unshifted GPU run."""
    vista = cuda_lib
    rng = np.random.default_rng(71)
    lens, S, H, d = [3000, 1, 129, 700], 256, 1, 128
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    q = (rng.integers(0, 17, size=(S, H, d)) / 8.0).astype(np.float32)   # >= 0: q.c ~ 8 * 128
    k = _grid8(rng, (off[-1], H, d))
    v = _grid8(rng, (off[-1], H, d)) + _grid8(rng, (1, H, d))
    ks = k + 8.0
    ot = torch.from_numpy(off).cuda()
    o0, l0 = vista.summarize(to_dev(q, "bf16"), to_dev(k, "bf16"), to_dev(v, "bf16"), ot, int(off[-1]),
                             scale=1.0, out_dtype=vista.F32)
    o1, l1 = vista.summarize(to_dev(q, "bf16"), to_dev(ks, "bf16"), to_dev(v, "bf16"), ot, int(off[-1]),
                             scale=1.0, out_dtype=vista.F32)
    torch.cuda.synchronize()
    ref, ref_lse = oracle.softmax_summarize(q, ks, v, off, scale=1.0)
    check_softmax(o1, l1, ref, ref_lse, lens, "bf16")
    shift = (q[:, 0].astype(np.float64) @ np.full(d, 8.0))  # [S]
    assert shift.min() > 500
    for u in range(len(lens)):
        assert block_err(o1[u].cpu().numpy(), o0[u].cpu().numpy()) <= 2e-2
        dl = l1[u, 0].double().cpu().numpy() - l0[u, 0].double().cpu().numpy()
        # lse is float32 near 1000: its own rounding is ~6e-5; the shift is exact in float64
        assert np.abs(dl - shift).max() <= 2e-3


def test_softmax_duplication_adds_ln2(cuda_lib):
    """Duplicating every history item leaves O unchanged and adds ln 2 to lse (P4(ii))."""
    vista = cuda_lib
    lens = [2500, 129, 1, 0]
    q, k, v, off = synth.make_batch(lens, 256, 2, 128, seed=72)
    lens2 = [2 * L for L in lens]
    off2 = np.concatenate([[0], np.cumsum(lens2)]).astype(np.int64)
    idx = np.concatenate([np.concatenate([np.arange(off[u], off[u + 1])] * 2) for u in range(len(lens))]).astype(np.int64)
    ot, ot2 = torch.from_numpy(off).cuda(), torch.from_numpy(off2).cuda()
    o1, l1 = vista.summarize(to_dev(q, "bf16"), to_dev(k, "bf16"), to_dev(v, "bf16"), ot, int(off[-1]), out_dtype=vista.F32)
    o2, l2 = vista.summarize(to_dev(q, "bf16"), to_dev(k[idx], "bf16"), to_dev(v[idx], "bf16"), ot2, int(off2[-1]),
                             out_dtype=vista.F32)
    torch.cuda.synchronize()
    for u in range(3):
        assert block_err(o2[u].cpu().numpy(), o1[u].cpu().numpy()) <= 2e-2
        assert (l2[u] - l1[u] - np.log(2.0)).abs().max().item() <= 1e-3
    assert torch.all(o2[3] == 0) and torch.all(l2[3] == -np.inf)


@pytest.mark.parametrize("attn", ["softmax", "qla"])
def test_user_and_row_independence_bitwise(cuda_lib, attn):
    """No leakage across users or seed rows: with the lengths (hence the stream-K partition) fixed,
    replacing every OTHER user's history values, or one seed row's values, leaves the remaining
    outputs bitwise unchanged (P4(iv), (v))."""
    vista = cuda_lib
    a = vista.SOFTMAX if attn == "softmax" else vista.QLA
    lens = [4000, 300, 0, 9000, 128]
    q, k, v, off = synth.make_batch(lens, 256, 2, 128, seed=73)
    ot = torch.from_numpy(off).cuda()
    run = lambda qq, kk, vv: vista.summarize(to_dev(qq, "bf16"), to_dev(kk, "bf16"), to_dev(vv, "bf16"), ot,  # noqa
                                             int(off[-1]), attn=a, out_dtype=vista.F32)
    o1, l1 = run(q, k, v)
    _, k2, v2, _ = synth.make_batch(lens, 256, 2, 128, seed=74)
    keep = slice(off[3], off[4])
    k2[keep], v2[keep] = k[keep], v[keep]
    o2, l2 = run(q, k2, v2)
    q3 = q.copy()
    q3[17] = q3[17][::-1].copy() * 0.5 + 0.25
    o3, l3 = run(q3, k, v)
    torch.cuda.synchronize()
    assert torch.equal(o1[3], o2[3])
    if attn == "softmax":
        assert torch.equal(l1[3], l2[3])
    rows = [i for i in range(256) if i != 17]
    if attn == "qla":
        assert torch.equal(o1[:, rows], o3[:, rows])
    else:
        # rows of other warps are bitwise unchanged; the 31 rows sharing row 17's warp share its
        # warp-uniform rescale decision, so their p are taken against a possibly
        # different running max: equal within rounding, not bitwise
        other = [i for i in range(256) if i // 32 != 17 // 32]
        assert torch.equal(o1[:, other], o3[:, other]) and torch.equal(l1[:, :, other], l3[:, :, other])
        for u in (0, 1, 3, 4):
            assert block_err(o3[u, rows].cpu().numpy(), o1[u, rows].cpu().numpy()) <= 1e-2


@pytest.mark.parametrize("attn", ["softmax", "qla"])
def test_all_empty_batch_and_zero_users(cuda_lib, attn):
    """Every user empty: softmax O = 0 and lse = -inf (R6); QLA O = phi1(Q) phi2(0) = 0 for SiLU.
    B = 0: a valid no-op (no launch, VISTA_OK)."""
    vista = cuda_lib
    a = vista.SOFTMAX if attn == "softmax" else vista.QLA
    q = to_dev(synth.make_q(256, 2, 128, seed=5), "bf16")
    k = torch.zeros((0, 2, 128), dtype=torch.bfloat16, device="cuda")
    off = torch.zeros(5, dtype=torch.int64, device="cuda")
    o, l = vista.summarize(q, k, k, off, 0, attn=a, out_dtype=vista.F32)
    torch.cuda.synchronize()
    assert o.shape == (4, 256, 2, 128) and torch.all(o == 0)
    if attn == "softmax":
        assert torch.all(l == -np.inf)
    o0, l0 = vista.summarize(q, k, k, torch.zeros(1, dtype=torch.int64, device="cuda"), 0, attn=a, out_dtype=vista.F32)
    torch.cuda.synchronize()
    assert o0.shape == (0, 256, 2, 128)


# ----------------------------------------------------------------------------- QLA rows from a saved state
@pytest.mark.parametrize("delta,normalize,dtype", [(True, True, "bf16"), (False, True, "bf16"), (True, False, "bf16"),
                                                   (True, True, "f32")])
def test_qla_rows_from_state(cuda_lib, delta, normalize, dtype):
    """vista_qla_rows_from_state on the state of vista_summarize_partial (QLA) and N_u = L_u gives
    the rows of vista_qla_rows bitwise (same W_u operands, same rows kernel) and matches the oracle
    (the state computed first, then multiplied with Q[S]_l, Q[T]_l)."""
    vista = cuda_lib
    lens = [300, 0, 129, 2049, 5, 1]
    rows = [130, 3, 0, 257, 1, 128]
    H, d = 2, 128 if dtype == "bf16" else 64
    q, roff, k, v, off, ks, vs = _rows_case(lens, rows, H, d, dtype, 66, delta)
    dev = lambda x: None if x is None else to_dev(x, dtype)  # noqa: E731
    kt, vt, ot, rt = dev(k), dev(v), torch.from_numpy(off).cuda(), torch.from_numpy(roff).cuda()
    seeds = dev(q[:1])  # any q: the partial state does not read it
    z, _ = vista.summarize_partial(seeds, kt, vt, ot, int(off[-1]), attn=vista.QLA, normalize=normalize)
    ulen = torch.from_numpy(np.diff(off)).cuda()
    a = vista.qla_rows_from_state(z, ulen, dev(q), rt, int(roff[-1]), k_self=dev(ks), v_self=dev(vs),
                                  normalize=normalize, out_dtype=vista.F32)
    b = vista.qla_rows(kt, vt, ot, int(off[-1]), dev(q), rt, int(roff[-1]), k_self=dev(ks), v_self=dev(vs),
                       normalize=normalize, out_dtype=vista.F32)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    ref = oracle.qla_rows(q, roff, k, v, off, "silu", "silu", normalize, k_self=ks, v_self=vs)
    g = a.cpu().numpy()
    tol = 2e-2 if dtype == "bf16" else 1e-4
    for u in range(len(lens)):
        for h in range(H):
            if roff[u + 1] > roff[u]:
                assert block_err(g[roff[u]:roff[u + 1], h], ref[roff[u]:roff[u + 1], h]) <= tol


def test_qla_target_rows_c2_full_size_from_state(cuda_lib):
    """The bench's --qla-rows target step at config 2 size: 256 target rows per user with the Delta
    term from the users' saved states; three users against the oracle."""
    vista = cuda_lib
    lens, S, H, d, q, K, V, off = _c2_full()
    ot = torch.from_numpy(off).cuda()
    B = len(lens)
    z, _ = vista.summarize_partial(q, K, V, ot, int(off[-1]), attn=vista.QLA)
    rng = np.random.default_rng(13)
    n = 256 * B
    qr, ks, vs = [(rng.integers(-128, 128, size=(n, H, d)) / 64.0).astype(np.float32) for _ in range(3)]
    roff = np.arange(B + 1, dtype=np.int64) * 256
    out = vista.qla_rows_from_state(z, torch.from_numpy(np.asarray(lens, np.int64)).cuda(), to_dev(qr, "bf16"),
                                    torch.from_numpy(roff).cuda(), n, k_self=to_dev(ks, "bf16"),
                                    v_self=to_dev(vs, "bf16"), out_dtype=vista.BF16)
    torch.cuda.synchronize()
    for u in (0, 31, 63):
        a, b = int(off[u]), int(off[u + 1])
        ref = oracle.qla_rows(qr[256 * u:256 * (u + 1)], [0, 256], K[a:b].float().cpu().numpy(),
                              V[a:b].float().cpu().numpy(), [0, b - a], k_self=ks[256 * u:256 * (u + 1)],
                              v_self=vs[256 * u:256 * (u + 1)])
        g = out[256 * u:256 * (u + 1)].float().cpu().numpy()
        for h in range(H):
            assert block_err(g[:, h], ref[:, h]) <= 2e-2, f"user {u} head {h}"


# ----------------------------------------------------------------------------- stage-2 target-aware attention (NEXT-4)
def _ta_case(rng, B, S, H, d, rows, dtype):
    codes = rng.integers(-127, 128, size=(B, S, H, d)).astype(np.int8)
    ts = (rng.integers(1, 64, size=(B, S, H)) / 1024.0).astype(np.float32)
    tz = (rng.integers(-64, 64, size=(B, S, H)) / 128.0).astype(np.float32)
    roff = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
    R = int(roff[-1])
    g = lambda: (rng.integers(-128, 128, size=(R, H, d)) / 64.0).astype(np.float32)  # noqa: E731
    return codes, ts, tz, g(), g(), g(), g(), roff


def _ta_check(vista, B, S, H, d, rows, dtype, seed, resid, out_dtype, tol, ltol):
    rng = np.random.default_rng(seed)
    codes, ts, tz, q, k, v, rs, roff = _ta_case(rng, B, S, H, d, rows, dtype)
    dev = lambda x: to_dev(x, dtype)  # noqa: E731
    out, lse = vista.target_attend(torch.from_numpy(codes).cuda(), torch.from_numpy(ts).cuda(),
                                   torch.from_numpy(tz).cuda(), dev(q), dev(k), dev(v), torch.from_numpy(roff).cuda(),
                                   resid=dev(rs) if resid else None, out_dtype=out_dtype)
    torch.cuda.synchronize()
    ref, ref_lse = oracle.target_attend(codes, ts, tz, q, k, v, roff, resid=rs if resid else None)
    g = out.float().cpu().numpy()
    # lse gate: the tensor-core path rounds the dequantized tokens to bf16 (relative 2^-9), so a logit
    # moves by at most scale * sum_e |q_e| * max |t| * 2^-9 (2^-8 with the f32 accumulation slack)
    t = codes.astype(np.float64) * ts[..., None] + tz[..., None]
    tmax = np.abs(t).max(axis=(1, 3))  # [B, H]
    for u in range(B):
        a, b = roff[u], roff[u + 1]
        for h in range(H):
            if b > a:
                e = block_err(g[a:b, h], ref[a:b, h])
                assert e <= tol, f"user {u} head {h}: {e:.3g}"
                bound = np.abs(q[a:b, h]).sum(-1) * tmax[u, h] * 2.0 ** -8 / np.sqrt(d) if dtype == "bf16" else 0.0
                assert np.all(np.abs(lse[a:b, h].cpu().numpy() - ref_lse[a:b, h]) <= ltol + bound)
    return out


@pytest.mark.parametrize("S,resid,out_bf16", [(256, False, True), (128, True, False), (256, True, True)])
def test_target_attend_tcgen05(cuda_lib, S, resid, out_bf16):
    """Ragged candidates per user (none, 1, a tile tail, several tiles), int8 tokens dequantized in
    the load path, the self key / value, an optional residual; bf16 and f32 out."""
    vista = cuda_lib
    _ta_check(vista, 5, S, 2, 128, [130, 0, 1, 300, 128], "bf16", 81, resid, vista.BF16 if out_bf16 else vista.F32,
              2e-2, 1e-3)


@pytest.mark.parametrize("S,d,dtype", [(17, 64, "bf16"), (256, 128, "f32"), (40, 32, "f32")])
def test_target_attend_simt(cuda_lib, S, d, dtype):
    vista = cuda_lib
    tol, ltol = (1e-4, 1e-5) if dtype == "f32" else (2e-2, 1e-3)
    _ta_check(vista, 3, S, 2, d, [5, 0, 9], dtype, 82, True, vista.F32, tol, ltol)


@pytest.mark.gpu
def test_target_attend_wide_logit_range(cuda_lib):
    """A token far above the row's first scores (here ~775 log2 units): the one-pass softmax's
    provisional offset would overflow, so the kernel must take its fallback (the row max, the pass
    again) and still match the oracle."""
    vista = cuda_lib
    rng = np.random.default_rng(85)
    B, S, H, d = 3, 256, 2, 128
    codes, ts, tz, q, k, v, rs, roff = _ta_case(rng, B, S, H, d, [130, 1, 256], "bf16")
    q = np.abs(q) * 0.5 + 0.5  # positive queries: the special tokens score high for every candidate
    codes[:, 100] = 127
    ts[:, 100] = 0.5
    tz[:, 100] = 0.0
    dev = lambda x: to_dev(x, "bf16")  # noqa: E731
    out, lse = vista.target_attend(torch.from_numpy(codes).cuda(), torch.from_numpy(ts).cuda(),
                                   torch.from_numpy(tz).cuda(), dev(q), dev(k), dev(v), torch.from_numpy(roff).cuda())
    torch.cuda.synchronize()
    ref, ref_lse = oracle.target_attend(codes, ts, tz, q, k, v, roff)
    g = out.float().cpu().numpy()
    assert np.all(np.isfinite(g)) and np.all(np.isfinite(lse.cpu().numpy()))
    for u in range(B):
        a, b = roff[u], roff[u + 1]
        for h in range(H):
            assert block_err(g[a:b, h], ref[a:b, h]) <= 2e-2
            # the logits are ~1e3 (natural units): the bf16 token rounding moves them by <= 2^-8 relative
            assert np.all(np.abs(lse[a:b, h].cpu().numpy() - ref_lse[a:b, h]) <= 2.0 ** -8 * np.abs(ref_lse[a:b, h]) + 1e-3)


def test_target_attend_candidate_independence_bitwise(cuda_lib):
    """PAPER.md:156 "the candidates cannot attend each other": a candidate's output is bitwise the same
    whatever the other candidates of the batch (here: their values replaced), on the tcgen05 path."""
    vista = cuda_lib
    rng = np.random.default_rng(83)
    codes, ts, tz, q, k, v, rs, roff = _ta_case(rng, 2, 256, 2, 128, [200, 57], "bf16")
    q2, k2, v2 = q.copy(), k.copy(), v.copy()
    keep = [3, 150, 230]
    others = np.setdiff1d(np.arange(257), keep)
    q2[others] = -q2[others]
    k2[others] = 0.5 * k2[others]
    v2[others] = v2[others][::-1]
    args = lambda qq, kk, vv: (torch.from_numpy(codes).cuda(), torch.from_numpy(ts).cuda(),  # noqa: E731
                               torch.from_numpy(tz).cuda(), to_dev(qq, "bf16"), to_dev(kk, "bf16"), to_dev(vv, "bf16"),
                               torch.from_numpy(roff).cuda())
    o1, l1 = vista.target_attend(*args(q, k, v), out_dtype=vista.F32)
    o2, l2 = vista.target_attend(*args(q2, k2, v2), out_dtype=vista.F32)
    torch.cuda.synchronize()
    assert torch.equal(o1[keep], o2[keep]) and torch.equal(l1[keep], l2[keep])


def test_target_attend_reads_the_summarize_int8_export(cuda_lib):
    """Stage 1 -> export -> stage 2 on the device: vista_summarize_fwd_int8's codes / scales feed
    vista_target_attend directly; checked against the oracle applied to the same exported codes."""
    vista = cuda_lib
    lens = [3000, 129, 700]
    S, H, d = 256, 2, 128
    q, k, v, off = synth.make_batch(lens, S, H, d, seed=84)
    qt, kt, vt = to_dev(q, "bf16"), to_dev(k, "bf16"), to_dev(v, "bf16")
    ot = torch.from_numpy(off).cuda()
    B = len(lens)
    desc = vista.make_desc(B, S, H, d, in_dtype=vista.BF16, out_dtype=vista.BF16)
    need = vista.vista_summarize_workspace_size(desc, int(off[-1]))
    ws = torch.empty(max(need, 16), dtype=torch.uint8, device="cuda")
    out = torch.empty((B, S, H, d), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((B, H, S), dtype=torch.float32, device="cuda")
    codes = torch.empty((B, S, H, d), dtype=torch.int8, device="cuda")
    sc = torch.empty((B, S, H), dtype=torch.float32, device="cuda")
    zp = torch.empty((B, S, H), dtype=torch.float32, device="cuda")
    vista.vista_summarize_fwd_int8(desc, qt, kt, vt, ot, int(off[-1]), out, lse, codes, sc, zp, ws, need)
    rng = np.random.default_rng(85)
    rows = [64, 200, 1]
    roff = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
    cq, ck, cv = [(rng.integers(-128, 128, size=(int(roff[-1]), H, d)) / 64.0).astype(np.float32) for _ in range(3)]
    o, l = vista.target_attend(codes, sc, zp, to_dev(cq, "bf16"), to_dev(ck, "bf16"), to_dev(cv, "bf16"),
                               torch.from_numpy(roff).cuda(), out_dtype=vista.F32)
    torch.cuda.synchronize()
    ref, _ = oracle.target_attend(codes.cpu().numpy(), sc.cpu().numpy(), zp.cpu().numpy(), cq, ck, cv, roff)
    g = o.cpu().numpy()
    for u in range(B):
        for h in range(H):
            assert block_err(g[roff[u]:roff[u + 1], h], ref[roff[u]:roff[u + 1], h]) <= 2e-2


# ----------------------------------------------------------------------------- multi-layer summarizer (NEXT-3)
def _layers_case(rng, lens, S, H, n_layers, d=128):
    D = H * d
    off = np.concatenate([[0], np.cumsum([S + L for L in lens])]).astype(np.int64)
    x = ((rng.integers(-128, 128, size=(int(off[-1]), D)) / 64.0)).astype(np.float32)
    # weights ~ U(-1, 1) / sqrt(D) / 2: activations stay O(1) through the layers (with twice that
    # scale they grow ~10^4-fold over three layers and bf16 rounding of the intermediates dominates)
    W = (rng.integers(-128, 128, size=(n_layers, 5, D, D)) / (128.0 * np.sqrt(D))).astype(np.float32)
    return x, off, W


@pytest.mark.parametrize("lens,S,H,n_layers", [([300, 0, 1000], 128, 1, 3), ([129, 2000], 256, 2, 2)])
def test_summarize_layers(cuda_lib, lens, S, H, n_layers):
    """3 (2) summarizer layers (projections, QLA over [seeds; history], SGLU, output projection,
    residual) on tcgen05 against the float64 oracle of the per-layer definition: the tokens (each
    user's first S rows) and every updated row, per (user, head-column block)."""
    vista = cuda_lib
    rng = np.random.default_rng(91)
    x, off, W = _layers_case(rng, lens, S, H, n_layers)
    xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
    x_bf = xt.float().cpu().numpy()  # the bf16-rounded input the GPU sees
    Wt = torch.from_numpy(W).cuda().to(torch.bfloat16)
    W_bf = Wt.float().cpu().numpy()
    tok = vista.summarize_layers(xt, torch.from_numpy(off).cuda(), Wt, S, H, out_dtype=vista.F32)
    torch.cuda.synchronize()
    ref = oracle.summarize_layers(x_bf, off, W_bf, S, H)
    g = xt.float().cpu().numpy()
    d = 128
    for u in range(len(lens)):
        a, b = off[u], off[u + 1]
        for h in range(H):
            c = slice(h * d, (h + 1) * d)
            assert block_err(g[a:b, c], ref[a:b, c]) <= 2e-2, f"user {u} head {h}"
            assert block_err(tok[u, :, h].cpu().numpy(), ref[a:a + S, c]) <= 2e-2


@pytest.mark.gpu
def test_softmax_cta_pair_mode(cuda_lib):
    """The cta_group::2 variant of the softmax kernel (VISTA_SOFTMAX_PAIR=1, off by default; the
    switch is read once per process, so it runs in a child process): the S = 256 parity cases
    (jagged edges, peaky / category inputs, stream-K splits, c2 at full size, large-logit shift)."""
    import subprocess
    import sys
    env = dict(os.environ, VISTA_SOFTMAX_PAIR="1")
    sel = ("test_softmax_tcgen05_jagged_edges and 256 or test_softmax_tcgen05_peaky or "
           "test_softmax_many_users_split or test_softmax_c2_full_size or test_softmax_key_shift or "
           "test_softmax_duplication or test_int8_export_fused_equals_separate and 256-2")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
                        os.path.abspath(__file__), "-k", sel], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.gpu
def test_target_attend_c2_full_size_sampled_users(cuda_lib):
    """Stage 2 in the launch configuration bench.py --stage2 times (c2: 64 users x 256 int8 summary
    tokens, H = 4, 256 candidates per user, bf16): the whole batch on the GPU, the oracle on sampled
    users (candidates never see another user's tokens, so a user's block is checked alone)."""
    vista = cuda_lib
    B, S, H, d, cpu = 64, 256, 4, 128, 256
    g = torch.Generator(device="cuda")
    g.manual_seed(2024)
    codes = torch.randint(-127, 128, (B, S, H, d), device="cuda", generator=g, dtype=torch.int8)
    sc = (torch.randint(1, 64, (B, S, H), device="cuda", generator=g).float() / 1024.0)
    zp = (torch.randint(-64, 64, (B, S, H), device="cuda", generator=g).float() / 128.0)
    R = B * cpu
    grid = lambda: (torch.randint(-128, 128, (R, H, d), device="cuda", generator=g).float() / 64).to(torch.bfloat16)  # noqa
    cq, ck, cv = grid(), grid(), grid()
    roff = torch.arange(B + 1, dtype=torch.int64, device="cuda") * cpu
    o, l = vista.target_attend(codes, sc, zp, cq, ck, cv, roff, out_dtype=vista.F32)
    torch.cuda.synchronize()
    for u in (0, 17, 63):
        a, b = u * cpu, (u + 1) * cpu
        ref, rl = oracle.target_attend(codes[u:u + 1].cpu().numpy(), sc[u:u + 1].cpu().numpy(),
                                       zp[u:u + 1].cpu().numpy(), cq[a:b].float().cpu().numpy(),
                                       ck[a:b].float().cpu().numpy(), cv[a:b].float().cpu().numpy(), [0, cpu])
        go, gl = o[a:b].cpu().numpy(), l[a:b].cpu().numpy()
        for h in range(H):
            assert block_err(go[:, h], ref[:, h]) <= 2e-2, f"user {u} head {h}"
        # lse: the bf16 rounding of the dequantized tokens bounds the logit error (|q|_1 max|t| 2^-8 / sqrt(d))
        tmax = (np.abs(codes[u].float().cpu().numpy()) * sc[u].cpu().numpy()[..., None]
                + np.abs(zp[u].cpu().numpy())[..., None]).max()
        bound = np.abs(cq[a:b].float().cpu().numpy()).sum(-1) * tmax * 2.0 ** -8 / np.sqrt(d) + 1e-3
        assert np.all(np.abs(gl - rl) <= bound)


@pytest.mark.gpu
def test_summarize_layers_c2_full_size_sampled_users(cuda_lib):
    """Two summarizer layers in the launch configuration bench.py --layers times (c2: 64 users x
    [256 seeds; 10,000 items], D = 512, CTA-pair projection GEMMs): the whole batch on the GPU, the
    oracle on sampled users (layers never mix users: a user's segment is checked alone)."""
    vista = cuda_lib
    B, S, H, d, L, n_layers = 64, 256, 4, 128, 10000, 2
    D = H * d
    off = np.arange(B + 1, dtype=np.int64) * (S + L)
    g = torch.Generator(device="cuda")
    g.manual_seed(77)
    x = (torch.randint(-128, 128, (int(off[-1]), D), device="cuda", generator=g).float() / 64).to(torch.bfloat16)
    W = (torch.randint(-128, 128, (n_layers, 5, D, D), device="cuda", generator=g).float()
         / (128.0 * np.sqrt(D))).to(torch.bfloat16)
    samples = (0, 41)
    x_in = {u: x[off[u]:off[u + 1]].float().cpu().numpy() for u in samples}
    tok = vista.summarize_layers(x, torch.from_numpy(off).cuda(), W, S, H, out_dtype=vista.F32)
    torch.cuda.synchronize()
    W_bf = W.float().cpu().numpy()
    for u in samples:
        ref = oracle.summarize_layers(x_in[u], [0, S + L], W_bf, S, H)
        gx = x[off[u]:off[u + 1]].float().cpu().numpy()
        for h in range(H):
            c = slice(h * d, (h + 1) * d)
            assert block_err(gx[:, c], ref[:, c]) <= 2e-2, f"user {u} head {h}"
            assert block_err(tok[u, :, h].cpu().numpy(), ref[:S, c]) <= 2e-2


@pytest.mark.gpu
def test_qla_target_rows_from_state_c2_full_size_sampled_users(cuda_lib):
    """QLA target rows with the Delta term (NEXT-4) in the launch configuration bench.py --qla-rows
    target times: the c2 states from vista_summarize_partial (QLA), then 256 target rows per user
    through vista_qla_rows_from_state (double-buffered W_u, v_self from global); sampled users vs the
    oracle computed from the users' full histories."""
    vista = cuda_lib
    lens, S, H, d, q, K, V, off = _c2_full()
    B = len(lens)
    ot = torch.from_numpy(off).cuda()
    z, _ = vista.summarize_partial(q, K, V, ot, int(off[-1]), attn=vista.QLA)
    rpu = 256
    roff = np.arange(B + 1, dtype=np.int64) * rpu
    rng = np.random.default_rng(13)
    qr, kr, vr = [((rng.integers(-128, 128, size=(B * rpu, H, d)) / 64.0)).astype(np.float32) for _ in range(3)]
    ulen = torch.from_numpy(np.asarray(lens, dtype=np.int64)).cuda()
    dev = lambda a: torch.from_numpy(a).cuda().to(torch.bfloat16)  # noqa: E731
    out = vista.qla_rows_from_state(z, ulen, dev(qr), torch.from_numpy(roff).cuda(), B * rpu, k_self=dev(kr),
                                    v_self=dev(vr), out_dtype=vista.F32)
    torch.cuda.synchronize()
    for u in (0, 33, 63):
        a, b = int(off[u]), int(off[u + 1])
        ra, rb = int(roff[u]), int(roff[u + 1])
        ref = oracle.qla_rows(qr[ra:rb], [0, rpu], K[a:b].float().cpu().numpy(), V[a:b].float().cpu().numpy(),
                              [0, b - a], k_self=kr[ra:rb], v_self=vr[ra:rb])
        go = out[ra:rb].cpu().numpy()
        for h in range(H):
            assert block_err(go[:, h], ref[:, h]) <= 2e-2, f"user {u} head {h}"


@pytest.mark.gpu
@pytest.mark.parametrize("attn,fused", [("softmax", True), ("softmax", False), ("qla", True), ("qla", False)])
def test_peer_exchange_single_rank(cuda_lib, attn, fused):
    """The peer-memory split-L exchange (vista_exchange_*, dist.PeerExchange) at world size 1 (one
    GPU: the rank pushes into its own receive buffer): bitwise equal to merging the partial directly,
    over several steps (device epochs and acks), eagerly and replayed from a CUDA graph.  fused: the
    partial's own kernels store into the receive buffers (vista_summarize_partial_peers; the batch
    has an empty user and split units, so the empty-user fill and the slot merge store there too) --
    the buffer must hold exactly the bytes of the plain partial."""
    from paper_2510_22049_b200 import dist as vdist
    vista = cuda_lib
    lens = [700, 0, 129, 2050]
    S, H, d = 256, 2, 128
    q, k, v, off = synth.make_batch(lens, S, H, d, seed=31, backend="torch", device="cuda")
    ot = torch.from_numpy(off).cuda()
    ulen = torch.tensor(lens, dtype=torch.int64, device="cuda")
    a = vista.SOFTMAX if attn == "softmax" else vista.QLA
    be = vdist.CudaBackend()
    po, pl = be.partial(q, k, v, ot, int(off[-1]), a)
    ref_o, ref_l = be.merge(po[None], pl[None] if a == vista.SOFTMAX else None, q, a, ulen)
    ex = vdist.PeerExchange(po.shape, pl.shape if a == vista.SOFTMAX else None)
    for _ in range(3):
        o, l = vdist.summarize_by_length(q, k, v, ot, ulen, attn=attn, total_len=int(off[-1]), exchange=ex,
                                         fused=fused)
        torch.cuda.synchronize()
        assert torch.equal(o, ref_o)
        if a == vista.SOFTMAX:
            assert torch.equal(l, ref_l)
        assert torch.equal(ex.recv_o[0], po)
        if a == vista.SOFTMAX:
            assert torch.equal(ex.recv_lse[0], pl)
    assert int(ex.epoch.item()) == 3 and int(ex.acks[0].item()) == 3 and int(ex.flags[0].item()) == 3
    # captured: the epoch is a device counter, so replays advance it
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        g.capture_begin()
        o2, l2 = vdist.summarize_by_length(q, k, v, ot, ulen, attn=attn, total_len=int(off[-1]), exchange=ex,
                                           fused=fused)
        g.capture_end()
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(o2, ref_o)
    assert int(ex.epoch.item()) == 5
