"""CPU-only checks of the C-ABI library: it builds, loads, exports every symbol include/vista.h
declares, and rejects bad arguments before any launch (no GPU needed for those paths)."""
import ctypes
import math
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as ge
    ge.build()
    import paper_2510_22049_b200 as vista
    return vista.load()


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "vista.h")).read()
    return sorted(set(re.findall(r"\b(vista_[a-z_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("vista_summarize_fwd", "vista_summarize_partial", "vista_summarize_merge",
              "vista_summarize_workspace_size", "vista_abi_version", "vista_status_string"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_library_is_sm100a_only():
    import subprocess
    import paper_2510_22049_b200 as vista
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", vista.lib_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out


def test_sass_has_tcgen05_and_tma():
    import subprocess
    import paper_2510_22049_b200 as vista
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", vista.lib_path()],
                          capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass or "UTCQMMA" in sass or "UTCMMA" in sass
    assert "UTMALDG" in sass
    assert "LDTM" in sass and "STTM" in sass
    assert "HGMMA" not in sass


def test_validation_errors_before_launch(lib):
    import paper_2510_22049_b200 as vista
    d = vista.make_desc(2, 256, 1, 128)
    assert vista.vista_abi_version() == 1
    n = vista.vista_summarize_workspace_size(d, 1000)
    assert n > 0
    # bad descriptor fields
    for field, val, code in [("num_summary", 0, 2), ("num_users", -1, 2), ("head_dim", 96, 3),
                             ("abi_version", 99, 2), ("attn", 7, 2), ("softmax_scale", -1.0, 2)]:
        dd = vista.make_desc(2, 256, 1, 128)
        setattr(dd, field, val)
        with pytest.raises(vista.VistaError) as e:
            vista.vista_summarize_workspace_size(dd, 1000)
        assert e.value.status == code, field
    # NULL pointers and misalignment are rejected before touching the device
    with pytest.raises(vista.VistaError) as e:
        vista.vista_summarize_fwd(d, 0, 0, 0, 0, 10, 0, 0, 0, 0, stream=0)
    assert e.value.status == 1
    with pytest.raises(vista.VistaError) as e:
        vista.vista_summarize_fwd(d, 16 * 1001 + 8, 4096, 4096, 4096, 10, 4096, 0, 4096, n, stream=0)
    assert e.value.status == 4
    with pytest.raises(vista.VistaError) as e:
        vista.vista_summarize_fwd(d, 4096, 4096, 4096, 4096, 10, 4096, 0, 4096, 1, stream=0)
    assert e.value.status == 5
    assert vista.vista_status_string(5) == "VISTA_ERR_WORKSPACE"


def test_qla_rows_and_bwd_validation_before_launch(lib):
    """NEXT-2/3/4 entry points: argument errors are returned before any launch."""
    import paper_2510_22049_b200 as vista
    dq = vista.make_desc(2, 1, 1, 128, attn=vista.QLA)
    n = vista.vista_qla_rows_workspace_size(dq, 1000, 500)
    assert n > 0
    with pytest.raises(vista.VistaError) as e:  # rows need the QLA form
        vista.vista_qla_rows_workspace_size(vista.make_desc(2, 1, 1, 128), 1000, 500)
    assert e.value.status == 2
    with pytest.raises(vista.VistaError) as e:  # negative row count
        vista.vista_qla_rows_workspace_size(dq, 1000, -1)
    assert e.value.status == 2
    with pytest.raises(vista.VistaError) as e:  # NULL row offsets
        vista.vista_qla_rows(dq, 4096, 4096, 4096, 10, 4096, 0, 5, 0, 0, 4096, 4096, n, stream=0)
    assert e.value.status == 1
    with pytest.raises(vista.VistaError) as e:  # k_self without v_self
        vista.vista_qla_rows(dq, 4096, 4096, 4096, 10, 4096, 4096, 5, 4096, 0, 4096, 4096, n, stream=0)
    assert e.value.status == 1
    with pytest.raises(vista.VistaError) as e:  # misaligned q rows
        vista.vista_qla_rows(dq, 4096, 4096, 4096, 10, 4104, 4096, 5, 0, 0, 4096, 4096, n, stream=0)
    assert e.value.status == 4
    with pytest.raises(vista.VistaError) as e:  # short workspace
        vista.vista_qla_rows(dq, 4096, 4096, 4096, 10, 4096, 4096, 5, 0, 0, 4096, 4096, 1, stream=0)
    assert e.value.status == 5
    # the softmax backward takes every shape the forward takes (tcgen05 or CUDA cores)
    for desc in (vista.make_desc(2, 200, 1, 128), vista.make_desc(2, 16, 1, 32, in_dtype=vista.F32),
                 vista.make_desc(2, 256, 1, 128)):
        assert vista.vista_summarize_bwd_workspace_size(desc, 100) > 0


def test_layers_stage2_rows_from_state_validation_before_launch(lib):
    """NEXT-3 layers, NEXT-4 stage 2 and rows from a saved state: argument errors are returned before
    any launch (no GPU here)."""
    import paper_2510_22049_b200 as vista
    E = vista.VistaError
    dl = vista.make_desc(2, 128, 1, 128, attn=vista.QLA)
    need = vista.vista_summarize_layers_workspace_size(dl, 3, 1000)
    assert need > 0
    cases = [
        (lambda: vista.vista_summarize_layers(dl, -1, 4096, 4096, 4096, 1000, 4096, 4096, need, stream=0), 2),  # layers < 0
        (lambda: vista.vista_summarize_layers(vista.make_desc(2, 128, 1, 128), 3, 4096, 4096, 4096, 1000, 4096, 4096,
                                              need, stream=0), 3),  # softmax form: the layers are QLA layers
        (lambda: vista.vista_summarize_layers(dl, 3, 4096, 4096, 0, 1000, 4096, 4096, need, stream=0), 1),  # no offsets
        (lambda: vista.vista_summarize_layers(dl, 3, 4096, 4104, 4096, 1000, 4096, 4096, need, stream=0), 4),  # misaligned x
        (lambda: vista.vista_summarize_layers(dl, 3, 4096, 4096, 4096, 1000, 4096, 4096, 64, stream=0), 5),  # short workspace
    ]
    ds = vista.make_desc(2, 256, 1, 128)
    ns = vista.vista_target_attend_workspace_size(ds, 512)
    cases += [
        (lambda: vista.vista_target_attend(ds, 4096, 4096, 4096, 4096, 4096, 4096, 0, 4096, -1, 4096, 0, 4096, ns, stream=0), 2),
        (lambda: vista.vista_target_attend(ds, 4096, 4096, 4096, 4096, 4096, 4096, 0, 0, 512, 4096, 0, 4096, ns, stream=0), 1),
        (lambda: vista.vista_target_attend(ds, 0, 4096, 4096, 4096, 4096, 4096, 0, 4096, 512, 4096, 0, 4096, ns, stream=0), 1),
        (lambda: vista.vista_target_attend(ds, 4096, 4098, 4096, 4096, 4096, 4096, 0, 4096, 512, 4096, 0, 4096, ns, stream=0), 4),
        (lambda: vista.vista_target_attend(ds, 4096, 4096, 4096, 4096, 4096, 4096, 0, 4096, 512, 4096, 0, 4096, 0, stream=0), 5),
    ]
    dq = vista.make_desc(2, 1, 1, 128, attn=vista.QLA)
    nr = vista.vista_qla_rows_from_state_workspace_size(dq, 500)
    cases += [
        (lambda: vista.vista_qla_rows_from_state(dq, 0, 4096, 4096, 4096, 500, 0, 0, 4096, 4096, nr, stream=0), 1),  # no z
        (lambda: vista.vista_qla_rows_from_state(dq, 4100, 4096, 4096, 4096, 500, 0, 0, 4096, 4096, nr, stream=0), 4),
        (lambda: vista.vista_qla_rows_from_state(dq, 4096, 4096, 4096, 4096, 500, 0, 0, 4096, 4096, 1, stream=0), 5),
    ]
    for fn, status in cases:
        with pytest.raises(E) as e:
            fn()
        assert e.value.status == status


def test_exchange_validation_before_launch(lib):
    """Peer-memory exchange entry points: argument errors are returned before any launch."""
    import paper_2510_22049_b200 as vista
    E = vista.VistaError
    cases = [
        (lambda: vista.vista_exchange_push(0, 0, 4096, 64, 4096, 16, [4096], [4096], 4096, 4096, stream=0), 2),
        (lambda: vista.vista_exchange_push(2, 2, 4096, 64, 4096, 16, [4096, 8192], [4096, 8192], 4096, 4096,
                                           stream=0), 2),  # rank >= world
        (lambda: vista.vista_exchange_push(9, 0, 4096, 64, 4096, 16, [4096] * 9, [4096] * 9, 4096, 4096,
                                           stream=0), 2),  # more than one node's ranks
        (lambda: vista.vista_exchange_push(1, 0, 4096, 63, 4096, 16, [4096], [4096], 4096, 4096, stream=0), 2),
        (lambda: vista.vista_exchange_push(1, 0, 0, 64, 4096, 16, [4096], [4096], 4096, 4096, stream=0), 1),
        (lambda: vista.vista_exchange_push(2, 0, 4096, 64, 4096, 16, [4096, 0], [4096, 8192], 4096, 4096,
                                           stream=0), 1),  # a NULL peer buffer
        (lambda: vista.vista_exchange_push(1, 0, 4100, 64, 4096, 16, [4096], [4096], 4096, 4096, stream=0), 4),
        (lambda: vista.vista_exchange_signal(1, 1, [4096], 4096, stream=0), 2),
        (lambda: vista.vista_exchange_signal(1, 0, [4096], 0, stream=0), 1),
        (lambda: vista.vista_exchange_wait(0, 4096, 4096, stream=0), 2),
        (lambda: vista.vista_exchange_wait(1, 0, 4096, stream=0), 1),
        (lambda: vista.vista_exchange_ack(1, 0, [0], 4096, stream=0), 1),
    ]
    d = vista.make_desc(2, 256, 2, 128)
    dq = vista.make_desc(2, 256, 2, 128, attn=vista.QLA)
    pp = lambda desc, world, rank, o, l, acks=4096, ep=4096: (  # noqa: E731
        lambda: vista.vista_summarize_partial_peers(desc, 4096, 4096, 4096, 4096, 64, world, rank, o, l, acks, ep,
                                                    4096, 1 << 20, stream=0))
    cases += [
        (pp(dq, 1, 0, [4100], None), 4),  # QLA: no lse buffers; Z buffer not 16-B aligned
        (pp(vista.make_desc(2, 256, 2, 64), 1, 0, [4096], [4096]), 3),  # d = 64: CUDA-core path, no fused stores
        (pp(vista.make_desc(2, 200, 2, 128), 1, 0, [4096], [4096]), 3),  # S % 128 != 0: likewise
        (pp(d, 0, 0, [4096], [4096]), 2),
        (pp(d, 2, 2, [4096, 8192], [4096, 8192]), 2),  # rank >= world
        (pp(d, 1, 0, [4096], [4096], acks=0), 1),
        (pp(d, 2, 0, [4096, 0], [4096, 8192]), 1),  # a NULL peer buffer
        (pp(d, 1, 0, [4100], [4096]), 4),  # receive buffer not 16-B aligned
    ]
    for fn, status in cases:
        with pytest.raises(E) as e:
            fn()
        assert e.value.status == status


def test_dispatch_by_shape(lib):
    import paper_2510_22049_b200 as vista
    assert vista.vista_dispatch_name(vista.make_desc(8, 256, 4, 128)) == "sm100_softmax"
    assert vista.vista_dispatch_name(vista.make_desc(8, 512, 1, 128)) == "sm100_softmax"
    assert vista.vista_dispatch_name(vista.make_desc(8, 256, 1, 128, attn=vista.QLA)) == "sm100_qla"
    assert vista.vista_dispatch_name(vista.make_desc(1, 16, 1, 32, in_dtype=vista.F32)) == "simt_softmax"
    assert vista.vista_dispatch_name(vista.make_desc(1, 100, 1, 128)) == "simt_softmax"
    assert vista.vista_dispatch_name(vista.make_desc(1, 16, 1, 64, attn=vista.QLA)) == "simt_qla"


def test_product_package_does_not_import_oracle():
    """The product path must not reach the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2510_22049_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", text).lower() or f == "__init__.py" and \
                    "import oracle" not in text, f
