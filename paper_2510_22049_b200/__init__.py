"""VISTA stage-1 user-history summarization on B200 -- Python binding of libvista (include/vista.h).

The binding only marshals arguments: every step of the hot path runs in the CUDA kernels of
``libvista.so`` (built in-tree from ``csrc/`` by ``__graft_entry__.build()``).  There is no CPU or
PyTorch fallback: ``load()`` raises if the library or a CUDA device is missing.  PyTorch is used
for device memory and streams only.

ABI entry points (same names as the C ABI):
    vista_abi_version, vista_status_string, vista_summarize_workspace_size,
    vista_summarize_fwd, vista_summarize_partial, vista_summarize_merge,
    vista_check_offsets, vista_dispatch_name
Convenience wrappers on torch tensors: ``make_desc``, ``summarize``, ``summarize_partial``,
``summarize_merge``.
"""
from __future__ import annotations

import ctypes
import math
import os

__all__ = [
    "VistaError", "Desc", "load", "lib_path", "make_desc",
    "vista_abi_version", "vista_status_string", "vista_summarize_workspace_size",
    "vista_summarize_fwd", "vista_summarize_partial", "vista_summarize_merge",
    "vista_summarize_merge_workspace_size",
    "vista_check_offsets", "vista_dispatch_name", "vista_time_next_main_kernel", "vista_launch_counter",
    "vista_quantize_rows_int8", "quantize_int8",
    "vista_summarize_prefix_workspace_size", "vista_summarize_fwd_prefix", "vista_summarize_partial_prefix",
    "vista_summarize_bwd_workspace_size", "vista_summarize_bwd", "vista_summarize_fwd_int8",
    "vista_qla_rows_workspace_size", "vista_qla_rows", "vista_summarize_bwd_qla_saved",
    "vista_qla_rows_from_state_workspace_size", "vista_qla_rows_from_state", "qla_rows_from_state",
    "vista_target_attend_workspace_size", "vista_target_attend", "target_attend",
    "vista_summarize_layers_workspace_size", "vista_summarize_layers", "summarize_layers",
    "summarize", "summarize_partial", "summarize_partial_peers", "summarize_merge", "summarize_bwd", "qla_rows",
    "vista_ipc_get_handle", "vista_ipc_open_handle", "vista_ipc_close", "vista_exchange_push",
    "vista_summarize_partial_peers",
    "vista_exchange_signal", "vista_exchange_wait", "vista_exchange_ack",
    "SOFTMAX", "QLA", "F32", "BF16", "ACT",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("VISTA_LIB") or os.path.join(_HERE, "libvista.so")  # VISTA_LIB: A/B builds

ABI_VERSION = 1
F32, BF16 = 0, 1
SOFTMAX, QLA = 0, 1
ACT = {"identity": 0, "silu": 1, "shifted_elu": 2}

_lib = None


class VistaError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = f"{where}: {_status_name(status)}"
        if status == 6 and _lib is not None:
            msg += f" ({_lib.vista_last_cuda_error().decode()})"
        super().__init__(msg)
        self.status = status


class Desc(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("num_users", ctypes.c_int32),
        ("num_summary", ctypes.c_int32),
        ("num_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("in_dtype", ctypes.c_int32),
        ("out_dtype", ctypes.c_int32),
        ("attn", ctypes.c_int32),
        ("softmax_scale", ctypes.c_float),
        ("qla_phi1", ctypes.c_int32),
        ("qla_phi2", ctypes.c_int32),
        ("qla_normalize", ctypes.c_int32),
        ("q_user_stride", ctypes.c_int64),
    ]


def lib_path() -> str:
    return _LIB_PATH


def load():
    """Load libvista.so (fails loudly: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"libvista.so not built ({_LIB_PATH}); run __graft_entry__.build()")
    lib = ctypes.CDLL(_LIB_PATH)
    P, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    DP = ctypes.POINTER(Desc)
    lib.vista_abi_version.restype = ctypes.c_int
    lib.vista_status_string.restype = ctypes.c_char_p
    lib.vista_status_string.argtypes = [ctypes.c_int]
    lib.vista_last_cuda_error.restype = ctypes.c_char_p
    lib.vista_dispatch_name.restype = ctypes.c_char_p
    lib.vista_dispatch_name.argtypes = [DP]
    lib.vista_summarize_workspace_size.argtypes = [DP, i64, ctypes.POINTER(sz)]
    lib.vista_summarize_fwd.argtypes = [DP, P, P, P, P, i64, P, P, P, sz, P]
    lib.vista_summarize_partial.argtypes = [DP, P, P, P, P, i64, P, P, P, sz, P]
    lib.vista_summarize_merge.argtypes = [DP, i32, P, P, P, P, P, P, P, sz, P]
    lib.vista_summarize_prefix_workspace_size.argtypes = [DP, i64, i64, ctypes.POINTER(sz)]
    lib.vista_summarize_bwd_workspace_size.argtypes = [DP, i64, ctypes.POINTER(sz)]
    lib.vista_summarize_fwd_int8.argtypes = [DP, P, P, P, P, i64, P, P, P, P, P, P, sz, P]
    lib.vista_summarize_bwd.argtypes = [DP, P, P, P, P, i64, P, P, P, P, P, P, P, sz, P]
    lib.vista_summarize_bwd_qla_saved.argtypes = [DP, P, P, P, P, i64, P, P, P, P, P, P, sz, P]
    lib.vista_qla_rows_workspace_size.argtypes = [DP, i64, i64, ctypes.POINTER(sz)]
    lib.vista_qla_rows.argtypes = [DP, P, P, P, i64, P, P, i64, P, P, P, P, sz, P]
    lib.vista_qla_rows_from_state_workspace_size.argtypes = [DP, i64, ctypes.POINTER(sz)]
    lib.vista_qla_rows_from_state.argtypes = [DP, P, P, P, P, i64, P, P, P, P, sz, P]
    lib.vista_target_attend_workspace_size.argtypes = [DP, i64, ctypes.POINTER(sz)]
    lib.vista_target_attend.argtypes = [DP, P, P, P, P, P, P, P, P, i64, P, P, P, sz, P]
    lib.vista_summarize_layers_workspace_size.argtypes = [DP, i32, i64, ctypes.POINTER(sz)]
    lib.vista_summarize_layers.argtypes = [DP, i32, P, P, P, i64, P, P, sz, P]
    lib.vista_summarize_fwd_prefix.argtypes = [DP, P, P, P, P, i64, P, P, i64, P, P, P, sz, P]
    lib.vista_summarize_partial_prefix.argtypes = [DP, P, P, P, P, i64, P, P, i64, P, P, P, sz, P]
    lib.vista_summarize_merge_workspace_size.argtypes = [DP, ctypes.POINTER(sz)]
    lib.vista_summarize_merge_workspace_size.restype = ctypes.c_int
    lib.vista_check_offsets.argtypes = [P, i32, i64, P]
    lib.vista_quantize_rows_int8.argtypes = [i64, i32, i32, P, P, P, P, P]
    lib.vista_quantize_rows_int8.restype = ctypes.c_int
    lib.vista_time_next_main_kernel.argtypes = [P, P]
    lib.vista_time_next_main_kernel.restype = ctypes.c_int
    lib.vista_launch_counter.restype = ctypes.c_uint64
    PP = ctypes.POINTER(ctypes.c_void_p)
    lib.vista_ipc_get_handle.argtypes = [P, P]
    lib.vista_ipc_open_handle.argtypes = [P, PP]
    lib.vista_ipc_close.argtypes = [P]
    lib.vista_exchange_push.argtypes = [i32, i32, P, i64, P, i64, PP, PP, P, P, P]
    lib.vista_exchange_signal.argtypes = [i32, i32, PP, P, P]
    lib.vista_exchange_wait.argtypes = [i32, P, P, P]
    lib.vista_exchange_ack.argtypes = [i32, i32, PP, P, P]
    lib.vista_summarize_partial_peers.argtypes = [DP, P, P, P, P, i64, i32, i32, PP, PP, P, P, P, sz, P]
    for f in ("vista_ipc_get_handle", "vista_ipc_open_handle", "vista_ipc_close", "vista_exchange_push",
              "vista_exchange_signal", "vista_exchange_wait", "vista_exchange_ack", "vista_summarize_partial_peers"):
        getattr(lib, f).restype = ctypes.c_int
    for f in ("vista_qla_rows_from_state_workspace_size", "vista_qla_rows_from_state",
              "vista_target_attend_workspace_size", "vista_target_attend",
              "vista_summarize_layers_workspace_size", "vista_summarize_layers",
              "vista_summarize_workspace_size", "vista_summarize_fwd", "vista_summarize_partial",
              "vista_summarize_merge", "vista_check_offsets", "vista_summarize_prefix_workspace_size",
              "vista_summarize_fwd_prefix", "vista_summarize_partial_prefix",
              "vista_summarize_bwd_workspace_size", "vista_summarize_bwd", "vista_summarize_fwd_int8"):
        getattr(lib, f).restype = ctypes.c_int
    if lib.vista_abi_version() != ABI_VERSION:
        raise RuntimeError("libvista ABI version mismatch")
    _lib = lib
    return lib


def _status_name(s: int) -> str:
    return load().vista_status_string(s).decode() if _lib else str(s)


def _check(status: int, where: str):
    if status != 0:
        raise VistaError(status, where)


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


# ----------------------------------------------------------------------------- raw ABI
def vista_abi_version() -> int:
    return load().vista_abi_version()


def vista_status_string(status: int) -> str:
    return load().vista_status_string(status).decode()


def vista_dispatch_name(desc: Desc) -> str | None:
    r = load().vista_dispatch_name(ctypes.byref(desc))
    return r.decode() if r else None


def vista_summarize_workspace_size(desc: Desc, total_len: int) -> int:
    n = ctypes.c_size_t(0)
    _check(load().vista_summarize_workspace_size(ctypes.byref(desc), int(total_len), ctypes.byref(n)),
           "vista_summarize_workspace_size")
    return n.value


def vista_summarize_fwd(desc, q, k, v, offsets, total_len, out, lse, workspace, workspace_bytes, stream=None):
    _check(load().vista_summarize_fwd(ctypes.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(offsets),
                                      int(total_len), _ptr(out), _ptr(lse), _ptr(workspace),
                                      int(workspace_bytes), _stream(stream)), "vista_summarize_fwd")


def vista_summarize_fwd_int8(desc, q, k, v, offsets, total_len, out, lse, codes, scale, zero_point, workspace,
                             workspace_bytes, stream=None):
    _check(load().vista_summarize_fwd_int8(ctypes.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(offsets),
                                           int(total_len), _ptr(out), _ptr(lse), _ptr(codes), _ptr(scale),
                                           _ptr(zero_point), _ptr(workspace), int(workspace_bytes), _stream(stream)),
           "vista_summarize_fwd_int8")


def vista_summarize_partial(desc, q, k, v, offsets, total_len, part_o, part_lse, workspace,
                            workspace_bytes, stream=None):
    _check(load().vista_summarize_partial(ctypes.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(offsets),
                                          int(total_len), _ptr(part_o), _ptr(part_lse), _ptr(workspace),
                                          int(workspace_bytes), _stream(stream)), "vista_summarize_partial")


def vista_summarize_prefix_workspace_size(desc: Desc, total_len: int, prefix_len: int) -> int:
    n = ctypes.c_size_t(0)
    _check(load().vista_summarize_prefix_workspace_size(ctypes.byref(desc), int(total_len), int(prefix_len),
                                                        ctypes.byref(n)), "vista_summarize_prefix_workspace_size")
    return n.value


def vista_summarize_fwd_prefix(desc, q, k, v, offsets, total_len, k_prefix, v_prefix, prefix_len, out, lse,
                               workspace, workspace_bytes, stream=None):
    _check(load().vista_summarize_fwd_prefix(ctypes.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(offsets),
                                             int(total_len), _ptr(k_prefix), _ptr(v_prefix), int(prefix_len),
                                             _ptr(out), _ptr(lse), _ptr(workspace), int(workspace_bytes),
                                             _stream(stream)), "vista_summarize_fwd_prefix")


def vista_summarize_partial_prefix(desc, q, k, v, offsets, total_len, k_prefix, v_prefix, prefix_len, part_o,
                                   part_lse, workspace, workspace_bytes, stream=None):
    _check(load().vista_summarize_partial_prefix(ctypes.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(offsets),
                                                 int(total_len), _ptr(k_prefix), _ptr(v_prefix), int(prefix_len),
                                                 _ptr(part_o), _ptr(part_lse), _ptr(workspace),
                                                 int(workspace_bytes), _stream(stream)),
           "vista_summarize_partial_prefix")


def vista_summarize_bwd_workspace_size(desc: Desc, total_len: int) -> int:
    n = ctypes.c_size_t(0)
    _check(load().vista_summarize_bwd_workspace_size(ctypes.byref(desc), int(total_len), ctypes.byref(n)),
           "vista_summarize_bwd_workspace_size")
    return n.value


def vista_summarize_bwd(desc, q, k, v, offsets, total_len, out, lse, dout, dq, dk, dv, workspace, workspace_bytes,
                        stream=None):
    _check(load().vista_summarize_bwd(ctypes.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(offsets), int(total_len),
                                      _ptr(out), _ptr(lse), _ptr(dout), _ptr(dq), _ptr(dk), _ptr(dv),
                                      _ptr(workspace), int(workspace_bytes), _stream(stream)),
           "vista_summarize_bwd")


def vista_summarize_bwd_qla_saved(desc, q, k, v, offsets, total_len, z_saved, dout, dq, dk, dv, workspace,
                                  workspace_bytes, stream=None):
    _check(load().vista_summarize_bwd_qla_saved(ctypes.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(offsets),
                                                int(total_len), _ptr(z_saved), _ptr(dout), _ptr(dq), _ptr(dk),
                                                _ptr(dv), _ptr(workspace), int(workspace_bytes), _stream(stream)),
           "vista_summarize_bwd_qla_saved")


def vista_qla_rows_workspace_size(desc, total_len, total_rows) -> int:
    n = ctypes.c_size_t(0)
    _check(load().vista_qla_rows_workspace_size(ctypes.byref(desc), int(total_len), int(total_rows), ctypes.byref(n)),
           "vista_qla_rows_workspace_size")
    return n.value


def vista_qla_rows(desc, k, v, offsets, total_len, q_rows, row_offsets, total_rows, k_self, v_self, out, workspace,
                   workspace_bytes, stream=None):
    _check(load().vista_qla_rows(ctypes.byref(desc), _ptr(k), _ptr(v), _ptr(offsets), int(total_len), _ptr(q_rows),
                                 _ptr(row_offsets), int(total_rows), _ptr(k_self), _ptr(v_self), _ptr(out),
                                 _ptr(workspace), int(workspace_bytes), _stream(stream)),
           "vista_qla_rows")


def vista_qla_rows_from_state_workspace_size(desc, total_rows) -> int:
    n = ctypes.c_size_t(0)
    _check(load().vista_qla_rows_from_state_workspace_size(ctypes.byref(desc), int(total_rows), ctypes.byref(n)),
           "vista_qla_rows_from_state_workspace_size")
    return n.value


def vista_qla_rows_from_state(desc, z, user_len, q_rows, row_offsets, total_rows, k_self, v_self, out, workspace,
                              workspace_bytes, stream=None):
    _check(load().vista_qla_rows_from_state(ctypes.byref(desc), _ptr(z), _ptr(user_len), _ptr(q_rows),
                                            _ptr(row_offsets), int(total_rows), _ptr(k_self), _ptr(v_self), _ptr(out),
                                            _ptr(workspace), int(workspace_bytes), _stream(stream)),
           "vista_qla_rows_from_state")


def vista_target_attend_workspace_size(desc, total_rows) -> int:
    n = ctypes.c_size_t(0)
    _check(load().vista_target_attend_workspace_size(ctypes.byref(desc), int(total_rows), ctypes.byref(n)),
           "vista_target_attend_workspace_size")
    return n.value


def vista_target_attend(desc, codes, token_scale, token_zero_point, q, k_self, v_self, resid, row_offsets, total_rows,
                        out, lse, workspace, workspace_bytes, stream=None):
    _check(load().vista_target_attend(ctypes.byref(desc), _ptr(codes), _ptr(token_scale), _ptr(token_zero_point),
                                      _ptr(q), _ptr(k_self), _ptr(v_self), _ptr(resid), _ptr(row_offsets),
                                      int(total_rows), _ptr(out), _ptr(lse), _ptr(workspace), int(workspace_bytes),
                                      _stream(stream)), "vista_target_attend")


def vista_summarize_layers_workspace_size(desc, num_layers, total_rows) -> int:
    n = ctypes.c_size_t(0)
    _check(load().vista_summarize_layers_workspace_size(ctypes.byref(desc), int(num_layers), int(total_rows),
                                                        ctypes.byref(n)), "vista_summarize_layers_workspace_size")
    return n.value


def vista_summarize_layers(desc, num_layers, weights, x, x_offsets, total_rows, tokens, workspace, workspace_bytes,
                           stream=None):
    _check(load().vista_summarize_layers(ctypes.byref(desc), int(num_layers), _ptr(weights), _ptr(x), _ptr(x_offsets),
                                         int(total_rows), _ptr(tokens), _ptr(workspace), int(workspace_bytes),
                                         _stream(stream)), "vista_summarize_layers")


def vista_summarize_merge_workspace_size(desc: Desc) -> int:
    n = ctypes.c_size_t(0)
    _check(load().vista_summarize_merge_workspace_size(ctypes.byref(desc), ctypes.byref(n)),
           "vista_summarize_merge_workspace_size")
    return n.value


def vista_summarize_merge(desc, num_parts, part_o, part_lse, q, user_len, out, lse, workspace=None,
                          workspace_bytes=0, stream=None):
    _check(load().vista_summarize_merge(ctypes.byref(desc), int(num_parts), _ptr(part_o), _ptr(part_lse),
                                        _ptr(q), _ptr(user_len), _ptr(out), _ptr(lse), _ptr(workspace),
                                        int(workspace_bytes), _stream(stream)), "vista_summarize_merge")


def vista_check_offsets(offsets, num_users, total_len, stream=None):
    _check(load().vista_check_offsets(_ptr(offsets), int(num_users), int(total_len), _stream(stream)),
           "vista_check_offsets")


def vista_quantize_rows_int8(n, d, in_dtype, x, codes, scale, zero_point, stream=None):
    _check(load().vista_quantize_rows_int8(int(n), int(d), int(in_dtype), _ptr(x), _ptr(codes), _ptr(scale),
                                           _ptr(zero_point), _stream(stream)), "vista_quantize_rows_int8")


def quantize_int8(x, stream=None):
    """Int8 export of rows of x [..., d] (bf16 or f32, device) -> (codes int8, scale f32, zero_point f32)."""
    import torch
    d = x.shape[-1]
    n = x.numel() // d
    codes = torch.empty(x.shape, dtype=torch.int8, device=x.device)
    scale = torch.empty(x.shape[:-1], dtype=torch.float32, device=x.device)
    zp = torch.empty(x.shape[:-1], dtype=torch.float32, device=x.device)
    vista_quantize_rows_int8(n, d, _dtype_code(x), x.contiguous(), codes, scale, zp, stream)
    return codes, scale, zp


def vista_time_next_main_kernel(start_event, stop_event):
    """Arm the one-shot timing hook (torch.cuda.Event objects or raw cudaEvent_t handles)."""
    h = [None if e is None else (e if isinstance(e, int) else e.cuda_event) for e in (start_event, stop_event)]
    _check(load().vista_time_next_main_kernel(h[0], h[1]), "vista_time_next_main_kernel")


def vista_launch_counter() -> int:
    return int(load().vista_launch_counter())


# ----------------------------------------------------------------------------- torch helpers
def make_desc(B, S, H, d, *, in_dtype=BF16, out_dtype=None, attn=SOFTMAX, scale=None,
              phi1="silu", phi2="silu", normalize=True, q_user_stride=0) -> Desc:
    return Desc(ABI_VERSION, int(B), int(S), int(H), int(d), int(in_dtype),
                int(in_dtype if out_dtype is None else out_dtype), int(attn),
                float("nan") if scale is None else float(scale), ACT[phi1], ACT[phi2],
                int(bool(normalize)), int(q_user_stride))


def _dtype_code(t):
    import torch
    if t.dtype == torch.bfloat16:
        return BF16
    if t.dtype == torch.float32:
        return F32
    raise TypeError(f"unsupported dtype {t.dtype}")


def _desc_for(q, k, offsets, attn, scale, phi1, phi2, normalize, out_dtype):
    B = offsets.numel() - 1
    S, H, d = q.shape[-3:]
    stride = S * H * d if q.dim() == 4 else 0
    return make_desc(B, S, H, d, in_dtype=_dtype_code(q), out_dtype=out_dtype, attn=attn, scale=scale,
                     phi1=phi1, phi2=phi2, normalize=normalize, q_user_stride=stride)


def _workspace(desc, total_len, device, workspace=None, prefix_len=0):
    import torch
    need = (vista_summarize_prefix_workspace_size(desc, total_len, prefix_len) if prefix_len
            else vista_summarize_workspace_size(desc, total_len))
    if workspace is not None and workspace.numel() >= need:
        return workspace, need
    return torch.empty(max(need, 16), dtype=torch.uint8, device=device), need


def summarize(q, k, v, offsets, total_len=None, *, attn=SOFTMAX, scale=None, phi1="silu", phi2="silu",
              normalize=True, out_dtype=None, workspace=None, stream=None, k_prefix=None, v_prefix=None):
    """Summary tokens of every user: out [B,S,H,d] (+ lse [B,H,S] for softmax).

    q: [S,H,d] shared seeds or [B,S,H,d]; k, v: [total_len,H,d]; offsets: int64 [B+1] on device.
    total_len (host int) avoids a device read; pass it on the hot path.
    k_prefix, v_prefix: optional shared key prefix [P,H,d] every user also attends to
    (vista_summarize_fwd_prefix).
    """
    import torch
    if total_len is None:
        total_len = k.shape[0]
    desc = _desc_for(q, k, offsets, attn, scale, phi1, phi2, normalize, out_dtype)
    B, S, H, d = desc.num_users, desc.num_summary, desc.num_heads, desc.head_dim
    odt = torch.bfloat16 if desc.out_dtype == BF16 else torch.float32
    out = torch.empty((B, S, H, d), dtype=odt, device=q.device)
    lse = torch.empty((B, H, S), dtype=torch.float32, device=q.device) if attn == SOFTMAX else None
    P = 0 if k_prefix is None else int(k_prefix.shape[0])
    ws, need = _workspace(desc, total_len, q.device, workspace, P)
    if k_prefix is not None:
        vista_summarize_fwd_prefix(desc, q, k, v, offsets, total_len, k_prefix, v_prefix, P, out, lse, ws,
                                   ws.numel(), stream)
    else:
        vista_summarize_fwd(desc, q, k, v, offsets, total_len, out, lse, ws, ws.numel(), stream)
    return out, lse


def summarize_partial(q, k, v, offsets, total_len=None, *, attn=SOFTMAX, scale=None, phi1="silu",
                      phi2="silu", normalize=True, workspace=None, stream=None, k_prefix=None, v_prefix=None):
    """Partial over one history shard: softmax -> (part_o [B,H,S,d] f32, part_lse [B,H,S]);
    QLA -> (Z [B,H,d,d] f32, None)."""
    import torch
    if total_len is None:
        total_len = k.shape[0]
    desc = _desc_for(q, k, offsets, attn, scale, phi1, phi2, normalize, None)
    B, S, H, d = desc.num_users, desc.num_summary, desc.num_heads, desc.head_dim
    if attn == SOFTMAX:
        po = torch.empty((B, H, S, d), dtype=torch.float32, device=q.device)
        pl = torch.empty((B, H, S), dtype=torch.float32, device=q.device)
    else:
        po = torch.empty((B, H, d, d), dtype=torch.float32, device=q.device)
        pl = None
    P = 0 if k_prefix is None else int(k_prefix.shape[0])
    ws, need = _workspace(desc, total_len, q.device, workspace, P)
    if k_prefix is not None:
        vista_summarize_partial_prefix(desc, q, k, v, offsets, total_len, k_prefix, v_prefix, P, po, pl, ws,
                                       ws.numel(), stream)
    else:
        vista_summarize_partial(desc, q, k, v, offsets, total_len, po, pl, ws, ws.numel(), stream)
    return po, pl


def summarize_partial_peers(q, k, v, offsets, total_len, exchange, *, attn=SOFTMAX, scale=None, phi1="silu",
                            phi2="silu", normalize=True, workspace=None, stream=None):
    """Partial over one history shard with the split-L exchange fused into its stores: softmax O_p / lse_p
    rows or QLA Z_p rows land in slot `exchange.rank` of every rank's receive buffer (exchange: a
    dist.PeerExchange).  Returns nothing; follow with exchange.signal_wait() and the merge."""
    if total_len is None:
        total_len = k.shape[0]
    desc = _desc_for(q, k, offsets, attn, scale, phi1, phi2, normalize, None)
    ws, need = _workspace(desc, total_len, q.device, workspace, 0)
    vista_summarize_partial_peers(desc, q, k, v, offsets, total_len, exchange.world, exchange.rank, exchange.o_ptrs,
                                  exchange.lse_ptrs if attn == SOFTMAX else None, exchange.acks, exchange.epoch, ws,
                                  ws.numel(), stream)


def summarize_bwd(q, k, v, offsets, total_len, dout, *, attn=QLA, phi1="silu", phi2="silu", normalize=True,
                  out=None, lse=None, z=None, workspace=None, stream=None):
    """Backward of summarize (NEXT-2): returns (dq, dk, dv).  dq float32 [S,H,d] (shared seeds,
    summed over users) or [B,S,H,d]; dk, dv like k, v.  Softmax needs the forward's out and lse;
    QLA may take the forward's saved state z ([B,H,d,d] f32 from summarize_partial) instead of
    recomputing it."""
    import torch
    if total_len is None:
        total_len = k.shape[0]
    desc = _desc_for(q, k, offsets, attn, None, phi1, phi2, normalize, _dtype_code(dout))
    dq = torch.empty(q.shape, dtype=torch.float32, device=q.device)
    dk = torch.empty_like(k)
    dv = torch.empty_like(v)
    need = vista_summarize_bwd_workspace_size(desc, total_len)
    ws = workspace if workspace is not None and workspace.numel() >= need else \
        torch.empty(max(need, 16), dtype=torch.uint8, device=q.device)
    if attn == QLA and z is not None:
        vista_summarize_bwd_qla_saved(desc, q, k, v, offsets, total_len, z, dout, dq, dk, dv, ws, ws.numel(), stream)
    else:
        vista_summarize_bwd(desc, q, k, v, offsets, total_len, out, lse, dout, dq, dk, dv, ws, ws.numel(), stream)
    return dq, dk, dv


def qla_rows(k, v, offsets, total_len, q_rows, row_offsets, total_rows=None, *, k_self=None, v_self=None,
             phi1="silu", phi2="silu", normalize=True, out_dtype=None, workspace=None, stream=None):
    """QLA at per-user query rows (NEXT-3 / NEXT-4): out [R,H,d] with out[r] = phi1(q_r) phi2(Z_u / N_u)
    (+ (phi1(q_r) . phi1(k_self_r)) v_self_r when k_self, v_self are given: the target rows' Delta
    term).  Rows [row_offsets[u], row_offsets[u+1]) belong to user u; Z_u is its history's state."""
    import torch
    if total_len is None:
        total_len = k.shape[0]
    if total_rows is None:
        total_rows = q_rows.shape[0]
    B = offsets.numel() - 1
    H, d = q_rows.shape[-2:]
    desc = make_desc(B, 1, H, d, in_dtype=_dtype_code(q_rows), out_dtype=out_dtype, attn=QLA, phi1=phi1, phi2=phi2,
                     normalize=normalize)
    odt = torch.bfloat16 if desc.out_dtype == BF16 else torch.float32
    out = torch.empty((q_rows.shape[0], H, d), dtype=odt, device=q_rows.device)
    need = vista_qla_rows_workspace_size(desc, total_len, total_rows)
    ws = workspace if workspace is not None and workspace.numel() >= need else \
        torch.empty(max(need, 16), dtype=torch.uint8, device=q_rows.device)
    vista_qla_rows(desc, k, v, offsets, total_len, q_rows, row_offsets, total_rows, k_self, v_self, out, ws,
                   ws.numel(), stream)
    return out


def qla_rows_from_state(z, user_len, q_rows, row_offsets, total_rows=None, *, k_self=None, v_self=None,
                        phi1="silu", phi2="silu", normalize=True, out_dtype=None, workspace=None, stream=None):
    """QLA rows from saved states z [B,H,d,d] (f32, unnormalized; e.g. summarize_partial(..., attn=QLA)[0])
    and user_len [B] (int64 N_u): the same rows as qla_rows without re-reading the histories."""
    import torch
    if total_rows is None:
        total_rows = q_rows.shape[0]
    B = z.shape[0]
    H, d = q_rows.shape[-2:]
    desc = make_desc(B, 1, H, d, in_dtype=_dtype_code(q_rows), out_dtype=out_dtype, attn=QLA, phi1=phi1, phi2=phi2,
                     normalize=normalize)
    odt = torch.bfloat16 if desc.out_dtype == BF16 else torch.float32
    out = torch.empty((q_rows.shape[0], H, d), dtype=odt, device=q_rows.device)
    need = vista_qla_rows_from_state_workspace_size(desc, total_rows)
    ws = workspace if workspace is not None and workspace.numel() >= need else \
        torch.empty(max(need, 16), dtype=torch.uint8, device=q_rows.device)
    vista_qla_rows_from_state(desc, z, user_len, q_rows, row_offsets, total_rows, k_self, v_self, out, ws, ws.numel(),
                              stream)
    return out


def target_attend(codes, token_scale, token_zero_point, q, k_self, v_self, row_offsets, total_rows=None, *,
                  resid=None, scale=None, out_dtype=None, with_lse=True, workspace=None, stream=None):
    """Stage-2 target-aware attention (NEXT-4): candidates q, k_self, v_self [R,H,d] attend to the int8
    summary tokens of their user (codes [B,S,H,d], token_scale / token_zero_point [B,S,H], e.g. the
    outputs of vista_summarize_fwd_int8) and to themselves.  Returns (out [R,H,d], lse [R,H] or None)."""
    import torch
    if total_rows is None:
        total_rows = q.shape[0]
    B, S, H, d = codes.shape
    desc = make_desc(B, S, H, d, in_dtype=_dtype_code(q), out_dtype=out_dtype, attn=SOFTMAX, scale=scale)
    odt = torch.bfloat16 if desc.out_dtype == BF16 else torch.float32
    out = torch.empty((q.shape[0], H, d), dtype=odt, device=q.device)
    lse = torch.empty((q.shape[0], H), dtype=torch.float32, device=q.device) if with_lse else None
    need = vista_target_attend_workspace_size(desc, total_rows)
    ws = workspace if workspace is not None and workspace.numel() >= need else \
        torch.empty(max(need, 16), dtype=torch.uint8, device=q.device)
    vista_target_attend(desc, codes, token_scale, token_zero_point, q, k_self, v_self, resid, row_offsets, total_rows,
                        out, lse, ws, ws.numel(), stream)
    return out, lse


# ----------------------------------------------------------------------------- peer-memory exchange
IPC_HANDLE_BYTES = 64


def vista_ipc_get_handle(tensor_or_ptr) -> bytes:
    """CUDA IPC handle (64 bytes) of a device allocation, to be opened by another process."""
    buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    _check(load().vista_ipc_get_handle(_ptr(tensor_or_ptr), buf), "vista_ipc_get_handle")
    return buf.raw


def vista_ipc_open_handle(handle: bytes) -> int:
    """Device pointer (in this process) of another process's allocation."""
    out = ctypes.c_void_p(0)
    buf = ctypes.create_string_buffer(bytes(handle), IPC_HANDLE_BYTES)
    _check(load().vista_ipc_open_handle(buf, ctypes.byref(out)), "vista_ipc_open_handle")
    return int(out.value)


def vista_ipc_close(ptr: int):
    _check(load().vista_ipc_close(ptr), "vista_ipc_close")


def _ptr_array(ptrs):
    return (ctypes.c_void_p * len(ptrs))(*[int(p) for p in ptrs])


def vista_exchange_push(world, rank, part_o, n_o, part_lse, n_lse, recv_o_ptrs, recv_lse_ptrs, acks, epoch,
                        stream=None):
    _check(load().vista_exchange_push(int(world), int(rank), _ptr(part_o), int(n_o), _ptr(part_lse), int(n_lse),
                                      _ptr_array(recv_o_ptrs), _ptr_array(recv_lse_ptrs) if recv_lse_ptrs else None,
                                      _ptr(acks), _ptr(epoch), _stream(stream)), "vista_exchange_push")


def vista_summarize_partial_peers(desc, q, k, v, offsets, total_len, world, rank, recv_o_ptrs, recv_lse_ptrs, acks,
                                  epoch, workspace, workspace_bytes, stream=None):
    """The softmax partial with the exchange fused into its stores (include/vista.h): every row goes
    straight into slot `rank` of every rank's receive buffer."""
    _check(load().vista_summarize_partial_peers(ctypes.byref(desc), _ptr(q), _ptr(k), _ptr(v), _ptr(offsets),
                                                int(total_len), int(world), int(rank), _ptr_array(recv_o_ptrs),
                                                _ptr_array(recv_lse_ptrs) if recv_lse_ptrs else None, _ptr(acks),
                                                _ptr(epoch), _ptr(workspace),
                                                int(workspace_bytes), _stream(stream)),
           "vista_summarize_partial_peers")


def vista_exchange_signal(world, rank, flag_ptrs, epoch, stream=None):
    _check(load().vista_exchange_signal(int(world), int(rank), _ptr_array(flag_ptrs), _ptr(epoch), _stream(stream)),
           "vista_exchange_signal")


def vista_exchange_wait(world, flags, epoch, stream=None):
    _check(load().vista_exchange_wait(int(world), _ptr(flags), _ptr(epoch), _stream(stream)), "vista_exchange_wait")


def vista_exchange_ack(world, rank, ack_ptrs, epoch, stream=None):
    _check(load().vista_exchange_ack(int(world), int(rank), _ptr_array(ack_ptrs), _ptr(epoch), _stream(stream)),
           "vista_exchange_ack")


def summarize_layers(x, x_offsets, weights, S, H, total_rows=None, *, phi1="silu", phi2="silu", normalize=True,
                     out_dtype=None, workspace=None, stream=None):
    """Multi-layer summarizer (NEXT-3): x [R, D] bf16 (user u = rows [x_offsets[u], x_offsets[u+1]), its
    first S rows the seed rows), weights [L, 5, D, D] bf16 (Wq, Wk, Wv, Wg, Wo as [out][in]).  x is
    updated in place; returns the summary tokens [B, S, H, d]."""
    import torch
    if total_rows is None:
        total_rows = x.shape[0]
    B = x_offsets.numel() - 1
    D = x.shape[1]
    d = D // H
    L = weights.shape[0]
    desc = make_desc(B, S, H, d, in_dtype=BF16, out_dtype=out_dtype, attn=QLA, phi1=phi1, phi2=phi2,
                     normalize=normalize)
    odt = torch.bfloat16 if desc.out_dtype == BF16 else torch.float32
    tokens = torch.empty((B, S, H, d), dtype=odt, device=x.device)
    need = vista_summarize_layers_workspace_size(desc, L, total_rows)
    ws = workspace if workspace is not None and workspace.numel() >= need else \
        torch.empty(max(need, 16), dtype=torch.uint8, device=x.device)
    vista_summarize_layers(desc, L, weights, x, x_offsets, total_rows, tokens, ws, ws.numel(), stream)
    return tokens


def summarize_merge(part_o, part_lse, *, q, attn=SOFTMAX, user_len=None, scale=None, phi1="silu",
                    phi2="silu", normalize=True, out_dtype=None, stream=None):
    """Merge stacked partials [P, ...] (e.g. all_gather output) into (out [B,S,H,d], lse)."""
    import torch
    P = part_o.shape[0]
    if attn == SOFTMAX:
        B, H, S, d = part_o.shape[1:]
    else:
        B, H, d, _ = part_o.shape[1:]
        S = q.shape[-3]
    in_dtype = _dtype_code(q)
    desc = make_desc(B, S, H, d, in_dtype=in_dtype, out_dtype=out_dtype, attn=attn, scale=scale, phi1=phi1,
                     phi2=phi2, normalize=normalize, q_user_stride=(S * H * d if q.dim() == 4 else 0))
    odt = torch.bfloat16 if desc.out_dtype == BF16 else torch.float32
    out = torch.empty((B, S, H, d), dtype=odt, device=part_o.device)
    lse = torch.empty((B, H, S), dtype=torch.float32, device=part_o.device) if attn == SOFTMAX else None
    need = vista_summarize_merge_workspace_size(desc)
    ws = torch.empty(max(need, 16), dtype=torch.uint8, device=part_o.device) if need else None
    vista_summarize_merge(desc, P, part_o, part_lse, q, user_len, out, lse, ws, need, stream)
    return out, lse
