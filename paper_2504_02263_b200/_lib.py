"""ctypes binding of libmsinfer.so (include/msinfer.h).

The extension is the only compute path: there is no CPU or PyTorch fallback.
If the library is missing or the device is not a B200 (sm_100), calls raise.
"""

from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libmsinfer.so")
MAX_RANKS = 8
IPC_HANDLE_BYTES = 64
ROW_ALIGN = 128
KV_PAGE = 64     # MSI_KV_PAGE
HEAD_DIM = 128   # MSI_HEAD_DIM

BUF_RECV, BUF_HBUF, BUF_CNTAB, BUF_TP_X = 0, 3, 4, 5
ERRORS = {-1: "MSI_EINVAL", -2: "MSI_EARCH", -3: "MSI_ESTATE", -4: "MSI_ETIMEOUT", -5: "MSI_EDRIVER"}


class MsiError(RuntimeError):
    """A libmsinfer call failed (rc > 0: cudaError_t, rc < 0: MSI_E*)."""

    def __init__(self, fn: str, rc: int, text: str):
        self.rc = rc
        super().__init__(f"{fn} failed: rc={rc} ({ERRORS.get(rc, 'cudaError')}): {text}")


class Plan(ctypes.Structure):
    _fields_ = [
        ("world", ctypes.c_int32), ("n_a", ctypes.c_int32), ("n_e", ctypes.c_int32),
        ("attn_ranks", ctypes.c_int32 * MAX_RANKS), ("expert_ranks", ctypes.c_int32 * MAX_RANKS),
        ("hidden", ctypes.c_int32), ("inter", ctypes.c_int32), ("experts", ctypes.c_int32),
        ("topk", ctypes.c_int32), ("max_tokens", ctypes.c_int32), ("slots", ctypes.c_int32),
        ("tp_e", ctypes.c_int32), ("tp_a", ctypes.c_int32),
    ]


class IpcHandle(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_ubyte * IPC_HANDLE_BYTES)]


# name -> (restype, argtypes); the exact exported surface of include/msinfer.h
_P, _I, _U32, _SZ, _U64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32, ctypes.c_size_t, ctypes.c_uint64
SIGNATURES = {
    "msi_version": (_I, []),
    "msi_last_error": (ctypes.c_char_p, []),
    "msi_check_device": (_I, []),
    "msi_ctx_create": (_I, [ctypes.POINTER(Plan), _I, ctypes.POINTER(_P)]),
    "msi_ctx_destroy": (_I, [_P]),
    "msi_ctx_export": (_I, [_P, ctypes.POINTER(IpcHandle)]),
    "msi_ctx_import": (_I, [_P, _I, ctypes.POINTER(IpcHandle)]),
    "msi_ctx_finalize": (_I, [_P]),
    "msi_ctx_buffer": (_I, [_P, _I, _I, ctypes.POINTER(_P), ctypes.POINTER(_SZ)]),
    "msi_ctx_reset": (_I, [_P]),
    "msi_poll_status": (_I, [_P, ctypes.POINTER(ctypes.c_int32)]),
    "msi_set_wait_timeout": (_I, [_P, _U64]),
    "msi_ctx_stats": (_I, [_P, ctypes.POINTER(_U64), ctypes.POINTER(_U64)]),
    "msi_set_trace": (_I, [_P, _I]),
    "msi_ctx_trace": (_I, [_P, ctypes.POINTER(_U64), _I]),
    "msi_ctx_workspace": (_I, [_P, ctypes.POINTER(_P), ctypes.POINTER(_SZ)]),
    "msi_gate_topk_workspace": (_SZ, [_I, _I]),
    "msi_gate_topk": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P]),
    "msi_gate_topk_placed": (_I, [_P, _P, _I, _I, _I, _I, _P, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "msi_dispatch": (_I, [_P, _P, _P, _P, _P, _I, _I, _U32, _P]),
    "msi_route_dispatch": (_I, [_P, _P, _P, _I, _I, _P, _I, _P, _P, _P, _P, _P, _I, _U32, _P]),
    "msi_expert_ffn": (_I, [_P, _P, _P, _I, _U32, _P]),
    "msi_expert_echo": (_I, [_P, _I, _U32, _P]),
    "msi_expert_wait": (_I, [_P, _I, _U32, _P]),
    "msi_combine": (_I, [_P, _P, _P, _P, _P, _P, _I, _I, _U32, _P]),
    "msi_gather_y": (_I, [_P, _P, _P, _P, _I, _I, _P]),
    "msi_pack_w13": (_I, [_P, _P, _P, _I, _I, _I, _P]),
    "msi_set_gemm_cta_group": (_I, [_I]),
    "msi_grouped_ffn": (_I, [_P, _P, _I, _I, _P, _P, _P, _P, _I, _I, _P]),
    "msi_combine_local": (_I, [_P, _P, _P, _P, _I, _I, _I, _P]),
    "msi_rope_append": (_I, [_P, ctypes.c_int64, _P, _I, _I, _I, ctypes.c_float, _P, _I, _P, _P,
                             ctypes.c_int64, _P, _P]),
    "msi_grouped_ffn_regions": (_I, [_P, _P, _I, ctypes.c_int64, _I, _P, _P, _P, ctypes.c_int64, _P, _I, _I, _I,
                                     _P, _P]),
    "msi_tp_publish": (_I, [_P, _P, _I, _I, _U32, _P]),
    "msi_tp_qkv": (_I, [_P, _P, _I, _I, _P, ctypes.c_float, _P, _I, _P, _P, _P, _I, _I, _U32, _P]),
    "msi_tp_oproj": (_I, [_P, _P, _P, _I, _I, _I, _U32, _P]),
    "msi_tp_reduce": (_I, [_P, _P, _P, _I, _I, _U32, _P]),
    "msi_dense_logits": (_I, [_P, ctypes.c_int64, _P, _I, _I, _P, _P, _P]),
    "msi_dense_gemm": (_I, [_P, ctypes.c_int64, _P, _I, _I, _P, ctypes.c_int64, _P, ctypes.c_int64, _P, _P]),
    "msi_qkv_rope_append": (_I, [_P, ctypes.c_int64, _I, _P, _I, _I, _P, ctypes.c_float, _P, _I, _P, _P, _P,
                                 _P, _P]),
    "msi_decode_attention_workspace": (_SZ, [_I, _I, _I, _I]),
    "msi_decode_attention": (_I, [_P, _P, _P, ctypes.c_int64, _P, _I, _P, _I, _I, _I, ctypes.c_float, _P, _P,
                                  _SZ, _P]),
}

_lib = None


def load(build_if_missing: bool = False):
    """Load libmsinfer.so (optionally building it with nvcc first)."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing and not os.path.exists(LIB_PATH):
        from . import build as _build
        _build.build()
    if not os.path.exists(LIB_PATH):
        raise MsiError("load", -3, f"{LIB_PATH} not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def call(name: str, *args) -> int:
    rc = getattr(load(), name)(*args)
    if rc != 0:
        raise MsiError(name, rc, load().msi_last_error().decode())
    return rc


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
