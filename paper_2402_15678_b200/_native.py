"""ctypes binding of libminions.so (the C-ABI declared in include/minions.h).

The product path has no CPU fallback: importing this module on a machine
without the built library raises, and every entry point raises when the
library reports an error.  Status codes map onto the reference's exception
classes (include/minions.h).
"""
from __future__ import annotations

import ctypes
import os

from .core import DistMismatch, LengthMismatch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MS_LIB") or os.path.join(_HERE, "lib", "libminions.so")  # MS_LIB: diagnostic builds

MS_OK, MS_ERR_VALUE, MS_ERR_LENGTH, MS_ERR_DIST, MS_ERR_UNSUPPORTED, MS_ERR_CUDA = 0, -1, -2, -3, -4, -5

_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_F = ctypes.c_float

# name -> argtypes (restype int unless listed in _RESTYPE)
_SIGS = {
    "ms_version": [],
    "ms_strerror": [_I],
    "ms_launch_count": [],
    "ms_reset_launch_count": [],
    "ms_preload": [],
    "ms_vote": [_P, _P, _P, _I, _I, _I, _P, _P, _P],
    "ms_accept_greedy": [_P, _P, _P, _I, _I, _I, _P, _P, _P, _P, _P, _P],
    "ms_argmax_rows": [_P, _I, _I, _I, _I64, _P, _P, _P],
    "ms_accept_greedy_logits": [_P, _P, _I, _I, _P, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P],
    "ms_softmax_sample": [_P, _I64, _I, _I, _P, _I64, _P, _I64, _P, _P],
    "ms_gather_voted": [_P, _P, _I, _I, _I, _I, _P, _P],
    "ms_accept_stochastic": [_P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P],
    "ms_linear": [_P, _I64, _P, _P, _P, _I64, _P, _I64, _I, _I, _I, _I, _I, _I, _P],
    "ms_linear_rms": [_P, _I64, _P, _P, _P, _I64, _P, _I64, _I, _I, _I, _I, _I, _I, _P, _I, _F, _P, _I64, _P],
    "ms_linear_wide": [_P, _I64, _P, _P, _P, _I64, _P, _I64, _I, _I, _I, _I, _I, _P],
    "ms_gemv": [_P, _I64, _P, _P, _P, _I64, _P, _I64, _I, _I, _I, _I, _I, _P],
    "ms_linear_splits": [_I, _I],
    "ms_set_gated_persistent": [_I],
    "ms_embed": [_P, _P, _I, _P, _P, _I, _I, _I, _P, _P],
    "ms_layernorm": [_P, _I64, _P, _P, _P, _F, _I, _I, _P, _I64, _P],
    "ms_kv_append": [_P, _I64, _I, _I, _I, _I, _P, _P, _I, _P, _P, _P],
    "ms_kv_append_gqa": [_P, _I64, _I, _I, _I, _I, _I, _P, _P, _I, _P, _P, _P, _P],
    "ms_rmsnorm": [_P, _I64, _P, _P, _F, _I, _I, _P, _I64, _P],
    "ms_gated_silu": [_P, _I64, _I, _I, _P, _I64, _P],
    "ms_attention_gqa": [_P, _I64, _I, _I, _I, _I, _I, _P, _P, _I, _P, _P, _P, _F, _I, _P, _I64, _P, _I64,
                         _P, _I, _P],
    "ms_draft_commit": [_P, _P, _I, _I, _I, _I, _I, _P, _I64, _P, _F, ctypes.c_uint64, _P, _P, _P],
    "ms_pack_verify": [_P, _P, _I, _I, _P, _P],
    "ms_attention": [_P, _I64, _I, _I, _I, _I, _P, _P, _I, _P, _P, _F, _I, _P, _I64, _P, _I64, _P, _I, _P],
    "ms_embed_f32": [_P, _P, _I, _P, _P, _I, _I, _I, _P, _P],
    "ms_norm_f32": [_P, _I64, _P, _P, _P, _F, _I, _I, _I, _P, _I64, _P],
    "ms_linear_f32": [_P, _I64, _P, _P, _P, _I64, _P, _I64, _I, _I, _I, _I, _P],
    "ms_attention_f32": [_P, _I64, _I, _I, _I, _I, _I, _P, _P, _I, _P, _P, _P, _F, _I, _P, _I64, _P],
    "ms_ipc_alloc": [_I64, ctypes.POINTER(ctypes.c_void_p), _P],
    "ms_ipc_handle_size": [],
    "ms_ipc_open": [_P, ctypes.POINTER(ctypes.c_void_p)],
    "ms_ipc_close": [_P],
    "ms_free": [_P],
    "ms_tp_signal": [_P, _I, _I, _P, _P],
    "ms_tp_reduce_gather": [_P, _I64, _P, _I64, _P, _P, _I, _I, _I, _I, _P, _I, _P],
    "ms_linear_tp_scatter": [_P, _I64, _P, _P, _I64, _I, _I, _I, _P, _I, _I, _I, _P],
    "ms_tp_reduce_recv_gather": [_P, _I, _I, _P, _I64, _P, _P, _I, _I, _I, _P, _I, _P],
    "ms_rmsnorm_wait": [_P, _I64, _P, _F, _I, _I, _P, _I64, _P, _P, _I, _P, _I, _P],
    "ms_tp_argmax_local": [_P, _I64, _I, _I, _I, _P, _P],
    "ms_tp_argmax_combine": [_P, _I, _I, _P, _P, _P, _P, _I, _P],
    "ms_linear_grouped": [_P, _I64, _P, _P, _P, _I64, _P, _I64, _I, _I, _I, _I, _I, _I, _I, _P],
    "ms_gemv_grouped": [_P, _I64, _P, _I64, _P, _P, _I64, _P, _I64, _I, _I, _I, _I, _I, _I, _P],
    "ms_gemv_rms_grouped": [_P, _I64, _P, _I64, _P, _I64, _P, _I64, _I, _I, _I, _I, _I, _I, _F, _P],
    "ms_embed_grouped": [_P, _P, _I, _P, _I64, _I, _P, _I, _I, _I, _P, _P],
    "ms_rmsnorm_grouped": [_P, _I64, _P, _P, _I64, _I, _F, _I, _I, _P, _I64, _P],
    "ms_draft_commit_grouped": [_P, _P, _I, _I, _I, _I, _P, _I64, _P, ctypes.POINTER(ctypes.c_float),
                                ctypes.c_uint64, _P, _P, _P],
    "ms_attention_tc": [_P, _I64, _I, _I, _I, _I, _I, _P, _P, _I, _I, _P, _P, _P, _F, _I, _P, _I64, _P, _I, _I, _P],
    "ms_attention_paged": [_P, _I64, _I, _I, _I, _I, _I, _P, _P, _I, _P, _P, _P, _F, _I, _P, _I64, _P, _I64,
                           _P, _I, _P, _I, _I, _P],
    "ms_kv_append_paged": [_P, _I64, _I, _I, _I, _I, _I, _P, _P, _I, _P, _P, _P, _P, _I, _I, _P],
    "ms_attention_workspace_gqa": [_I, _I, _I, _I, _I, _I, ctypes.POINTER(ctypes.c_int64),
                                   ctypes.POINTER(ctypes.c_int)],
    "ms_set_pdl": [_I],
    "ms_set_coresident": [_I],
    "ms_sm_partition": [_I, _I, _I, _I, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p),
                        ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)],
    "ms_attention_workspace": [_I, _I, _I, _I, _I, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)],
}
_RESTYPE = {"ms_strerror": ctypes.c_char_p, "ms_launch_count": ctypes.c_int64,
            "ms_reset_launch_count": None}


class NativeLibraryMissing(RuntimeError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} is not built; run `python -m paper_2402_15678_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)  # AttributeError = header/library drift
        fn.argtypes = args
        fn.restype = _RESTYPE.get(name, ctypes.c_int)
    return lib


lib = _load()


def exported_symbols() -> list[str]:
    return sorted(_SIGS)


def check(status: int, what: str = "") -> None:
    if status == MS_OK:
        return
    msg = f"{what}: {lib.ms_strerror(status).decode()}"
    if status == MS_ERR_VALUE:
        raise ValueError(msg)
    if status == MS_ERR_LENGTH:
        raise LengthMismatch(msg)
    if status == MS_ERR_DIST:
        raise DistMismatch(msg)
    if status == MS_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib, name)(*args), name)


def launch_count() -> int:
    return int(lib.ms_launch_count())


def reset_launch_count() -> None:
    lib.ms_reset_launch_count()
