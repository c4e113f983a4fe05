"""ctypes binding of liblasp.so -- argument marshalling only (include/lasp.h is the contract).

The names mirror the C ABI one to one. Every step of the path runs in the CUDA library; this
module never computes. If liblasp.so is missing the import fails loudly (there is no fallback).
"""
from __future__ import annotations

import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LASP_LIB") or os.path.join(HERE, "liblasp.so")  # LASP_LIB: debug builds
HEADER = os.path.join(os.path.dirname(HERE), "include", "lasp.h")

LASP_BF16, LASP_FP32 = 0, 1
LASP_EXCHANGE_RING, LASP_EXCHANGE_ALLGATHER, LASP_EXCHANGE_P2P, LASP_EXCHANGE_P2P_ALLGATHER = 0, 1, 2, 3
STATUS = {0: "LASP_OK", 1: "LASP_ERR_SHAPE", 2: "LASP_ERR_DOMAIN", 3: "LASP_ERR_PARTITION", 4: "LASP_ERR_STATE",
          5: "LASP_ERR_COMM", 6: "LASP_ERR_CUDA", 7: "LASP_ERR_UNSUPPORTED"}


class lasp_shape_t(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int64), ("n_local", ctypes.c_int64), ("heads", ctypes.c_int64),
                ("head_dim", ctypes.c_int64), ("dtype", ctypes.c_int), ("kv_heads", ctypes.c_int64)]


class LaspError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


_vp = ctypes.c_void_p
_sp = ctypes.POINTER(lasp_shape_t)
_fp = ctypes.POINTER(ctypes.c_float)
_i64p = ctypes.POINTER(ctypes.c_int64)

_SIGS = {
    "lasp_last_error": ([], ctypes.c_char_p),
    "lasp_version": ([], ctypes.c_char_p),
    "lasp_cache_bytes": ([_sp], ctypes.c_size_t),
    "lasp_launch_count": ([], ctypes.c_uint64),
    "lasp_profile_enable": ([ctypes.c_int], None),
    "lasp_profile_read": ([ctypes.c_char_p, ctypes.c_size_t], ctypes.c_int),
    "lasp_debug_trace": ([_vp], None),
    "lasp_debug_occupy": ([ctypes.c_int, ctypes.c_int, ctypes.c_double, _vp], ctypes.c_int),
    "lasp_workspace_bytes": ([_sp], ctypes.c_size_t),
    "lasp_workspace_status": ([_vp, _vp], ctypes.c_int),
    "lasp_segment_len": ([_sp], ctypes.c_int64),
    "lasp_fwd_local": ([_sp, _vp, _vp, _vp, _fp, _vp, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "lasp_bwd_local": ([_sp, _vp, _vp, _vp, _fp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "lasp_unique_id": ([ctypes.c_char_p], ctypes.c_int),
    "lasp_ctx_create": ([ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(_vp)],
                        ctypes.c_int),
    "lasp_ctx_create_loopback": ([ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(_vp)],
                                 ctypes.c_int),
    "lasp_ctx_destroy": ([_vp], ctypes.c_int),
    "lasp_ctx_set_exchange": ([_vp, ctypes.c_int], ctypes.c_int),
    "lasp_ctx_create_p2p": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)], ctypes.c_int),
    "lasp_ctx_p2p_setup": ([_vp, ctypes.c_size_t, ctypes.c_char_p], ctypes.c_int),
    "lasp_ctx_p2p_connect": ([_vp, ctypes.c_char_p], ctypes.c_int),
    "lasp_ctx_protocol": ([_vp, _sp, _i64p, _i64p, _i64p], ctypes.c_int),
    "lasp_ring_peers": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                         ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "lasp_topology": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                       ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "lasp_fwd": ([_vp, _sp, _vp, _vp, _vp, _fp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "lasp_layer_workspace_bytes": ([_sp], ctypes.c_size_t),
    "lasp_layer_fwd": ([_vp, _sp, ctypes.c_int64] + [_vp] * 4 + [_fp] + [_vp] * 4 + [_vp] * 4, ctypes.c_int),
    "lasp_layer_bwd": ([_vp, _sp, ctypes.c_int64] + [_vp] * 4 + [_fp] + [_vp] * 5 + [_vp] * 2 + [_vp] * 4 +
                       [_vp] * 4 + [_vp, _vp], ctypes.c_int),
    "lasp_bwd": ([_vp, _sp, _vp, _vp, _vp, _fp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "lasp_gla_cache_bytes": ([_sp], ctypes.c_size_t),
    "lasp_gla_workspace_bytes": ([_sp], ctypes.c_size_t),
    "lasp_gla_segment_len": ([_sp], ctypes.c_int64),
    "lasp_gla_fwd_local": ([_sp] + [_vp] * 10, ctypes.c_int),
    "lasp_gla_bwd_local": ([_sp] + [_vp] * 14, ctypes.c_int),
    "lasp_gla_fwd": ([_vp, _sp] + [_vp] * 8, ctypes.c_int),
    "lasp_gla_bwd": ([_vp, _sp] + [_vp] * 12, ctypes.c_int),
}

_lib = None


def header_functions() -> list[str]:
    """Every function name include/lasp.h declares (used by the export test)."""
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lasp_[a-z_0-9]+)\s*\(", text)))


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(the LASP path has no CPU fallback)")
        if not os.environ.get("LASP_CUBLAS_LIB"):
            # the layer entry points' projection GEMMs: torch's bundled cuBLAS (already loaded by torch)
            try:
                import nvidia.cublas
                cand = os.path.join(list(nvidia.cublas.__path__)[0], "lib", "libcublas.so.12")
                if os.path.exists(cand):
                    os.environ["LASP_CUBLAS_LIB"] = cand
            except ImportError:
                pass
        if not os.environ.get("LASP_NCCL_LIB"):
            # the ring loads NCCL lazily (dlopen): point it at torch's bundled copy, the one torch.distributed uses
            try:
                import nvidia.nccl
                cand = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
                if os.path.exists(cand):
                    os.environ["LASP_NCCL_LIB"] = cand
            except ImportError:
                pass
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            if os.environ.get("LASP_LIB") and not hasattr(L, name):
                continue  # an older build loaded for a same-box A/B (tools/cmp_libs.sh)
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        raise LaspError(status, lib().lasp_last_error().decode())


def shape(batch: int, n_local: int, heads: int, head_dim: int, dtype: int, kv_heads: int = 0) -> lasp_shape_t:
    return lasp_shape_t(batch, n_local, heads, head_dim, dtype, kv_heads)
