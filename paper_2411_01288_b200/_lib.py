"""ctypes binding of libhexamoe.so (the C ABI declared in include/hexamoe.h).

The product path has exactly one implementation: the CUDA kernels in this
library.  If the library is missing or the process has no CUDA device, the
operator calls raise -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# HXM_LIB: an alternative in-tree build of the same library (A/B experiments)
LIB_PATH = os.environ.get("HXM_LIB") or os.path.join(HERE, "libhexamoe.so")

HXM_OK, HXM_ERR_SHAPE, HXM_ERR_INVALID_ARG, HXM_ERR_CUDA = 0, 1, 2, 3
HXM_ERR_NCCL, HXM_ERR_CACHE, HXM_ERR_UNSUPPORTED = 4, 5, 6
HXM_F32, HXM_BF16 = 0, 1
ACT = {"relu": 0, "gelu": 1, "identity": 2}
HXM_WRITE, HXM_ACCUMULATE = 0, 1


class ShapeError(ValueError):
    """moekit::ShapeError (reference core/include/moekit/tensor.hpp:12-15)."""


class CacheError(RuntimeError):
    """moekit::CacheError (reference core/include/moekit/dist_sim.hpp:55-58)."""


class NcclError(RuntimeError):
    """HXM_ERR_NCCL: an NCCL collective of the C ABI failed (or NCCL is absent)."""


class HexaMoeCudaError(RuntimeError):
    pass


class LayerDesc(C.Structure):
    """hxm_layer_desc (include/hexamoe.h)."""
    _fields_ = [("n_tokens", C.c_int64), ("n_experts", C.c_int64), ("k", C.c_int64),
                ("d_in", C.c_int64), ("hidden", C.c_int64), ("d_out", C.c_int64),
                ("activation", C.c_int32), ("dtype", C.c_int32), ("add_b2", C.c_int32),
                ("capacity", C.c_int32), ("weight_shards", C.c_int32),
                ("reserved0", C.c_int32), ("weights_ready", C.c_void_p)]


MAX_PEERS = 8


class PeerRows(C.Structure):
    """hxm_peer_rows (include/hexamoe.h): the token owners' receive buffers."""
    _fields_ = [("n_ranks", C.c_int32), ("reserved", C.c_int32), ("rows_per_rank", C.c_int64),
                ("ptrs", C.c_void_p * MAX_PEERS)]


class PeerFlags(C.Structure):
    """hxm_peer_flags (include/hexamoe.h): every rank's barrier flag array."""
    _fields_ = [("n_ranks", C.c_int32), ("rank", C.c_int32), ("ptrs", C.c_void_p * MAX_PEERS)]


_p = C.c_void_p
_i64 = C.c_int64
_sz = C.c_size_t

# name -> (restype, argtypes); every symbol include/hexamoe.h declares
SIGNATURES = {
    "hxm_last_error": (C.c_char_p, []),
    "hxm_version": (C.c_int, []),
    "hxm_device_sm_count": (C.c_int, []),
    "hxm_reindex_bound": (_sz, [_i64, _i64, _i64]),
    "hxm_reindex_workspace_bytes": (_sz, [_i64, _i64]),
    "hxm_build_reindex": (C.c_int, [_p, _i64, _i64, _i64, _p, _p, _p, _sz, _p, _p]),
    "hxm_reindex_all_workspace_bytes": (_sz, [_i64, _i64, _i64]),
    "hxm_build_reindex_all": (C.c_int, [_p, _i64, _i64, _i64, _i64, _p, _i64, _p, _p, _sz, _p,
                                        _p]),
    "hxm_op_workspace_bytes": (_sz, [_i64, _i64, _i64, _i64, _i64]),
    "hxm_esmm": (C.c_int, [C.c_int, _p, _i64, _i64, _p, _i64, _i64, C.c_int, _p, _p, _p, _i64,
                           C.c_int, _p, _p, _sz, _p]),
    "hxm_ess": (C.c_int, [C.c_int, _p, _i64, _i64, _p, _p, _i64, _i64, _p, _p, _sz, _p]),
    "hxm_estmm": (C.c_int, [C.c_int, _p, _p, _i64, _i64, _i64, _p, _p, _i64, _i64, _p, _p, _sz,
                            _p]),
    "hxm_esfk": (C.c_int, [C.c_int, _p, _p, _i64, _i64, _i64, _p, C.c_int, _p, _p, _i64, _i64,
                           _p, _p, _p, _p, _sz, _p]),
    "hxm_layer_workspace_bytes": (_sz, [C.POINTER(LayerDesc)]),
    "hxm_moe_forward": (C.c_int, [C.POINTER(LayerDesc), _p, _p, _p, _p, _p, _p, _p, _p, _sz, _p,
                                  _p]),
    "hxm_moe_backward": (C.c_int, [C.POINTER(LayerDesc), _p, _p, _p, _p, _p, _sz, _p, _p, _p, _p,
                                   _p, _p]),
    "hxm_moe_stash_export": (C.c_int, [C.POINTER(LayerDesc), _p, _i64, _p, _p, _p]),
    "hxm_layer_forward_macs": (C.c_uint64, [C.POINTER(LayerDesc)]),
    "hxm_layer_path": (C.c_int, [C.POINTER(LayerDesc)]),
    "hxm_layer_weight_shards_ok": (C.c_int, [C.POINTER(LayerDesc), C.c_int32]),
    "hxm_nccl_get_unique_id": (C.c_int, [_p]),
    "hxm_nccl_comm_init": (C.c_int, [_p, C.c_int32, _p, C.c_int32]),
    "hxm_nccl_comm_destroy": (C.c_int, [_p]),
    "hxm_dc_cache_bytes": (_sz, [C.POINTER(LayerDesc)]),
    "hxm_dc_cache_views": (C.c_int, [C.POINTER(LayerDesc), _p, _p, _p, _p]),
    "hxm_dc_fill_cache": (C.c_int, [_p, C.POINTER(LayerDesc), _p, _p, _p, _p, _sz, _p]),
    "hxm_dc_allreduce_grads": (C.c_int, [_p, C.POINTER(LayerDesc), _p, _p, _p, _p, _p]),
    "hxm_tp_allgather_rows": (C.c_int, [_p, _p, _i64, _i64, _p, _p]),
    "hxm_tp_allgather_assignments": (C.c_int, [_p, _p, _i64, _i64, _p, _p]),
    "hxm_tp_allreduce_sum": (C.c_int, [_p, _p, _i64, _p]),
    "hxm_op_stats_add": (None, [C.c_int, _i64, _i64, _i64, _i64, _p]),
    "hxm_synthesize_routing": (C.c_int, [_i64, _i64, _i64, C.c_char_p, C.c_uint64, _p]),
    "hxm_make_layer_inputs": (None, [C.c_uint64, _i64, _i64, _i64, _i64, _i64, C.c_double, _p,
                                     _p, _p, _p, _p]),
    "hxm_profile_enable": (None, [C.c_int]),
    "hxm_profile_reset": (None, []),
    "hxm_profile_read": (C.c_int, [C.c_int, C.c_char_p, C.c_int, _p, _p, _p, _p]),
    "hxm_profile_read2": (C.c_int, [C.c_int, C.c_char_p, C.c_int, _p, _p, _p, _p, _p]),
    "hxm_launch_count": (C.c_uint64, []),
    "hxm_moe_forward_tp": (C.c_int, [C.POINTER(LayerDesc), _p, _p, _p, _p, _p, _p,
                                     C.POINTER(PeerRows), _p, _sz, _p, _p]),
    "hxm_moe_backward_tp": (C.c_int, [C.POINTER(LayerDesc), _p, _p, _p, _p, _p, _sz, _p, _p, _p,
                                      _p, C.POINTER(PeerRows), _p]),
    "hxm_moe_backward_dc": (C.c_int, [C.POINTER(LayerDesc), _p, _p, _p, _p, _p, _sz,
                                      C.POINTER(PeerRows), _p, C.POINTER(PeerRows), _p, _p, _p]),
    "hxm_peer_malloc": (C.c_int, [_sz, C.POINTER(C.c_void_p)]),
    "hxm_peer_free": (C.c_int, [_p]),
    "hxm_ipc_get_handle": (C.c_int, [_p, C.c_char_p]),
    "hxm_ipc_open_handle": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "hxm_ipc_close_handle": (C.c_int, [_p]),
    "hxm_peer_barrier": (C.c_int, [C.POINTER(PeerFlags), C.c_int32, _p]),
}


def profile_read(max_names: int = 64, name_len: int = 64):
    """{name: (total_ms, launches, work, kind, bytes)} for regions recorded since reset
    (bytes: algorithmic HBM bytes of FLOP-counted regions, 0 if not stated)."""
    import numpy as np
    names = C.create_string_buffer(max_names * name_len)
    ms = np.zeros(max_names, np.float64)
    n = np.zeros(max_names, np.int64)
    work = np.zeros(max_names, np.float64)
    kind = np.zeros(max_names, np.int32)
    nbytes = np.zeros(max_names, np.float64)
    cnt = lib().hxm_profile_read2(max_names, names, name_len, ms.ctypes.data, n.ctypes.data,
                                  work.ctypes.data, kind.ctypes.data, nbytes.ctypes.data)
    if cnt < 0:
        raise HexaMoeCudaError("hxm_profile_read failed")
    out = {}
    raw = names.raw
    for i in range(cnt):
        nm = raw[i * name_len:(i + 1) * name_len].split(b"\0", 1)[0].decode()
        out[nm] = (float(ms[i]), int(n[i]), float(work[i]), int(kind[i]), float(nbytes[i]))
    return out

_lib = None


def lib() -> C.CDLL:
    """Load libhexamoe.so.  Raises ImportError if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not built: run `python -m paper_2411_01288_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int, what: str = "") -> None:
    if status == HXM_OK:
        return
    msg = lib().hxm_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if status == HXM_ERR_SHAPE:
        raise ShapeError(msg)
    if status == HXM_ERR_INVALID_ARG:
        raise ValueError(msg)
    if status == HXM_ERR_CACHE:
        raise CacheError(msg)
    if status == HXM_ERR_NCCL:
        raise NcclError(msg)
    raise HexaMoeCudaError(f"[status {status}] {msg}")
