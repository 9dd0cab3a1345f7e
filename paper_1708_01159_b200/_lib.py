"""ctypes binding of libabfs.so (include/abfs.h).

The shared library is built in-tree by `__graft_entry__.build()` (nvcc,
sm_100a).  There is no CPU fallback: if the library or a CUDA device is
missing, every engine entry point raises immediately.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ABFS_LIB: an alternative build of the same library (A/B experiments, tools/)
LIB_PATH = os.environ.get("ABFS_LIB") or os.path.join(_HERE, "libabfs.so")

ABFS_OK, ABFS_EINVAL, ABFS_ECUDA, ABFS_ENCCL, ABFS_ENOMEM, ABFS_EFEATURE = range(6)

u32p = ctypes.POINTER(ctypes.c_uint32)
i32p = ctypes.POINTER(ctypes.c_int32)
u64p = ctypes.POINTER(ctypes.c_uint64)
i64p = ctypes.POINTER(ctypes.c_int64)
f64p = ctypes.POINTER(ctypes.c_double)
u16p = ctypes.POINTER(ctypes.c_uint16)
u8p = ctypes.POINTER(ctypes.c_uint8)
vpp = ctypes.POINTER(ctypes.c_void_p)


class AbfsTree(ctypes.Structure):
    _fields_ = [("node_count", ctypes.c_uint32), ("n_selection", ctypes.c_uint32),
                ("selection", u16p), ("features", u16p), ("thresholds", f64p),
                ("lefts", u32p), ("rights", u32p), ("leaf_classes", u8p)]


class AbfsGenSpec(ctypes.Structure):
    """abfs_gen_spec (include/abfs.h): a device generator as data."""
    _fields_ = [("kind", ctypes.c_int32), ("symmetrize", ctypes.c_int32),
                ("scale", ctypes.c_uint32), ("rows", ctypes.c_uint32), ("cols", ctypes.c_uint32),
                ("n", ctypes.c_uint64), ("edges", ctypes.c_uint64),
                ("a", ctypes.c_double), ("b", ctypes.c_double), ("c", ctypes.c_double),
                ("pcg_state", ctypes.c_uint64 * 2), ("pcg_inc", ctypes.c_uint64 * 2)]


class AbfsLevelRecord(ctypes.Structure):
    _fields_ = [("level", ctypes.c_int64), ("kernel", ctypes.c_int32),
                ("variant", ctypes.c_int32), ("fallback", ctypes.c_int32),
                ("converted", ctypes.c_int32), ("frontier_size", ctypes.c_uint64),
                ("new_count", ctypes.c_uint64), ("elapsed_ns", ctypes.c_uint64),
                ("prediction_ns", ctypes.c_uint64), ("unvisited", ctypes.c_uint64),
                ("next_out_edges", ctypes.c_uint64)]


# name -> (restype, argtypes); every symbol declared in include/abfs.h.
_SIGNATURES = {
    "abfs_last_error": (ctypes.c_char_p, []),
    "abfs_version": (ctypes.c_int, []),
    "abfs_graph_upload": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                         u32p, u32p, u32p, u32p, u32p, vpp]),
    "abfs_graph_build": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                        u32p, u32p, vpp]),
    "abfs_graph_generate_rmat": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64,
                                                ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                                u64p, u64p, ctypes.c_int, vpp]),
    "abfs_graph_generate_uniform": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                                   u64p, u64p, vpp]),
    "abfs_graph_generate_mesh": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32, vpp]),
    "abfs_graph_read": (ctypes.c_int, [ctypes.c_int, ctypes.c_char_p, vpp]),
    "abfs_graph_write": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p]),
    "abfs_tree_read": (ctypes.c_int, [ctypes.c_char_p, vpp]),
    "abfs_tree_file_view": (ctypes.POINTER(AbfsTree), [ctypes.c_void_p]),
    "abfs_tree_file_free": (None, [ctypes.c_void_p]),
    "abfs_tree_write": (ctypes.c_int, [ctypes.POINTER(AbfsTree), ctypes.c_char_p]),
    "abfs_trace_write": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(AbfsLevelRecord),
                                        ctypes.c_size_t]),
    "abfs_trace_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(AbfsLevelRecord),
                                       ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "abfs_graph_info": (ctypes.c_int, [ctypes.c_void_p, u64p, u64p, ctypes.POINTER(ctypes.c_int)]),
    "abfs_graph_download": (ctypes.c_int, [ctypes.c_void_p, u32p, u32p, u32p, u32p, u32p, u32p]),
    "abfs_graph_destroy": (None, [ctypes.c_void_p]),
    "abfs_traversal_create": (ctypes.c_int, [ctypes.c_void_p, vpp]),
    "abfs_traversal_destroy": (None, [ctypes.c_void_p]),
    "abfs_traversal_set_stream": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "abfs_init_depths": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64]),
    "abfs_load_depths": (ctypes.c_int, [ctypes.c_void_p, i32p]),
    "abfs_read_depths": (ctypes.c_int, [ctypes.c_void_p, i32p]),
    "abfs_level": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int64, u64p, u64p]),
    "abfs_run_level": (ctypes.c_int, [ctypes.c_void_p, i32p, ctypes.c_int64, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int64, u64p, u64p]),
    "abfs_bfs_full": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int64, i32p, u64p, u64p, ctypes.c_size_t,
                                     ctypes.POINTER(ctypes.c_size_t)]),
    "abfs_adaptive_bfs": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64,
                                         ctypes.POINTER(AbfsTree), f64p, ctypes.c_int64, i32p,
                                         ctypes.POINTER(AbfsLevelRecord), ctypes.c_size_t,
                                         ctypes.POINTER(ctypes.c_size_t)]),
    "abfs_adaptive_bfs_batch": (ctypes.c_int, [ctypes.c_void_p, i64p, ctypes.c_size_t,
                                               ctypes.POINTER(AbfsTree), f64p, ctypes.c_int64,
                                               u64p, u64p, u64p]),
    "abfs_adaptive_bfs_batch_check": (ctypes.c_int, [ctypes.c_void_p, i64p, ctypes.c_size_t,
                                                     ctypes.POINTER(AbfsTree), f64p, ctypes.c_int64,
                                                     u64p, u64p, u64p, ctypes.c_size_t,
                                                     ctypes.POINTER(ctypes.c_size_t)]),
    "abfs_last_traversal_ns": (ctypes.c_int, [ctypes.c_void_p, u64p]),
    "abfs_traversal_set_mode": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "abfs_traversal_launches": (ctypes.c_int, [ctypes.c_void_p, u64p]),
    "abfs_traversal_batch_ways": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t,
                                                 ctypes.POINTER(ctypes.c_int)]),
    "abfs_traversal_set_batch_ways": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "abfs_traversal_instrument": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "abfs_traversal_level_stats": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t, u64p, u64p,
                                                  u64p, u64p]),
    "abfs_reached_edges": (ctypes.c_int, [ctypes.c_void_p, u64p, u64p]),
    "abfs_aggregate_count": (ctypes.c_int, [ctypes.c_int, i64p, ctypes.c_size_t, ctypes.c_int,
                                            i64p]),
    "abfs_tree_predict": (ctypes.c_int, [ctypes.POINTER(AbfsTree), f64p,
                                         ctypes.POINTER(ctypes.c_int)]),
    "abfs_features": (ctypes.c_int, [f64p, ctypes.c_uint64, ctypes.c_uint64, f64p]),
    "abfs_part_create": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, vpp]),
    "abfs_part_destroy": (None, [ctypes.c_void_p]),
    "abfs_gen_size": (ctypes.c_int, [ctypes.POINTER(AbfsGenSpec), u64p, u64p]),
    "abfs_gen_degrees": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(AbfsGenSpec), u32p, u32p]),
    "abfs_part_create_generated": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(AbfsGenSpec),
                                                  ctypes.c_uint64, ctypes.c_uint64, vpp]),
    "abfs_part_download": (ctypes.c_int, [ctypes.c_void_p, u32p, u32p, u32p, u32p, u32p, u32p,
                                          u32p]),
    "abfs_part_info": (ctypes.c_int, [ctypes.c_void_p, u64p, u64p, u64p, u64p]),
    "abfs_part_set_stream": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "abfs_part_init": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64]),
    "abfs_part_level": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int64, ctypes.c_void_p, ctypes.c_uint64]),
    "abfs_part_exchange": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, u64p, ctypes.c_uint32,
                                          ctypes.c_uint64, u64p, u64p, u64p]),
    "abfs_part_read_depths": (ctypes.c_int, [ctypes.c_void_p, i32p]),
    "abfs_part_depths_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "abfs_part_launches": (ctypes.c_int, [ctypes.c_void_p, u64p]),
    "abfs_part_peer_buffers": (ctypes.c_int, [ctypes.c_void_p, vpp, vpp, vpp]),
    "abfs_part_set_peers": (ctypes.c_int, [ctypes.c_void_p, vpp, vpp, vpp, ctypes.c_uint32,
                                           ctypes.c_uint32]),
    "abfs_part_ipc_export": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p]),
    "abfs_part_ipc_open": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_uint32,
                                          ctypes.c_uint32]),
    "abfs_part_level_p2p": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_int64]),
    "abfs_part_p2p_finish": (ctypes.c_int, [ctypes.c_void_p, u64p, u64p, u64p]),
    "abfs_parts_adaptive_bfs": (ctypes.c_int, [vpp, ctypes.c_uint32, ctypes.c_int64,
                                               ctypes.POINTER(AbfsTree), f64p, ctypes.c_int64,
                                               ctypes.POINTER(AbfsLevelRecord), u64p, ctypes.c_size_t,
                                               ctypes.POINTER(ctypes.c_size_t)]),
    "abfs_part_mega_adaptive_bfs": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64,
                                                   ctypes.POINTER(AbfsTree), f64p, ctypes.c_int64,
                                                   ctypes.POINTER(AbfsLevelRecord), u64p,
                                                   ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "abfs_part_mega_bfs_full": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                               ctypes.c_int, ctypes.c_int64,
                                               ctypes.POINTER(AbfsLevelRecord), u64p, ctypes.c_size_t,
                                               ctypes.POINTER(ctypes.c_size_t)]),
    "abfs_parts_bfs_full": (ctypes.c_int, [vpp, ctypes.c_uint32, ctypes.c_int64, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_int64,
                                           ctypes.POINTER(AbfsLevelRecord), u64p, ctypes.c_size_t,
                                           ctypes.POINTER(ctypes.c_size_t)]),
    "abfs_host_register": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t]),
    "abfs_host_unregister": (ctypes.c_int, [ctypes.c_void_p]),
}

_lib = None


class EngineUnavailable(RuntimeError):
    """libabfs.so is missing or no CUDA device is usable (no CPU fallback)."""


def lib():
    """Load libabfs.so once; raise loudly if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise EngineUnavailable(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return sorted(_SIGNATURES)


def check(rc: int, what: str = "") -> None:
    """Map abfs_status to the reference's exception types."""
    if rc == ABFS_OK:
        return
    msg = lib().abfs_last_error().decode("utf-8", "replace")
    if rc in (ABFS_EINVAL, ABFS_EFEATURE):
        raise ValueError(msg)
    if rc == ABFS_ENOMEM:
        raise MemoryError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: abfs status {rc}: {msg}")


def ptr(arr: np.ndarray, typ):
    return arr.ctypes.data_as(typ)
