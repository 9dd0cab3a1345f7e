"""ctypes binding of the CPU oracle (oracle/abfs_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, always as the checker or as
the timed CPU port of the reference -- never by the product package.  Each
wrapper names the reference function (file:line, relative to
/root/reference/pkg/src/adaptive_bfs/) it restates.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

INF_DEPTH = 2**31 - 1

_u32p = ctypes.POINTER(ctypes.c_uint32)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


class _Graph(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("m", ctypes.c_uint64),
                ("out_offsets", _u32p), ("destinations", _u32p),
                ("origins", _u32p), ("in_offsets", _u32p),
                ("sources", _u32p), ("rev_owner", _u32p)]


class _Tree(ctypes.Structure):
    _fields_ = [("node_count", ctypes.c_uint32), ("n_selection", ctypes.c_uint32),
                ("selection", ctypes.POINTER(ctypes.c_uint16)),
                ("features", ctypes.POINTER(ctypes.c_uint16)),
                ("thresholds", _f64p), ("lefts", _u32p), ("rights", _u32p),
                ("leaf_classes", ctypes.POINTER(ctypes.c_uint8))]


class _Record(ctypes.Structure):
    _fields_ = [("level", ctypes.c_int64), ("kernel", ctypes.c_int32),
                ("variant", ctypes.c_int32), ("fallback", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("frontier_size", ctypes.c_uint64),
                ("new_count", ctypes.c_uint64), ("elapsed_ns", ctypes.c_uint64),
                ("prediction_ns", ctypes.c_uint64)]


def build() -> str:
    """Compile liboracle.so with the committed Makefile."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
    return _lib


def _p(arr, typ):
    return arr.ctypes.data_as(typ)


class OracleGraph:
    """Host arrays of the combined representation (graph.py:27-69)."""

    def __init__(self, n, m, out_offsets, destinations, origins, in_offsets,
                 sources, rev_owner=None):
        self.n, self.m = int(n), int(m)
        c = lambda a: np.ascontiguousarray(a, dtype=np.uint32)
        self.out_offsets, self.destinations = c(out_offsets), c(destinations)
        self.origins, self.in_offsets, self.sources = c(origins), c(in_offsets), c(sources)
        if rev_owner is None:
            rev_owner = np.repeat(np.arange(self.n, dtype=np.uint32),
                                  np.diff(self.in_offsets.astype(np.int64)))
        self.rev_owner = c(rev_owner)
        self._s = _Graph(self.n, self.m, _p(self.out_offsets, _u32p),
                         _p(self.destinations, _u32p), _p(self.origins, _u32p),
                         _p(self.in_offsets, _u32p), _p(self.sources, _u32p),
                         _p(self.rev_owner, _u32p))

    @classmethod
    def from_graph(cls, g):
        return cls(g.vertex_count, g.edge_count, g.out_offsets, g.destinations,
                   g.origins, g.in_offsets, g.sources)


def _check(rc, what):
    if rc == 1:
        raise ValueError(f"oracle {what}: invalid argument")
    if rc == 5:
        raise ValueError(f"oracle {what}: invalid feature state")
    if rc != 0:
        raise RuntimeError(f"oracle {what}: rc={rc}")


def reference_bfs(g: OracleGraph, root: int) -> np.ndarray:
    """kernels.py:374-391."""
    d = np.empty(g.n, dtype=np.int32)
    _check(lib().orc_reference_bfs(ctypes.c_uint64(g.n), _p(g.out_offsets, _u32p),
                                   _p(g.destinations, _u32p), ctypes.c_int64(root),
                                   _p(d, _i32p)), "reference_bfs")
    return d


def run_level(g: OracleGraph, depths: np.ndarray, level: int, kernel: int,
              variant: int, chunk_size: int = 32, threads: int = 1):
    """kernels.py:340-353; mutates int32 `depths` in place -> (count, ns)."""
    assert depths.dtype == np.int32 and depths.flags.c_contiguous
    c, el = ctypes.c_uint64(), ctypes.c_uint64()
    _check(lib().orc_run_level(ctypes.byref(g._s), _p(depths, _i32p),
                               ctypes.c_int64(level), int(kernel), int(variant),
                               ctypes.c_int64(chunk_size), int(threads),
                               ctypes.byref(c), ctypes.byref(el)), "run_level")
    return c.value, el.value


def bfs_full(g: OracleGraph, root: int, kernel: int, variant: int,
             chunk_size: int = 32, threads: int = 1):
    """kernels.py:356-371 -> (depths, counts[], elapsed_ns[])."""
    d = np.empty(g.n, dtype=np.int32)
    cap = 1 << 16
    counts = np.zeros(cap, dtype=np.uint64)
    el = np.zeros(cap, dtype=np.uint64)
    nl = ctypes.c_uint64()
    _check(lib().orc_bfs_full(ctypes.byref(g._s), ctypes.c_int64(root), int(kernel),
                              int(variant), ctypes.c_int64(chunk_size), int(threads),
                              _p(d, _i32p), _p(counts, _u64p), _p(el, _u64p),
                              ctypes.c_uint64(cap), ctypes.byref(nl)), "bfs_full")
    k = min(nl.value, cap)
    return d, counts[:k].copy(), el[:k].copy()


def aggregate_count(counts, variant: int) -> int:
    """kernels.py:143-170."""
    a = np.ascontiguousarray(counts, dtype=np.int64)
    t = ctypes.c_int64()
    _check(lib().orc_aggregate_count(_p(a, _i64p), ctypes.c_uint64(a.size),
                                     int(variant), ctypes.byref(t)), "aggregate_count")
    return t.value


class OracleTree:
    """FlatTree arrays (tree.py:303-359) + canonical selection indices."""

    def __init__(self, selection_idx, features, thresholds, lefts, rights, classes):
        self.sel = np.ascontiguousarray(selection_idx, dtype=np.uint16)
        self.features = np.ascontiguousarray(features, dtype=np.uint16)
        self.thresholds = np.ascontiguousarray(thresholds, dtype=np.float64)
        self.lefts = np.ascontiguousarray(lefts, dtype=np.uint32)
        self.rights = np.ascontiguousarray(rights, dtype=np.uint32)
        self.classes = np.ascontiguousarray(classes, dtype=np.uint8)
        self._s = _Tree(len(self.classes), len(self.sel),
                        _p(self.sel, ctypes.POINTER(ctypes.c_uint16)),
                        _p(self.features, ctypes.POINTER(ctypes.c_uint16)),
                        _p(self.thresholds, _f64p), _p(self.lefts, _u32p),
                        _p(self.rights, _u32p),
                        _p(self.classes, ctypes.POINTER(ctypes.c_uint8)))


def adaptive_bfs(g: OracleGraph, root: int, tree: OracleTree, static24,
                 chunk_size: int = 32, threads: int = 1):
    """adaptive.py:83-129 with a FlatTree model -> (depths, records)."""
    d = np.empty(g.n, dtype=np.int32)
    st = np.ascontiguousarray(static24, dtype=np.float64)
    cap = 1 << 16
    recs = (_Record * cap)()
    nl = ctypes.c_uint64()
    _check(lib().orc_adaptive_bfs(ctypes.byref(g._s), ctypes.c_int64(root),
                                  ctypes.byref(tree._s), _p(st, _f64p),
                                  ctypes.c_int64(chunk_size), int(threads),
                                  _p(d, _i32p), recs, ctypes.c_uint64(cap),
                                  ctypes.byref(nl)), "adaptive_bfs")
    out = [(r.level, r.kernel, r.variant, bool(r.fallback), r.frontier_size,
            r.new_count, r.elapsed_ns, r.prediction_ns)
           for r in recs[:min(nl.value, cap)]]
    return d, out


def pcg_state(seed: int):
    """(state[2], inc[2]) u64 words of numpy default_rng(seed)'s PCG64."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, i = st["state"], st["inc"]
    m64 = (1 << 64) - 1
    return (np.array([s >> 64, s & m64], dtype=np.uint64),
            np.array([i >> 64, i & m64], dtype=np.uint64))


def generate_rmat_pairs(scale, m, seed, a=0.57, b=0.19, c=0.19, threads=8):
    """graph.py:232-252 (edge pairs before build_combined)."""
    st, inc = pcg_state(seed)
    src = np.empty(m, dtype=np.uint32)
    dst = np.empty(m, dtype=np.uint32)
    _check(lib().orc_generate_rmat(ctypes.c_uint32(scale), ctypes.c_uint64(m),
                                   ctypes.c_double(a), ctypes.c_double(b),
                                   ctypes.c_double(c), _p(st, _u64p), _p(inc, _u64p),
                                   _p(src, _u32p), _p(dst, _u32p), int(threads)),
           "generate_rmat")
    return src, dst


def generate_uniform_pairs(n, m, seed, threads=8):
    """graph.py:226-231 for power-of-two n."""
    st, inc = pcg_state(seed)
    src = np.empty(m, dtype=np.uint32)
    dst = np.empty(m, dtype=np.uint32)
    _check(lib().orc_generate_uniform(ctypes.c_uint64(n), ctypes.c_uint64(m),
                                      _p(st, _u64p), _p(inc, _u64p),
                                      _p(src, _u32p), _p(dst, _u32p), int(threads)),
           "generate_uniform")
    return src, dst


def build_combined(n, src, dst) -> OracleGraph:
    """graph.py:93-134 via stable counting sorts."""
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    m = src.size
    oo = np.empty(n + 1, dtype=np.uint32)
    io = np.empty(n + 1, dtype=np.uint32)
    de = np.empty(m, dtype=np.uint32)
    og = np.empty(m, dtype=np.uint32)
    so = np.empty(m, dtype=np.uint32)
    _check(lib().orc_build_combined(ctypes.c_uint64(n), ctypes.c_uint64(m),
                                    _p(src, _u32p), _p(dst, _u32p), _p(oo, _u32p),
                                    _p(de, _u32p), _p(og, _u32p), _p(io, _u32p),
                                    _p(so, _u32p)), "build_combined")
    return OracleGraph(n, m, oo, de, og, io, so)
