"""Device-resident graph and traversal handles over libabfs.so.

`DeviceGraph` owns the combined representation in HBM (out-CSR, origins,
in-CSR, rev_owner); `Traversal` owns one BFS state (depths, visited bitmap,
frontier queue/bitmap pair, counters) and a CUDA stream.  These are the
objects the reference-named functions in kernels.py / adaptive.py drive.
"""

from __future__ import annotations

import contextlib
import ctypes
import threading

import numpy as np

from . import _lib as L


class DeviceGraph:
    """A Graph (graph.py:27-69) resident on one GPU."""

    def __init__(self, handle: ctypes.c_void_p):
        self._h = handle
        n, m, dev = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_int()
        L.check(L.lib().abfs_graph_info(handle, ctypes.byref(n), ctypes.byref(m),
                                        ctypes.byref(dev)), "graph_info")
        self.vertex_count = n.value
        self.edge_count = m.value
        self.device = dev.value
        self._scratch = None
        # traversal pool of the stateless reference-style calls: the primary
        # (`scratch()`) serves single-threaded use; concurrent callers on the
        # same graph get their own Traversal (distinct
        # traversals of one immutable Graph may run concurrently)
        self._pool_lock = threading.Lock()
        self._idle: list = []
        self._primary_busy = False

    # -- constructors -------------------------------------------------------
    @classmethod
    def upload(cls, graph, device: int = 0) -> "DeviceGraph":
        a = [np.ascontiguousarray(getattr(graph, k), dtype=np.uint32) for k in
             ("out_offsets", "destinations", "origins", "in_offsets", "sources")]
        h = ctypes.c_void_p()
        L.check(L.lib().abfs_graph_upload(device, graph.vertex_count, graph.edge_count,
                                          *[L.ptr(x, L.u32p) for x in a], ctypes.byref(h)),
                "graph_upload")
        return cls(h)

    @classmethod
    def build(cls, vertex_count: int, src, dst, device: int = 0) -> "DeviceGraph":
        """Device build_combined (graph.py:93-134) from range-checked pairs."""
        s = np.ascontiguousarray(src, dtype=np.uint32)
        d = np.ascontiguousarray(dst, dtype=np.uint32)
        h = ctypes.c_void_p()
        L.check(L.lib().abfs_graph_build(device, vertex_count, s.size, L.ptr(s, L.u32p),
                                         L.ptr(d, L.u32p), ctypes.byref(h)), "graph_build")
        return cls(h)

    @classmethod
    def rmat(cls, scale: int, edges: int, seed: int, a=0.57, b=0.19, c=0.19,
             symmetrize: bool = False, device: int = 0, permute: bool = False) -> "DeviceGraph":
        """generate_graph("rmat-like", ...) (graph.py:232-252) on the device,
        optionally symmetrised by appending reversed pairs;
        permute=True relabels the ids by a fixed bijection (no reference
        counterpart: robustness runs with hubs spread over the id space)."""
        st, inc = pcg_words(seed)
        h = ctypes.c_void_p()
        L.check(L.lib().abfs_graph_generate_rmat(device, scale, edges, a, b, c,
                                                 L.ptr(st, L.u64p), L.ptr(inc, L.u64p),
                                                 int(bool(symmetrize)) | (2 if permute else 0),
                                                 ctypes.byref(h)),
                "generate_rmat")
        return cls(h)

    @classmethod
    def uniform(cls, n: int, edges: int, seed: int, device: int = 0) -> "DeviceGraph":
        """generate_graph("uniform-random", ...) (graph.py:226-231), n = 2^k."""
        st, inc = pcg_words(seed)
        h = ctypes.c_void_p()
        L.check(L.lib().abfs_graph_generate_uniform(device, n, edges, L.ptr(st, L.u64p),
                                                    L.ptr(inc, L.u64p), ctypes.byref(h)),
                "generate_uniform")
        return cls(h)

    @classmethod
    def mesh(cls, rows: int, cols: int, device: int = 0) -> "DeviceGraph":
        h = ctypes.c_void_p()
        L.check(L.lib().abfs_graph_generate_mesh(device, rows, cols, ctypes.byref(h)),
                "generate_mesh")
        return cls(h)

    # -- host views -----------------------------------------------------------
    def download(self, rev_owner: bool = False) -> dict:
        n, m = self.vertex_count, self.edge_count
        out = {"out_offsets": np.empty(n + 1, np.uint32), "destinations": np.empty(m, np.uint32),
               "origins": np.empty(m, np.uint32), "in_offsets": np.empty(n + 1, np.uint32),
               "sources": np.empty(m, np.uint32)}
        ro = np.empty(m, np.uint32) if rev_owner else None
        L.check(L.lib().abfs_graph_download(
            self._h, L.ptr(out["out_offsets"], L.u32p), L.ptr(out["destinations"], L.u32p),
            L.ptr(out["origins"], L.u32p), L.ptr(out["in_offsets"], L.u32p),
            L.ptr(out["sources"], L.u32p), L.ptr(ro, L.u32p) if ro is not None else None),
            "graph_download")
        if ro is not None:
            out["rev_owner"] = ro
        return out

    def offsets(self):
        """(out_offsets, in_offsets) on the host -- enough for compute_stats."""
        n = self.vertex_count
        oo, io = np.empty(n + 1, np.uint32), np.empty(n + 1, np.uint32)
        L.check(L.lib().abfs_graph_download(self._h, L.ptr(oo, L.u32p), None, None,
                                            L.ptr(io, L.u32p), None, None), "graph_download")
        return oo, io

    def to_graph(self):
        from .graph import Graph
        a = self.download()
        return Graph(self.vertex_count, self.edge_count, a["out_offsets"], a["destinations"],
                     a["origins"], a["in_offsets"], a["sources"])

    def scratch(self) -> "Traversal":
        """The primary traversal of the stateless reference-style calls
        (its level-loop mode is inherited by the pool's other traversals)."""
        with self._pool_lock:
            if self._scratch is None:
                self._scratch = Traversal(self)
            return self._scratch

    @contextlib.contextmanager
    def borrow(self):
        """A traversal no other thread is using, for one reference-style call
        (the primary when it is free, else a pooled or new one)."""
        with self._pool_lock:
            if self._scratch is None:
                self._scratch = Traversal(self)
            t = None
            if not self._primary_busy:
                self._primary_busy = True
                t = self._scratch
            elif self._idle:
                t = self._idle.pop()
            mode = self._scratch.mode
        if t is None:
            t = Traversal(self)
        if t is not self._scratch and t.mode != mode:
            t.set_device_loop(mode)
        try:
            yield t
        finally:
            with self._pool_lock:
                if t is self._scratch:
                    self._primary_busy = False
                else:
                    self._idle.append(t)

    def close(self):
        for t in self._idle:
            t.close()
        self._idle = []
        if self._scratch is not None:
            self._scratch.close()
            self._scratch = None
        if self._h:
            L.lib().abfs_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Traversal:
    """Device BFS state over a DeviceGraph (depths + frontier + counters)."""

    def __init__(self, dgraph: DeviceGraph):
        self.graph = dgraph
        self.mode = 1
        self._h = ctypes.c_void_p()
        L.check(L.lib().abfs_traversal_create(dgraph._h, ctypes.byref(self._h)),
                "traversal_create")

    def set_stream(self, cuda_stream_ptr: int | None):
        L.check(L.lib().abfs_traversal_set_stream(self._h, ctypes.c_void_p(cuda_stream_ptr or 0)),
                "set_stream")

    def init(self, root: int):
        L.check(L.lib().abfs_init_depths(self._h, int(root)), "init_depths")

    def load(self, depths: np.ndarray):
        d = np.ascontiguousarray(depths, dtype=np.int32)
        L.check(L.lib().abfs_load_depths(self._h, L.ptr(d, L.i32p)), "load_depths")

    def read(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.graph.vertex_count, dtype=np.int32)
        L.check(L.lib().abfs_read_depths(self._h, L.ptr(out, L.i32p)), "read_depths")
        return out

    def level(self, level: int, kernel: int, variant: int, chunk_size: int = 32):
        c, el = ctypes.c_uint64(), ctypes.c_uint64()
        L.check(L.lib().abfs_level(self._h, int(level), int(kernel), int(variant),
                                   int(chunk_size), ctypes.byref(c), ctypes.byref(el)),
                "level")
        return c.value, el.value

    def run_level_host(self, depths: np.ndarray, level: int, kernel: int, variant: int,
                       chunk_size: int = 32):
        assert depths.dtype == np.int32 and depths.flags.c_contiguous and depths.flags.writeable
        c, el = ctypes.c_uint64(), ctypes.c_uint64()
        L.check(L.lib().abfs_run_level(self._h, L.ptr(depths, L.i32p), int(level), int(kernel),
                                       int(variant), int(chunk_size), ctypes.byref(c),
                                       ctypes.byref(el)), "run_level")
        return c.value, el.value

    def bfs_full(self, root: int, kernel: int, variant: int, chunk_size: int = 32,
                 depths_out: np.ndarray | None = None, cap: int = 1 << 16):
        """Every level's (count, ns); a traversal with more than `cap` levels
        is re-run with room for all of them (the reference returns every
        level, kernels.py:356-371)."""
        while True:
            counts, el = self._level_arrays(cap)
            nl = ctypes.c_size_t()
            L.check(L.lib().abfs_bfs_full(self._h, int(root), int(kernel), int(variant),
                                          int(chunk_size),
                                          L.ptr(depths_out, L.i32p) if depths_out is not None else None,
                                          L.ptr(counts, L.u64p), L.ptr(el, L.u64p), cap,
                                          ctypes.byref(nl)), "bfs_full")
            if nl.value <= cap:
                return counts[:nl.value].copy(), el[:nl.value].copy()
            cap = nl.value

    def adaptive(self, root: int, tree: L.AbfsTree, static24: np.ndarray, chunk_size: int = 32,
                 depths_out: np.ndarray | None = None, cap: int = 1 << 16):
        st = np.ascontiguousarray(static24, dtype=np.float64)
        while True:
            recs = self._records(cap)
            nl = ctypes.c_size_t()
            L.check(L.lib().abfs_adaptive_bfs(
                self._h, int(root), ctypes.byref(tree), L.ptr(st, L.f64p), int(chunk_size),
                L.ptr(depths_out, L.i32p) if depths_out is not None else None, recs, cap,
                ctypes.byref(nl)), "adaptive_bfs")
            if nl.value <= cap:
                return [L.AbfsLevelRecord.from_buffer_copy(r) for r in recs[:nl.value]]
            cap = nl.value   # more levels than records: re-run with room for all

    def adaptive_batch(self, roots, tree: L.AbfsTree, static24: np.ndarray,
                       chunk_size: int = 32):
        """Tree-switched BFS from every root in one persistent launch
        (abfs_adaptive_bfs_batch): returns (levels, bfs_ns per root, total_ns)."""
        r = np.ascontiguousarray(roots, dtype=np.int64)
        lv = np.zeros(r.size, np.uint64)
        ns = np.zeros(r.size, np.uint64)
        tot = ctypes.c_uint64()
        st = np.ascontiguousarray(static24, dtype=np.float64)
        L.check(L.lib().abfs_adaptive_bfs_batch(self._h, L.ptr(r, L.i64p), r.size, ctypes.byref(tree),
                                                L.ptr(st, L.f64p), int(chunk_size), L.ptr(lv, L.u64p),
                                                L.ptr(ns, L.u64p), ctypes.byref(tot)),
                "adaptive_bfs_batch")
        return lv, ns, tot.value

    def adaptive_batch_check(self, roots, tree: L.AbfsTree, static24: np.ndarray,
                             chunk_size: int = 32):
        """The batch with per-root parity evidence: (levels, depth checksums,
        per-root lists of per-level new counts).  See depth_checksum()."""
        r = np.ascontiguousarray(roots, dtype=np.int64)
        lv = np.zeros(r.size, np.uint64)
        cs = np.zeros(r.size, np.uint64)
        cap = 1 << 16
        nc = np.zeros(cap, np.uint64)
        n = ctypes.c_size_t()
        st = np.ascontiguousarray(static24, dtype=np.float64)
        L.check(L.lib().abfs_adaptive_bfs_batch_check(
            self._h, L.ptr(r, L.i64p), r.size, ctypes.byref(tree), L.ptr(st, L.f64p),
            int(chunk_size), L.ptr(lv, L.u64p), L.ptr(cs, L.u64p), L.ptr(nc, L.u64p), cap,
            ctypes.byref(n)), "adaptive_bfs_batch_check")
        per, off = [], 0
        for k in lv.tolist():
            per.append(nc[off:off + k].tolist() if off + k <= min(n.value, cap) else None)
            off += k
        return lv, cs, per

    def _records(self, cap: int):
        # one record buffer per traversal (allocating 3.6 MB per call would
        # dominate short traversals)
        buf = getattr(self, "_recbuf", None)
        if buf is None or len(buf) < cap:
            buf = (L.AbfsLevelRecord * cap)()
            self._recbuf = buf
        return buf

    def _level_arrays(self, cap: int):
        arr = getattr(self, "_lvlbuf", None)
        if arr is None or arr[0].size < cap:
            arr = (np.empty(cap, np.uint64), np.empty(cap, np.uint64))
            self._lvlbuf = arr
        return arr

    def last_ns(self) -> int:
        v = ctypes.c_uint64()
        L.check(L.lib().abfs_last_traversal_ns(self._h, ctypes.byref(v)), "last_ns")
        return v.value

    def set_device_loop(self, on):
        """True/1 (default): whole traversals run in the persistent megakernel
        (2: its 64-register variant); False/0: per-level launches."""
        L.check(L.lib().abfs_traversal_set_mode(self._h, int(on)), "set_mode")
        self.mode = int(on)

    def set_batch_ways(self, ways: int = 0):
        """Fix adaptive_batch's split (1 = one full-grid launch; 0 = automatic)."""
        L.check(L.lib().abfs_traversal_set_batch_ways(self._h, int(ways)), "set_batch_ways")

    def batch_ways(self, nroots: int) -> int:
        """Concurrent launches adaptive_batch splits nroots roots into."""
        v = ctypes.c_int()
        L.check(L.lib().abfs_traversal_batch_ways(self._h, int(nroots), ctypes.byref(v)),
                "batch_ways")
        return v.value

    def launches(self) -> int:
        v = ctypes.c_uint64()
        L.check(L.lib().abfs_traversal_launches(self._h, ctypes.byref(v)), "launches")
        return v.value

    def instrument(self, on: bool = True):
        L.check(L.lib().abfs_traversal_instrument(self._h, int(on)), "instrument")

    def level_stats(self, nlev: int):
        """Per-depth (count, Σ out-degree, Σ in-degree) for depths < nlev plus
        an unreached slot, and per-level pull-scanned edges (instrumented)."""
        a = [np.zeros(nlev + 1, np.uint64) for _ in range(4)]
        L.check(L.lib().abfs_traversal_level_stats(self._h, nlev, *[L.ptr(x, L.u64p) for x in a]),
                "level_stats")
        return {"count": a[0], "out_deg": a[1], "in_deg": a[2], "scanned": a[3][:nlev]}

    def reached(self):
        e, v = ctypes.c_uint64(), ctypes.c_uint64()
        L.check(L.lib().abfs_reached_edges(self._h, ctypes.byref(e), ctypes.byref(v)), "reached")
        return e.value, v.value

    def close(self):
        if self._h:
            L.lib().abfs_traversal_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pcg_words(seed: int):
    """numpy default_rng(seed)'s PCG64 (state, inc) as (hi, lo) u64 words."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    m64 = (1 << 64) - 1
    s, i = st["state"], st["inc"]
    return (np.array([s >> 64, s & m64], dtype=np.uint64),
            np.array([i >> 64, i & m64], dtype=np.uint64))


def depth_checksum(depths: np.ndarray) -> int:
    """Host restatement of the batch kernel's per-root depth checksum:
    sum over v of (uint64(uint32(d[v])) + 1) * ((v + 1) * 0x9E3779B97F4A7C15)
    mod 2^64 (abfs_adaptive_bfs_batch_check)."""
    d = np.asarray(depths).astype(np.int64).astype(np.uint32).astype(np.uint64) + np.uint64(1)
    w = (np.arange(1, d.size + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15))
    with np.errstate(over="ignore"):
        return int((d * w).sum(dtype=np.uint64))
