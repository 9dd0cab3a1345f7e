"""1-D vertex-partitioned tree-switched BFS over several GPUs.

The reference runs one process over one graph (kernels.py:82-127); this is
the multi-GPU form of the same level loop (adaptive.py:83-129,
kernels.py:356-371).  Vertices are split into P contiguous, edge-balanced
destination ranges; rank p's `abfs_part` holds the destination-filtered
out-CSR over all sources, the in-CSR rows of its owned vertices, its owned
depths and a replicated global frontier bitmap.  Per level:

  1. every rank runs the chosen (kernel, variant) on its slice and packs its
     next-frontier bitmap slice (`abfs_part_level`);
  2. the slices are all-gathered (NCCL over NVLink between processes; a
     device concat when several partitions share one GPU);
  3. every rank unpacks the gathered bitmap and popc-counts it
     (`abfs_part_exchange`) -- the same global count everywhere, hence the
     same float64 features and the same tree decision, with no broadcast.

Level semantics, counts and traces equal the single-GPU engine's (and the
reference's) for the same tree: the per-level global count is exactly the
number of INF -> level+1 transitions.

The driver is independent of where the local level runs: `PartitionedBFS`
takes local partition objects with the `DevicePartition` interface and an
exchange with the `Exchange` interface (the CPU tests plug in world-size-2
gloo processes).
"""

from __future__ import annotations

import ctypes
import time
from typing import Sequence

import numpy as np

from . import _lib as L
from .adaptive import DEFAULT_KERNEL, AdaptiveTrace, LevelTrace
from .features import extract_runtime_features
from .graph import GraphStats
from .kernels import GROUP_SIZE, CountVariant, KernelId, LevelOutcome
from .tree import UNKNOWN, FlatTree, predict

ALIGN = 32


def edge_balanced_bounds(in_offsets, parts: int, align: int = ALIGN) -> np.ndarray:
    """Vertex bounds b[0..parts] of contiguous destination ranges with about
    equal owned in-edge counts (the probe found vertex-equal ranges 3.5x
    imbalanced on Kronecker at P=8).  Inner bounds are multiples
    of `align` (whole bitmap words); b[0] = 0, b[parts] = |V|."""
    if parts < 1:
        raise ValueError("need at least one partition")
    if align < 32 or align % 32:
        raise ValueError("align must be a positive multiple of 32")
    io = np.asarray(in_offsets, dtype=np.int64)
    n = io.size - 1
    m = int(io[-1]) if n >= 0 else 0
    targets = (np.arange(1, parts, dtype=np.int64) * m) // parts
    b = np.searchsorted(io, targets, side="left").astype(np.int64)
    b = (b + align // 2) // align * align
    b = np.minimum(b, n // align * align)
    b = np.maximum.accumulate(np.concatenate([[0], b, [n]]))
    return b


def word_bounds(bounds: np.ndarray) -> np.ndarray:
    """Global bitmap-word offsets of each range (inner bounds are word
    aligned; the last ends at ceil(|V|/32))."""
    b = np.asarray(bounds, dtype=np.int64)
    w = b // 32
    w[-1] = (b[-1] + 31) // 32
    return w.astype(np.uint64)


# ---- generator specs: a rank builds its slice without the whole graph -------

def gen_spec(kind: str, **kw) -> L.AbfsGenSpec:
    """An `abfs_gen_spec` for the device generators (DeviceGraph.rmat /
    .uniform / .mesh take the same parameters):
    gen_spec("rmat", scale=, edges=, seed=, symmetrize=, a=.57, b=.19, c=.19),
    gen_spec("uniform", n=, edges=, seed=), gen_spec("mesh", rows=, cols=)."""
    from .engine import pcg_words
    sp = L.AbfsGenSpec()
    if kind == "rmat":
        sp.kind, sp.scale, sp.edges = 0, int(kw["scale"]), int(kw["edges"])
        sp.symmetrize = int(bool(kw.get("symmetrize", False)))
        sp.a, sp.b, sp.c = kw.get("a", 0.57), kw.get("b", 0.19), kw.get("c", 0.19)
    elif kind == "uniform":
        sp.kind, sp.n, sp.edges = 1, int(kw["n"]), int(kw["edges"])
    elif kind == "mesh":
        sp.kind, sp.rows, sp.cols = 2, int(kw["rows"]), int(kw["cols"])
        return sp
    else:
        raise ValueError(f"unknown generator {kind!r}")
    st, inc = pcg_words(int(kw["seed"]))
    sp.pcg_state[0], sp.pcg_state[1] = int(st[0]), int(st[1])
    sp.pcg_inc[0], sp.pcg_inc[1] = int(inc[0]), int(inc[1])
    return sp


def gen_size(spec: L.AbfsGenSpec) -> tuple[int, int]:
    n, m = ctypes.c_uint64(), ctypes.c_uint64()
    L.check(L.lib().abfs_gen_size(ctypes.byref(spec), ctypes.byref(n), ctypes.byref(m)), "gen_size")
    return n.value, m.value


def gen_offsets(spec: L.AbfsGenSpec, device: int = 0):
    """(out_offsets, in_offsets) of the generated graph from one streaming
    degree pass on `device` (no edge arrays): compute_stats's and
    edge_balanced_bounds's inputs."""
    n, m = gen_size(spec)
    od, id_ = np.empty(n, np.uint32), np.empty(n, np.uint32)
    L.check(L.lib().abfs_gen_degrees(device, ctypes.byref(spec), L.ptr(od, L.u32p),
                                     L.ptr(id_, L.u32p)), "gen_degrees")
    oo, io = np.zeros(n + 1, np.uint32), np.zeros(n + 1, np.uint32)
    np.cumsum(od, out=oo[1:], dtype=np.uint32)
    np.cumsum(id_, out=io[1:], dtype=np.uint32)
    if int(oo[-1]) != m or int(io[-1]) != m:
        raise RuntimeError(f"degree pass counted {int(oo[-1])}/{int(io[-1])} slots, expected {m}")
    return oo, io


class DevicePartition:
    """One rank's slice on its GPU (`abfs_part`, include/abfs.h): cut from a
    DeviceGraph, or (``spec=``) built straight from the generator stream on
    ``device`` without the whole graph ever being resident."""

    def __init__(self, dgraph, lo: int, hi: int, stream_ptr: int | None = None, *,
                 spec: L.AbfsGenSpec | None = None, device: int | None = None):
        self.lo, self.hi = int(lo), int(hi)
        self._h = ctypes.c_void_p()
        if spec is not None:
            self.device = int(device or 0)
            L.check(L.lib().abfs_part_create_generated(self.device, ctypes.byref(spec), self.lo,
                                                       self.hi, ctypes.byref(self._h)),
                    "part_create_generated")
        else:
            self.device = dgraph.device
            L.check(L.lib().abfs_part_create(dgraph._h, self.lo, self.hi, ctypes.byref(self._h)),
                    "part_create")
        mf, mr = ctypes.c_uint64(), ctypes.c_uint64()
        L.check(L.lib().abfs_part_info(self._h, None, None, ctypes.byref(mf), ctypes.byref(mr)),
                "part_info")
        self.m_fwd, self.m_rev = mf.value, mr.value
        self.n_total = gen_size(spec)[0] if spec is not None else dgraph.vertex_count
        if stream_ptr is not None:
            self.set_stream(stream_ptr)

    @property
    def owned(self) -> int:
        return self.hi - self.lo

    def set_stream(self, stream_ptr: int | None):
        L.check(L.lib().abfs_part_set_stream(self._h, ctypes.c_void_p(stream_ptr or 0)),
                "part_set_stream")

    def init(self, root: int):
        L.check(L.lib().abfs_part_init(self._h, int(root)), "part_init")

    def level(self, level: int, kernel: int, variant: int, chunk_size: int, send) -> None:
        """Enqueue one level; `send` is a device int32/uint32 tensor of stride words."""
        L.check(L.lib().abfs_part_level(self._h, int(level), int(kernel), int(variant),
                                        int(chunk_size), ctypes.c_void_p(send.data_ptr()),
                                        send.numel()), "part_level")

    def exchange(self, gathered, wbounds: np.ndarray, stride: int):
        """Unpack the gathered slices; returns (global_count, local_count, ns)."""
        g, lc, ns = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        wb = np.ascontiguousarray(wbounds, dtype=np.uint64)
        L.check(L.lib().abfs_part_exchange(self._h, ctypes.c_void_p(gathered.data_ptr()),
                                           L.ptr(wb, L.u64p), wb.size - 1, int(stride),
                                           ctypes.byref(g), ctypes.byref(lc), ctypes.byref(ns)),
                "part_exchange")
        return g.value, lc.value, ns.value

    # -- fused peer exchange ---------------------------------------------------
    def peer_buffers(self):
        f0, f1, mb = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        L.check(L.lib().abfs_part_peer_buffers(self._h, ctypes.byref(f0), ctypes.byref(f1),
                                               ctypes.byref(mb)), "part_peer_buffers")
        return f0.value, f1.value, mb.value

    def set_peers(self, buffers, rank: int):
        n = len(buffers)
        arr = [(ctypes.c_void_p * n)(*[b[k] for b in buffers]) for k in range(3)]
        L.check(L.lib().abfs_part_set_peers(self._h, *arr, n, rank), "part_set_peers")

    def ipc_export(self) -> bytes:
        buf = ctypes.create_string_buffer(192)
        L.check(L.lib().abfs_part_ipc_export(self._h, buf), "part_ipc_export")
        return buf.raw

    def ipc_open(self, handles: Sequence[bytes], rank: int):
        blob = b"".join(handles)
        L.check(L.lib().abfs_part_ipc_open(self._h, blob, len(handles), rank), "part_ipc_open")

    def level_p2p(self, level: int, kernel: int, variant: int, chunk_size: int) -> None:
        L.check(L.lib().abfs_part_level_p2p(self._h, int(level), int(kernel), int(variant),
                                            int(chunk_size)), "part_level_p2p")

    def p2p_finish(self):
        g, lc, ns = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        L.check(L.lib().abfs_part_p2p_finish(self._h, ctypes.byref(g), ctypes.byref(lc),
                                             ctypes.byref(ns)), "part_p2p_finish")
        return g.value, lc.value, ns.value

    def read_depths(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.owned, np.int32)
        L.check(L.lib().abfs_part_read_depths(self._h, L.ptr(out, L.i32p)), "part_read_depths")
        return out

    def depths_to(self, dev_tensor) -> None:
        L.check(L.lib().abfs_part_depths_device(self._h, ctypes.c_void_p(dev_tensor.data_ptr())),
                "part_depths_device")

    def launches(self) -> int:
        v = ctypes.c_uint64()
        L.check(L.lib().abfs_part_launches(self._h, ctypes.byref(v)), "part_launches")
        return v.value

    def download(self) -> dict:
        """The slice's arrays on the host (tests)."""
        n = int(self.n_total)
        out = {"fo_off": np.empty(n + 1, np.uint32), "fo_dst": np.empty(self.m_fwd, np.uint32),
               "fo_org": np.empty(self.m_fwd, np.uint32), "r_off": np.empty(self.owned + 1, np.uint32),
               "r_src": np.empty(self.m_rev, np.uint32), "r_own": np.empty(self.m_rev, np.uint32),
               "r_first": np.empty(self.owned, np.uint32)}
        L.check(L.lib().abfs_part_download(self._h, *[L.ptr(out[k], L.u32p) for k in
                                                      ("fo_off", "fo_dst", "fo_org", "r_off",
                                                       "r_src", "r_own", "r_first")]),
                "part_download")
        return out

    def close(self):
        if self._h:
            L.lib().abfs_part_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LocalExchange:
    """All partitions live in this process on one device: the all-gather is
    a device concat on the current stream."""

    def __init__(self, torch_mod):
        self.torch = torch_mod

    def allgather(self, sends: Sequence):
        return self.torch.cat(list(sends))

    def max_over_ranks(self, x: float) -> float:
        return x

    def gather_depths(self, slices: Sequence, bounds, n: int):
        return np.concatenate([s for s in slices]) if slices else np.empty(0, np.int32)


class LocalPeerExchange(LocalExchange):
    """Fused exchange between partitions of this process: every partition's
    level-ending kernel stores its slice into all partitions' bitmaps."""

    fused = True

    def __init__(self, torch_mod, parts):
        super().__init__(torch_mod)
        bufs = [p.peer_buffers() for p in parts]
        for r, p in enumerate(parts):
            p.set_peers(bufs, r)


class DistPeerExchange:
    """Fused exchange, one partition per process (one GPU each): peers'
    bitmaps and mailboxes are mapped by CUDA IPC (handles travel once over
    torch.distributed); per level each rank's kernel stores its slice into
    every peer's bitmap over NVLink -- no NCCL call on the data path."""

    fused = True

    def __init__(self, torch_mod, dist_mod, part, group=None):
        self.torch, self.dist, self.group = torch_mod, dist_mod, group
        self.world = dist_mod.get_world_size(group)
        rank = dist_mod.get_rank(group)
        handles = [None] * self.world
        dist_mod.all_gather_object(handles, part.ipc_export(), group=group)
        part.ipc_open(handles, rank)
        dist_mod.barrier(group=group)

    def max_over_ranks(self, x: float) -> float:
        return DistExchange.max_over_ranks(self, x)

    def gather_depths(self, slices, bounds, n: int):
        return DistExchange.gather_depths(self, slices, bounds, n)


class DistExchange:
    """One partition per process; all-gather over torch.distributed (NCCL
    between GPUs, gloo in CPU tests)."""

    def __init__(self, torch_mod, dist_mod, group=None):
        self.torch, self.dist, self.group = torch_mod, dist_mod, group
        self.world = dist_mod.get_world_size(group)

    def allgather(self, sends: Sequence):
        (send,) = sends
        out = self.torch.empty(self.world * send.numel(), dtype=send.dtype, device=send.device)
        self.dist.all_gather_into_tensor(out, send, group=self.group)
        return out

    def max_over_ranks(self, x: float) -> float:
        t = self.torch.tensor([x], dtype=self.torch.float64,
                              device="cuda" if self.torch.cuda.is_available() and
                              self.dist.get_backend(self.group) == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def gather_depths(self, slices: Sequence, bounds, n: int):
        (mine,) = slices
        width = int(np.max(np.diff(bounds)))
        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        buf = self.torch.full((width,), -1, dtype=self.torch.int32, device=dev)
        buf[:mine.size] = self.torch.from_numpy(np.ascontiguousarray(mine)).to(dev)
        out = self.torch.empty(self.world * width, dtype=self.torch.int32, device=dev)
        self.dist.all_gather_into_tensor(out, buf, group=self.group)
        allv = out.cpu().numpy().reshape(self.world, width)
        return np.concatenate([allv[r, :bounds[r + 1] - bounds[r]] for r in range(self.world)])


class PartitionedBFS:
    """Vertex-partitioned bfs_full / adaptive_bfs over the partitions this
    process drives (one per process under torch.distributed, or all P in
    one process on one GPU).

    `parts` must cover this process's share of `bounds` in rank order; the
    send buffers come from `alloc(stride)` (device tensors in production).
    """

    def __init__(self, parts: Sequence, bounds, exchange, alloc, stream=None):
        self.parts = list(parts)
        self.bounds = np.asarray(bounds, dtype=np.int64)
        self.n = int(self.bounds[-1])
        self.wbounds = word_bounds(self.bounds)
        self.stride = int(np.max(np.diff(self.wbounds))) if self.bounds.size > 1 else 0
        self.stride = max(self.stride, 1)
        self.exchange = exchange
        self.fused = bool(getattr(exchange, "fused", False))
        self.sends = [] if self.fused else [alloc(self.stride) for _ in self.parts]
        # fused exchange over engine partitions: whole traversals run in C
        # (abfs_parts_*), no Python between levels
        self.native = self.fused and all(isinstance(p, DevicePartition) for p in self.parts)
        # one partition per process (one per GPU): the whole per-rank level
        # loop, exchange included, runs in one persistent kernel
        self.persistent = self.native and len(self.parts) == 1
        self.stream = stream
        self.last_local_counts: list[list[int]] = []
        # optional: CUDA-event time of the all-gathers (bench NVLink figure)
        self.time_exchange = False
        self.exchange_ms = 0.0
        self.exchange_calls = 0

    # -- one level ------------------------------------------------------------
    def _level(self, level: int, kernel: int, variant: int, chunk: int):
        if self.fused:
            for p in self.parts:
                p.level_p2p(level, kernel, variant, chunk)
            res = [p.p2p_finish() for p in self.parts]
            counts = {r[0] for r in res}
            if len(counts) != 1:
                raise RuntimeError(f"partitions disagree on the level count: {sorted(counts)}")
            self.last_local_counts.append([r[1] for r in res])
            return res[0][0], max(r[2] for r in res)
        for p, s in zip(self.parts, self.sends):
            p.level(level, kernel, variant, chunk, s)
        if self.time_exchange:
            import torch
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        gathered = self.exchange.allgather(self.sends)
        if self.time_exchange:
            ev[1].record()
        res = [p.exchange(gathered, self.wbounds, self.stride) for p in self.parts]
        if self.time_exchange:
            self.exchange_ms += ev[0].elapsed_time(ev[1])
            self.exchange_calls += 1
        counts = {r[0] for r in res}
        if len(counts) != 1:
            raise RuntimeError(f"partitions disagree on the level count: {sorted(counts)}")
        self.last_local_counts.append([r[1] for r in res])
        return res[0][0], max(r[2] for r in res)

    def _init(self, root: int):
        if not 0 <= root < self.n:
            raise ValueError(f"root {root} out of range for |V|={self.n}")
        self.last_local_counts = []
        for p in self.parts:
            p.init(root)

    # -- reference-shaped entry points ------------------------------------------
    def _native_records(self, fn, *args, single=False):
        cap = 1 << 16
        if getattr(self, "_native_buf", None) is None:
            self._native_buf = ((L.AbfsLevelRecord * cap)(),
                                np.zeros(cap * len(self.parts), np.uint64))
        recs, loc = self._native_buf
        nl = ctypes.c_size_t()
        if single:   # one partition per process: the persistent per-rank loop
            L.check(fn(self.parts[0]._h, *args, recs, L.ptr(loc, L.u64p), cap, ctypes.byref(nl)),
                    fn.__name__)
        else:
            handles = (ctypes.c_void_p * len(self.parts))(*[p._h.value for p in self.parts])
            L.check(fn(handles, len(self.parts), *args, recs, L.ptr(loc, L.u64p), cap,
                       ctypes.byref(nl)), fn.__name__)
        k = min(nl.value, cap)
        self.last_local_counts = loc[:k * len(self.parts)].reshape(k, len(self.parts)).tolist()
        return [L.AbfsLevelRecord.from_buffer_copy(r) for r in recs[:k]]

    def bfs_full(self, root: int, kernel: KernelId, variant: CountVariant,
                 chunk_size: int = GROUP_SIZE) -> list[LevelOutcome]:
        """bfs_full (kernels.py:356-371) over the partitions; depths stay
        distributed (see `depths`)."""
        if self.native:
            if not 0 <= root < self.n:
                raise ValueError(f"root {root} out of range for |V|={self.n}")
            if self.persistent:
                recs = self._native_records(L.lib().abfs_part_mega_bfs_full, int(root), int(kernel),
                                            int(variant), int(chunk_size), single=True)
            else:
                recs = self._native_records(L.lib().abfs_parts_bfs_full, int(root), int(kernel),
                                            int(variant), int(chunk_size))
            return [LevelOutcome(new_frontier_count=int(r.new_count), elapsed_ns=int(r.elapsed_ns))
                    for r in recs]
        self._init(root)
        outs = []
        level = 0
        while True:
            c, ns = self._level(level, int(kernel), int(variant), chunk_size)
            outs.append(LevelOutcome(new_frontier_count=int(c), elapsed_ns=int(ns)))
            if c == 0:
                return outs
            level += 1

    def adaptive(self, root: int, model, stats: GraphStats,
                 chunk_size: int = GROUP_SIZE) -> AdaptiveTrace:
        """adaptive_bfs (adaptive.py:83-129): features from the global counts,
        UNKNOWN falls back to the previous pair, seeded with DEFAULT_KERNEL."""
        if isinstance(model, FlatTree) and self.native:
            if not 0 <= root < self.n:
                raise ValueError(f"root {root} out of range for |V|={self.n}")
            from .features import static_vector
            st = np.ascontiguousarray(static_vector(stats), dtype=np.float64)
            if self.persistent:
                recs = self._native_records(L.lib().abfs_part_mega_adaptive_bfs, int(root),
                                            ctypes.byref(model.as_abfs()), L.ptr(st, L.f64p),
                                            int(chunk_size), single=True)
            else:
                recs = self._native_records(L.lib().abfs_parts_adaptive_bfs, int(root),
                                            ctypes.byref(model.as_abfs()), L.ptr(st, L.f64p),
                                            int(chunk_size))
            return AdaptiveTrace(tuple(
                LevelTrace(level=int(r.level), kernel=KernelId(r.kernel),
                           variant=CountVariant(r.variant), fallback_used=bool(r.fallback),
                           frontier_size=int(r.frontier_size), elapsed_ns=int(r.elapsed_ns),
                           prediction_ns=int(r.prediction_ns)) for r in recs))
        if isinstance(model, FlatTree):
            policy = lambda level, fv: predict(model, fv)  # noqa: E731
        else:
            policy = model
        self._init(root)
        records = []
        frontier, discovered, level = 1, 1, 0
        previous = DEFAULT_KERNEL
        while True:
            t0 = time.perf_counter_ns()
            fv = extract_runtime_features(stats, frontier, discovered)
            raw = policy(level, fv)
            pred_ns = time.perf_counter_ns() - t0
            fallback = raw is UNKNOWN
            pair = previous if fallback else raw
            c, ns = self._level(level, int(pair[0]), int(pair[1]), chunk_size)
            records.append(LevelTrace(level=level, kernel=KernelId(pair[0]),
                                      variant=CountVariant(pair[1]), fallback_used=fallback,
                                      frontier_size=frontier, elapsed_ns=int(ns),
                                      prediction_ns=max(pred_ns, 1)))
            previous = pair
            if c == 0:
                return AdaptiveTrace(tuple(records))
            frontier = int(c)
            discovered += int(c)
            level += 1

    def depths(self) -> np.ndarray:
        """The full depth array (gathered from every partition)."""
        slices = [p.read_depths() for p in self.parts]
        return self.exchange.gather_depths(slices, self.bounds, self.n)


def local_partitions(dgraph, parts: int, stream_ptr: int | None = None):
    """P DevicePartitions of one DeviceGraph on its GPU (edge-balanced)."""
    _, io = dgraph.offsets()
    bounds = edge_balanced_bounds(io, parts)
    ps = [DevicePartition(dgraph, int(bounds[i]), int(bounds[i + 1]), stream_ptr)
          for i in range(parts)]
    return ps, bounds


__all__ = ["ALIGN", "gen_spec", "gen_size", "gen_offsets", "edge_balanced_bounds", "word_bounds", "DevicePartition", "LocalExchange",
           "LocalPeerExchange", "DistExchange", "DistPeerExchange", "PartitionedBFS",
           "local_partitions"]
