"""Level-synchronous BFS kernels: 5 strategies x 3 frontier-count variants.

Same names, signatures, argument meaning and error texts as
/root/reference/pkg/src/adaptive_bfs/kernels.py; every level runs as
hand-written sm_100a CUDA in libabfs.so (paper_1708_01159_b200/csrc/):

  EDGE_LIST         k_edge<.., false>  item per forward slot     (kernels.py:212-219)
  REV_EDGE_LIST     k_edge<.., true>   item per reverse slot     (kernels.py:222-231)
  VERTEX_PUSH       k_push             thread per frontier vertex (kernels.py:260-267)
  VERTEX_PULL       k_pull             warp per 32-vertex word    (kernels.py:270-300)
  VERTEX_PUSH_WARP  k_push_warp+k_heavy virtual warp + CTA units (kernels.py:303-322)

  DIRECT_ATOMIC / GROUP_REDUCE / TWO_LEVEL_REDUCE are the count epilogues
  (1 atomic per discovery / per warp / per CTA; kernels.py:143-170).

`run_level` mutates the caller's host depth array in place, exactly like the
reference (H2D -> level on the GPU -> D2H).  `bfs_full` keeps the state in
HBM for the whole traversal and copies the depths back once.
"""

from __future__ import annotations

import ctypes
import threading
from collections import deque
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from .hostmem import depth_array
from . import _lib as L

INF_DEPTH = np.iinfo(np.int32).max
DEPTH_DTYPE = np.int32

#: Work-item group width of the hierarchical count reductions and the
#: default virtual-warp width (kernels.py:33-35).
GROUP_SIZE = 32


class KernelId(IntEnum):
    EDGE_LIST = 0
    REV_EDGE_LIST = 1
    VERTEX_PUSH = 2
    VERTEX_PULL = 3
    VERTEX_PUSH_WARP = 4


class CountVariant(IntEnum):
    DIRECT_ATOMIC = 0
    GROUP_REDUCE = 1
    TWO_LEVEL_REDUCE = 2


ALL_PAIRS: tuple[tuple[KernelId, CountVariant], ...] = tuple(
    (k, v) for k in KernelId for v in CountVariant)


def pair_index(kernel: KernelId, variant: CountVariant) -> int:
    return int(kernel) * len(CountVariant) + int(variant)


def pair_from_index(index: int) -> tuple[KernelId, CountVariant]:
    return ALL_PAIRS[index]


@dataclass(frozen=True)
class LevelOutcome:
    new_frontier_count: int
    elapsed_ns: int


_worker_count = 1


def set_worker_count(count: int) -> None:
    """API parity with kernels.py:88-97.  The GPU engine sizes its grids from
    the SM count; the value is validated and recorded but does not change
    the schedule (schedules never change results)."""
    global _worker_count
    if count < 1:
        raise ValueError("worker count must be >= 1")
    _worker_count = int(count)


def worker_count() -> int:
    return _worker_count


_foreign_uploads: dict = {}
_foreign_lock = threading.Lock()


def _device(graph):
    """DeviceGraph for a host Graph (cached upload), a DeviceGraph, or any
    object with the reference Graph's fields (e.g. an adaptive_bfs.Graph).

    A foreign graph's upload is cached under id(graph) together with a weak
    reference to it, and evicted when the graph is collected; every hit is
    checked against the weak reference, so a recycled id never maps to
    another graph's device copy.  Objects that cannot be weakly referenced
    are uploaded per call (correct, uncached)."""
    if hasattr(graph, "device_graph"):
        return graph.device_graph()
    if hasattr(graph, "out_offsets") and hasattr(graph, "sources"):
        import weakref
        from .engine import DeviceGraph
        key = id(graph)
        with _foreign_lock:
            hit = _foreign_uploads.get(key)
            if hit is not None and hit[0]() is graph:
                return hit[1]
        try:
            ref = weakref.ref(graph)
        except TypeError:
            return DeviceGraph.upload(graph)
        dg = DeviceGraph.upload(graph)
        with _foreign_lock:
            _foreign_uploads[key] = (ref, dg)
        weakref.finalize(graph, _evict_foreign, key, ref)
        return dg
    return graph


def _evict_foreign(key, ref) -> None:
    with _foreign_lock:
        hit = _foreign_uploads.get(key)
        if hit is not None and hit[0] is ref:
            del _foreign_uploads[key]


def _check_root(graph, root: int) -> None:
    if not 0 <= root < graph.vertex_count:
        raise ValueError(f"root {root} out of range for |V|={graph.vertex_count}")


def init_depths(graph, root: int) -> np.ndarray:
    """INF everywhere except depth 0 at root (kernels.py:134-140), built on
    the device and copied back."""
    _check_root(graph, root)
    with _device(graph).borrow() as t:
        t.init(root)
        return t.read(depth_array(graph.vertex_count))


def aggregate_count(local_counts, variant: CountVariant) -> int:
    """Exact total of per-item counts with the variant's reduction shape
    (kernels.py:143-161), computed by the device count kernels."""
    counts = np.ascontiguousarray(np.asarray(local_counts, dtype=np.int64).ravel())
    if int(variant) not in (0, 1, 2):
        raise ValueError(f"unknown count variant {variant!r}")
    total = ctypes.c_int64()
    L.check(L.lib().abfs_aggregate_count(0, L.ptr(counts, L.i64p), counts.size, int(variant),
                                         ctypes.byref(total)), "aggregate_count")
    return int(total.value)


def _validate(kernel, variant, chunk_size) -> tuple[int, int]:
    try:
        k = int(KernelId(kernel))
    except ValueError:
        raise ValueError(f"unknown kernel {kernel!r}") from None
    try:
        v = int(CountVariant(variant))
    except ValueError:
        raise ValueError(f"unknown count variant {variant!r}") from None
    if k == KernelId.VERTEX_PUSH_WARP and chunk_size < 1:
        raise ValueError("chunk_size must be >= 1")
    return k, v


def run_level(graph, depths: np.ndarray, level: int, kernel: KernelId,
              variant: CountVariant, chunk_size: int = GROUP_SIZE) -> LevelOutcome:
    """Run one level on the GPU and update `depths` in place (kernels.py:340-353).

    `depths` may be any caller-built array (tests/test_kernels.py:209-236);
    int32 C-contiguous arrays are transferred directly, other integer dtypes
    (duck typing, e.g. int64) through an int32 staging copy.
    """
    k, v = _validate(kernel, variant, chunk_size)
    with _device(graph).borrow() as t:
        if (isinstance(depths, np.ndarray) and depths.dtype == np.int32
                and depths.flags.c_contiguous and depths.flags.writeable):
            c, el = t.run_level_host(depths, level, k, v, chunk_size)
        else:
            stage = np.ascontiguousarray(depths, dtype=np.int32)
            c, el = t.run_level_host(stage, level, k, v, chunk_size)
            depths[...] = stage
    return LevelOutcome(new_frontier_count=int(c), elapsed_ns=int(el))


def run_level_edge_list(graph, depths, level, variant) -> LevelOutcome:
    return run_level(graph, depths, level, KernelId.EDGE_LIST, variant)


def run_level_rev_edge_list(graph, depths, level, variant) -> LevelOutcome:
    return run_level(graph, depths, level, KernelId.REV_EDGE_LIST, variant)


def run_level_vertex_push(graph, depths, level, variant) -> LevelOutcome:
    return run_level(graph, depths, level, KernelId.VERTEX_PUSH, variant)


def run_level_vertex_pull(graph, depths, level, variant) -> LevelOutcome:
    return run_level(graph, depths, level, KernelId.VERTEX_PULL, variant)


def run_level_push_warp(graph, depths, level, variant,
                        chunk_size: int = GROUP_SIZE) -> LevelOutcome:
    if chunk_size < 1:
        raise ValueError("chunk_size must be >= 1")
    return run_level(graph, depths, level, KernelId.VERTEX_PUSH_WARP, variant, chunk_size)


def bfs_full(graph, root: int, kernel: KernelId, variant: CountVariant,
             chunk_size: int = GROUP_SIZE) -> tuple[np.ndarray, list[LevelOutcome]]:
    """Levels until one discovers nothing; the terminating zero level is run
    and recorded (kernels.py:356-371).  State stays in HBM throughout."""
    _check_root(graph, root)
    k, v = _validate(kernel, variant, chunk_size)
    depths = depth_array(graph.vertex_count)
    with _device(graph).borrow() as t:
        counts, elapsed = t.bfs_full(root, k, v, chunk_size, depths_out=depths)
    return depths, [LevelOutcome(int(c), int(e)) for c, e in zip(counts, elapsed)]


def reference_bfs(graph, root: int) -> np.ndarray:
    """The reference's sequential FIFO correctness oracle (kernels.py:374-391),
    kept for API parity.  The engine never calls it."""
    _check_root(graph, root)
    depths = np.full(graph.vertex_count, INF_DEPTH, dtype=DEPTH_DTYPE)
    depths[root] = 0
    offsets = graph.out_offsets.tolist()
    dest = graph.destinations.tolist()
    queue = deque([root])
    while queue:
        u = queue.popleft()
        d = depths[u] + 1
        for e in range(offsets[u], offsets[u + 1]):
            w = dest[e]
            if depths[w] == INF_DEPTH:
                depths[w] = d
                queue.append(w)
    return depths
