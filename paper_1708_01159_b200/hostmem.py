"""Recycled page-locked host arrays for depth results.

The reference returns a fresh int32[V] depth array per BFS
(kernels.py:356-371, adaptive.py:83-129).  At Kronecker scale 24 that is
64 MiB per call: a fresh numpy allocation costs ~16k first-touch page faults
plus a staged (pageable) copy.  `depth_array(n)` instead hands out an
ordinary writable numpy array whose memory is an anonymous huge-page mapping
registered with CUDA (so the read-back is direct DMA), and returns the
mapping to a small pool once the array -- and every view of it -- is
garbage.  Semantics are unchanged: each call gets memory no live array uses.
"""

from __future__ import annotations

import ctypes
import mmap
import threading
import weakref

import numpy as np

from . import _lib as L

MIN_POOLED_BYTES = 4 << 20     # smaller results use plain numpy arrays
_HUGE = 2 << 20
_KEEP_PER_SIZE = 4

_lock = threading.Lock()
_free: dict[int, list] = {}


class _Mapping:
    __slots__ = ("mm", "addr", "size", "registered")

    def __init__(self, size: int):
        self.size = size
        self.mm = mmap.mmap(-1, size)
        if hasattr(mmap, "MADV_HUGEPAGE"):
            try:
                self.mm.madvise(mmap.MADV_HUGEPAGE)
            except OSError:
                pass
        self.addr = ctypes.addressof(ctypes.c_char.from_buffer(self.mm))
        ctypes.memset(self.addr, 0, size)   # fault the pages in once
        self.registered = L.lib().abfs_host_register(ctypes.c_void_p(self.addr), size) == L.ABFS_OK


def _release(size: int, m: _Mapping) -> None:
    with _lock:
        lst = _free.setdefault(size, [])
        if len(lst) < _KEEP_PER_SIZE:
            lst.append(m)
            return
    if m.registered:
        L.lib().abfs_host_unregister(ctypes.c_void_p(m.addr))


def depth_array(n: int) -> np.ndarray:
    """A writable int32[n] array for a depth read-back (pooled when large)."""
    nbytes = 4 * n
    if nbytes < MIN_POOLED_BYTES:
        return np.empty(n, dtype=np.int32)
    size = (nbytes + _HUGE - 1) // _HUGE * _HUGE
    with _lock:
        lst = _free.get(size)
        m = lst.pop() if lst else None
    if m is None:
        m = _Mapping(size)
    owner = (ctypes.c_int32 * n).from_address(m.addr)
    owner._mapping = m                       # keep the mapping alive with the owner
    weakref.finalize(owner, _release, size, m)
    return np.ctypeslib.as_array(owner)


__all__ = ["depth_array", "MIN_POOLED_BYTES"]
