"""numpy restatement of one rank's level of the 1-D vertex-partitioned BFS.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): the CPU gloo tests plug
this in as the local partition of paper_1708_01159_b200.partition's
PartitionedBFS driver, so the multi-process host logic (exchange, global
counts, tree decisions, fallback, termination) is checked without a GPU.

Level semantics from a consistent state (init_depths, kernels.py:134-140):
an owned vertex v joins level+1 iff depth[v] is INF and some in-edge u -> v
has u in the global frontier -- what every strategy computes
(_relax_from_edges kernels.py:196-209, _push_block :234-257, vertex pull
:270-300, _claim :177-193), restricted to destinations in [lo, hi).
"""

from __future__ import annotations

import numpy as np

INF = 2**31 - 1


def _pack(bits: np.ndarray, words: int) -> np.ndarray:
    pad = np.zeros(words * 32, dtype=bool)
    pad[:bits.size] = bits
    return np.packbits(pad, bitorder="little").view("<u4")


def _unpack(words: np.ndarray, nbits: int) -> np.ndarray:
    return np.unpackbits(np.ascontiguousarray(words, dtype="<u4").view(np.uint8),
                         bitorder="little")[:nbits].astype(bool)


class OraclePartition:
    def __init__(self, n: int, in_offsets, sources, lo: int, hi: int):
        self.n, self.lo, self.hi = int(n), int(lo), int(hi)
        io = np.asarray(in_offsets, dtype=np.int64)
        src = np.asarray(sources, dtype=np.int64)
        b, e = int(io[self.lo]), int(io[self.hi])
        self.r_src = src[b:e]
        self.r_own = np.repeat(np.arange(self.lo, self.hi, dtype=np.int64),
                               np.diff(io[self.lo:self.hi + 1]))
        self.nwl = (self.hi + 31) // 32 - self.lo // 32
        self.depth = np.full(self.hi - self.lo, INF, dtype=np.int32)
        self.frontier = np.zeros(self.n, dtype=bool)
        self.new = np.zeros(self.hi - self.lo, dtype=bool)

    def init(self, root: int):
        self.depth[:] = INF
        self.frontier[:] = False
        self.frontier[root] = True
        if self.lo <= root < self.hi:
            self.depth[root - self.lo] = 0

    def level(self, level: int, kernel: int, variant: int, chunk: int, send) -> None:
        hit = self.r_own[self.frontier[self.r_src]] - self.lo
        cand = np.zeros(self.hi - self.lo, dtype=bool)
        cand[hit] = True
        self.new = cand & (self.depth == INF)
        self.depth[self.new] = level + 1
        words = _pack(self.new, self.nwl)
        out = np.zeros(send.numel(), dtype=np.uint32)
        out[:words.size] = words
        send.copy_(_as_tensor(out, send))

    def exchange(self, gathered, wbounds, stride: int):
        g = gathered.cpu().numpy().view(np.uint32)
        wb = np.asarray(wbounds, dtype=np.int64)
        words = np.concatenate([g[r * stride: r * stride + (wb[r + 1] - wb[r])]
                                for r in range(wb.size - 1)])
        self.frontier = _unpack(words, self.n)
        return int(self.frontier.sum()), int(self.new.sum()), 1

    def read_depths(self) -> np.ndarray:
        return self.depth.copy()


def _as_tensor(arr: np.ndarray, like):
    import torch
    return torch.from_numpy(arr.view(np.int32)).to(like.device)
