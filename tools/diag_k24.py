"""Diagnostics on the GPU box: per-level records of the switched run, the
host gap between traversals, the e2e breakdown, and every fixed pair's
whole-BFS time (not a bench number).

    python tools/diag_k24.py --scale 24 --roots 4
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_01159_b200 as P  # noqa: E402
from paper_1708_01159_b200 import DeviceGraph, Traversal  # noqa: E402
from paper_1708_01159_b200.features import static_vector  # noqa: E402

KN = ["EDGE", "REV", "PUSH", "PULL", "PUSHW"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--roots", type=int, default=4)
    ap.add_argument("--model", default="models/gpu_tree.tree")
    ap.add_argument("--fixed", action="store_true")
    ap.add_argument("--mode", type=int, default=1)
    a = ap.parse_args()
    dg = DeviceGraph.rmat(a.scale, 16 << a.scale, 1, symmetrize=True)
    stats = P.compute_stats(dg)
    st = static_vector(stats)
    flat = P.deserialize(a.model)
    tree = flat.as_abfs()
    oo, _ = dg.offsets()
    deg = np.diff(oo.astype(np.int64))
    rng = np.random.default_rng(1)
    roots = sorted(int(x) for x in rng.choice(np.flatnonzero(deg > 0), 64, replace=False))[:a.roots]
    t = Traversal(dg)
    t.set_device_loop(a.mode)
    for r in roots[:2]:
        t.adaptive(r, tree, st)
    for r in roots:
        w0 = time.perf_counter()
        recs = t.adaptive(r, tree, st)
        wall = (time.perf_counter() - w0) * 1e6
        dev = t.last_ns() / 1e3
        print(f"root {r}: device {dev:.1f} us wall {wall:.1f} us levels {len(recs)}")
        for x in recs:
            print(f"   L{x.level} {KN[x.kernel]}/{x.variant} F={x.frontier_size} new={x.new_count} "
                  f"{x.elapsed_ns/1e3:.1f}us conv={x.converted}")
    # e2e breakdown
    d = np.empty(dg.vertex_count, np.int32)
    for k in range(3):
        w0 = time.perf_counter()
        t.read(d)
        print(f"read_depths pageable(reused): {(time.perf_counter()-w0)*1e3:.2f} ms")
    from paper_1708_01159_b200.hostmem import depth_array
    for k in range(4):
        w0 = time.perf_counter()
        x = depth_array(dg.vertex_count)
        w1 = time.perf_counter()
        t.read(x)
        w2 = time.perf_counter()
        print(f"depth_array alloc {(w1-w0)*1e3:.2f} ms read {(w2-w1)*1e3:.2f} ms")
        del x
    for k in range(4):
        w0 = time.perf_counter()
        dd, tr = P.adaptive_bfs(dg, roots[k % len(roots)], flat, stats)
        print(f"adaptive_bfs public call: {(time.perf_counter()-w0)*1e3:.2f} ms")
        del dd
    if a.fixed:
        for k, v in P.ALL_PAIRS:
            ts = []
            for r in roots:
                t.bfs_full(r, int(k), int(v))
                ts.append(t.last_ns() / 1e3)
            print(f"fixed {KN[int(k)]}/{int(v)}: " + " ".join(f"{x:.0f}" for x in ts) + " us")


if __name__ == "__main__":
    main()
