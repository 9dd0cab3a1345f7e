"""Run fixed-pair BFS traversals on the per-level launch path so ncu can
capture each level as its own kernel launch (profiling helper).

    ncu ... -k regex:k_pull python tools/prof_levels.py --pair 3 2 --scale 24
    ncu ... python tools/prof_levels.py --graph er --pair 4 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_01159_b200 import DeviceGraph, Traversal  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--pair", type=int, nargs=2, action="append", required=True)
ap.add_argument("--root", type=int, default=185441)
ap.add_argument("--graph", default="kron", choices=["kron", "er"])
a = ap.parse_args()
if a.graph == "er":   # config 5 (ER-32M); root 665133 is the bench's first
    dg = DeviceGraph.uniform(1 << 25, 1 << 30, 1)
    if a.root == 185441:
        a.root = 665133
else:
    dg = DeviceGraph.rmat(a.scale, 16 << a.scale, 1, symmetrize=True)
t = Traversal(dg)
t.set_device_loop(0)
for k, v in a.pair:
    counts, el = t.bfs_full(a.root, k, v)
    print(k, v, counts.tolist(), (el / 1e3).round(1).tolist())
