"""Fixed edge-list levels: megakernel (mode 1) vs launch path (mode 0)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1708_01159_b200 import DeviceGraph, Traversal
dg = DeviceGraph.rmat(24, 16 << 24, 1, symmetrize=True)
t = Traversal(dg)
for mode in (1, 0):
    t.set_device_loop(mode)
    for k, v in [(0, 2), (1, 1)]:
        t.bfs_full(185441, k, v)
        c, el = t.bfs_full(185441, k, v)
        print("mode", mode, (k, v), (el / 1e3).round(1).tolist(), "total", round(el.sum() / 1e3, 1))
