"""e2e breakdown of the public adaptive_bfs call at K24 (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1708_01159_b200 as P
from paper_1708_01159_b200 import DeviceGraph, Traversal
from bench import pick_roots
dg = DeviceGraph.rmat(24, 16 << 24, 1, symmetrize=True)
oo, _ = dg.offsets()
stats = P.compute_stats(dg)
flat = P.deserialize("models/gpu_tree.tree")
roots = pick_roots(oo, 64, 1)
dg._scratch = Traversal(dg)
for r in roots[:2]:
    P.adaptive_bfs(dg, r, flat, stats)
ts = []
for r in roots[:16]:
    t0 = time.perf_counter()
    d, tr = P.adaptive_bfs(dg, r, flat, stats)
    ts.append((time.perf_counter() - t0) * 1e3)
print("adaptive_bfs ms:", np.round(ts, 2).tolist())
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for r in roots[:8]:
    d, tr = P.adaptive_bfs(dg, r, flat, stats)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
