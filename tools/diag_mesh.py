"""Mesh: switched vs fixed per-level times for one root (diagnostic)."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1708_01159_b200 as P
from paper_1708_01159_b200 import DeviceGraph, Traversal
from paper_1708_01159_b200.features import static_vector
from bench import pick_roots
dg = DeviceGraph.mesh(4096, 4096)
oo, _ = dg.offsets()
stats = P.compute_stats(dg)
flat = P.deserialize("models/gpu_tree.tree")
t = Traversal(dg)
r = pick_roots(oo, 64, 1)[0]
recs = t.adaptive(r, flat.as_abfs(), static_vector(stats))
recs = t.adaptive(r, flat.as_abfs(), static_vector(stats))
sw = np.array([x.elapsed_ns for x in recs])
pairs = collections.Counter((x.kernel, x.variant) for x in recs)
print("root", r, "levels", len(recs), "switched sum us", sw.sum() / 1e3, "last_ns", t.last_ns() / 1e3, pairs)
for k, v in [(4, 1), (4, 2), (2, 1), (2, 2)]:
    c, el = t.bfs_full(r, k, v)
    c, el = t.bfs_full(r, k, v)
    print((k, v), "sum us", el.sum() / 1e3, "last_ns", t.last_ns() / 1e3, "median level", np.median(el) / 1e3)
print("switched median level", np.median(sw) / 1e3, "median prediction ns", np.median([x.prediction_ns for x in recs]))
# per-level comparison vs fixed PUSHW/2 for the levels the tree ran as PUSHW/2
c, el = t.bfs_full(r, 4, 2)
m = np.array([(x.kernel, x.variant) == (4, 2) for x in recs])
print("PUSHW/2 levels in switched:", m.sum(), "switched", sw[m].sum() / 1e3, "fixed same levels", el[m].sum() / 1e3)
# levels the tree ran as PUSH/GROUP vs the fixed PUSH/GROUP run, and the rest
c, el = t.bfs_full(r, 2, 1)
m = np.array([(x.kernel, x.variant) == (2, 1) for x in recs])
print("PUSH/1 levels in switched:", m.sum(), "switched", sw[m].sum() / 1e3, "fixed same levels", el[m].sum() / 1e3,
      "| other levels: switched", sw[~m].sum() / 1e3, "fixed PUSH/1", el[~m].sum() / 1e3,
      "levels", np.flatnonzero(~m)[:20], "frontiers", [recs[i].frontier_size for i in np.flatnonzero(~m)[:20]])
