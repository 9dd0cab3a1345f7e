"""Mesh 4096^2 per-root device times (switched and two fixed pairs) for A/B
runs of alternative library builds (ABFS_LIB)."""
import os, sys
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
roots = pick_roots(oo, 64, 1)[:3]
out = {"switched": 0.0, (2, 1): 0.0, (2, 2): 0.0}
for r in roots:
    t.adaptive(r, flat.as_abfs(), static_vector(stats))
    out["switched"] += t.last_ns() / 1e3
    for kv in [(2, 1), (2, 2)]:
        t.bfs_full(r, *kv)
        out[kv] += t.last_ns() / 1e3
print(os.environ.get("ABFS_LIB", "default"), {str(k): round(v) for k, v in out.items()})
