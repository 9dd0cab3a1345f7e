"""Mesh 4096^2: which pairs the tree picks per level (switched run) and how
each level's time compares with the same level under fixed PUSH/GROUP."""
import collections
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_01159_b200 as P  # noqa: E402
from bench import default_model  # noqa: E402
from paper_1708_01159_b200 import DeviceGraph, Traversal  # noqa: E402
from paper_1708_01159_b200.features import static_vector  # noqa: E402

dg = DeviceGraph.mesh(4096, 4096)
st = static_vector(P.compute_stats(dg))
tree = P.deserialize(default_model()).as_abfs()
t = Traversal(dg)
KN = ["EDGE", "REV", "PUSH", "PULL", "PUSHW"]
for r in (0, 4096 * 2048 + 2048):
    t.adaptive(r, tree, st, 32)
    recs = t.adaptive(r, tree, st, 32)
    sw = np.array([x.elapsed_ns for x in recs], np.float64)
    t.bfs_full(r, 2, 1, 32)
    _, fx = t.bfs_full(r, 2, 1, 32)
    fx = np.asarray(fx, np.float64)[:len(sw)]
    by = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for x, a, b in zip(recs, sw, fx):
        k = (KN[x.kernel], x.variant, "solo" if x.frontier_size <= 4096 else "grid")
        by[k][0] += 1
        by[k][1] += a
        by[k][2] += b
    print(f"root {r}: switched {sw.sum() / 1e6:.2f} ms, PUSH/GROUP {fx.sum() / 1e6:.2f} ms")
    for k, (n, a, b) in sorted(by.items(), key=lambda kv: -kv[1][1]):
        print(f"   {k}: levels {n}  switched {a / 1e3:9.1f} us  push/group {b / 1e3:9.1f} us")
