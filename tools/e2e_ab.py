"""Per-call wall time of the public adaptive_bfs (host int32 depths) on
Kronecker-24 under environment settings, interleaved:

    python tools/e2e_ab.py "ABFS_SNAP_DIV=0" "ABFS_SNAP_DIV=8" ...
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_01159_b200 as P  # noqa: E402
from bench import default_model, pick_roots  # noqa: E402
from paper_1708_01159_b200 import DeviceGraph, Traversal  # noqa: E402

dg = DeviceGraph.rmat(24, 16 << 24, 1, symmetrize=True)
oo, _ = dg.offsets()
stats = P.compute_stats(dg)
flat = P.deserialize(default_model())
dg._scratch = Traversal(dg)
roots = pick_roots(oo, 64, 1)[:16]
settings = sys.argv[1:] or ["ABFS_SNAP_DIV=8"]
res = {s: [] for s in settings}
for r in roots[:3]:
    d, _ = P.adaptive_bfs(dg, r, flat, stats)
for rep in range(6):
    for s in settings:
        k, v = s.split("=", 1)
        os.environ[k] = v
        for r in roots:
            t0 = time.perf_counter()
            d, _ = P.adaptive_bfs(dg, r, flat, stats)
            res[s].append(time.perf_counter() - t0)
for s in settings:
    x = sorted(res[s])
    print(f"{s}: median {statistics.median(x) * 1e3:.3f} ms  p10 {x[len(x) // 10] * 1e3:.3f} ms")
