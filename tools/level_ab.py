"""Per-level device times of tree-switched BFSs under several environment
settings (A/B of engine knobs read per call, e.g. ABFS_RED_*):

    python tools/level_ab.py [--graph kron|er|mesh] [--roots N] "ENV=a" "ENV=b;ENV2=c" ...

Prints, per root and level, the pair, frontier and each setting's level time."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_01159_b200 as P  # noqa: E402
from bench import default_model, pick_roots  # noqa: E402
from paper_1708_01159_b200 import DeviceGraph, Traversal  # noqa: E402
from paper_1708_01159_b200.features import static_vector  # noqa: E402

KN = ["EDGE", "REV", "PUSH", "PULL", "PUSHW"]
ap = argparse.ArgumentParser()
ap.add_argument("--graph", default="kron")
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--roots", type=int, default=8)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("settings", nargs="+")
a = ap.parse_args()
if a.graph == "er":
    dg = DeviceGraph.uniform(1 << 25, 1 << 30, 1)
elif a.graph == "mesh":
    dg = DeviceGraph.mesh(4096, 4096)
else:
    dg = DeviceGraph.rmat(a.scale, 16 << a.scale, 1, symmetrize=True)
oo, _ = dg.offsets()
st = static_vector(P.compute_stats(dg))
tree = P.deserialize(default_model()).as_abfs()
t = Traversal(dg)
roots = pick_roots(oo, 64, 1)[:a.roots]
res = {}
for s in a.settings:
    kv = dict(x.split("=", 1) for x in s.split(";"))   # "A=1;B=2" sets several
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update(kv)
    for r in roots:
        t.adaptive(r, tree, st, 32)
        best = None
        for _ in range(a.reps):
            recs = t.adaptive(r, tree, st, 32)
            ns = np.array([x.elapsed_ns for x in recs], np.float64)
            best = ns if best is None else np.minimum(best, ns)
        res[(s, r)] = (recs, best)
    for k, v in old.items():
        if v is None:
            del os.environ[k]
        else:
            os.environ[k] = v
tot = {s: 0.0 for s in a.settings}
for r in roots:
    recs0 = res[(a.settings[0], r)][0]
    print(f"root {r}")
    for i, x in enumerate(recs0):
        ts = [res[(s, r)][1][i] / 1e3 if i < len(res[(s, r)][1]) else float("nan") for s in a.settings]
        print(f"  L{x.level} {KN[x.kernel]}/{x.variant} F={x.frontier_size} new={x.new_count} " +
              " ".join(f"{v:8.1f}" for v in ts))
    for s in a.settings:
        tot[s] += res[(s, r)][1].sum() / 1e3
print("total us:", {s: round(v, 1) for s, v in tot.items()})
