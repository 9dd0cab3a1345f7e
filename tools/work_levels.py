"""Per-level work model of tree-switched BFSs (instrumented replay): F, N, U,
EF, ES, algorithmic bytes (bench.py level_bytes) and achieved GB/s of each
level -- which levels hold the time and how far each is from the HBM roofline.

    python tools/work_levels.py [--graph kron|er|mesh] [--roots N]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_01159_b200 as P  # noqa: E402
from bench import KERNEL_NAMES, default_model, level_bytes, pick_roots  # noqa: E402
from paper_1708_01159_b200 import DeviceGraph, Traversal  # noqa: E402
from paper_1708_01159_b200.features import static_vector  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--graph", default="kron")
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--roots", type=int, default=4)
a = ap.parse_args()
if a.graph == "er":
    dg = DeviceGraph.uniform(1 << 25, 1 << 30, 1)
elif a.graph == "mesh":
    dg = DeviceGraph.mesh(4096, 4096)
else:
    dg = DeviceGraph.rmat(a.scale, 16 << a.scale, 1, symmetrize=True)
V, E = dg.vertex_count, dg.edge_count
oo, io = dg.offsets()
st = static_vector(P.compute_stats(dg))
tree = P.deserialize(default_model()).as_abfs()
t = Traversal(dg)
for r in pick_roots(oo, 64, 1)[:a.roots]:
    t.adaptive(r, tree, st, 32)
    recs = t.adaptive(r, tree, st, 32)              # timed (uninstrumented)
    t.instrument(True)
    t.adaptive(r, tree, st, 32)
    s = t.level_stats(len(recs))
    t.instrument(False)
    cnt, od, idg, es = s["count"], s["out_deg"], s["in_deg"], s["scanned"]
    print(f"root {r}")
    disc, unv_in = 0, int(idg.sum())
    for L, x in enumerate(recs):
        F = int(cnt[L])
        N = int(cnt[L + 1]) if L + 1 < len(recs) else 0
        disc += F
        unv_in -= int(idg[L])
        U = V - disc
        b = level_bytes(int(x.kernel), V, E, F, N, int(od[L]), U, unv_in, int(es[L]), bool(x.converted))
        print(f"  L{L} {KERNEL_NAMES[x.kernel]:>16}/{x.variant} F={F:>9} N={N:>9} U={U:>9} "
              f"EF={int(od[L]):>10} ES={int(es[L]):>10} {x.elapsed_ns / 1e3:7.1f}us "
              f"{b / 1e6:8.1f}MB {b / x.elapsed_ns:7.1f}GB/s")
