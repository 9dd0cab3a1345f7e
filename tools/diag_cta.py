"""Per-level CTA finish-time spread inside the megakernel (diagnostic build):

    tools/build_variant.sh diag -DABFS_DIAG_CTA
    ABFS_LIB=build/diag.so python tools/diag_cta.py [scale] [roots]

For each level of a tree-switched BFS: level start (record t_start), the
spread of the CTAs' light-pass end times (min / median / p90 / max, us after
start) and of the unit-pass end -- i.e. how much of the level the grid idles
at its barriers because of load imbalance."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_01159_b200 as P  # noqa: E402
from bench import default_model, pick_roots  # noqa: E402
from paper_1708_01159_b200 import DeviceGraph, Traversal, _lib  # noqa: E402
from paper_1708_01159_b200.features import static_vector  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
nroots = int(sys.argv[2]) if len(sys.argv) > 2 else 3
graph = os.environ.get("ABFS_DIAG_GRAPH", "kron")
if graph == "er":
    dg = DeviceGraph.uniform(1 << 25, 1 << 30, 1)
elif graph == "mesh":
    dg = DeviceGraph.mesh(4096, 4096)
else:
    dg = DeviceGraph.rmat(scale, 16 << scale, 1, symmetrize=True)
oo, _ = dg.offsets()
st = static_vector(P.compute_stats(dg))
tree = P.deserialize(default_model()).as_abfs()
t = Traversal(dg)
lib = _lib.lib()
buf = np.zeros(128 * 1024, np.uint64)
KN = ["EDGE", "REV", "PUSH", "PULL", "PUSHW"]
for r in pick_roots(oo, 64, 1)[:nroots]:
    t.adaptive(r, tree, st, 32)
    ctypes.CDLL(_lib.LIB_PATH).abfs_debug_diag_cta(buf.ctypes.data_as(ctypes.c_void_p))   # clear
    recs = t.adaptive(r, tree, st, 32)
    ctypes.CDLL(_lib.LIB_PATH).abfs_debug_diag_cta(buf.ctypes.data_as(ctypes.c_void_p))
    print(f"root {r}")
    # the records' t_start is not exported; use the previous level's unit-pass end max
    prev_end = None
    for x in recs:
        L = x.level
        a = buf[(2 * L) * 1024:(2 * L) * 1024 + 1024].astype(np.int64)
        b = buf[(2 * L + 1) * 1024:(2 * L + 1) * 1024 + 1024].astype(np.int64)
        a, b = a[a > 0], b[b > 0]
        if not a.size:
            continue
        base = int(a.min()) if prev_end is None else prev_end
        pa = (np.percentile(a - base, [0, 50, 90, 100]) / 1e3).round(1)
        pb = (np.percentile(b - base, [0, 50, 90, 100]) / 1e3).round(1) if b.size else None
        print(f"  L{L} {KN[x.kernel]}/{x.variant} F={x.frontier_size} new={x.new_count} "
              f"level {x.elapsed_ns / 1e3:.1f}us | light end min/med/p90/max {pa.tolist()} | "
              f"units end {pb.tolist() if pb is not None else '-'}")
        prev_end = int(b.max()) if b.size else int(a.max())
