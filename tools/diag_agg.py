"""Where the switched K24 traversal spends its time over the 64 bench roots:
level time aggregated by strategy and frontier size (diagnostic)."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1708_01159_b200 as P
from paper_1708_01159_b200 import DeviceGraph, Traversal
from paper_1708_01159_b200.features import static_vector
from bench import pick_roots
KN = ["EDGE", "REV", "PUSH", "PULL", "PUSHW"]
arg = sys.argv[1] if len(sys.argv) > 1 else "24"
if arg == "er":
    dg = DeviceGraph.uniform(1 << 25, 1 << 30, 1)
else:
    scale = int(arg)
    dg = DeviceGraph.rmat(scale, 16 << scale, 1, symmetrize=True)
oo, _ = dg.offsets()
stats = P.compute_stats(dg)
flat = P.deserialize("models/gpu_tree.tree")
t = Traversal(dg)
roots = pick_roots(oo, 64, 1)
for r in roots[:4]:
    t.adaptive(r, flat.as_abfs(), static_vector(stats))
agg = collections.defaultdict(lambda: [0, 0])
total = 0
for r in roots:
    recs = t.adaptive(r, flat.as_abfs(), static_vector(stats))
    for x in recs:
        F = x.frontier_size
        b = "F<1e3" if F < 1000 else "F<1e5" if F < 100000 else "F<1e6" if F < 1000000 else "F>=1e6"
        key = (KN[x.kernel], b, "conv" if x.converted else "")
        agg[key][0] += x.elapsed_ns
        agg[key][1] += 1
        total += x.elapsed_ns
print(f"total level time over {len(roots)} roots: {total/1e3:.0f} us ({total/len(roots)/1e3:.1f} us/root)")
for k, (ns, c) in sorted(agg.items(), key=lambda z: -z[1][0]):
    print(f"{k[0]:6s} {k[1]:7s} {k[2]:5s} levels={c:4d} total={ns/1e3:9.0f}us share={ns/total:.3f} mean={ns/c/1e3:7.1f}us")
