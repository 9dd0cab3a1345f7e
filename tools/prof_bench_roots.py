"""The bench's tree-switched traversals (same graph, tree and first roots) on
the per-level launch path, so ncu sees each level's kernels separately
(profiling helper for profiles/: per-level DRAM traffic of each strategy)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_01159_b200 as P  # noqa: E402
from bench import pick_roots  # noqa: E402
from paper_1708_01159_b200 import DeviceGraph, Traversal  # noqa: E402
from paper_1708_01159_b200.features import static_vector  # noqa: E402

n_roots = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dg = DeviceGraph.rmat(24, 16 << 24, 1, symmetrize=True)
oo, _ = dg.offsets()
stats = P.compute_stats(dg)
flat = P.deserialize(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                  "models", "gpu_tree.tree"))
t = Traversal(dg)
t.set_device_loop(0)
for r in pick_roots(oo, 64, seed=1)[:n_roots]:
    recs = t.adaptive(r, flat.as_abfs(), static_vector(stats), 32)
    print(r, [(x.kernel, x.variant, x.frontier_size, x.elapsed_ns) for x in recs])
