"""Per-level device times: single-graph megakernel vs the persistent
partition loop with one partition (fused peer exchange), same graph, tree
and roots -- the partition machinery's own overhead, level by level.

    python tools/part_levels.py [scale] [roots]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_01159_b200 as P  # noqa: E402
from bench import default_model, pick_roots  # noqa: E402
from paper_1708_01159_b200 import DeviceGraph, Traversal  # noqa: E402
from paper_1708_01159_b200.features import static_vector  # noqa: E402
from paper_1708_01159_b200.partition import LocalPeerExchange, PartitionedBFS, local_partitions  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dg = DeviceGraph.rmat(scale, 16 << scale, 1, symmetrize=True)
oo, _ = dg.offsets()
stats = P.compute_stats(dg)
st = static_vector(stats)
flat = P.deserialize(default_model())
tree = flat.as_abfs()
t = Traversal(dg)
stream = torch.cuda.current_stream().cuda_stream
ps, bounds = local_partitions(dg, 1, stream)
bfs = PartitionedBFS(ps, bounds, LocalPeerExchange(torch, ps), alloc=None)
KN = ["EDGE", "REV", "PUSH", "PULL", "PUSHW"]
tot = [0.0, 0.0]
for r in pick_roots(oo, 64, 1)[24:24 + nr]:
    a = b = pb = None
    for _ in range(4):
        ra = t.adaptive(r, tree, st, 32)
        rb = bfs.adaptive(r, flat, stats).records
        ea = np.array([x.elapsed_ns for x in ra], float)
        eb = np.array([x.elapsed_ns for x in rb], float)
        ep = np.array([x.prediction_ns for x in rb], float)
        a = ea if a is None else np.minimum(a, ea)
        b = eb if b is None else np.minimum(b, eb)
        pb = ep if pb is None else np.minimum(pb, ep)
    print("root", r)
    for i, x in enumerate(ra):
        print(f"  L{i} {KN[x.kernel]}/{x.variant} F={x.frontier_size} single {a[i]/1e3:7.1f}  part {b[i]/1e3:7.1f} (t_pred {pb[i]/1e3:6.1f})")
    tot[0] += a.sum()
    tot[1] += b.sum()
print(f"total us single {tot[0]/1e3:.1f} partition(P=1) {tot[1]/1e3:.1f}")
