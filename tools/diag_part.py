"""Per-level trace of the partitioned BFS vs the single-GPU engine (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1708_01159_b200 as P
from paper_1708_01159_b200 import DeviceGraph, Traversal
from paper_1708_01159_b200.features import static_vector
from paper_1708_01159_b200.partition import LocalExchange, PartitionedBFS, local_partitions
KN = ["EDGE", "REV", "PUSH", "PULL", "PUSHW"]
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
parts = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dg = DeviceGraph.rmat(scale, 16 << scale, 1, symmetrize=True)
stats = P.compute_stats(dg)
flat = P.deserialize("models/gpu_tree.tree")
t = Traversal(dg)
for r in (1, 123457):
    recs = t.adaptive(r, flat.as_abfs(), static_vector(stats), 32)
    recs = t.adaptive(r, flat.as_abfs(), static_vector(stats), 32)
    print("single", r, t.last_ns() / 1e3, "us")
    for x in recs:
        print(f"   L{x.level} {KN[x.kernel]}/{x.variant} F={x.frontier_size} new={x.new_count} {x.elapsed_ns/1e3:.1f}us")
t.close()
ps, bounds = local_partitions(dg, parts, torch.cuda.current_stream().cuda_stream)
bfs = PartitionedBFS(ps, bounds, LocalExchange(torch), alloc=lambda s: torch.zeros(s, dtype=torch.int32, device="cuda"))
for r in (1, 123457):
    bfs.adaptive(r, flat, stats)
    w0 = time.perf_counter()
    tr = bfs.adaptive(r, flat, stats)
    print("partitioned", parts, r, (time.perf_counter() - w0) * 1e3, "ms wall")
    for x in tr.records:
        print(f"   L{x.level} {x.kernel.name}/{int(x.variant)} F={x.frontier_size} {x.elapsed_ns/1e3:.1f}us")
