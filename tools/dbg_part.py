import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import golden_util as G
import paper_1708_01159_b200 as P
from paper_1708_01159_b200 import DeviceGraph
from paper_1708_01159_b200.partition import LocalExchange, PartitionedBFS, local_partitions
n, m, a = G.graph_arrays("kron10")
dg = DeviceGraph.upload(P.Graph(n, m, *[a[k].copy() for k in G.ARRAYS]))
stream = torch.cuda.current_stream().cuda_stream
for seq in ([(1,0)], [(0,0),(1,0)], [(0,2),(1,0)], [(1,1)], [(3,0),(1,0)]):
    ps, bounds = local_partitions(dg, 1, stream)
    bfs = PartitionedBFS(ps, bounds, LocalExchange(torch), alloc=lambda s: torch.zeros(s, dtype=torch.int32, device="cuda"))
    for k, v in seq:
        outs = bfs.bfs_full(0, k, v)
        print(seq, (k, v), [o.new_frontier_count for o in outs], bfs.last_local_counts, "want", G.counts("kron10", 0).tolist())
