import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import golden_util as G
import paper_1708_01159_b200 as P
from paper_1708_01159_b200 import DeviceGraph, Traversal
n, m, a = G.graph_arrays("kron10")
dg = DeviceGraph.upload(P.Graph(n, m, *[a[k].copy() for k in G.ARRAYS]))
t = Traversal(dg)
mode = int(sys.argv[1])
t.set_device_loop(mode)
print("V", n, "E", m, "mode", mode, flush=True)
for k, v in [(a_, b_) for a_ in (0, 1) for b_ in (0, 1, 2)]:
    c, el = t.bfs_full(G.roots("kron10")[0], k, v)
    print(k, v, c.tolist(), G.counts("kron10", G.roots("kron10")[0]).tolist(), flush=True)
