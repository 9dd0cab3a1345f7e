import sys, os, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import golden_util as G
import paper_1708_01159_b200 as P
from paper_1708_01159_b200 import DeviceGraph, Traversal
name, mode, k, v = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
n, m, a = G.graph_arrays(name)
dg = DeviceGraph.upload(P.Graph(n, m, *[a[x].copy() for x in G.ARRAYS]))
t = Traversal(dg)
t.set_device_loop(mode)
print(name, "V", n, "E", m, flush=True)
for r in G.roots(name):
    t0 = time.time()
    c, el = t.bfs_full(r, k, v)
    print(r, c.tolist() == G.counts(name, r).tolist(), round(time.time() - t0, 4), (el / 1e3).round(1).tolist(), flush=True)
