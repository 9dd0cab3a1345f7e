import sys, os, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import golden_util as G
import paper_1708_01159_b200 as P
name = sys.argv[1] if len(sys.argv) > 1 else "kron10"
n, m, a = G.graph_arrays(name)
g = P.Graph(n, m, *[a[k].copy() for k in G.ARRAYS])
for r in G.roots(name):
    for k, v in P.ALL_PAIRS:
        print(name, r, k.name, v.name, end=" ", flush=True)
        t0 = time.time()
        d, outs = P.bfs_full(g, r, k, v)
        print([o.new_frontier_count for o in outs] == G.counts(name, r).tolist(), round(time.time() - t0, 3), flush=True)
