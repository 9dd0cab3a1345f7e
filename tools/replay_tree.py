"""Replay trees on a measured levels.csv (per graph: geomean tree/optimum and
best-single/tree), using the reference's own read_samples / FlatTree.

    python tools/replay_tree.py --levels L.csv --stats S.json tree1 tree2 ...
"""
import argparse, collections, json, math, sys
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, __file__.rsplit("/", 2)[0])
import adaptive_bfs as ab  # noqa: E402
from tools.train_tree import replay, stats_from_vec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--levels", required=True)
ap.add_argument("--stats", required=True)
ap.add_argument("trees", nargs="+")
a = ap.parse_args()
raw = ab.read_samples(a.levels)
with open(a.stats) as fh:
    stats_map = {k: stats_from_vec(v) for k, v in json.load(fh).items()}
table = {(s.graph_id, s.root, s.level, ab.pair_index(s.kernel, s.variant)): s.min_ns for s in raw}
levels = ab.training_samples_from(raw, stats_map, metric="min")
opt, single = {}, collections.defaultdict(lambda: collections.Counter())
for t in levels:
    key = (t.graph_id, t.root)
    opt[key] = opt.get(key, 0) + min(table[(t.graph_id, t.root, t.level, i)] for i in range(15))
    for i in range(15):
        single[key][i] += table[(t.graph_id, t.root, t.level, i)]
for path in a.trees:
    cost = replay(ab.deserialize(path), levels, table)
    g = collections.defaultdict(list)
    for k, c in cost.items():
        g[k[0]].append((c / opt[k], min(single[k].values()) / c))
    print(path, {k: (round(math.exp(sum(math.log(x) for x, _ in v) / len(v)), 3),
                     round(math.exp(sum(math.log(y) for _, y in v) / len(v)), 2)) for k, v in sorted(g.items())})
