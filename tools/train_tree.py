"""Train the GPU switching tree with the UNMODIFIED reference trainer.

Runs in the build container (the reference exists only here), on the
levels.csv + stats.json that tools/gpu_levels.py measured on a B200:

    PYTHONDONTWRITEBYTECODE=1 python tools/train_tree.py \
        --levels gpurun_out/levels.csv --stats gpurun_out/stats.json \
        --out models/gpu_tree.tree

Pipeline = the reference's own cmd_train path (src/cli.py:275-348):
read_samples -> training_samples_from (argmin labels, features.py:145-162)
-> split_train_test -> to_matrix -> fit -> evaluate -> flatten -> serialize.
It also prints, per (graph, root), the per-level optimum, the best single
pair and the tree's replayed choice cost (from the same measured table).
"""

from __future__ import annotations

import argparse
import json
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import adaptive_bfs as ab  # noqa: E402


def stats_from_vec(v):
    s = [ab.DegreeSummary(*v[6 + 6 * i: 12 + 6 * i]) for i in range(3)]
    return ab.GraphStats(int(v[0]), int(v[1]), s[0], s[1], s[2])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", required=True)
    ap.add_argument("--stats", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--max-depth", type=int, default=8)
    ap.add_argument("--min-leaf", type=int, default=2)
    ap.add_argument("--min-split", type=int, default=4)
    ap.add_argument("--metric", default="min")
    a = ap.parse_args()
    samples = ab.read_samples(a.levels)
    with open(a.stats) as fh:
        stats_map = {k: stats_from_vec(v) for k, v in json.load(fh).items()}
    training = ab.training_samples_from(samples, stats_map, metric=a.metric)
    cfg = ab.TrainConfig(max_depth=a.max_depth, min_samples_leaf=a.min_leaf,
                         min_samples_split=a.min_split)
    x, y = ab.to_matrix(training, ab.DEFAULT_MODEL_FEATURES)
    tree = ab.fit(x, y, ab.DEFAULT_MODEL_FEATURES, cfg)
    flat = ab.flatten(tree)
    rep = ab.evaluate(flat, x, y)
    print(f"samples={len(training)} nodes={flat.node_count} train_acc={rep.top1_accuracy:.3f} "
          f"unknown={rep.unknown_rate:.3f}")
    if len(training) >= 10:
        tr, te = ab.split_train_test(training, 0.7, seed=0)
        xt, yt = ab.to_matrix(tr, ab.DEFAULT_MODEL_FEATURES)
        xe, ye = ab.to_matrix(te, ab.DEFAULT_MODEL_FEATURES)
        held = ab.evaluate(ab.fit(xt, yt, ab.DEFAULT_MODEL_FEATURES, cfg), xe, ye)
        print(f"held-out top1={held.top1_accuracy:.3f} (70/30 split)")
    ab.serialize(flat, a.out)
    # replay: cost of the tree's per-level choice from the measured table
    table = {}
    for s in samples:
        table[(s.graph_id, s.root, s.level, ab.pair_index(s.kernel, s.variant))] = s.min_ns
    opt = ab.compute_optimal(samples)
    orc = ab.compute_oracle(samples)
    by_run = {}
    for t in training:
        by_run.setdefault((t.graph_id, t.root), []).append(t)
    for key in sorted(by_run):
        prev = 0
        cost = 0
        for t in sorted(by_run[key], key=lambda t: t.level):
            c = flat.predict_one(t.features)
            c = prev if c == 254 else c
            prev = c
            cost += table[(key[0], key[1], t.level, c)]
        k, v, o = orc[key]
        print(f"{key[0]:10s} root={key[1]:9d} optimal={opt[key]/1e3:9.1f}us "
              f"best_single={o/1e3:9.1f}us ({k.name}/{v.name}) tree={cost/1e3:9.1f}us "
              f"tree/opt={cost/opt[key]:.3f} single/tree={o/cost:.2f}")


if __name__ == "__main__":
    main()
