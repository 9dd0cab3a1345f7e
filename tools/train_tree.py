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


def quantize(samples, q):
    """Round level times to a geometric grid of ratio (1+q): variants whose
    times differ by less than the GPU's run-to-run noise then tie, and the
    reference's label_level breaks the tie toward the lowest ordinal, which
    gives consistent labels for similar levels (the trainer is unchanged)."""
    import dataclasses
    import math
    if q <= 0:
        return samples
    out = []
    for s_ in samples:
        b = lambda t: float((1 + q) ** round(math.log(max(t, 1.0)) / math.log(1 + q)))
        out.append(dataclasses.replace(s_, mean_ns=b(s_.mean_ns), min_ns=int(b(s_.min_ns))))
    return out


def greedy_menu(samples, k):
    """Greedy set of k pairs minimising the geomean (over runs) of the
    per-level best-in-menu cost relative to the per-level optimum."""
    import math
    lv = {}
    for s_ in samples:
        lv.setdefault((s_.graph_id, s_.root, s_.level), {})[ab.pair_index(s_.kernel, s_.variant)] = s_.min_ns
    def score(menu):
        tot, opt = {}, {}
        for key, d in lv.items():
            r = key[:2]
            tot[r] = tot.get(r, 0) + min(d[p] for p in menu)
            opt[r] = opt.get(r, 0) + min(d.values())
        return math.exp(sum(math.log(tot[r] / opt[r]) for r in tot) / len(tot))
    menu = []
    for _ in range(k):
        menu.append(min((p for p in range(15) if p not in menu), key=lambda p: score(menu + [p])))
    return menu, score(menu)


def restrict(samples, menu):
    """Labels may only name menu pairs: the other pairs are made infinitely
    slow before the reference's argmin labelling (label_level)."""
    import dataclasses
    keep = set(menu)
    return [s_ if ab.pair_index(s_.kernel, s_.variant) in keep else
            dataclasses.replace(s_, mean_ns=1e30, min_ns=2**62) for s_ in samples]


def replay(flat, training, table):
    """Σ over runs of the measured cost of the tree's per-level choices."""
    by_run = {}
    for t in training:
        by_run.setdefault((t.graph_id, t.root), []).append(t)
    cost = {}
    for key in sorted(by_run):
        prev, c_ = 0, 0
        for t in sorted(by_run[key], key=lambda t: t.level):
            c = flat.predict_one(t.features)
            c = prev if c == 254 else c
            prev = c
            c_ += table[(key[0], key[1], t.level, c)]
        cost[key] = c_
    return cost


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--levels", required=True)
    ap.add_argument("--stats", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--metric", default="min")
    ap.add_argument("--max-levels", type=int, default=64)
    ap.add_argument("--menu", type=int, default=6,
                    help="restrict labels to a greedy menu of this many pairs (0 = all 15)")
    ap.add_argument("--seed-menu", default="",
                    help="comma list of pair ordinals the menu starts from")
    ap.add_argument("--grid", default="0,0.03,0.06,0.1/4,6,8,12/1,2,4",
                    help="quantisations / max depths / min leaf sizes to search")
    a = ap.parse_args()
    raw = ab.read_samples(a.levels)
    with open(a.stats) as fh:
        stats_map = {k: stats_from_vec(v) for k, v in json.load(fh).items()}
    # measured table and the feature vector of every level of every run
    table = {(s_.graph_id, s_.root, s_.level, ab.pair_index(s_.kernel, s_.variant)): s_.min_ns
             for s_ in raw}
    all_levels = ab.training_samples_from(raw, stats_map, metric=a.metric)
    opt = {}
    for t in all_levels:
        best = min(table[(t.graph_id, t.root, t.level, i)] for i in range(15))
        opt[(t.graph_id, t.root)] = opt.get((t.graph_id, t.root), 0) + best
    depth = {}
    for s_ in raw:
        depth[(s_.graph_id, s_.root)] = max(depth.get((s_.graph_id, s_.root), 0), s_.level + 1)
    sub = [s_ for s_ in raw if depth[(s_.graph_id, s_.root)] <= a.max_levels
           or s_.level % (depth[(s_.graph_id, s_.root)] // a.max_levels + 1) == 0]
    qs, depths, leaves = (list(map(float if i == 0 else int, g.split(",")))
                          for i, g in enumerate(a.grid.split("/")))
    # model selection on held-out roots: every other root of each graph
    runs = sorted({(s_.graph_id, s_.root) for s_ in raw})
    held = {r for i, r in enumerate(runs) if i % 2 == 1}
    fit_part = [s_ for s_ in sub if (s_.graph_id, s_.root) not in held]
    val_levels = [t for t in all_levels if (t.graph_id, t.root) in held]
    if a.menu:
        # greedy menu, each candidate scored by the held-out replay cost of a
        # tree fitted on it: a pair whose bad levels the features cannot
        # predict (e.g. thread-per-vertex push on a hub frontier of size 1)
        # is not worth adding, however fast it is on average
        def menu_score(menu):
            tr_ = ab.training_samples_from(quantize(restrict(fit_part, menu), 0.05), stats_map,
                                           metric=a.metric)
            x_, y_ = ab.to_matrix(tr_, ab.DEFAULT_MODEL_FEATURES)
            fl = ab.flatten(ab.fit(x_, y_, ab.DEFAULT_MODEL_FEATURES,
                                   ab.TrainConfig(max_depth=6, min_samples_leaf=2,
                                                  min_samples_split=4)))
            c_ = replay(fl, val_levels, table)
            r_ = [c_[k] / opt[k] for k in c_]
            return float(np.exp(np.mean(np.log(r_)))), max(r_)
        menu = [int(x) for x in a.seed_menu.split(",") if x]
        cur = menu_score(menu) if menu else None
        for _ in range(a.menu):
            cands = [(menu_score(menu + [p]), p) for p in range(15) if p not in menu]
            (sc, p) = min(cands, key=lambda z: (z[0][1] > 2.0, z[0][0]))
            if cur is not None and sc[0] >= cur[0] * 0.999:
                break
            menu.append(p)
            cur = sc
            print("menu +", f"{ab.ALL_PAIRS[p][0].name}/{ab.ALL_PAIRS[p][1].name}",
                  f"held-out geomean {sc[0]:.4f} worst {sc[1]:.3f}", flush=True)
        fit_part = restrict(fit_part, menu)
        sub = restrict(sub, menu)
    best = None
    for q in qs:
        training = ab.training_samples_from(quantize(fit_part, q), stats_map, metric=a.metric)
        x, y = ab.to_matrix(training, ab.DEFAULT_MODEL_FEATURES)
        for d in depths:
            for leaf in leaves:
                cfg = ab.TrainConfig(max_depth=d, min_samples_leaf=leaf,
                                     min_samples_split=max(2, 2 * leaf))
                flat = ab.flatten(ab.fit(x, y, ab.DEFAULT_MODEL_FEATURES, cfg))
                cost = replay(flat, val_levels, table)
                ratios = [cost[k] / opt[k] for k in cost]
                score = float(np.exp(np.mean(np.log(ratios))))
                worst = max(ratios)
                print(f"q={q:<5} depth={d:<3} leaf={leaf}: nodes={flat.node_count:4d} "
                      f"held-out geomean tree/opt={score:.4f} worst={worst:.3f}", flush=True)
                if best is None or (worst > 2.0, score, worst) < best[0]:
                    best = ((worst > 2.0, score, worst), q, d, leaf)
    (_, score, worst), q, d, leaf = best
    training = ab.training_samples_from(quantize(sub, q), stats_map, metric=a.metric)
    x, y = ab.to_matrix(training, ab.DEFAULT_MODEL_FEATURES)
    cfg = ab.TrainConfig(max_depth=d, min_samples_leaf=leaf, min_samples_split=max(2, 2 * leaf))
    flat = ab.flatten(ab.fit(x, y, ab.DEFAULT_MODEL_FEATURES, cfg))
    cost = replay(flat, all_levels, table)
    ab.serialize(flat, a.out)
    print(f"\nchosen: q={q} max_depth={d} min_leaf={leaf} (held-out geomean {score:.4f}, "
          f"worst {worst:.3f}); refit on all runs: nodes={flat.node_count} -> {a.out}")
    orc = ab.compute_oracle(raw)
    for key in sorted(cost):
        k, v, o = orc[key]
        print(f"{key[0]:10s} root={key[1]:9d} optimal={opt[key]/1e3:9.1f}us "
              f"best_single={o/1e3:9.1f}us ({k.name}/{v.name}) tree={cost[key]/1e3:9.1f}us "
              f"tree/opt={cost[key]/opt[key]:.3f} single/tree={o/cost[key]:.2f}")


if __name__ == "__main__":
    main()
