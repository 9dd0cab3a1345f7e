"""Per-level timing of all 15 pairs on a device-generated graph (quick probe;
the reference's benchmark_graph schema, src/bench.py:102-165).

    python tools/probe_levels.py --config k24 --roots 4 --out gpurun_out/levels_k24.csv
"""

from __future__ import annotations

import argparse
import csv
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_01159_b200 as P  # noqa: E402
from paper_1708_01159_b200 import DeviceGraph, Traversal  # noqa: E402


def make(config):
    t0 = time.time()
    if config.startswith("k"):
        s = int(config[1:])
        dg = DeviceGraph.rmat(s, 16 << s, 1, symmetrize=True)
    elif config == "er":
        dg = DeviceGraph.uniform(1 << 25, 1 << 30, 1)
    elif config.startswith("er"):
        s = int(config[2:])
        dg = DeviceGraph.uniform(1 << s, 32 << s, 1)
    elif config == "mesh":
        dg = DeviceGraph.mesh(4096, 4096)
    else:
        r = int(config[4:])
        dg = DeviceGraph.mesh(r, r)
    print(f"# {config}: V={dg.vertex_count} E={dg.edge_count} gen+build {time.time()-t0:.2f}s",
          flush=True)
    return dg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="k24")
    ap.add_argument("--roots", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="")
    ap.add_argument("--pairs", default="all")
    a = ap.parse_args()
    dg = make(a.config)
    oo, _ = dg.offsets()
    deg = np.diff(oo.astype(np.int64))
    rng = np.random.default_rng(1)
    roots = sorted(int(x) for x in rng.choice(np.flatnonzero(deg > 0), size=a.roots, replace=False))
    t = Traversal(dg)
    rows = []
    pairs = P.ALL_PAIRS if a.pairs == "all" else [P.ALL_PAIRS[int(i)] for i in a.pairs.split(",")]
    for root in roots:
        for k, v in pairs:
            best = None
            for _ in range(a.reps):
                counts, el = t.bfs_full(root, k, v, 32, cap=100000)
                tot = t.last_ns()
                if best is None or tot < best[0]:
                    best = (tot, counts.copy(), el.copy())
            tot, counts, el = best
            e, rv = t.reached()
            gteps = e / 2 / (tot * 1e-9) / 1e9
            print(f"root={root} {k.name:17s} {v.name:16s} levels={len(counts):5d} "
                  f"total={tot/1e3:10.1f}us  GTEPS={gteps:8.2f}  per-level(us)="
                  f"{[round(x/1e3,1) for x in el[:12]]}", flush=True)
            disc = 1
            for lvl, (c, x) in enumerate(zip(counts, el)):
                fr = 1 if lvl == 0 else int(counts[lvl - 1])
                rows.append((a.config, root, k.name, v.name, lvl, int(x), int(x), fr, disc, int(c)))
                disc += int(c)
    if a.out:
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["graph_id", "root", "kernel", "variant", "level", "mean_ns", "min_ns",
                        "frontier_size", "discovered_before", "new_count"])
            w.writerows(rows)


if __name__ == "__main__":
    main()
