"""Run the GPU benchmark harness over a graph corpus (on the GPU box).

    python tools/gpu_levels.py --configs k20,k22,k24,er22,mesh1024 --roots 4 \
        --out gpurun_out/levels.csv --stats gpurun_out/stats.json

Outputs the reference levels.csv schema plus a stats JSON (graph_id ->
compute_stats as 18 floats + V, E) for tools/train_tree.py.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_01159_b200 as P  # noqa: E402
from paper_1708_01159_b200 import DeviceGraph, Traversal  # noqa: E402
from paper_1708_01159_b200.bench_levels import benchmark_graph_gpu, export_levels  # noqa: E402
from paper_1708_01159_b200.features import static_vector  # noqa: E402


def make(config: str) -> DeviceGraph:
    if config.startswith("k"):
        s = int(config[1:])
        return DeviceGraph.rmat(s, 16 << s, 1, symmetrize=True)
    if config == "er":
        return DeviceGraph.uniform(1 << 25, 1 << 30, 1)
    if config.startswith("er"):
        s = int(config[2:])
        return DeviceGraph.uniform(1 << s, 32 << s, 1)
    if config == "mesh":
        return DeviceGraph.mesh(4096, 4096)
    r = int(config[4:])
    return DeviceGraph.mesh(r, r)


def pick_roots(dg, k, seed=1):
    oo, _ = dg.offsets()
    deg = np.diff(oo.astype(np.int64))
    cand = np.flatnonzero(deg > 0)
    rng = np.random.default_rng(seed)
    return sorted(int(x) for x in rng.choice(cand, size=min(k, cand.size), replace=False))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="k20,k22,k24")
    ap.add_argument("--roots", type=int, default=4)
    ap.add_argument("--root-seed", type=int, default=1)
    ap.add_argument("--mesh-roots", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--out", default="gpurun_out/levels.csv")
    ap.add_argument("--stats", default="gpurun_out/stats.json")
    ap.add_argument("--mode", type=int, default=1,
                    help="1 megakernel (40 regs), 2 megakernel (64 regs), 0 per-level launches")
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    stats = {}
    first = True
    for cfg in a.configs.split(","):
        t0 = time.time()
        dg = make(cfg)
        st = P.compute_stats(dg)
        stats[cfg] = static_vector(st).tolist()
        roots = pick_roots(dg, a.roots if not cfg.startswith("mesh") else a.mesh_roots,
                           seed=a.root_seed)
        if cfg.startswith("mesh"):
            roots = sorted(set([0, *roots]))
        t = Traversal(dg)
        t.set_device_loop(a.mode)
        rows = benchmark_graph_gpu(dg, roots, cfg, a.reps, a.warmup, traversal=t)
        export_levels(rows, a.out, append=not first)
        first = False
        best = {}
        for r in rows:
            best.setdefault((r.root, r.level), []).append(r.mean_ns)
        opt = sum(min(v) for v in best.values())
        print(f"{cfg}: V={dg.vertex_count} E={dg.edge_count} roots={roots} rows={len(rows)} "
              f"optimal_sum={opt/1e3:.1f}us time={time.time()-t0:.1f}s", flush=True)
        t.close()
        dg.close()
    with open(a.stats, "w") as fh:
        json.dump(stats, fh)


if __name__ == "__main__":
    main()
