#!/usr/bin/env python
"""bench.py -- tree-switched BFS GTEPS, Kronecker scale 24, B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1]): Kronecker scale 24, edgefactor 16,
symmetrised (rmat-like a,b,c = .57/.19/.19, seed 1, generated bit-exactly on
the device), tree-switched BFS from 64 seeded non-isolated roots.  A step = one batched
launch of tree-switched BFSs from --roots-per-step (8) roots, init_depths of
each included (rotating through the 64; the default 8 steps time each once).  GTEPS = Σ_roots (Σ out-degree of reached vertices / 2) / device time
of the K timed steps (CUDA events on the traversal's stream, init_depths
included).  The graph (8.1 GB of arrays) is larger than L2 and stays
resident, like model weights.

With N > 1 ranks (torchrun, one per GPU) the same workload runs as ONE
tree-switched BFS at a time over a 1-D edge-balanced vertex partition of the
graph: each rank builds only its slice from the generator
stream, and the per-level frontier exchange is fused NVLink peer stores
inside the persistent per-rank megakernel (scaling "strong"); the NCCL
all-gather exchange and config 3 (Kronecker-26) are secondary keys.
`--root-sharded` instead replicates the graph and shards the roots.

`--impl reference` times the reference algorithm's CPU port (oracle/, C +
OpenMP, all host cores) on the same config: the reference is pure Python +
numpy and cannot travel to the GPU box.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BFS GTEPS (Kronecker scale 24, 1/2/4/8 B200); HBM GB/s vs peak"
UNIT = "GTEPS"
HBM_FALLBACK = 6650.0


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def pick_roots(out_offsets, k=64, seed=1):
    deg = np.diff(out_offsets.astype(np.int64))
    cand = np.flatnonzero(deg > 0)
    rng = np.random.default_rng(seed)
    return sorted(int(x) for x in rng.choice(cand, size=min(k, cand.size), replace=False))


def default_model():
    for p in ("models/gpu_tree.tree", "tests/golden/trees/t1.tree"):
        q = os.path.join(ROOT, p)
        if os.path.exists(q):
            return q
    raise FileNotFoundError("no tree model")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 5 + i and r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# Work model: algorithmic bytes of one level.
# ---------------------------------------------------------------------------
def level_bytes(kernel, V, E, F, N, EF, U, A_rev, ES, converted):
    bm = (V + 7) // 8
    if kernel in (0,):
        b = 4 * E + 4 * EF + 4 * N + 2 * bm
    elif kernel == 1:
        b = 4 * E + 4 * A_rev + 4 * N + 2 * bm
    elif kernel in (2, 4):
        b = 4 * F + 8 * F + 4 * EF + 4 * N + 4 * N + bm
    else:
        b = bm + 8 * U + 4 * ES + bm + 4 * N
    if converted:
        b += bm + 4 * F
    return b


def work_model(t, records, V, E):
    """Per-level (kernel, ns, bytes) from one instrumented replay."""
    nlev = len(records)
    st = t.level_stats(nlev)
    cnt, od, idg, es = st["count"], st["out_deg"], st["in_deg"], st["scanned"]
    out = []
    discovered = 0
    unvisited_in = int(idg.sum())
    for lvl, r in enumerate(records):
        F = int(cnt[lvl])
        N = int(cnt[lvl + 1]) if lvl + 1 < nlev else 0
        discovered += F
        unvisited_in -= int(idg[lvl])
        U = V - discovered
        b = level_bytes(int(r.kernel), V, E, F, N, int(od[lvl]), U, unvisited_in,
                        int(es[lvl]), bool(r.converted))
        out.append((int(r.kernel), int(r.variant), int(r.elapsed_ns), b))
    return out


KERNEL_NAMES = ["EDGE_LIST", "REV_EDGE_LIST", "VERTEX_PUSH", "VERTEX_PULL", "VERTEX_PUSH_WARP"]


# ---------------------------------------------------------------------------
def make_graph(a, dev):
    """(DeviceGraph, symmetric, workload name) for --graph."""
    from paper_1708_01159_b200 import DeviceGraph
    if a.graph == "er":        # config 5: uniform-random, 32M vertices, avg degree 32
        return (DeviceGraph.uniform(1 << 25, 1 << 30, 1, device=dev), False,
                "erdos-renyi-32M-deg32 (directed)")
    if a.graph == "mesh":      # config 4: 4096 x 4096 4-neighbour grid
        return DeviceGraph.mesh(4096, 4096, device=dev), True, "mesh-4096x4096"
    return (DeviceGraph.rmat(a.scale, 16 << a.scale, 1, symmetrize=True, device=dev,
                             permute=a.permute), True,
            f"kronecker-{a.scale}-ef16-symmetrised" + ("-permuted-ids" if a.permute else ""))


def workload_config(a, wname, V, E, symmetric, R):
    """The workload both arms time (identical dicts): graph, tree, root pool
    and the step's roots -- implementation details live beside it."""
    return {"workload": f"{wname} tree-switched BFS",
            "graph": a.graph, "scale": a.scale, "vertices": V, "directed_edge_slots": E,
            "teps_basis": "sum of out-degree of reached vertices" + (" / 2" if symmetric else ""),
            "roots_per_step": R, "roots_pool": 64,
            "root_order": "64 seeded non-isolated roots (seed 1); step s times roots "
                          "[s*R, (s+1)*R) of the pool repeated, after the warm-up steps",
            "model": os.path.relpath(a.model, ROOT)}


def run_ours(a):
    import torch
    import torch.distributed as dist

    import paper_1708_01159_b200 as P
    from paper_1708_01159_b200 import DeviceGraph, Traversal
    from paper_1708_01159_b200.features import static_vector

    rank, world, local = env_rank()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local if world > 1 else 0
    torch.cuda.set_device(dev)

    t_setup = time.time()
    dg, symmetric, wname = make_graph(a, dev)
    V, E = dg.vertex_count, dg.edge_count
    oo, io = dg.offsets()
    stats = P.compute_stats(dg)
    static24 = static_vector(stats)
    roots_all = pick_roots(oo, 64, seed=1)
    my_roots = roots_all[rank::world] if world > 1 else roots_all
    flat = P.deserialize(a.model)
    tree = flat.as_abfs()
    trav = Traversal(dg)
    trav.set_device_loop(a.mode)
    stream = torch.cuda.Stream(device=dev)
    trav.set_stream(stream.cuda_stream)
    # the headline keeps per-BFS semantics (GTEPS over t_bfs):
    # every batch is ONE full-grid launch, its BFSs back to back; the split
    # batch (concurrent partial-grid launches) is timed after, as a
    # throughput key
    trav.set_batch_ways(1)

    # traversed edges per root (Graph500 undirected basis: Σ out-degree / 2)
    m_trav = {}
    for r in my_roots:
        trav.adaptive(r, tree, static24, 32)
        e, _ = trav.reached()
        m_trav[r] = e / 2 if symmetric else float(e)
    setup_s = time.time() - t_setup

    R = a.roots_per_step
    order = [my_roots[i % len(my_roots)] for i in range(R * (a.warmup + a.steps))]
    for s in range(a.warmup):
        trav.adaptive_batch(order[s * R:(s + 1) * R], tree, static24, 32)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = trav.launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    edges = 0.0
    bfs_ns = 0
    per_root = []
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for s in range(a.warmup, a.warmup + a.steps):
            # one step = one batched launch: R tree-switched BFSs back to back
            batch = order[s * R:(s + 1) * R]
            _, ns_b, _ = trav.adaptive_batch(batch, tree, static24, 32)
            for r, ns_r in zip(batch, ns_b.tolist()):
                bfs_ns += ns_r
                edges += m_trav[r]
                per_root.append(m_trav[r] / (ns_r * 1e-9) / 1e9)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = trav.launches() - launches0
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        ee = torch.tensor([edges], device="cuda", dtype=torch.float64)
        dist.all_reduce(ee)
        edges = float(ee.item())
    gteps = edges / (ms * 1e-3) / 1e9

    # ---- multi-BFS throughput: the same steps as S concurrent launches ----
    concurrent = None
    if world == 1 and a.mode:
        trav.set_batch_ways(0)
        S = trav.batch_ways(R)
        if S > 1:
            for s in range(a.warmup):
                trav.adaptive_batch(order[s * R:(s + 1) * R], tree, static24, 32)
            c_edges = 0.0
            torch.cuda.synchronize()
            ev0.record(stream)
            for s in range(a.warmup, a.warmup + a.steps):
                batch = order[s * R:(s + 1) * R]
                trav.adaptive_batch(batch, tree, static24, 32)
                c_edges += sum(m_trav[r] for r in batch)
            ev1.record(stream)
            torch.cuda.synchronize()
            c_ms = ev0.elapsed_time(ev1)
            concurrent = {"value": round(c_edges / (c_ms * 1e-3) / 1e9, 3), "unit": UNIT,
                          "ms_per_step": round(c_ms / a.steps, 4), "ways": S,
                          "basis": "the same steps' R BFSs dealt round-robin to S concurrent "
                                   "persistent launches of 1/S of the grid (abfs_adaptive_bfs_batch "
                                   "default): multi-BFS throughput, each BFS's own t_bfs is longer"}
        trav.set_batch_ways(1)

    # ---- roofline of the dominant kernel (instrumented replay, untimed) ----
    peak, peak_kind = measured_peak_hbm()
    per_kernel = {}
    trav.instrument(True)
    for r in my_roots[:R]:
        recs = trav.adaptive(r, tree, static24, 32)
        for k, v, ns, b in work_model(trav, recs, V, E):
            agg = per_kernel.setdefault(k, [0, 0, 0])
            agg[0] += ns
            agg[1] += b
            agg[2] += 1
    trav.instrument(False)
    # per-level times of the (uninstrumented) switched run for the same roots
    lv_ns = {}
    trace_pairs = None
    for r in my_roots[:R]:
        recs = trav.adaptive(r, tree, static24, 32)
        trace_pairs = trace_pairs or [(KERNEL_NAMES[x.kernel], x.variant) for x in recs]
        for x in recs:
            lv_ns[x.kernel] = lv_ns.get(x.kernel, 0) + x.elapsed_ns
    dom = max(per_kernel, key=lambda k: lv_ns.get(k, 0))
    dom_ns = lv_ns[dom]
    dom_bytes = per_kernel[dom][1]
    achieved = dom_bytes / (dom_ns * 1e-9) / 1e9
    total_ns = sum(lv_ns.values())
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            with open(tf) as fh:
                tr = json.load(fh).get(KERNEL_NAMES[dom])
                traffic = round(tr["bytes_per_launch_mean"]) if tr else None
        except Exception:
            traffic = None
    kmega = None
    kf = os.path.join(ROOT, "profiles", "kmega_traffic.json")
    if os.path.exists(kf) and a.graph == "kronecker" and a.scale == 24:
        try:
            with open(kf) as fh:
                kmega = json.load(fh)
        except Exception:
            kmega = None
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": traffic, "kernel": KERNEL_NAMES[dom],
                "kernel_share_of_step": round(dom_ns / total_ns, 3),
                "launches_measured": per_kernel[dom][2],
                "algorithmic_bytes": int(dom_bytes),
                "algorithmic_bytes_per_launch": int(dom_bytes / max(1, per_kernel[dom][2])),
                "whole_traversal_GBps": round(sum(v[1] for v in per_kernel.values()) /
                                              (total_ns * 1e-9) / 1e9, 1),
                # the timed step's aggregate: R roots' algorithmic bytes over
                # ms_per_step (the concurrent launches together)
                "step_GBps": round(sum(v[1] for v in per_kernel.values()) /
                                   (ms / a.steps * 1e-3) / 1e9, 1) if world == 1 else None,
                "timed_kernel_ncu": kmega}

    # ---- every fixed pair vs the switched run (same roots, untimed extra) ----
    from types import SimpleNamespace as NS
    sample = my_roots[:max(1, min(len(my_roots), a.fixed_roots))]
    fixed = {}
    sw_ns, sw_e = 0, 0.0
    for r in sample:
        trav.adaptive(r, tree, static24, 32)
        sw_ns += trav.last_ns()
        sw_e += m_trav[r]
    for k, v in P.ALL_PAIRS:
        # best of the two level drivers per pair: the device loop (megakernel
        # bodies) and the per-level launch path (stand-alone kernels, e.g. the
        # bulk-copy edge stream)
        drv = {}
        for mode in (a.mode, 0) if a.mode else (0,):
            trav.set_device_loop(mode)
            ns_m, e_tot = 0, 0.0
            for r in sample:
                trav.bfs_full(r, int(k), int(v), 32)
                ns_m += trav.last_ns()
                e_tot += m_trav[r]
            drv[mode] = ns_m
        trav.set_device_loop(a.mode)
        best_mode = min(drv, key=drv.get)
        ns_tot = drv[best_mode]
        trav.instrument(True)
        _, el = trav.bfs_full(sample[0], int(k), int(v), 32)
        wm = work_model(trav, [NS(kernel=int(k), variant=int(v), elapsed_ns=int(x), converted=False)
                               for x in el], V, E)
        trav.instrument(False)
        byt, t_ns = sum(x[3] for x in wm), sum(x[2] for x in wm)
        fixed[f"{k.name}/{v.name}"] = {"gteps": round(e_tot / (ns_tot * 1e-9) / 1e9, 3),
                                       "driver": "device loop" if best_mode else "launch path",
                                       "roofline_frac": round(byt / (t_ns * 1e-9) / 1e9 / peak, 4)}
    best_fixed = max(fixed, key=lambda x: fixed[x]["gteps"])
    sw_gteps = sw_e / (sw_ns * 1e-9) / 1e9
    fixed_block = {"roots": len(sample), "basis": "device time after init_depths (t_bfs); "
                                                  "each pair: best of the two level drivers",
                   "switched_gteps": round(sw_gteps, 3), "best_fixed": best_fixed,
                   "best_fixed_gteps": fixed[best_fixed]["gteps"],
                   "switched_over_best_fixed": round(sw_gteps / fixed[best_fixed]["gteps"], 3),
                   "pairs": fixed}

    # ---- e2e through the public API with host results ----------------------
    e2e = None
    dg_api = dg
    dg_api._scratch = Traversal(dg)
    n_e2e = min(len(my_roots), R * max(1, a.steps // 2))
    # warm-up in the timed loop's own pattern (the previous result is still
    # alive during the next call), so the recycled page-locked result
    # arrays are allocated before timing
    depths = None
    for r in my_roots[:3]:
        depths, _ = P.adaptive_bfs(dg_api, r, flat, stats)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e_edges = 0.0
    for i in range(n_e2e):
        r = my_roots[i % len(my_roots)]
        depths, _ = P.adaptive_bfs(dg_api, r, flat, stats)
        e_edges += m_trav[r]
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if world > 1:   # whole-job: edges summed over ranks / slowest rank's time
        te = torch.tensor([e_edges, el], dtype=torch.float64, device="cuda")
        tmax = te.clone()
        dist.all_reduce(te)
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        e_edges, el = float(te[0].item()), float(tmax[1].item())
    e2e = {"value": round(e_edges / el / 1e9, 3), "unit": UNIT,
           "h2d_bytes_per_step": int(R * 8 + flat.node_count * 19 + 24 * 8),
           "d2h_bytes_per_step": int(R * 4 * V),
           "api": "paper_1708_01159_b200.adaptive_bfs(graph, root, FlatTree, stats) -> host int32 depths",
           "bfs_per_sample": n_e2e}

    # ---- CPU baseline: oracle port of the reference algorithm --------------
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(dg, roots_all, a.model, static24, a.cpu_seconds, symmetric)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(gteps, 3), "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms / a.steps, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (device-generated Kronecker, bit-exact to the reference generator"
                    + (", ids relabelled by a fixed bijection)" if a.permute else ")"),
            "config": workload_config(a, wname, V, E, symmetric, R),
            "implementation": {"step": "abfs_adaptive_bfs_batch: R tree-switched BFSs (init_depths "
                                       "included) back to back in one persistent full-grid launch",
                               "level_loop": "device (persistent megakernel)" if a.mode
                               else "host (per-level launches)",
                               "parallelism": f"roots sharded over {world} GPU(s), graph replicated",
                               "l2": "inputs larger than L2 (graph arrays 8.1 GB)"},
            "gteps_graph500_tbfs": round(edges / (bfs_ns * 1e-9) / 1e9, 3) if world == 1 else None,
            "gteps_per_root": {"median": round(statistics.median(per_root), 3),
                               "harmonic_mean": round(len(per_root) / sum(1 / x for x in per_root), 3),
                               "bfs": len(per_root)} if per_root else None,
            "fixed_vs_switched": fixed_block,
            "gpu_launches": int(launches),
            "concurrent_batch": concurrent,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk.summary(),
            "trace_first_root": {"levels": len(trace_pairs), "first_16": trace_pairs[:16]}
            if trace_pairs else None,
            "setup_s": round(setup_s, 1),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_partitioned(a):
    """--partition: config 3 -- one tree-switched BFS over a 1-D vertex
    partition (edge-balanced destination ranges, one rank per GPU, frontier
    bitmap slices all-gathered over NCCL every level).  At N=1,
    --virtual-parts P runs P partitions on the one GPU (device concat)."""
    import torch
    import torch.distributed as dist

    import paper_1708_01159_b200 as P
    from paper_1708_01159_b200 import DeviceGraph
    from paper_1708_01159_b200.partition import (DevicePartition, DistExchange,
                                                 DistPeerExchange, LocalExchange,
                                                 LocalPeerExchange, PartitionedBFS,
                                                 edge_balanced_bounds)

    rank, world, local = env_rank()
    dev = local if world > 1 else 0
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    parts_n = world if world > 1 else max(1, a.virtual_parts)
    t_setup = time.time()
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        dg = DeviceGraph.rmat(a.scale, 16 << a.scale, 1, symmetrize=True, device=dev)
        V, E = dg.vertex_count, dg.edge_count
        oo, io = dg.offsets()
        stats = P.compute_stats(dg)
        bounds = edge_balanced_bounds(io, parts_n)
        mine = [rank] if world > 1 else list(range(parts_n))
        parts = [DevicePartition(dg, int(bounds[i]), int(bounds[i + 1]), stream.cuda_stream)
                 for i in mine]
        dg.close()
        if a.exchange == "peer":
            exch = (DistPeerExchange(torch, dist, parts[0]) if world > 1
                    else LocalPeerExchange(torch, parts))
        else:
            exch = DistExchange(torch, dist) if world > 1 else LocalExchange(torch)
        bfs = PartitionedBFS(parts, bounds, exch,
                             alloc=lambda s: torch.zeros(s, dtype=torch.int32, device=f"cuda:{dev}"))
        flat = P.deserialize(a.model)
        roots = pick_roots(oo, 64, seed=1)
        deg = np.diff(oo.astype(np.int64))
        order = [roots[i % len(roots)] for i in range(a.warmup + a.steps)]
        m_trav, levels = {}, {}
        for r in sorted(set(order)):
            tr = bfs.adaptive(r, flat, stats)
            d = bfs.depths()
            m_trav[r] = float(deg[d != 2**31 - 1].sum()) / 2
            levels[r] = tr.level_count
        setup_s = time.time() - t_setup
        for r in order[:a.warmup]:
            bfs.adaptive(r, flat, stats)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        l0 = sum(p.launches() for p in parts)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        edges, nlev = 0.0, 0
        with ClockSampler(dev) as clk:
            torch.cuda.synchronize()
            ev0.record(stream)
            for r in order[a.warmup:]:
                bfs.adaptive(r, flat, stats)
                edges += m_trav[r]
                nlev += levels[r]
            ev1.record(stream)
            torch.cuda.synchronize()
        launches = sum(p.launches() for p in parts) - l0
        ms = exch.max_over_ranks(ev0.elapsed_time(ev1))
        gteps = edges / (ms * 1e-3) / 1e9
        # exchange share (untimed replay with all-gather events; the fused
        # peer exchange has no separate collective to time)
        ex_ms = 0.0
        if a.exchange != "peer":
            bfs.time_exchange = True
            for r in order[a.warmup:a.warmup + min(4, a.steps)]:
                bfs.adaptive(r, flat, stats)
            bfs.time_exchange = False
            ex_ms = exch.max_over_ranks(bfs.exchange_ms / max(1, bfs.exchange_calls))
            recv = (parts_n - 1) * bfs.stride * 4
        else:
            recv = int((V + 31) // 32 * 4 * (parts_n - 1) / parts_n)
        # e2e: the partitioned call + gathered host depths
        t0 = time.perf_counter()
        ne = min(4, a.steps)
        e_edges = 0.0
        for r in order[a.warmup:a.warmup + ne]:
            bfs.adaptive(r, flat, stats)
            bfs.depths()
            e_edges += m_trav[r]
        torch.cuda.synchronize()
        e_el = exch.max_over_ranks(time.perf_counter() - t0)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(gteps, 3), "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms / a.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (device-generated Kronecker, bit-exact to the reference generator)",
            "config": {"workload": f"kronecker-{a.scale}-ef16-symmetrised tree-switched BFS, "
                                   f"1-D vertex partition",
                       "scale": a.scale, "vertices": V, "directed_edge_slots": E,
                       "partitions": parts_n, "roots_per_step": 1,
                       "parallelism": (f"1-D edge-balanced vertex partition over {world} GPUs, "
                                       "NCCL all-gather of frontier bitmap slices per level")
                       if world > 1 else f"{parts_n} partitions on one GPU (device concat)",
                       "model": os.path.relpath(a.model, ROOT),
                       "l2": "inputs larger than L2"},
            "gpu_launches": int(launches),
            "exchange": {"kind": "fused peer stores over NVLink + mailbox signal (no collective)"
                         if a.exchange == "peer" else "NCCL all-gather of padded bitmap slices",
                         "bytes_received_per_rank_per_level": int(recv),
                         "mean_allgather_us": round(ex_ms * 1e3, 2) if ex_ms else None,
                         "GBps_received_per_rank": round(recv / (ex_ms * 1e-3) / 1e9, 2)
                         if ex_ms > 0 else None,
                         "nvlink_peak_GBps_per_direction": 900.0,
                         "levels_timed": nlev},
            "e2e": {"value": round(e_edges / e_el / 1e9, 3), "unit": UNIT,
                    "h2d_bytes_per_step": 8, "d2h_bytes_per_step": int(4 * V),
                    "api": "PartitionedBFS.adaptive + depths() (gathered host int32 depths)"},
            "cpu_baseline": None,
            "clocks": clk.summary(),
            "setup_s": round(setup_s, 1),
        }
        print(json.dumps(line), flush=True)
    for p in parts:
        p.close()
    if world > 1:
        dist.destroy_process_group()


def bench_spec(graph, scale):
    """Generator spec of the bench graph (configs 2/3: Kronecker; 5: ER; 4: mesh)."""
    from paper_1708_01159_b200.partition import gen_spec
    if graph == "er":
        return gen_spec("uniform", n=1 << 25, edges=1 << 30, seed=1), False, "erdos-renyi-32M-deg32 (directed)"
    if graph == "mesh":
        return gen_spec("mesh", rows=4096, cols=4096), True, "mesh-4096x4096"
    return (gen_spec("rmat", scale=scale, edges=16 << scale, seed=1, symmetrize=True), True,
            f"kronecker-{scale}-ef16-symmetrised")


class PartitionedRun:
    """One rank of the 1-D partitioned BFS on its own GPU: the
    slice is built from the generator stream (the whole graph is never on a
    GPU), the frontier exchange is `exchange` ("peer": fused NVLink peer
    stores inside the persistent per-rank megakernel; "nccl": NCCL
    all-gather of the bitmap slices between per-level launches)."""

    def __init__(self, torch, dist, a, graph, scale, exchange, dev):
        from paper_1708_01159_b200.graph import stats_from_offsets
        from paper_1708_01159_b200.partition import (DevicePartition, DistExchange,
                                                     DistPeerExchange, PartitionedBFS,
                                                     edge_balanced_bounds, gen_offsets, gen_size)
        self.torch, self.dist = torch, dist
        rank, world, _ = env_rank()
        t0 = time.time()
        self.spec, self.symmetric, self.wname = bench_spec(graph, scale)
        self.V, self.E = gen_size(self.spec)
        self.oo, io = gen_offsets(self.spec, dev)          # one streaming degree pass
        self.stats = stats_from_offsets(self.V, self.E, self.oo, io)
        self.bounds = edge_balanced_bounds(io, world)
        self.lo, self.hi = int(self.bounds[rank]), int(self.bounds[rank + 1])
        self.stream = torch.cuda.Stream(device=dev)
        self.part = DevicePartition(None, self.lo, self.hi, self.stream.cuda_stream, spec=self.spec,
                                    device=dev)
        self.exch = (DistPeerExchange(torch, dist, self.part) if exchange == "peer"
                     else DistExchange(torch, dist))
        self.bfs = PartitionedBFS([self.part], self.bounds, self.exch,
                                  alloc=lambda s: torch.zeros(s, dtype=torch.int32, device=f"cuda:{dev}"))
        self.deg_owned = np.diff(self.oo[self.lo:self.hi + 1].astype(np.int64))
        self.roots = pick_roots(self.oo, 64, seed=1)
        self.setup_s = time.time() - t0
        self.exchange = exchange

    def traversed(self, root, flat):
        """Traversed edges of one tree-switched BFS from root (Σ out-degree of
        reached vertices, / 2 if symmetric), summed over the ranks' slices."""
        tr = self.bfs.adaptive(root, flat, self.stats)
        d = self.part.read_depths()
        e = float(self.deg_owned[d != 2**31 - 1].sum())
        t = self.torch.tensor([e], dtype=self.torch.float64,
                              device="cuda" if self.dist.get_backend() == "nccl" else "cpu")
        self.dist.all_reduce(t)
        e = float(t.item())
        return (e / 2 if self.symmetric else e), tr

    def time_roots(self, order, flat):
        torch = self.torch
        torch.cuda.synchronize()
        self.dist.barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record(self.stream)
        for r in order:
            self.bfs.adaptive(r, flat, self.stats)
        ev1.record(self.stream)
        torch.cuda.synchronize()
        return self.exch.max_over_ranks(ev0.elapsed_time(ev1))

    def close(self):
        self.part.close()


def run_multi(a):
    """--gpus N > 1: one tree-switched BFS at a time over the 1-D
    edge-balanced vertex partition of the bench graph across the N GPUs
    (strong scaling of configs[1]'s Kronecker-24 workload; config 3's
    Kronecker-26 run as a secondary key), fused NVLink peer exchange, with
    the NCCL all-gather exchange and root-sharded replicas as secondary
    lines."""
    import torch
    import torch.distributed as dist

    import paper_1708_01159_b200 as P

    rank, world, local = env_rank()
    if a.shared_gpu:   # test mode: every rank on GPU 0, gloo control plane, no NCCL line
        local = 0
        a.no_secondary = True
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    flat = P.deserialize(a.model)
    run = PartitionedRun(torch, dist, a, a.graph, a.scale, "peer", local)
    m_trav, levels = {}, {}
    for r in run.roots:
        m_trav[r], tr = run.traversed(r, flat)
        levels[r] = tr.level_count
    R = a.roots_per_step
    order = [run.roots[i % len(run.roots)] for i in range(R * (a.warmup + a.steps))]
    run.time_roots(order[:R * a.warmup], flat)
    l0 = run.part.launches()
    with ClockSampler(local) as clk:
        ms = run.time_roots(order[R * a.warmup:], flat)
    launches = run.part.launches() - l0
    timed = order[R * a.warmup:]
    edges = sum(m_trav[r] for r in timed)
    nlev = sum(levels[r] for r in timed)
    gteps = edges / (ms * 1e-3) / 1e9
    words = (run.V + 31) // 32
    recv = int(words * 4 * (world - 1) / world)
    # e2e: the public partitioned call + the gathered host depth array
    ne = min(len(run.roots), R)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    e_edges = 0.0
    for r in run.roots[:ne]:
        run.bfs.adaptive(r, flat, run.stats)
        run.bfs.depths()
        e_edges += m_trav[r]
    torch.cuda.synchronize()
    e_el = run.exch.max_over_ranks(time.perf_counter() - t0)

    # ---- secondary: the same BFS with the NCCL all-gather exchange --------
    nccl = None
    if a.nccl_line and not a.no_secondary:
      try:
        from paper_1708_01159_b200.partition import DistExchange, PartitionedBFS
        torch.cuda.set_stream(run.stream)   # the all-gathers must follow the levels' kernels
        nb = PartitionedBFS([run.part], run.bounds, DistExchange(torch, dist),
                            alloc=lambda s: torch.zeros(s, dtype=torch.int32, device=f"cuda:{local}"))
        nb.time_exchange = True
        sample = run.roots[:4]
        for r in sample[:1]:
            nb.adaptive(r, flat, run.stats)
        nb.exchange_ms, nb.exchange_calls = 0.0, 0
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for r in sample:
            nb.adaptive(r, flat, run.stats)
        torch.cuda.synchronize()
        el = run.exch.max_over_ranks(time.perf_counter() - t0)
        ex_us = run.exch.max_over_ranks(nb.exchange_ms / max(1, nb.exchange_calls)) * 1e3
        nrecv = (world - 1) * nb.stride * 4
        nccl = {"gteps": round(sum(m_trav[r] for r in sample) / el / 1e9, 3),
                "basis": "host wall clock of per-level launches + NCCL all_gather_into_tensor",
                "mean_allgather_us": round(ex_us, 2),
                "bytes_received_per_rank_per_level": int(nrecv),
                "GBps_received_per_rank": round(nrecv / (ex_us * 1e-6) / 1e9, 2) if ex_us else None,
                "nvlink_peak_GBps_per_direction": 900.0, "roots": len(sample)}
      except Exception as exc:   # a secondary line never costs the headline
        nccl = {"error": f"{type(exc).__name__}: {exc}"[:300]}
      finally:
        torch.cuda.set_stream(torch.cuda.default_stream(local))

    # ---- secondary: config 3 (Kronecker-26) over the same partition -------
    k26 = None
    run.close()
    if not a.no_secondary and a.graph == "kronecker" and a.scale != 26:
        try:
            r26 = PartitionedRun(torch, dist, a, "kronecker", 26, "peer", local)
            m26 = {r: r26.traversed(r, flat)[0] for r in r26.roots[:4]}
            o26 = [r26.roots[i % 4] for i in range(8)]
            ms26 = r26.time_roots(o26, flat)
            k26 = {"workload": r26.wname, "vertices": r26.V, "directed_edge_slots": r26.E,
                   "gteps": round(sum(m26[r] for r in o26) / (ms26 * 1e-3) / 1e9, 3),
                   "ms_per_bfs": round(ms26 / len(o26), 4), "bfs_timed": len(o26),
                   "setup_s": round(r26.setup_s, 1)}
            r26.close()
        except Exception as exc:
            k26 = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(gteps, 3), "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms / a.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (device-generated, bit-exact to the reference generator)",
            "config": {"workload": f"{run.wname} tree-switched BFS, 1-D vertex partition over "
                                   f"{world} GPUs",
                       "graph": a.graph, "scale": a.scale, "vertices": run.V,
                       "directed_edge_slots": run.E, "roots_per_step": R, "roots_pool": 64,
                       "step": f"{R} tree-switched BFSs, one at a time over all ranks (one "
                               "persistent per-rank launch each)",
                       "parallelism": f"1-D edge-balanced destination partition, {world} ranks x 1 GPU; "
                                      "per-level frontier exchange = fused NVLink peer stores "
                                      "inside the per-rank megakernel (LL words across devices)",
                       "slices": "built per rank from the generator stream (whole graph never resident)",
                       "model": os.path.relpath(a.model, ROOT),
                       "l2": "inputs larger than L2"},
            "gpu_launches": int(launches),
            "exchange": {"kind": "fused peer stores over NVLink (CUDA IPC) inside the per-rank megakernel: "
                                 "LL words (epoch | bitmap word, one 8-byte store, no fence) between "
                                 "devices, GPU-scoped release/acquire arrival counters on one device",
                         "bytes_received_per_rank_per_level": recv,
                         "levels_timed": nlev,
                         "nvlink_peak_GBps_per_direction": 900.0,
                         "nccl_allgather_line": nccl},
            "config3_k26": k26,
            "roofline": None,
            "cpu_baseline": None,
            "e2e": {"value": round(e_edges / e_el / 1e9, 3), "unit": UNIT,
                    "h2d_bytes_per_step": 8 * ne, "d2h_bytes_per_step": int(4 * run.V * ne),
                    "api": "PartitionedBFS.adaptive + depths() (gathered host int32 depths)",
                    "bfs_per_sample": ne},
            "clocks": clk.summary(),
            "setup_s": round(run.setup_s, 1),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_baseline(dg, roots, model, static24, budget_s, symmetric=True):
    """The reference algorithm's CPU port (oracle/) on the host cores, same
    graph / tree / roots, bounded to ~budget_s seconds (>= 1 root)."""
    import oracle
    import paper_1708_01159_b200 as P
    from paper_1708_01159_b200.features import canonical_indices

    a = dg.download(rev_owner=True)
    og = oracle.OracleGraph(dg.vertex_count, dg.edge_count, a["out_offsets"], a["destinations"],
                            a["origins"], a["in_offsets"], a["sources"], a["rev_owner"])
    del a
    flat = P.deserialize(model)
    ot = oracle.OracleTree(canonical_indices(flat.selection), flat.features, flat.thresholds,
                           flat.lefts, flat.rights, flat.leaf_classes)
    threads = os.cpu_count() or 1
    deg = np.diff(og.out_offsets.astype(np.int64))
    done, edges, el = 0, 0.0, 0.0
    for r in roots:
        t0 = time.perf_counter()
        d, _ = oracle.adaptive_bfs(og, r, ot, static24, threads=threads)
        el += time.perf_counter() - t0
        edges += deg[d != 2**31 - 1].sum() / (2 if symmetric else 1)
        done += 1
        if el >= budget_s:
            break
    return {"value": round(edges / el / 1e9, 5), "unit": UNIT, "cores": threads, "kind": "port",
            "cpu_model": cpu_model(), "numpy": np.__version__,
            "sample": f"{done} tree-switched BFS root(s) on the full {dg.vertex_count}-vertex "
                      f"graph, same tree; C+OpenMP port of the reference level kernels "
                      f"(oracle/abfs_oracle.c), {el:.1f}s wall"}


def run_reference(a):
    """--impl reference: the reference algorithm's CPU port, rank 0 only."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    import oracle
    import paper_1708_01159_b200.graph as G
    from paper_1708_01159_b200.features import canonical_indices, static_vector
    from paper_1708_01159_b200.tree import deserialize

    t0 = time.time()
    threads = os.cpu_count() or 1
    src, dst = oracle.generate_rmat_pairs(a.scale, 16 << a.scale, 1, threads=threads)
    og = oracle.build_combined(1 << a.scale, np.concatenate([src, dst]), np.concatenate([dst, src]))
    del src, dst
    stats = G.stats_from_offsets(og.n, og.m, og.out_offsets, og.in_offsets)
    static24 = static_vector(stats)
    roots = pick_roots(og.out_offsets, 64, seed=1)
    flat = deserialize(a.model)
    ot = oracle.OracleTree(canonical_indices(flat.selection), flat.features, flat.thresholds,
                           flat.lefts, flat.rights, flat.leaf_classes)
    deg = np.diff(og.out_offsets.astype(np.int64))
    setup = time.time() - t0
    # the same steps as the GPU arm: R roots per step, rotating through the
    # 64-root pool in the same order, warm-up steps first
    R = a.roots_per_step
    order = [roots[i % len(roots)] for i in range(R * (a.warmup + a.steps))]
    edges_tot, el_tot, times = 0.0, 0.0, []
    for s in range(a.warmup + a.steps):
        t1 = time.perf_counter()
        e_step = 0.0
        for r in order[s * R:(s + 1) * R]:
            d, _ = oracle.adaptive_bfs(og, r, ot, static24, threads=threads)
            e_step += deg[d != 2**31 - 1].sum() / 2
        el = time.perf_counter() - t1
        if s >= a.warmup:
            edges_tot += e_step
            el_tot += el
            times.append(el)
    gteps = edges_tot / el_tot / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": round(gteps, 5), "unit": UNIT,
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": round(1e3 * el_tot / max(1, a.steps), 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (host-generated Kronecker, same generator/seed)",
            "config": workload_config(a, f"kronecker-{a.scale}-ef16-symmetrised", og.n, og.m, True, R),
            "implementation": {"step": f"{R} tree-switched BFSs per step, one after the other, "
                                       "C+OpenMP port of the reference level kernels (oracle/)",
                               "parallelism": f"{threads} host threads"},
            "cpu_baseline": {"value": round(gteps, 5), "unit": UNIT, "cores": threads,
                             "kind": "port", "cpu_model": cpu_model(), "numpy": np.__version__,
                             "sample": f"{R} tree-switched BFSs per step ({a.steps} steps) on the "
                                       f"full graph; C+OpenMP port of the reference kernels"},
            "e2e": {"value": round(gteps, 5), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "setup_s": round(setup, 1)}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=int, default=None)
    ap.add_argument("--roots-per-step", type=int, default=8)
    ap.add_argument("--model", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--fixed-roots", type=int, default=4,
                    help="roots for the per-pair fixed-variant comparison")
    ap.add_argument("--graph", default="kronecker", choices=["kronecker", "er", "mesh"],
                    help="workload graph (configs 2 / 5 / 4); the headline is kronecker")
    ap.add_argument("--partition", action="store_true",
                    help="config 3: one BFS over a 1-D vertex partition (default scale 26)")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="--partition frontier exchange: fused peer stores or NCCL all-gather")
    ap.add_argument("--virtual-parts", type=int, default=8,
                    help="--partition at N=1: partitions sharing the one GPU")
    ap.add_argument("--permute", action="store_true",
                    help="Kronecker with ids relabelled by a fixed bijection (hubs spread over the "
                         "id space; a robustness run, not the reference's generator)")
    ap.add_argument("--root-sharded", action="store_true",
                    help="N > 1: replicate the graph and shard the roots (no exchange) instead of "
                         "the 1-D partitioned BFS")
    ap.add_argument("--shared-gpu", action="store_true",
                    help="N > 1 test mode: all ranks on GPU 0 (gloo control plane; the peer "
                         "exchange still runs through CUDA IPC)")
    ap.add_argument("--nccl-line", action="store_true",
                    help="N > 1: also time the BFS with the NCCL all-gather exchange (per-level "
                         "launches + all_gather_into_tensor; not verifiable on a one-GPU box)")
    ap.add_argument("--no-secondary", action="store_true",
                    help="N > 1: skip the NCCL-exchange and Kronecker-26 secondary lines")
    ap.add_argument("--mode", type=int, default=1,
                    help="1: device-resident level loop (megakernel); 0: per-level launches")
    a = ap.parse_args()
    a.model = os.path.abspath(a.model) if a.model else default_model()
    if a.warmup < 3:
        a.warmup = 3
    if a.scale is None:
        a.scale = 26 if a.partition else 24
    if a.impl == "reference":
        run_reference(a)
    elif a.partition:
        run_partitioned(a)
    elif env_rank()[1] > 1 and not a.root_sharded:
        run_multi(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
