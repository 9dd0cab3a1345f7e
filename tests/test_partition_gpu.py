"""GPU parity of the 1-D vertex-partitioned BFS: P partitions
of one graph on one B200 (the exchange is a device concat; across GPUs it is
the NCCL all-gather over the same buffers) reproduce the reference's golden
depths, per-level counts and adaptive traces for every (kernel, variant),
and equal the single-GPU engine on larger device-generated graphs."""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch

import golden_util as G
import paper_1708_01159_b200 as P
from paper_1708_01159_b200 import DeviceGraph, Traversal
from paper_1708_01159_b200.features import static_vector
from paper_1708_01159_b200.graph import stats_from_offsets
from paper_1708_01159_b200.partition import (LocalExchange, LocalPeerExchange, PartitionedBFS,
                                             local_partitions)

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODEL = os.path.join(ROOT, "models", "gpu_tree.tree")


def make_bfs(dg, parts, exchange="gather"):
    """exchange: "gather" = send buffers + all-gather (device concat here, NCCL
    across GPUs); "peer" = fused kernel stores into every partition's bitmap."""
    stream = torch.cuda.current_stream().cuda_stream
    ps, bounds = local_partitions(dg, parts, stream)
    ex = LocalExchange(torch) if exchange == "gather" else LocalPeerExchange(torch, ps)
    return PartitionedBFS(ps, bounds, ex,
                          alloc=lambda s: torch.zeros(s, dtype=torch.int32, device="cuda"))


@pytest.mark.parametrize("exchange", ["gather", "peer"])
@pytest.mark.parametrize("parts", [1, 2, 3, 4])
@pytest.mark.parametrize("name", ["kron10", "kron12", "u1000", "er12", "mesh64", "hand1",
                                  "unreach", "dup", "selfloop", "star7", "single", "path9"])
def test_partitions_all_pairs_match_golden(name, parts, exchange):
    n, m, a = G.graph_arrays(name)
    g = P.Graph(n, m, *[a[k].copy() for k in G.ARRAYS])
    dg = DeviceGraph.upload(g)
    bfs = make_bfs(dg, parts, exchange)
    stats = stats_from_offsets(n, m, a["out_offsets"], a["in_offsets"])
    traces = G.traces()["small"]
    for r in G.roots(name):
        want = G.depth(name, r)
        cnt = G.counts(name, r).tolist()
        for k, v in P.ALL_PAIRS:
            outs = bfs.bfs_full(r, k, v)
            assert [o.new_frontier_count for o in outs] == cnt, (name, parts, r, k, v)
            assert [sum(x) for x in bfs.last_local_counts] == cnt, (name, parts, r, k, v)
            np.testing.assert_array_equal(bfs.depths(), want, err_msg=f"{name} {parts} {r} {k} {v}")
        for key, tree in G.trees_for(name):
            tr = bfs.adaptive(r, P.deserialize(G.tree_path(tree)), stats)
            got = [[int(x.kernel), int(x.variant), int(x.fallback_used), x.frontier_size]
                   for x in tr.records]
            assert got == traces[name][str(r)][key], (name, parts, r, key)
            np.testing.assert_array_equal(bfs.depths(), want)


@pytest.mark.parametrize("exchange", ["gather", "peer"])
@pytest.mark.parametrize("cfg,parts", [("k18", 8), ("er18", 4), ("mesh256", 3)])
def test_partitions_equal_single_gpu_engine(cfg, parts, exchange):
    if cfg.startswith("k"):
        dg = DeviceGraph.rmat(18, 16 << 18, 1, symmetrize=True)
    elif cfg.startswith("er"):
        dg = DeviceGraph.uniform(1 << 18, 32 << 18, 1)
    else:
        dg = DeviceGraph.mesh(256, 256)
    stats = P.compute_stats(dg)
    flat = P.deserialize(MODEL)
    t = Traversal(dg)
    bfs = make_bfs(dg, parts, exchange)
    oo, _ = dg.offsets()
    cand = np.flatnonzero(np.diff(oo.astype(np.int64)) > 0)
    for r in [int(cand[0]), int(cand[len(cand) // 2]), int(cand[-1])]:
        want = np.empty(dg.vertex_count, np.int32)
        recs = t.adaptive(r, flat.as_abfs(), static_vector(stats), 32, depths_out=want)
        tr = bfs.adaptive(r, flat, stats)
        assert [(int(x.kernel), int(x.variant), int(x.fallback_used), x.frontier_size)
                for x in tr.records] == \
               [(x.kernel, x.variant, x.fallback, x.frontier_size) for x in recs]
        np.testing.assert_array_equal(bfs.depths(), want)
        for k, v in [(P.KernelId.VERTEX_PUSH_WARP, P.CountVariant.TWO_LEVEL_REDUCE),
                     (P.KernelId.REV_EDGE_LIST, P.CountVariant.GROUP_REDUCE)]:
            outs = bfs.bfs_full(r, k, v)
            assert sum(o.new_frontier_count for o in outs) + 1 == int((want != G.INF).sum())
            np.testing.assert_array_equal(bfs.depths(), want)


@pytest.mark.parametrize("xsys", ["0", "1", "2"])
def test_persistent_partition_loop_exchange_scopes(xsys, monkeypatch):
    """The persistent per-rank loop's exchange: GPU-scoped release/acquire when
    every peer bitmap is on this device (0), system-scoped (1), or the LL
    words (epoch | bitmap word in one 8-byte store, no fence) used across
    devices (2); ABFS_XSYS forces each; all must give the single-engine
    traversal."""
    monkeypatch.setenv("ABFS_XSYS", xsys)
    dg = DeviceGraph.rmat(18, 16 << 18, 1, symmetrize=True)
    stats = P.compute_stats(dg)
    flat = P.deserialize(MODEL)
    t = Traversal(dg)
    bfs = make_bfs(dg, 1, "peer")
    assert bfs.persistent
    oo, _ = dg.offsets()
    cand = np.flatnonzero(np.diff(oo.astype(np.int64)) > 0)
    for r in [int(cand[0]), int(cand[len(cand) // 2]), int(cand[-1])]:
        want = np.empty(dg.vertex_count, np.int32)
        recs = t.adaptive(r, flat.as_abfs(), static_vector(stats), 32, depths_out=want)
        for _ in range(2):   # back-to-back launches continue the exchange sequence
            tr = bfs.adaptive(r, flat, stats)
            assert [(int(x.kernel), int(x.variant), x.frontier_size) for x in tr.records] == \
                   [(x.kernel, x.variant, x.frontier_size) for x in recs]
            np.testing.assert_array_equal(bfs.depths(), want)
        outs = bfs.bfs_full(r, P.KernelId.VERTEX_PULL, P.CountVariant.GROUP_REDUCE)
        assert sum(o.new_frontier_count for o in outs) + 1 == int((want != G.INF).sum())


def test_partition_rejects_misaligned_range():
    n, m, a = G.graph_arrays("kron10")
    dg = DeviceGraph.upload(P.Graph(n, m, *[a[k].copy() for k in G.ARRAYS]))
    from paper_1708_01159_b200.partition import DevicePartition
    with pytest.raises(ValueError, match="multiple of 32"):
        DevicePartition(dg, 5, 64)
    with pytest.raises(ValueError, match="out of bounds"):
        DevicePartition(dg, 0, n + 1)


@pytest.mark.parametrize("xsys", [None, "2"])
def test_peer_exchange_over_cuda_ipc_two_processes(xsys, monkeypatch):
    """DistPeerExchange: two processes (one GPU here; one per GPU in
    production) map each other's bitmaps/mailboxes by CUDA IPC and exchange
    frontier slices with the fused peer-store kernel (xsys "2": the LL-word
    exchange cross-device ranks use, forced on the shared GPU)."""
    if xsys is not None:
        monkeypatch.setenv("ABFS_XSYS", xsys)
    import sys
    sys.path.insert(0, ROOT)
    from tools import ipc_two_ranks
    for rank, status, checked in ipc_two_ranks.main():
        assert status == "ok", f"rank {rank}:\n{status}"
        assert checked > 0


# ---- slices built from the generator stream (no whole graph on the GPU) ------

GEN_CASES = [
    ("rmat", dict(scale=12, edges=16 << 12, seed=1, symmetrize=True),
     lambda: DeviceGraph.rmat(12, 16 << 12, 1, symmetrize=True)),
    ("rmat", dict(scale=11, edges=8 << 11, seed=7, symmetrize=False),
     lambda: DeviceGraph.rmat(11, 8 << 11, 7)),
    ("uniform", dict(n=1 << 12, edges=20 << 12, seed=3),
     lambda: DeviceGraph.uniform(1 << 12, 20 << 12, 3)),
    ("uniform", dict(n=1 << 10, edges=4099, seed=2),   # odd edge count: dst stream starts mid-draw
     lambda: DeviceGraph.uniform(1 << 10, 4099, 2)),
    ("mesh", dict(rows=37, cols=70), lambda: DeviceGraph.mesh(37, 70)),
]


@pytest.mark.parametrize("case", range(len(GEN_CASES)))
def test_generated_degrees_and_slices_equal_full_graph_slices(case):
    from paper_1708_01159_b200.partition import (DevicePartition, edge_balanced_bounds,
                                                 gen_offsets, gen_spec)
    kind, kw, full = GEN_CASES[case]
    spec = gen_spec(kind, **kw)
    dg = full()
    oo, io = dg.offsets()
    goo, gio = gen_offsets(spec)
    np.testing.assert_array_equal(goo, oo)
    np.testing.assert_array_equal(gio, io)
    for parts in (1, 3, 5):
        bounds = edge_balanced_bounds(io, parts)
        for i in range(parts):
            lo, hi = int(bounds[i]), int(bounds[i + 1])
            a = DevicePartition(dg, lo, hi).download()
            b = DevicePartition(None, lo, hi, spec=spec, device=0).download()
            for k in a:
                np.testing.assert_array_equal(b[k], a[k], err_msg=f"{kind} P={parts} part {i} {k}")


def test_generated_partitions_bfs_equal_single_gpu_engine():
    from paper_1708_01159_b200.partition import (DevicePartition, edge_balanced_bounds,
                                                 gen_offsets, gen_spec)
    spec = gen_spec("rmat", scale=16, edges=16 << 16, seed=1, symmetrize=True)
    oo, io = gen_offsets(spec)
    stats = stats_from_offsets(1 << 16, 32 << 16, oo, io)
    bounds = edge_balanced_bounds(io, 4)
    stream = torch.cuda.current_stream().cuda_stream
    ps = [DevicePartition(None, int(bounds[i]), int(bounds[i + 1]), stream, spec=spec, device=0)
          for i in range(4)]
    bfs = PartitionedBFS(ps, bounds, LocalPeerExchange(torch, ps), alloc=None)
    dg = DeviceGraph.rmat(16, 16 << 16, 1, symmetrize=True)
    t = Traversal(dg)
    flat = P.deserialize(MODEL)
    cand = np.flatnonzero(np.diff(oo.astype(np.int64)) > 0)
    for r in [int(cand[0]), int(cand[len(cand) // 3]), int(cand[-1])]:
        want = np.empty(dg.vertex_count, np.int32)
        recs = t.adaptive(r, flat.as_abfs(), static_vector(stats), 32, depths_out=want)
        tr = bfs.adaptive(r, flat, stats)
        assert [(int(x.kernel), int(x.variant), x.frontier_size) for x in tr.records] == \
               [(x.kernel, x.variant, x.frontier_size) for x in recs]
        np.testing.assert_array_equal(bfs.depths(), want)


@pytest.mark.parametrize("xsys", [None, "2"])
def test_multi_gpu_bench_runs_end_to_end_with_ranks_sharing_one_gpu(xsys, monkeypatch):
    """bench.py --gpus 2 under torchrun (the driver's SCALE launch) with both
    ranks on GPU 0 (--shared-gpu: gloo control plane; slices from the
    generator stream; fused peer exchange over CUDA IPC): one JSON line
    (xsys "2": with the cross-device LL-word exchange forced)."""
    if xsys is not None:
        monkeypatch.setenv("ABFS_XSYS", xsys)
    import json
    import subprocess
    import sys
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29533 + (xsys is not None)),
           "bench.py", "--gpus", "2",
           "--shared-gpu", "--scale", "14", "--steps", "1", "--warmup", "3",
           "--roots-per-step", "2"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["gpu_launches"] > 0 and d["e2e"]["value"] > 0
    assert "1-D edge-balanced" in d["config"]["parallelism"]
