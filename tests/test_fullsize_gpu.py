"""Full-size configurations (BASELINE.json configs 2-5) on one B200: depth
arrays from the tree-switched BFS and from fixed pairs equal the CPU oracle's
reference_bfs (exact), plus size-independent properties (frontier
conservation, mesh closed form, relaxation |d(u) - d(v)| <= 1 on every
symmetric edge)."""

from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
import paper_1708_01159_b200 as P
from paper_1708_01159_b200 import DeviceGraph, Traversal
from paper_1708_01159_b200.features import static_vector

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODEL = os.path.join(ROOT, "models", "gpu_tree.tree")
INF = 2**31 - 1


def check_graph(dg, roots, pairs, symmetric):
    oo, io = dg.offsets()
    a = dg.download()
    og = oracle.OracleGraph(dg.vertex_count, dg.edge_count, a["out_offsets"], a["destinations"],
                            a["origins"], a["in_offsets"], a["sources"], rev_owner=np.zeros(1, np.uint32))
    flat = P.deserialize(MODEL)
    stats = P.compute_stats(dg)
    t = Traversal(dg)
    for r in roots:
        want = oracle.reference_bfs(og, r)
        hist = np.bincount(want[want != INF])
        d = np.empty(dg.vertex_count, np.int32)
        recs = t.adaptive(r, flat.as_abfs(), static_vector(stats), 32, depths_out=d)
        np.testing.assert_array_equal(d, want)
        assert [int(x.frontier_size) for x in recs] == hist.tolist()
        assert sum(int(x.new_count) for x in recs) + 1 == int((want != INF).sum())
        if symmetric:
            du = want[a["origins"]].astype(np.int64)
            dv = want[a["destinations"]].astype(np.int64)
            reach = du != INF
            assert (dv[reach] != INF).all() and (np.abs(du[reach] - dv[reach]) <= 1).all()
        for k, v in pairs:
            counts, _ = t.bfs_full(r, k, v, 32, depths_out=d)
            np.testing.assert_array_equal(d, want, err_msg=f"{k} {v} root {r}")
            assert counts.tolist()[:-1] == hist[1:].tolist()
    t.close()


def test_config2_kronecker24():
    dg = DeviceGraph.rmat(24, 16 << 24, 1, symmetrize=True)
    check_graph(dg, [0, 6391562], [(4, 2), (3, 2), (0, 2), (1, 1)], symmetric=True)


def test_config4_mesh_4096():
    dg = DeviceGraph.mesh(4096, 4096)
    t = Traversal(dg)
    d = np.empty(dg.vertex_count, np.int32)
    counts, _ = t.bfs_full(0, 2, 1, 32, depths_out=d)
    r, c = np.divmod(np.arange(dg.vertex_count, dtype=np.int64), 4096)
    np.testing.assert_array_equal(d, (r + c).astype(np.int32))   # Manhattan distance
    assert len(counts) == 8191
    t.close()
    check_graph(dg, [4096 * 2048 + 2048], [(4, 2)], symmetric=True)


def test_config5_erdos_renyi_32m():
    dg = DeviceGraph.uniform(1 << 25, 1 << 30, 1)
    check_graph(dg, [12345], [(3, 2), (4, 2)], symmetric=False)


def test_config3_kronecker26_single_gpu():
    dg = DeviceGraph.rmat(26, 16 << 26, 1, symmetrize=True)
    assert dg.edge_count == 1 << 31
    check_graph(dg, [1], [(4, 2)], symmetric=False)


def test_config3_kronecker26_partitioned_8():
    """Config 3's 1-D vertex partition (8 edge-balanced ranges, exchanged by
    device concat on one GPU -- the same buffers NCCL all-gathers across
    GPUs) equals the single-GPU engine: traces and depths."""
    import torch

    from paper_1708_01159_b200.partition import LocalExchange, PartitionedBFS, local_partitions
    dg = DeviceGraph.rmat(26, 16 << 26, 1, symmetrize=True)
    stats = P.compute_stats(dg)
    flat = P.deserialize(MODEL)
    want = {}
    t = Traversal(dg)
    for r in (1, 123457):
        d = np.empty(dg.vertex_count, np.int32)
        recs = t.adaptive(r, flat.as_abfs(), static_vector(stats), 32, depths_out=d)
        want[r] = (d, [(x.kernel, x.variant, x.fallback, x.frontier_size) for x in recs])
    t.close()
    ps, bounds = local_partitions(dg, 8, torch.cuda.current_stream().cuda_stream)
    dg.close()
    bfs = PartitionedBFS(ps, bounds, LocalExchange(torch),
                         alloc=lambda s: torch.zeros(s, dtype=torch.int32, device="cuda"))
    for r, (d, tr) in want.items():
        got = bfs.adaptive(r, flat, stats)
        assert [(int(x.kernel), int(x.variant), int(x.fallback_used), x.frontier_size)
                for x in got.records] == tr
        np.testing.assert_array_equal(bfs.depths(), d)
    for p in ps:
        p.close()
