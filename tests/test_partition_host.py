"""1-D vertex partition host logic on CPU: edge-balanced
bounds, word bounds, and the PartitionedBFS driver over world-size-2 gloo
processes and over P in-process partitions, each local level restated by
the numpy oracle, against the reference's golden depths / counts / traces."""

from __future__ import annotations

import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import golden_util as G
import paper_1708_01159_b200 as P
from oracle.partition import OraclePartition
from paper_1708_01159_b200.graph import stats_from_offsets
from paper_1708_01159_b200.partition import (LocalExchange, PartitionedBFS,
                                             edge_balanced_bounds, word_bounds)

import partition_worker


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
@pytest.mark.parametrize("name", ["kron12", "u1000", "mesh64", "star7", "single"])
def test_edge_balanced_bounds(name, parts):
    n, m, a = G.graph_arrays(name)
    b = edge_balanced_bounds(a["in_offsets"], parts)
    assert b.size == parts + 1 and b[0] == 0 and b[-1] == n
    assert np.all(np.diff(b) >= 0)
    assert np.all(b[1:-1] % 32 == 0)
    wb = word_bounds(b)
    assert wb[0] == 0 and wb[-1] == (n + 31) // 32 and np.all(np.diff(wb.astype(np.int64)) >= 0)


def test_edge_balance_beats_vertex_split():
    n, m, a = G.graph_arrays("kron12")
    io = a["in_offsets"].astype(np.int64)
    b = edge_balanced_bounds(io, 8)
    share = np.diff(io[b]) / (m / 8)
    vb = np.linspace(0, n, 9).astype(np.int64)
    vshare = np.diff(io[vb]) / (m / 8)
    assert share.max() < vshare.max()
    assert share.max() < 1.25


def test_bounds_reject_bad_arguments():
    with pytest.raises(ValueError):
        edge_balanced_bounds(np.array([0, 1]), 0)
    with pytest.raises(ValueError):
        edge_balanced_bounds(np.array([0, 1]), 2, align=48)


@pytest.mark.parametrize("parts", [2, 3, 5])
@pytest.mark.parametrize("name", ["kron10", "u60", "hand1", "path9", "unreach", "er12"])
def test_in_process_partitions_match_golden(name, parts):
    n, m, a = G.graph_arrays(name)
    bounds = edge_balanced_bounds(a["in_offsets"], parts)
    ps = [OraclePartition(n, a["in_offsets"], a["sources"], int(bounds[i]), int(bounds[i + 1]))
          for i in range(parts)]
    bfs = PartitionedBFS(ps, bounds, LocalExchange(torch),
                         alloc=lambda s: torch.zeros(s, dtype=torch.int32))
    stats = stats_from_offsets(n, m, a["out_offsets"], a["in_offsets"])
    traces = G.traces()["small"]
    for r in G.roots(name):
        outs = bfs.bfs_full(r, P.KernelId.EDGE_LIST, P.CountVariant.DIRECT_ATOMIC)
        assert [o.new_frontier_count for o in outs] == G.counts(name, r).tolist()
        # local counts of every level add up to the global count
        assert [sum(x) for x in bfs.last_local_counts] == G.counts(name, r).tolist()
        np.testing.assert_array_equal(bfs.depths(), G.depth(name, r))
        flat = P.deserialize(G.tree_path("t1"))
        tr = bfs.adaptive(r, flat, stats)
        got = [[int(x.kernel), int(x.variant), int(x.fallback_used), x.frontier_size]
               for x in tr.records]
        assert got == traces[name][str(r)]["t1"]


def test_partitioned_rejects_bad_root():
    n, m, a = G.graph_arrays("hand1")
    bounds = edge_balanced_bounds(a["in_offsets"], 1)
    ps = [OraclePartition(n, a["in_offsets"], a["sources"], 0, n)]
    bfs = PartitionedBFS(ps, bounds, LocalExchange(torch),
                         alloc=lambda s: torch.zeros(s, dtype=torch.int32))
    with pytest.raises(ValueError, match="out of range"):
        bfs.bfs_full(n, P.KernelId.EDGE_LIST, P.CountVariant.DIRECT_ATOMIC)


def test_gloo_world_size_2_matches_golden():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    names = ["kron10", "u60", "hand1", "mesh7x13", "unreach", "dup", "star7"]
    procs = [ctx.Process(target=partition_worker.run_rank, args=(r, 2, port, names, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, checked in res:
        assert status == "ok", f"rank {rank}:\n{status}"
        assert checked > 0


def test_gen_spec_sizes_and_validation():
    """abfs_gen_size needs no GPU: |V| / |E| of each generator spec, and the
    generators' argument errors (graph.py:211-252's configs)."""
    from paper_1708_01159_b200.partition import gen_size, gen_spec
    assert gen_size(gen_spec("rmat", scale=24, edges=16 << 24, seed=1, symmetrize=True)) == \
        (1 << 24, 32 << 24)
    assert gen_size(gen_spec("rmat", scale=10, edges=1000, seed=1)) == (1024, 1000)
    assert gen_size(gen_spec("uniform", n=1 << 25, edges=1 << 30, seed=1)) == (1 << 25, 1 << 30)
    assert gen_size(gen_spec("mesh", rows=4096, cols=4096)) == (4096 * 4096, 2 * 2 * 4096 * 4095)
    with pytest.raises(ValueError, match="power-of-two"):
        gen_size(gen_spec("uniform", n=1000, edges=10, seed=1))
    with pytest.raises(ValueError, match="scale"):
        gen_size(gen_spec("rmat", scale=0, edges=10, seed=1))
    with pytest.raises(ValueError, match="2\\^32"):
        gen_size(gen_spec("rmat", scale=28, edges=16 << 28, seed=1, symmetrize=True))
    with pytest.raises(ValueError, match="unknown generator"):
        gen_spec("kron", scale=3)
