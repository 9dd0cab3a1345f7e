"""Worker of the world-size-2 gloo tests (tests/test_partition_host.py):
each rank drives one OraclePartition through the production
PartitionedBFS driver + DistExchange and checks depths, per-level counts
and adaptive traces against the reference's golden vectors."""

from __future__ import annotations

import os
import sys
import traceback

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)


def run_rank(rank, world, port, names, queue):
    import numpy as np
    import torch
    import torch.distributed as dist

    import golden_util as G
    import paper_1708_01159_b200 as P
    from oracle.partition import OraclePartition
    from paper_1708_01159_b200.graph import stats_from_offsets
    from paper_1708_01159_b200.partition import (DistExchange, PartitionedBFS,
                                                 edge_balanced_bounds)

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    checked = 0
    try:
        traces = G.traces()["small"]
        for name in names:
            n, m, a = G.graph_arrays(name)
            bounds = edge_balanced_bounds(a["in_offsets"], world)
            part = OraclePartition(n, a["in_offsets"], a["sources"], int(bounds[rank]),
                                   int(bounds[rank + 1]))
            bfs = PartitionedBFS([part], bounds, DistExchange(torch, dist),
                                 alloc=lambda s: torch.zeros(s, dtype=torch.int32))
            stats = stats_from_offsets(n, m, a["out_offsets"], a["in_offsets"])
            for r in G.roots(name):
                outs = bfs.bfs_full(r, P.KernelId.VERTEX_PULL, P.CountVariant.GROUP_REDUCE)
                assert [o.new_frontier_count for o in outs] == G.counts(name, r).tolist(), (name, r)
                np.testing.assert_array_equal(bfs.depths(), G.depth(name, r))
                for key, tree in G.trees_for(name):
                    flat = P.deserialize(G.tree_path(tree))
                    tr = bfs.adaptive(r, flat, stats)
                    got = [[int(x.kernel), int(x.variant), int(x.fallback_used), x.frontier_size]
                           for x in tr.records]
                    assert got == traces[name][str(r)][key], (name, r, key)
                    np.testing.assert_array_equal(bfs.depths(), G.depth(name, r))
                    checked += 1
        queue.put((rank, "ok", checked))
    except Exception:
        queue.put((rank, traceback.format_exc(), checked))
    finally:
        dist.destroy_process_group()
