"""Two processes on one GPU driving the fused peer exchange through CUDA IPC
(the one-process-per-GPU path of partition.DistPeerExchange), checked
against the golden depths.  Used by tests/test_partition_gpu.py."""
import os
import socket
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def worker(rank, world, port, q):
    import numpy as np
    import torch
    import torch.distributed as dist

    import golden_util as G
    import paper_1708_01159_b200 as P
    from paper_1708_01159_b200 import DeviceGraph
    from paper_1708_01159_b200.graph import stats_from_offsets
    from paper_1708_01159_b200.partition import (DevicePartition, DistPeerExchange,
                                                 PartitionedBFS, edge_balanced_bounds)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        torch.cuda.set_device(0)
        checked = 0
        for name in ("kron10", "u1000", "mesh64"):
            n, m, a = G.graph_arrays(name)
            dg = DeviceGraph.upload(P.Graph(n, m, *[a[k].copy() for k in G.ARRAYS]))
            bounds = edge_balanced_bounds(a["in_offsets"], world)
            part = DevicePartition(dg, int(bounds[rank]), int(bounds[rank + 1]),
                                   torch.cuda.current_stream().cuda_stream)
            bfs = PartitionedBFS([part], bounds, DistPeerExchange(torch, dist, part), alloc=None)
            stats = stats_from_offsets(n, m, a["out_offsets"], a["in_offsets"])
            flat = P.deserialize(G.tree_path("t1"))
            for r in G.roots(name)[:3]:
                tr = bfs.adaptive(r, flat, stats)
                got = [[int(x.kernel), int(x.variant), int(x.fallback_used), x.frontier_size]
                       for x in tr.records]
                assert got == G.traces()["small"][name][str(r)]["t1"], (name, r)
                np.testing.assert_array_equal(bfs.depths(), G.depth(name, r))
                checked += 1
            dist.barrier()
            part.close()
        q.put((rank, "ok", checked))
    except Exception:
        q.put((rank, traceback.format_exc(), 0))
    finally:
        dist.destroy_process_group()


def main(world=2, timeout=300):
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=timeout) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    return res


if __name__ == "__main__":
    for r in main():
        print(r)
