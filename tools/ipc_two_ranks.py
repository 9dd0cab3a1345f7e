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
        # slices built from the generator stream on each rank (bench --gpus N path)
        from paper_1708_01159_b200.partition import gen_offsets, gen_spec
        spec = gen_spec("rmat", scale=12, edges=16 << 12, seed=1, symmetrize=True)
        oo, io = gen_offsets(spec, 0)
        bounds = edge_balanced_bounds(io, world)
        part = DevicePartition(None, int(bounds[rank]), int(bounds[rank + 1]),
                               torch.cuda.current_stream().cuda_stream, spec=spec, device=0)
        bfs = PartitionedBFS([part], bounds, DistPeerExchange(torch, dist, part), alloc=None)
        stats = stats_from_offsets(1 << 12, 32 << 12, oo, io)
        host = DeviceGraph.rmat(12, 16 << 12, 1, symmetrize=True).to_graph()
        flat = P.deserialize(os.path.join(ROOT, "models", "gpu_tree.tree"))
        cand = np.flatnonzero(np.diff(oo.astype(np.int64)) > 0)
        for r in (int(cand[0]), int(cand[len(cand) // 2]), int(cand[-1])):
            bfs.adaptive(r, flat, stats)
            np.testing.assert_array_equal(bfs.depths(), P.reference_bfs(host, r))
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
