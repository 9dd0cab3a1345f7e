"""One bench step (an 8-root `abfs_adaptive_bfs_batch` launch of `k_mega` on
Kronecker-24, the bench's graph, tree and roots) bracketed by
cudaProfilerStart/Stop, so ncu captures exactly the kernel bench.py times:

    ncu --profile-from-start off --set full --clock-control none \
        --import-source on -k regex:k_mega -o gpurun_out/kmega \
        python tools/prof_kmega.py [R] [first_root_index]

ABFS_PROF_GRAPH=mesh profiles the 4096^2 mesh (config 4) instead.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1708_01159_b200 as P  # noqa: E402
from bench import default_model, pick_roots  # noqa: E402
from paper_1708_01159_b200 import DeviceGraph, Traversal  # noqa: E402
from paper_1708_01159_b200.features import static_vector  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
first = int(sys.argv[2]) if len(sys.argv) > 2 else 24   # bench's first timed step: roots 24..31
scale = int(os.environ.get("ABFS_PROF_SCALE", "24"))
if os.environ.get("ABFS_PROF_GRAPH") == "mesh":   # config 4 (ABFS_PROF_GRAPH=mesh, R=1)
    dg = DeviceGraph.mesh(4096, 4096)
else:
    dg = DeviceGraph.rmat(scale, 16 << scale, 1, symmetrize=True)
oo, _ = dg.offsets()
stats = P.compute_stats(dg)
tree = P.deserialize(default_model()).as_abfs()
st = static_vector(stats)
roots = pick_roots(oo, 64, seed=1)
batch = [roots[(first + i) % len(roots)] for i in range(R)]
t = Traversal(dg)
stream = torch.cuda.Stream()
t.set_stream(stream.cuda_stream)
t.adaptive_batch(batch, tree, st, 32)      # warm-up (untimed, not profiled)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
_, ns, _ = t.adaptive_batch(batch, tree, st, 32)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("roots", batch, "bfs ns", ns.tolist())
