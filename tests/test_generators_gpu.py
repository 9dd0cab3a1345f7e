"""Device generators + device build_combined are bit-exact to the reference
generate_graph/build_combined (golden sha256 pins, K16 config 1 included)."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import golden_util as G
import paper_1708_01159_b200 as P
from paper_1708_01159_b200 import DeviceGraph

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def assert_pinned(dg, spec):
    assert (dg.vertex_count, dg.edge_count) == (spec["V"], spec["E"])
    a = dg.download(rev_owner=True)
    for k in G.ARRAYS:
        assert sha(a[k]) == spec["sha256"][k], k
    want_owner = np.repeat(np.arange(dg.vertex_count, dtype=np.uint32),
                           np.diff(a["in_offsets"].astype(np.int64)))
    np.testing.assert_array_equal(a["rev_owner"], want_owner)


@pytest.mark.parametrize("label", ["rmat_s8", "rmat_s12_sym", "uniform_n1024", "uniform_n2p16"])
def test_generator_pins(label):
    spec = G.meta()["generators"][label]
    p = spec["params"]
    if spec["model"] == "rmat-like":
        dg = DeviceGraph.rmat(p["scale"], p["edges"], spec["seed"], symmetrize=spec["sym"])
    else:
        dg = DeviceGraph.uniform(p["n"], p["edges"], spec["seed"])
    assert_pinned(dg, spec)


def test_k16_config1_generator():
    meta = G.traces()["k16"]
    dg = DeviceGraph.rmat(16, 16 << 16, 1, symmetrize=True)
    assert_pinned(dg, meta)


def test_mesh_4096_config4_generator():
    dg = DeviceGraph.mesh(4096, 4096)
    assert_pinned(dg, G.meta()["generators"]["mesh4096"])


@pytest.mark.parametrize("name", G.graph_names())
def test_device_build_combined_and_upload(name):
    n, m, a = G.graph_arrays(name)
    rng = np.random.default_rng(1)
    perm = rng.permutation(m)
    dg = DeviceGraph.build(n, a["origins"][perm], a["destinations"][perm])
    got = dg.download(rev_owner=True)
    for k in G.ARRAYS + ("rev_owner",):
        np.testing.assert_array_equal(got[k], a[k], err_msg=k)
    up = DeviceGraph.upload(P.Graph(n, m, *[a[k].copy() for k in G.ARRAYS]))
    got = up.download(rev_owner=True)
    for k in G.ARRAYS + ("rev_owner",):
        np.testing.assert_array_equal(got[k], a[k], err_msg=k)


def test_reference_named_construction_routes_to_the_device(monkeypatch):
    """build_combined / generate_graph (graph.py:93-134, 211-252) build large
    inputs in HBM: the arrays equal the host construction's, stats are taken
    from the offsets only, and traversals use the resident copy (no upload)."""
    from paper_1708_01159_b200.graph import DeviceResidentGraph
    rng = np.random.default_rng(5)
    n = 5000
    pairs = rng.integers(0, n, size=(40000, 2))
    host = P.build_combined(pairs, n)
    monkeypatch.setenv("ABFS_DEVICE_BUILD_MIN_EDGES", "1000")
    dev = P.build_combined(pairs, n)
    assert isinstance(dev, DeviceResidentGraph) and not isinstance(host, DeviceResidentGraph)
    st = P.compute_stats(dev)
    assert dev._host is None          # stats did not download the edge arrays
    assert st == P.compute_stats(host)
    for k in ("out_offsets", "destinations", "origins", "in_offsets", "sources"):
        np.testing.assert_array_equal(getattr(dev, k), getattr(host, k), err_msg=k)
    np.testing.assert_array_equal(dev.rev_owner(), host.rev_owner())
    for r in (0, 17, 4999):
        d1, _ = P.bfs_full(dev, r, P.KernelId.VERTEX_PULL, P.CountVariant.GROUP_REDUCE)
        np.testing.assert_array_equal(d1, P.reference_bfs(host, r))
    assert dev.device_graph() is dev._dg
    # generators: rmat-like and uniform-random straight on the device
    for model, params in (("rmat-like", {"scale": 12, "edges": 16 << 12}),
                          ("uniform-random", {"n": 1 << 12, "edges": 20 << 12})):
        g_dev = P.generate_graph(model, params, 3)
        assert isinstance(g_dev, DeviceResidentGraph)
        monkeypatch.setenv("ABFS_DEVICE_BUILD_MIN_EDGES", str(1 << 40))
        g_host = P.generate_graph(model, params, 3)
        monkeypatch.setenv("ABFS_DEVICE_BUILD_MIN_EDGES", "1000")
        assert not isinstance(g_host, DeviceResidentGraph)
        for k in ("out_offsets", "destinations", "origins", "in_offsets", "sources"):
            np.testing.assert_array_equal(getattr(g_dev, k), getattr(g_host, k), err_msg=(model, k))
    # non-power-of-two uniform: host draws (the device stream needs 2^k), then
    # the device build of the pairs -- still the reference's arrays
    g = P.generate_graph("uniform-random", {"n": 3000, "edges": 5000}, 1)
    monkeypatch.setenv("ABFS_DEVICE_BUILD_MIN_EDGES", str(1 << 40))
    h = P.generate_graph("uniform-random", {"n": 3000, "edges": 5000}, 1)
    assert isinstance(g, DeviceResidentGraph) and not isinstance(h, DeviceResidentGraph)
    for k in ("out_offsets", "destinations", "origins", "in_offsets", "sources"):
        np.testing.assert_array_equal(getattr(g, k), getattr(h, k), err_msg=k)


def test_permuted_kronecker_is_the_relabelled_graph():
    """bench.py --permute's graph: the same Kronecker edges with ids mapped by
    v -> (v * 0x9E3779B1 + 0x7F4A7C15) mod 2^scale; BFS depths commute with
    the relabelling (both level drivers, tree-switched)."""
    scale = 12
    base = DeviceGraph.rmat(scale, 16 << scale, 1, symmetrize=True)
    perm = DeviceGraph.rmat(scale, 16 << scale, 1, symmetrize=True, permute=True)
    ids = ((np.arange(1 << scale, dtype=np.uint64) * 0x9E3779B1 + 0x7F4A7C15) &
           np.uint64((1 << scale) - 1)).astype(np.int64)
    assert np.unique(ids).size == 1 << scale
    ob, _ = base.offsets()
    op, _ = perm.offsets()
    np.testing.assert_array_equal(np.diff(op.astype(np.int64))[ids], np.diff(ob.astype(np.int64)))
    gb, gp = base.to_graph(), perm.to_graph()
    flat = P.deserialize(G.tree_path("t1"))
    for r in (0, 5, 777):
        want = P.reference_bfs(gb, r)
        d, _ = P.adaptive_bfs(gp, int(ids[r]), flat, P.compute_stats(gp))
        np.testing.assert_array_equal(d[ids], want)
