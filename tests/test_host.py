"""Host-side logic of the package (no GPU): graph model/formats, features,
FlatTree + ADBT, error texts, and the C-ABI export surface."""

from __future__ import annotations

import ctypes
import hashlib
import os
import re

import numpy as np
import pytest

import golden_util as G
import paper_1708_01159_b200 as P
from paper_1708_01159_b200 import _lib
from paper_1708_01159_b200.features import canonical_indices, static_vector
from paper_1708_01159_b200.graph import mesh_pairs, symmetrised

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", G.graph_names())
def test_build_combined_matches_reference_arrays(name):
    n, m, a = G.graph_arrays(name)
    pairs = np.stack([a["origins"], a["destinations"]], axis=1)
    rng = np.random.default_rng(0)
    g = P.build_combined(pairs[rng.permutation(m)], n)   # order-independent
    for k in G.ARRAYS:
        np.testing.assert_array_equal(getattr(g, k), a[k], err_msg=k)
    np.testing.assert_array_equal(g.rev_owner(), a["rev_owner"])


def test_generate_graph_matches_reference():
    cases = {"star7": ("star", {"leaves": 7}, 1), "path9": ("path", {"n": 9}, 1),
             "bip3x4": ("complete-bipartite", {"a": 3, "b": 4}, 1),
             "u60": ("uniform-random", {"n": 60, "edges": 240}, 5),
             "u1000": ("uniform-random", {"n": 1000, "edges": 7000}, 11),
             "rmat5": ("rmat-like", {"scale": 5, "edges": 120}, 2),
             "rmat9": ("rmat-like", {"scale": 9, "edges": 6000}, 26),
             "er12": ("uniform-random", {"n": 4096, "edges": 131072}, 1)}
    for name, (model, params, seed) in cases.items():
        g = P.generate_graph(model, params, seed)
        _, _, a = G.graph_arrays(name)
        for k in G.ARRAYS:
            np.testing.assert_array_equal(getattr(g, k), a[k], err_msg=f"{name} {k}")
    g = symmetrised(P.generate_graph("rmat-like", {"scale": 10, "edges": 16 << 10}, 1))
    _, _, a = G.graph_arrays("kron10")
    for k in G.ARRAYS:
        np.testing.assert_array_equal(getattr(g, k), a[k])
    g = P.build_combined(mesh_pairs(64, 64), 4096)
    _, _, a = G.graph_arrays("mesh64")
    for k in G.ARRAYS:
        np.testing.assert_array_equal(getattr(g, k), a[k])


@pytest.mark.parametrize("label", ["rmat_s8", "uniform_n1024", "uniform_n2p16"])
def test_generator_pins(label):
    spec = G.meta()["generators"][label]
    g = P.generate_graph(spec["model"], spec["params"], spec["seed"])
    for k in G.ARRAYS:
        assert sha(getattr(g, k)) == spec["sha256"][k]


def test_compute_stats_matches_reference():
    for name in G.graph_names():
        n, m, a = G.graph_arrays(name)
        g = P.Graph(n, m, *[a[k].copy() for k in G.ARRAYS])
        np.testing.assert_array_equal(static_vector(P.compute_stats(g))[6:], G.stats(name))


def test_graph_errors():
    with pytest.raises(ValueError, match="out of range"):
        P.build_combined([(0, 3)], 3)
    with pytest.raises(ValueError, match=r"\(n, 2\)"):
        P.build_combined(np.zeros((2, 3)), 3)
    with pytest.raises(ValueError, match="unknown graph model"):
        P.generate_graph("nope", {}, 0)
    with pytest.raises(ValueError, match="missing generator parameter"):
        P.generate_graph("path", {}, 0)
    with pytest.raises(ValueError, match="rmat probabilities"):
        P.generate_graph("rmat-like", {"scale": 3, "edges": 4, "a": 0.9, "b": 0.2}, 0)
    with pytest.raises(ValueError, match="line 2"):
        P.load_edge_list("1 2\nx y\n")
    with pytest.raises(ValueError, match="no edges"):
        P.load_edge_list("% only a comment\n")
    with pytest.raises(ValueError):
        P.extra_memory_cost(P.generate_graph("path", {"n": 2}, 0), 3)
    assert P.extra_memory_cost(P.generate_graph("path", {"n": 3}, 0), 4) == 8


def test_load_edge_list_remap():
    g = P.load_edge_list("% c\n10 20 7\n20 30\n# x\n10 30\n")
    assert g.vertex_count == 3 and g.edge_count == 3
    np.testing.assert_array_equal(g.destinations, [1, 2, 2])


def test_adgr_round_trip_and_errors(tmp_path):
    n, m, a = G.graph_arrays("kron10")
    g = P.Graph(n, m, *[a[k].copy() for k in G.ARRAYS])
    p = str(tmp_path / "g.graph")
    P.write_graph(g, p)
    h = P.read_graph(p)
    for k in G.ARRAYS:
        np.testing.assert_array_equal(getattr(h, k), a[k])
    raw = open(p, "rb").read()
    for bad, msg in ((b"XXXX" + raw[4:], "bad magic"), (raw[:10], "truncated graph header"),
                     (raw[:-1], "truncated graph file"), (raw + b"\0", "trailing bytes"),
                     (raw[:4] + b"\x02" + raw[5:], "unsupported graph format version")):
        q = tmp_path / "bad.graph"
        q.write_bytes(bad)
        with pytest.raises(ValueError, match=msg):
            P.read_graph(str(q))


def test_features():
    st = P.compute_stats(P.generate_graph("star", {"leaves": 9}, 0))
    v = P.extract_runtime_features(st, 1, 3)
    assert v.vertex_count == 10 and v.frontier_pct == 0.1 and v.discovered_pct == 0.3
    assert len(P.FEATURE_NAMES) == 24
    with pytest.raises(ValueError):
        P.extract_runtime_features(st, 4, 3)
    with pytest.raises(ValueError):
        P.extract_runtime_features(st, -1, 3)
    with pytest.raises(ValueError, match="exceeds"):
        P.extract_runtime_features(st, 1, 11)
    with pytest.raises(ValueError, match="non-empty"):
        P.validate_selection([])
    with pytest.raises(ValueError, match="duplicate"):
        P.validate_selection(["vertex_count", "vertex_count"])
    with pytest.raises(ValueError, match="unknown"):
        P.validate_selection(["colour"])
    idx = canonical_indices(P.DEFAULT_MODEL_FEATURES)
    assert [P.FEATURE_NAMES[i] for i in idx] == list(P.DEFAULT_MODEL_FEATURES)


def _shortcut_trace(flat, stats, depths):
    finite = depths[depths != G.INF]
    hist = np.bincount(finite)
    out, prev, fr, disc, lvl = [], (0, 0), 1, 1, 0
    while True:
        cls = flat.predict_one(P.extract_runtime_features(stats, fr, disc))
        fb = cls == 254
        pair = prev if fb else (cls // 3, cls % 3)
        out.append([pair[0], pair[1], int(fb), fr])
        prev = pair
        new = int(hist[lvl + 1]) if lvl + 1 < hist.size else 0
        if new == 0:
            return out
        fr, disc, lvl = new, disc + new, lvl + 1


def test_flat_tree_predictions_match_reference_traces():
    """Host FlatTree + features reproduce the reference traces (pairs,
    fallbacks, frontier sizes) from the golden depth histograms."""
    tr = G.traces()
    for name in G.graph_names():
        n, m, a = G.graph_arrays(name)
        stats = P.compute_stats(P.Graph(n, m, *[a[k].copy() for k in G.ARRAYS]))
        for r in G.roots(name):
            for key, fname in G.trees_for(name):
                flat = P.deserialize(G.tree_path(fname))
                assert _shortcut_trace(flat, stats, G.depth(name, r)) == tr["small"][name][str(r)][key]


def test_adbt_round_trip_and_errors(tmp_path):
    for f in sorted(os.listdir(os.path.join(G.GOLDEN, "trees"))):
        p = os.path.join(G.GOLDEN, "trees", f)
        q = str(tmp_path / f)
        P.serialize(P.deserialize(p), q)
        assert open(p, "rb").read() == open(q, "rb").read()
    raw = open(G.tree_path("t1"), "rb").read()
    for bad, msg in ((b"XXXX" + raw[4:], "bad magic"), (raw[:6], "truncated model header"),
                     (raw[:-3], "truncated node records"), (raw + b"\0", "trailing bytes")):
        q = tmp_path / "bad.tree"
        q.write_bytes(bad)
        with pytest.raises(ValueError, match=msg):
            P.deserialize(str(q))
    flat = P.deserialize(G.tree_path("t1"))
    x = np.random.default_rng(1).uniform(0, 1e5, size=(500, len(flat.selection)))
    assert [flat.predict_one(v) for v in x] == flat.predict_batch(x).tolist()


def test_enumerations():
    assert len(P.ALL_PAIRS) == 15
    for i, (k, v) in enumerate(P.ALL_PAIRS):
        assert P.pair_index(k, v) == i and P.pair_from_index(i) == (k, v)
    assert P.INF_DEPTH == 2**31 - 1
    with pytest.raises(ValueError):
        P.set_worker_count(0)


def test_abi_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "abfs.h")).read()
    declared = sorted(set(re.findall(r"ABFS_API\s+[\w\s\*]*?\b(abfs_\w+)\s*\(", header)))
    assert len(declared) >= 20
    assert declared == _lib.exported_symbols()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert _lib.lib().abfs_version() == 1


def test_abi_host_helpers_without_gpu():
    """Pure-host ABI entry points (features, tree descent) work without a GPU."""
    L = _lib.lib()
    st = np.arange(24, dtype=np.float64)
    st[0] = 10.0
    out = np.zeros(24)
    _lib.check(L.abfs_features(_lib.ptr(st, _lib.f64p), 2, 5, _lib.ptr(out, _lib.f64p)))
    assert out[2] == 2 and out[3] == 0.2 and out[4] == 5 and out[5] == 0.5
    with pytest.raises(ValueError, match="discovered"):
        _lib.check(L.abfs_features(_lib.ptr(st, _lib.f64p), 6, 5, _lib.ptr(out, _lib.f64p)))
    flat = P.deserialize(G.tree_path("t1"))
    x = np.random.default_rng(2).uniform(0, 1e5, size=(200, len(flat.selection)))
    leaf = ctypes.c_int()
    for v in x:
        v = np.ascontiguousarray(v)
        _lib.check(L.abfs_tree_predict(ctypes.byref(flat.as_abfs()), _lib.ptr(v, _lib.f64p),
                                       ctypes.byref(leaf)))
        assert leaf.value == flat.predict_one(v)
