"""Engine-side reference artefacts: the C library reads and
writes ADBT models and trace CSVs byte-identically to the reference's Python
(tree.py:389-447, adaptive.py:225-254), and ADGR graph files straight into
HBM (graph.py:292-324, GPU tests at the bottom)."""

from __future__ import annotations

import ctypes
import glob
import os

import numpy as np
import pytest

import golden_util as G
import paper_1708_01159_b200 as P
from paper_1708_01159_b200 import _lib as L
from paper_1708_01159_b200.features import canonical_indices

TREES = sorted(glob.glob(os.path.join(G.GOLDEN, "trees", "*.tree")))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def c_read_tree(path):
    h = ctypes.c_void_p()
    L.check(L.lib().abfs_tree_read(path.encode(), ctypes.byref(h)), "tree_read")
    return h


@pytest.mark.parametrize("path", TREES + [os.path.join(ROOT, "models", "gpu_tree.tree")])
def test_tree_read_matches_python_and_write_is_byte_identical(path, tmp_path):
    flat = P.deserialize(path)
    h = c_read_tree(path)
    try:
        v = L.lib().abfs_tree_file_view(h).contents
        n = v.node_count
        assert n == flat.node_count and v.n_selection == len(flat.selection)
        assert [v.selection[i] for i in range(v.n_selection)] == list(canonical_indices(flat.selection))
        np.testing.assert_array_equal(np.ctypeslib.as_array(v.features, (n,)), flat.features)
        np.testing.assert_array_equal(np.ctypeslib.as_array(v.thresholds, (n,)).view(np.uint64),
                                      flat.thresholds.view(np.uint64))
        np.testing.assert_array_equal(np.ctypeslib.as_array(v.lefts, (n,)), flat.lefts)
        np.testing.assert_array_equal(np.ctypeslib.as_array(v.rights, (n,)), flat.rights)
        np.testing.assert_array_equal(np.ctypeslib.as_array(v.leaf_classes, (n,)), flat.leaf_classes)
        out = str(tmp_path / "c.tree")
        L.check(L.lib().abfs_tree_write(ctypes.byref(v), out.encode()), "tree_write")
        with open(out, "rb") as a, open(path, "rb") as b:
            assert a.read() == b.read()
    finally:
        L.lib().abfs_tree_file_free(h)


def _err(fn, *args):
    rc = fn(*args)
    assert rc == L.ABFS_EINVAL
    return L.lib().abfs_last_error().decode()


def test_tree_read_errors_match_reference_texts(tmp_path):
    good = open(TREES[0], "rb").read()
    cases = {
        "magic": (b"XDBT" + good[4:], "bad magic b'XDBT' in model file {p}"),
        "hdr": (good[:7], "truncated model header in {p}"),
        "ver": (good[:4] + (2).to_bytes(4, "little") + good[8:], "unsupported model format version 2"),
        "sel": (good[:12], "truncated selection header in {p}"),
        "body": (good[:-3], "truncated node records in {p}"),
        "trail": (good + b"\0", "trailing bytes in model file {p}"),
    }
    for name, (blob, msg) in cases.items():
        p = str(tmp_path / f"{name}.tree")
        open(p, "wb").write(blob)
        with pytest.raises(ValueError) as ref:
            P.deserialize(p)
        h = ctypes.c_void_p()
        got = _err(L.lib().abfs_tree_read, p.encode(), ctypes.byref(h))
        assert got == msg.format(p=p) == str(ref.value), name


def _trace():
    recs = []
    rng = np.random.default_rng(3)
    for lvl in range(9):
        k, v = P.ALL_PAIRS[int(rng.integers(15))]
        recs.append(P.LevelTrace(level=lvl, kernel=k, variant=v, fallback_used=bool(lvl % 3 == 1),
                                 frontier_size=int(rng.integers(1, 10**9)),
                                 elapsed_ns=int(rng.integers(1, 10**12)),
                                 prediction_ns=int(rng.integers(1, 10**6))))
    return P.AdaptiveTrace(tuple(recs))


def test_trace_csv_write_read_byte_identical(tmp_path):
    tr = _trace()
    py = str(tmp_path / "py.csv")
    P.write_trace(tr, py)
    arr = (L.AbfsLevelRecord * len(tr.records))()
    for i, r in enumerate(tr.records):
        arr[i].level, arr[i].kernel, arr[i].variant = r.level, int(r.kernel), int(r.variant)
        arr[i].fallback, arr[i].frontier_size = int(r.fallback_used), r.frontier_size
        arr[i].elapsed_ns, arr[i].prediction_ns = r.elapsed_ns, r.prediction_ns
    c = str(tmp_path / "c.csv")
    L.check(L.lib().abfs_trace_write(c.encode(), arr, len(arr)), "trace_write")
    assert open(c, "rb").read() == open(py, "rb").read()
    n = ctypes.c_size_t()
    back = (L.AbfsLevelRecord * 16)()
    L.check(L.lib().abfs_trace_read(py.encode(), back, 16, ctypes.byref(n)), "trace_read")
    assert n.value == len(tr.records)
    for b, r in zip(back, P.read_trace(py).records):
        assert (b.level, b.kernel, b.variant, bool(b.fallback), b.frontier_size, b.elapsed_ns,
                b.prediction_ns) == (r.level, int(r.kernel), int(r.variant), r.fallback_used,
                                     r.frontier_size, r.elapsed_ns, r.prediction_ns)
    bad = str(tmp_path / "bad.csv")
    open(bad, "w").write("level,kernel\n")
    assert _err(L.lib().abfs_trace_read, bad.encode(), None, 0, ctypes.byref(n)) == \
        f"unexpected trace header in {bad}"


# ---- ADGR: streamed into HBM --------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("name", ["kron12", "er12", "mesh64", "hand1", "selfloop", "single"])
def test_graph_read_write_on_device(name, tmp_path):
    n, m, a = G.graph_arrays(name)
    g = P.Graph(n, m, *[a[k].copy() for k in G.ARRAYS])
    py = str(tmp_path / "g.adgr")
    P.write_graph(g, py)
    h = ctypes.c_void_p()
    L.check(L.lib().abfs_graph_read(0, py.encode(), ctypes.byref(h)), "graph_read")
    dg = P.DeviceGraph(h)
    got = dg.download(rev_owner=True)
    for k in G.ARRAYS + ("rev_owner",):
        np.testing.assert_array_equal(got[k], a[k], err_msg=k)
    r = G.roots(name)[0]
    d, _ = P.bfs_full(dg, r, P.KernelId.VERTEX_PULL, P.CountVariant.GROUP_REDUCE)
    np.testing.assert_array_equal(d, G.depth(name, r))
    c = str(tmp_path / "c.adgr")
    L.check(L.lib().abfs_graph_write(dg._h, c.encode()), "graph_write")
    assert open(c, "rb").read() == open(py, "rb").read()
    dg.close()


@pytest.mark.gpu
def test_graph_read_errors_match_reference_texts(tmp_path):
    n, m, a = G.graph_arrays("kron10")
    py = str(tmp_path / "g.adgr")
    P.write_graph(P.Graph(n, m, *[a[k].copy() for k in G.ARRAYS]), py)
    good = open(py, "rb").read()
    cases = {"magic": b"AD\x00R" + good[4:], "hdr": good[:20],
             "ver": good[:4] + (7).to_bytes(4, "little") + good[8:],
             "trunc": good[:-4], "trail": good + b"x"}
    for name, blob in cases.items():
        p = str(tmp_path / f"{name}.adgr")
        open(p, "wb").write(blob)
        with pytest.raises(ValueError) as ref:
            P.read_graph(p)
        h = ctypes.c_void_p()
        assert _err(L.lib().abfs_graph_read, 0, p.encode(), ctypes.byref(h)) == str(ref.value), name


@pytest.mark.gpu
def test_python_free_pipeline_from_files(tmp_path):
    """Graph file -> device, model file -> tree, adaptive BFS, trace CSV:
    all through the C ABI; the CSV equals the reference writer's output for
    the same records and the trace equals the golden T1 trace."""
    name = "kron12"
    n, m, a = G.graph_arrays(name)
    g = P.Graph(n, m, *[a[k].copy() for k in G.ARRAYS])
    gp = str(tmp_path / "g.adgr")
    P.write_graph(g, gp)
    lib = L.lib()
    h, t, tf = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    L.check(lib.abfs_graph_read(0, gp.encode(), ctypes.byref(h)), "graph_read")
    L.check(lib.abfs_traversal_create(h, ctypes.byref(t)), "traversal_create")
    L.check(lib.abfs_tree_read(G.tree_path("t1").encode(), ctypes.byref(tf)), "tree_read")
    st = G.static24(G.stats(name), n, m)
    recs = (L.AbfsLevelRecord * 64)()
    nl = ctypes.c_size_t()
    d = np.empty(n, np.int32)
    r = G.roots(name)[0]
    L.check(lib.abfs_adaptive_bfs(t, r, lib.abfs_tree_file_view(tf), L.ptr(st, L.f64p), 32,
                                  L.ptr(d, L.i32p), recs, 64, ctypes.byref(nl)), "adaptive")
    np.testing.assert_array_equal(d, G.depth(name, r))
    rows = [[recs[i].kernel, recs[i].variant, recs[i].fallback, recs[i].frontier_size]
            for i in range(nl.value)]
    assert rows == G.traces()["small"][name][str(r)]["t1"]
    cp = str(tmp_path / "trace.csv")
    L.check(lib.abfs_trace_write(cp.encode(), recs, nl.value), "trace_write")
    tr = P.read_trace(cp)
    assert [[int(x.kernel), int(x.variant), int(x.fallback_used), x.frontier_size]
            for x in tr.records] == rows
    lib.abfs_tree_file_free(tf)
    lib.abfs_traversal_destroy(t)
    lib.abfs_graph_destroy(h)
