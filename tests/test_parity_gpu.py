"""GPU parity: the CUDA engine (through the reference-named API, i.e. the
C ABI) against the reference's golden vectors and the CPU oracle.

Bit-exact bar: depth arrays, per-level new counts, and the
adaptive trace (kernel, variant, fallback, frontier) given the same tree.
"""

from __future__ import annotations

import os

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import golden_util as G
import oracle
import paper_1708_01159_b200 as P
from paper_1708_01159_b200.graph import stats_from_offsets

pytestmark = pytest.mark.gpu

_GRAPHS = {}


def graph(name):
    if name not in _GRAPHS:
        n, m, a = G.graph_arrays(name)
        _GRAPHS[name] = P.Graph(n, m, *[a[k].copy() for k in G.ARRAYS])
    return _GRAPHS[name]


NAMES = G.graph_names()


@pytest.mark.parametrize("name", NAMES)
def test_all_15_pairs_match_reference(name):
    g = graph(name)
    for r in G.roots(name):
        want = G.depth(name, r)
        cnt = G.counts(name, r).tolist()
        for k, v in P.ALL_PAIRS:
            d, outs = P.bfs_full(g, r, k, v)
            np.testing.assert_array_equal(d, want, err_msg=f"{name} root={r} {k.name} {v.name}")
            assert [o.new_frontier_count for o in outs] == cnt, (name, r, k, v)
            assert all(o.elapsed_ns >= 1 for o in outs)


@pytest.mark.parametrize("name", ["u1000", "kron10", "mesh64"])
def test_push_warp_chunk_sizes(name):
    g = graph(name)
    r = G.roots(name)[1]
    for chunk in (1, 2, 3, 5, 8, 16, 32, 33, 1000):
        for v in P.CountVariant:
            d, outs = P.bfs_full(g, r, P.KernelId.VERTEX_PUSH_WARP, v, chunk_size=chunk)
            np.testing.assert_array_equal(d, G.depth(name, r))
            assert [o.new_frontier_count for o in outs] == G.counts(name, r).tolist()


@pytest.mark.parametrize("name", [n for n in NAMES if G.level_cases(n)])
def test_level_contract_and_inconsistent_inputs(name):
    """run_level on caller arrays (consistent partial rings and random
    inconsistent arrays) mutates in place exactly like the reference."""
    g = graph(name)
    for arr, level, per_kernel in G.level_cases(name):
        for k, (want, cnt) in enumerate(per_kernel):
            for v in range(3):
                d = arr.copy()
                out = P.run_level(g, d, level, k, v)
                np.testing.assert_array_equal(d, want, err_msg=f"{name} L{level} k{k} v{v}")
                assert out.new_frontier_count == cnt, (name, level, k, v)
            d64 = arr.astype(np.int64)
            P.run_level(g, d64, level, k, 0)
            np.testing.assert_array_equal(d64, want)


@pytest.mark.parametrize("name", NAMES)
def test_adaptive_traces_match_reference(name):
    g = graph(name)
    tr = G.traces()["small"][name]
    stats = P.compute_stats(g)
    for r in G.roots(name):
        for key, fname in G.trees_for(name):
            flat = P.deserialize(G.tree_path(fname))
            d, trace = P.adaptive_bfs(g, r, flat, stats)
            np.testing.assert_array_equal(d, G.depth(name, r))
            got = [[int(x.kernel), int(x.variant), int(x.fallback_used), x.frontier_size]
                   for x in trace.records]
            assert got == tr[str(r)][key], (name, r, key)
            assert all(x.elapsed_ns >= 1 and x.prediction_ns >= 1 for x in trace.records)
            # the Python-policy path over the same device traversal agrees
            d2, trace2 = P.adaptive_bfs(
                g, r, lambda lvl, fv, f=flat: P.tree._class_to_result(f.predict_one(fv)), stats)
            np.testing.assert_array_equal(d2, d)
            assert trace2.pairs == trace.pairs
            assert [x.fallback_used for x in trace2.records] == [x.fallback_used for x in trace.records]


def test_fallback_chain_and_policies():
    g = P.generate_graph("path", {"n": 6}, 0)
    a, b = P.ALL_PAIRS[7], P.ALL_PAIRS[11]
    _, tr = P.adaptive_bfs(g, 0, lambda lvl, f: {0: a, 2: b}.get(lvl, P.UNKNOWN))
    assert tr.pairs[:4] == [a, a, b, b]
    assert [r.fallback_used for r in tr.records][:4] == [False, True, False, True]
    g = P.generate_graph("uniform-random", {"n": 60, "edges": 300}, 3)
    d, tr = P.adaptive_bfs(g, 10, lambda lvl, f: P.pair_from_index((lvl * 7 + 3) % 15))
    np.testing.assert_array_equal(d, P.reference_bfs(g, 10))
    _, tr = P.adaptive_bfs(P.generate_graph("path", {"n": 8}, 0), 0, P.tree.leaf_tree(0))
    assert tr.level_count == 8 and [r.frontier_size for r in tr.records] == [1] * 8


def test_errors_match_reference():
    g = graph("hand1")
    with pytest.raises(ValueError, match="out of range"):
        P.bfs_full(g, 6, 0, 0)
    with pytest.raises(ValueError, match="out of range"):
        P.init_depths(g, -1)
    with pytest.raises(ValueError, match="chunk_size must be >= 1"):
        P.bfs_full(g, 0, P.KernelId.VERTEX_PUSH_WARP, 0, chunk_size=0)
    with pytest.raises(ValueError, match="unknown kernel"):
        P.run_level(g, P.init_depths(g, 0), 0, 7, 0)
    with pytest.raises(ValueError, match="unknown count variant"):
        P.run_level(g, P.init_depths(g, 0), 0, 0, 5)
    d = P.init_depths(g, 1)
    assert d[1] == 0 and (np.delete(d, 1) == P.INF_DEPTH).all()


def test_aggregate_count_device_variants():
    rng = np.random.default_rng(7)
    for size in [0, 1, 31, 32, 33, 1023, 1024, 1025, 100_000]:
        c = rng.integers(0, 5, size=size)
        for v in P.CountVariant:
            assert P.aggregate_count(c, v) == int(c.sum())
    big = rng.integers(0, 2**40, size=200)
    assert P.aggregate_count(big, 2) == int(big.sum())


@settings(max_examples=40)
@given(data=st.data())
def test_random_multigraphs_all_pairs(data):
    n = data.draw(st.integers(1, 14))
    pairs = data.draw(st.lists(st.tuples(st.integers(0, n - 1), st.integers(0, n - 1)),
                               max_size=50))
    g = P.build_combined(np.array(pairs, dtype=np.int64).reshape(-1, 2), n)
    root = data.draw(st.integers(0, n - 1))
    og = oracle.OracleGraph.from_graph(g)
    want = oracle.reference_bfs(og, root)
    hist = np.bincount(want[want != G.INF])
    for k, v in P.ALL_PAIRS:
        d, outs = P.bfs_full(g, root, k, v)
        np.testing.assert_array_equal(d, want)
        assert [o.new_frontier_count for o in outs[:-1]] == hist[1:].tolist()
        assert outs[-1].new_frontier_count == 0


@settings(max_examples=25)
@given(data=st.data())
def test_random_level_contract(data):
    n = data.draw(st.integers(2, 12))
    pairs = data.draw(st.lists(st.tuples(st.integers(0, n - 1), st.integers(0, n - 1)),
                               min_size=1, max_size=40))
    g = P.build_combined(np.array(pairs, dtype=np.int64), n)
    root = data.draw(st.integers(0, n - 1))
    og = oracle.OracleGraph.from_graph(g)
    ref = oracle.reference_bfs(og, root)
    level = data.draw(st.integers(0, int(ref[ref != G.INF].max())))
    part = np.where(ref <= level, ref, G.INF).astype(np.int32)
    for k in range(5):
        for v in range(3):
            d = part.copy()
            out = P.run_level(g, d, level, k, v)
            e = part.copy()
            c, _ = oracle.run_level(og, e, level, k, v)
            np.testing.assert_array_equal(d, e)
            assert out.new_frontier_count == c


def test_larger_random_graphs_vs_oracle():
    rng = np.random.default_rng(20260819)
    for n, m in ((800, 6000), (5000, 20000), (20000, 400000)):
        g = P.build_combined(rng.integers(0, n, size=(m, 2)), n)
        og = oracle.OracleGraph.from_graph(g)
        stats = P.compute_stats(g)
        flat = P.deserialize(G.tree_path("t1"))
        for root in (0, n - 1, n // 3):
            want = oracle.reference_bfs(og, root)
            for k, v in P.ALL_PAIRS:
                d, _ = P.bfs_full(g, root, k, v)
                np.testing.assert_array_equal(d, want)
            d, tr = P.adaptive_bfs(g, root, flat, stats)
            np.testing.assert_array_equal(d, want)
            _, orecs = oracle.adaptive_bfs(og, root, oracle.OracleTree(
                P.features.canonical_indices(flat.selection), flat.features, flat.thresholds,
                flat.lefts, flat.rights, flat.leaf_classes),
                np.array([n, m, 0, 0, 0, 0, *P.features.static_vector(stats)[6:]]))
            assert [(int(r.kernel), int(r.variant), r.fallback_used, r.frontier_size)
                    for r in tr.records] == [(k_, v_, fb, fr) for (_, k_, v_, fb, fr, *_x) in orecs]


def test_push_level_of_mid_degree_hubs():
    """A push level whose frontier is thousands of vertices of degree 65..255
    (each one CTA work unit: more units than m / kHeavy) -- the unit buffer
    is sized for m / kPushHub.  Both level drivers, all variants."""
    rng = np.random.default_rng(7)
    n = 4096
    half = np.stack([np.repeat(np.arange(n), 50), rng.integers(0, n, n * 50)], axis=1)
    g = P.build_combined(np.concatenate([half, half[:, ::-1]]), n)
    deg = np.diff(np.asarray(g.out_offsets, dtype=np.int64))
    assert deg.min() > 64 and deg.max() < 256
    og = oracle.OracleGraph.from_graph(g)
    for root in (0, 1234):
        want = oracle.reference_bfs(og, root)
        for k in (P.KernelId.VERTEX_PUSH, P.KernelId.VERTEX_PUSH_WARP):
            for v in P.CountVariant:
                d, outs = P.bfs_full(g, root, k, v)
                np.testing.assert_array_equal(d, want)
                t = P.Traversal(P.DeviceGraph.upload(g))
                t.set_device_loop(0)
                counts, _ = t.bfs_full(root, int(k), int(v))
                assert counts.tolist() == [o.new_frontier_count for o in outs]


@pytest.mark.parametrize("name", ["kron12", "er12", "mesh64", "u1000", "path9", "star7"])
def test_device_loop_and_launch_loop_agree(name):
    """The persistent megakernel (default) and the per-level launch chain give
    identical depths, counts and adaptive traces."""
    g = graph(name)
    t = g.device_graph().scratch()
    flat = P.deserialize(G.tree_path("t1"))
    stats = P.compute_stats(g)
    try:
        for r in G.roots(name):
            res = {}
            for loop in (True, False):
                t.set_device_loop(loop)
                pairs = []
                for k, v in P.ALL_PAIRS:
                    d, outs = P.bfs_full(g, r, k, v)
                    pairs.append((d.copy(), [o.new_frontier_count for o in outs]))
                d, tr = P.adaptive_bfs(g, r, flat, stats)
                res[loop] = (pairs, d.copy(), tr.pairs, [x.frontier_size for x in tr.records])
            for (d1, c1), (d2, c2) in zip(res[True][0], res[False][0]):
                np.testing.assert_array_equal(d1, d2)
                assert c1 == c2
            np.testing.assert_array_equal(res[True][1], res[False][1])
            assert res[True][2:] == res[False][2:]
    finally:
        t.set_device_loop(True)


@pytest.mark.parametrize("name", ["kron12", "u1000", "mesh64", "unreach", "star7"])
def test_adaptive_batch_matches_single_traversals(name):
    """abfs_adaptive_bfs_batch: several tree-switched BFSs in one launch
    (in-kernel init per root) give each root's level count, and the final
    depth array equals the last root's golden depths."""
    from paper_1708_01159_b200 import DeviceGraph, Traversal
    from paper_1708_01159_b200.features import static_vector
    g = graph(name)
    dg = DeviceGraph.upload(g)
    t = Traversal(dg)
    flat = P.deserialize(G.tree_path("t1"))
    stats = P.compute_stats(g)
    roots = G.roots(name)
    order = roots + roots[::-1]
    lv, ns, tot = t.adaptive_batch(order, flat.as_abfs(), static_vector(stats))
    want = [len(G.traces()["small"][name][str(r)]["t1"]) for r in order]
    assert lv.tolist() == want
    assert (ns > 0).all() and tot > 0
    np.testing.assert_array_equal(t.read(), G.depth(name, order[-1]))
    with pytest.raises(ValueError, match="out of range"):
        t.adaptive_batch([0, g.vertex_count], flat.as_abfs(), static_vector(stats))
    t.close()


@pytest.mark.parametrize("name", ["kron12", "mesh64", "unreach"])
def test_split_batch_equals_one_launch(name, monkeypatch):
    """A batch split over S concurrent partial-grid megakernels (roots dealt
    round-robin, ABFS_BATCH_SPLIT) returns the same per-root level counts,
    depth checksums and per-level new counts, in the caller's root order, as
    the single launch; the final depths are the last root's."""
    from paper_1708_01159_b200 import DeviceGraph, Traversal
    from paper_1708_01159_b200.features import static_vector
    g = graph(name)
    dg = DeviceGraph.upload(g)
    flat = P.deserialize(G.tree_path("t1"))
    st = static_vector(P.compute_stats(g))
    roots = G.roots(name)
    order = (roots * 4)[:7]
    base = None
    for ways in ("1", "2", "3", "4"):
        monkeypatch.setenv("ABFS_BATCH_SPLIT", ways)
        t = Traversal(dg)
        for batch in (order, order[:1], order[:2]):
            lv, sums, per = t.adaptive_batch_check(batch, flat.as_abfs(), st)
            got = (lv.tolist(), [int(x) for x in sums], per)
            if ways == "1":
                base = base or {}
                base[len(batch)] = got
            else:
                assert got == base[len(batch)], (ways, len(batch))
            np.testing.assert_array_equal(t.read(), G.depth(name, batch[-1]))
        lv, ns, tot = t.adaptive_batch(order, flat.as_abfs(), st)
        assert (ns > 0).all() and tot > 0 and lv.tolist() == base[len(order)][0]
        assert t.batch_ways(len(order)) == min(int(ways), len(order)) and t.batch_ways(1) == 1
        t.set_batch_ways(1)   # the explicit setting wins over ABFS_BATCH_SPLIT
        assert t.batch_ways(len(order)) == 1
        with pytest.raises(Exception):
            t.set_batch_ways(-1)
        t.close()
    dg.close()


def _random_tree(rng, selection, values, depth):
    """Preorder FlatTree of the given depth; thresholds drawn from the exact
    feature values a traversal produces and their float64 neighbours (the
    boundary cases of `x < thr`), leaves random pairs or UNKNOWN."""
    feats, thrs, lefts, rights, cls = [], [], [], [], []

    def node(d):
        i = len(cls)
        feats.append(0), thrs.append(0.0), lefts.append(0), rights.append(0), cls.append(255)
        if d == depth or rng.random() < 0.15:
            cls[i] = int(rng.choice([*range(15), 254]))
            return i
        f = int(rng.integers(len(selection)))
        base = float(rng.choice(values[selection[f]]))
        feats[i] = f
        thrs[i] = float(rng.choice([base, np.nextafter(base, np.inf), np.nextafter(base, -np.inf)]))
        lefts[i] = node(d + 1)
        rights[i] = node(d + 1)
        return i

    node(0)
    return P.FlatTree(tuple(selection), np.array(feats, np.uint16), np.array(thrs, np.float64),
                      np.array(lefts, np.uint32), np.array(rights, np.uint32),
                      np.array(cls, np.uint8))


@pytest.mark.parametrize("name", ["mesh64", "kron12", "u1000"])
def test_device_tree_cutoffs_match_float64_walk(name):
    """The megakernel walks an integer-cutoff form of the tree (static nodes
    resolved per graph, float64 tests on frontier/discovered turned into
    exact integer cutoffs); its traces must equal the launch path's float64
    walk for random trees whose thresholds sit exactly on, and one ulp around,
    the feature values the traversal produces."""
    g = graph(name)
    t = g.device_graph().scratch()
    stats = P.compute_stats(g)
    r = G.roots(name)[0]
    cnt = G.counts(name, r).tolist()
    fr = [1] + cnt[:-1]
    disc = list(np.cumsum([1] + cnt[:-1]))
    n = g.vertex_count
    from paper_1708_01159_b200.features import FEATURE_NAMES
    fv = P.extract_runtime_features(stats, 1, 1)
    values = {nm: [fv.scalar(nm)] for nm in FEATURE_NAMES}
    values["frontier_abs"] = [float(x) for x in fr]
    values["frontier_pct"] = [x / n for x in fr]
    values["discovered_abs"] = [float(x) for x in disc]
    values["discovered_pct"] = [x / n for x in disc]
    rng = np.random.default_rng(7)
    sel = ["vertex_count", "frontier_abs", "frontier_pct", "discovered_abs", "discovered_pct",
           "out_deg.median", "edge_count"]
    try:
        for _ in range(12):
            flat = _random_tree(rng, sel, values, depth=5)
            res = {}
            for loop in (True, False):
                t.set_device_loop(loop)
                d, tr = P.adaptive_bfs(g, r, flat, stats)
                res[loop] = ([(int(x.kernel), int(x.variant), x.fallback_used, x.frontier_size)
                              for x in tr.records], d.copy())
            assert res[True][0] == res[False][0]
            np.testing.assert_array_equal(res[True][1], res[False][1])
    finally:
        t.set_device_loop(True)


@pytest.mark.parametrize("deg", [1025, 1040, 1057, 2049, 2081, 3000, 5000])
def test_pull_cta_units_cover_the_in_list_tail(deg):
    """A pull remainder above kPullHeavy goes to 1024-edge CTA units; the
    units must cover exactly the unscanned tail.  Vertex `deg` has in-edges
    from 0..deg-1 and only the LAST one is in the frontier (in-
    degrees 1024k+1..1024k+33 lost their last in-neighbours)."""
    src = np.arange(deg, dtype=np.int64)
    g = P.build_combined(np.stack([src, np.full(deg, deg)], axis=1), deg + 1)
    root = deg - 1
    dg = P.DeviceGraph.upload(g)
    t = P.Traversal(dg)
    try:
        for loop in (True, False):
            t.set_device_loop(loop)
            for v in P.CountVariant:
                d = np.empty(g.vertex_count, np.int32)
                counts, _ = t.bfs_full(root, int(P.KernelId.VERTEX_PULL), int(v), 32, depths_out=d)
                assert counts.tolist() == [1, 0], (deg, loop, v)
                assert d[deg] == 1 and d[root] == 0
        depths = np.full(g.vertex_count, G.INF, np.int32)
        depths[root] = 0
        out = P.run_level(g, depths, 0, P.KernelId.VERTEX_PULL, P.CountVariant.DIRECT_ATOMIC)
        assert out.new_frontier_count == 1 and depths[deg] == 1
    finally:
        t.close()
        dg.close()


def test_more_levels_than_megakernel_records():
    """A traversal with more than 65536 level calls (the megakernel's record
    capacity) still reports every level: path of 70000."""
    n = 70000
    g = P.generate_graph("path", {"n": n}, 0)
    d, outs = P.bfs_full(g, 0, P.KernelId.VERTEX_PUSH, P.CountVariant.GROUP_REDUCE)
    assert len(outs) == n
    assert [o.new_frontier_count for o in outs] == [1] * (n - 1) + [0]
    np.testing.assert_array_equal(d, np.arange(n, dtype=np.int32))
    d, tr = P.adaptive_bfs(g, 0, P.tree.leaf_tree(6))
    assert tr.level_count == n and d[-1] == n - 1
    assert [r.frontier_size for r in tr.records[-3:]] == [1, 1, 1]


def test_concurrent_traversals_on_one_graph():
    """SPEC.md:243 / SURVEY §8b: distinct traversals may run concurrently on
    the same immutable Graph.  4 threads x (adaptive_bfs, bfs_full, run_level)
    on different roots of one Graph; ctypes releases the GIL, so the calls
    really overlap.  Every result equals the golden vectors."""
    import threading
    name = "kron12"
    g = graph(name)
    stats = P.compute_stats(g)
    flat = P.deserialize(G.tree_path("t1"))
    roots = G.roots(name)
    tr = G.traces()["small"][name]
    errors = []

    def worker(i):
        try:
            for it in range(6):
                r = roots[(i + it) % len(roots)]
                d, trace = P.adaptive_bfs(g, r, flat, stats)
                np.testing.assert_array_equal(d, G.depth(name, r))
                got = [[int(x.kernel), int(x.variant), int(x.fallback_used), x.frontier_size]
                       for x in trace.records]
                assert got == tr[str(r)]["t1"]
                k, v = P.ALL_PAIRS[(3 * i + it) % 15]
                d, outs = P.bfs_full(g, r, k, v)
                np.testing.assert_array_equal(d, G.depth(name, r))
                assert [o.new_frontier_count for o in outs] == G.counts(name, r).tolist()
                d = P.init_depths(g, r)
                for level in range(len(outs)):
                    P.run_level(g, d, level, k, v)
                np.testing.assert_array_equal(d, G.depth(name, r))
        except BaseException as e:   # noqa: BLE001
            errors.append((i, repr(e)))

    th = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors
    assert len(g.device_graph()._idle) >= 1   # the pool really handed out extra traversals


def test_foreign_graph_upload_cache_is_identity_checked():
    """kernels._device caches uploads of foreign (reference-shaped) graphs by
    id with a weak reference; a recycled id never returns another graph."""
    import gc
    from types import SimpleNamespace

    from paper_1708_01159_b200 import kernels as K

    class RefGraph(SimpleNamespace):
        pass

    def mk(name):
        n, m, a = G.graph_arrays(name)
        return RefGraph(vertex_count=n, edge_count=m, **{k: a[k] for k in G.ARRAYS})

    for name in ("kron10", "mesh64", "u60", "star7"):
        fg = mk(name)
        r = G.roots(name)[0]
        d, _ = P.bfs_full(fg, r, P.KernelId.VERTEX_PULL, P.CountVariant.GROUP_REDUCE)
        np.testing.assert_array_equal(d, G.depth(name, r))
        key = id(fg)
        assert key in K._foreign_uploads
        del fg, d
        gc.collect()
        assert key not in K._foreign_uploads


@pytest.fixture(params=[("1", "1"), ("1000000000000", "1")], ids=["red-every-level", "red-units-only"])
def red_mode(request, monkeypatch):
    """Force the megakernel's RED-mode top-down claims (fire-and-forget OR
    reductions + one bitmap settle pass) onto small graphs: on every top-down
    level, or only on CTA-unit passes (read per call by the engine)."""
    f, u = request.param
    monkeypatch.setenv("ABFS_RED_F", f)
    monkeypatch.setenv("ABFS_RED_UNITS", u)
    yield request.param


@pytest.mark.parametrize("name", NAMES)
def test_red_mode_all_pairs_and_traces_match_reference(name, red_mode):
    g = graph(name)
    t = g.device_graph().scratch()
    assert t.mode  # device loop (RED mode lives in the megakernel)
    stats = P.compute_stats(g)
    traces = G.traces()["small"]
    for r in G.roots(name):
        want = G.depth(name, r)
        cnt = G.counts(name, r).tolist()
        for k, v in P.ALL_PAIRS:
            d, outs = P.bfs_full(g, r, k, v)
            np.testing.assert_array_equal(d, want, err_msg=f"{name} root={r} {k.name} {v.name}")
            assert [o.new_frontier_count for o in outs] == cnt, (name, r, k, v)
        for key, tree in G.trees_for(name):
            d, tr = P.adaptive_bfs(g, r, P.deserialize(G.tree_path(tree)), stats)
            got = [[int(x.kernel), int(x.variant), int(x.fallback_used), x.frontier_size]
                   for x in tr.records]
            assert got == traces[name][str(r)][key], (name, r, key)
            np.testing.assert_array_equal(d, want)


@pytest.fixture(params=[("1", "8", "1"), ("1", "16", "1"), ("1", "16", "0"), ("1", "4", "1")],
                ids=["solo8", "solo16", "solo16-filtered", "solo4"])
def solo_forced(request, monkeypatch):
    """Force the megakernel's cluster solo mode (small top-down levels on one
    cluster with DSMEM tails) on every graph, hubs included: solo levels that
    meet a hub hand the level back to the grid mid-flight."""
    on, cl, direct = request.param
    monkeypatch.setenv("ABFS_SOLO", on)
    monkeypatch.setenv("ABFS_SOLO_CLUSTER", cl)
    monkeypatch.setenv("ABFS_SOLO_DIRECT", direct)
    yield request.param


@pytest.mark.parametrize("name", ["kron10", "kron12", "star7", "u1000", "mesh64", "unreach", "hand1"])
def test_forced_solo_mode_all_pairs_and_traces_match_reference(name, solo_forced):
    g = graph(name)
    t = g.device_graph().scratch()
    assert t.mode
    stats = P.compute_stats(g)
    traces = G.traces()["small"]
    for r in G.roots(name):
        want = G.depth(name, r)
        cnt = G.counts(name, r).tolist()
        for k, v in P.ALL_PAIRS:
            if k in (P.KernelId.VERTEX_PUSH, P.KernelId.VERTEX_PUSH_WARP):   # solo-eligible
                d, outs = P.bfs_full(g, r, k, v)
                np.testing.assert_array_equal(d, want, err_msg=f"{name} root={r} {k.name} {v.name}")
                assert [o.new_frontier_count for o in outs] == cnt, (name, r, k, v)
        for key, tree in G.trees_for(name):
            d, tr = P.adaptive_bfs(g, r, P.deserialize(G.tree_path(tree)), stats)
            got = [[int(x.kernel), int(x.variant), int(x.fallback_used), x.frontier_size]
                   for x in tr.records]
            assert got == traces[name][str(r)][key], (name, r, key)
            np.testing.assert_array_equal(d, want)


def test_red_mode_batch_checksums_k18(red_mode):
    """RED mode through the batched launch the bench times: per-root depth
    checksums and per-level counts equal the oracle's on Kronecker-18."""
    from paper_1708_01159_b200 import DeviceGraph, Traversal
    from paper_1708_01159_b200.engine import depth_checksum
    from paper_1708_01159_b200.features import static_vector
    dg = DeviceGraph.rmat(18, 16 << 18, 1, symmetrize=True)
    g = dg.to_graph()
    og = oracle.OracleGraph.from_graph(g)
    flat = P.deserialize(G.tree_path("t1"))
    t = Traversal(dg)
    deg = np.diff(g.out_offsets.astype(np.int64))
    roots = [int(x) for x in np.flatnonzero(deg > 0)[[0, 7, 1000, 5000]]]
    lv, sums, per = t.adaptive_batch_check(roots, flat.as_abfs(),
                                           static_vector(P.compute_stats(g)))
    for i, r in enumerate(roots):
        want = oracle.reference_bfs(og, r)
        assert int(sums[i]) == depth_checksum(want), r
        n = int(lv[i])
        hist = np.bincount(want[want != G.INF], minlength=n)
        assert per[i] == hist[1:n].tolist() + [0], r
    t.close()


@pytest.mark.skipif(os.environ.get("ABFS_TEST_PULL2_BUILD") != "1",
                    reason="list-based pull is an opt-in build (-DABFS_PULL2_CODE=1 via "
                           "tools/build_variant.sh; run with ABFS_LIB=<that build> and "
                           "ABFS_TEST_PULL2_BUILD=1)")
@pytest.mark.parametrize("name", NAMES)
def test_list_pull_all_pairs_and_traces_match_reference(name, monkeypatch):
    """The megakernel's list-based pull (pull2.cuh, ABFS_PULL2=1: grid-wide
    probe-0 sweep or carried candidate list, then the survivors' scans)
    reproduces every golden depth array, count and trace."""
    monkeypatch.setenv("ABFS_PULL2", "1")
    g = graph(name)
    stats = P.compute_stats(g)
    traces = G.traces()["small"]
    for r in G.roots(name):
        want = G.depth(name, r)
        for v in P.CountVariant:
            d, outs = P.bfs_full(g, r, P.KernelId.VERTEX_PULL, v)
            np.testing.assert_array_equal(d, want, err_msg=f"{name} root={r} {v.name}")
            assert [o.new_frontier_count for o in outs] == G.counts(name, r).tolist()
        for key, tree in G.trees_for(name):
            d, tr = P.adaptive_bfs(g, r, P.deserialize(G.tree_path(tree)), stats)
            got = [[int(x.kernel), int(x.variant), int(x.fallback_used), x.frontier_size]
                   for x in tr.records]
            assert got == traces[name][str(r)][key], (name, r, key)
            np.testing.assert_array_equal(d, want)
