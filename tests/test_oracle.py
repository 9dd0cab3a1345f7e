"""Pin the CPU oracle (oracle/abfs_oracle.c) to the reference's own outputs.

Golden vectors come from the unmodified reference (tools/make_golden.py);
the oracle must reproduce them exactly before it is trusted as the checker
for the CUDA engine (tests/test_parity_gpu.py) and as the timed CPU port.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import oracle
import golden_util as G
from paper_1708_01159_b200.features import canonical_indices
from paper_1708_01159_b200.tree import deserialize


def ograph(name):
    n, m, a = G.graph_arrays(name)
    return oracle.OracleGraph(n, m, a["out_offsets"], a["destinations"], a["origins"],
                              a["in_offsets"], a["sources"], a["rev_owner"])


def otree(path):
    t = deserialize(path)
    return oracle.OracleTree(canonical_indices(t.selection), t.features, t.thresholds,
                             t.lefts, t.rights, t.leaf_classes)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


NAMES = G.graph_names()


@pytest.mark.parametrize("name", NAMES)
def test_reference_bfs_matches_golden(name):
    g = ograph(name)
    for r in G.roots(name):
        np.testing.assert_array_equal(oracle.reference_bfs(g, r), G.depth(name, r))


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("threads", [1, 3])
def test_all_pairs_depths_and_counts(name, threads):
    g = ograph(name)
    for r in G.roots(name)[:3]:
        for k in range(5):
            for v in range(3):
                d, c, el = oracle.bfs_full(g, r, k, v, chunk_size=3 if k == 4 else 32,
                                           threads=threads)
                np.testing.assert_array_equal(d, G.depth(name, r), err_msg=f"{name} {r} {k} {v}")
                np.testing.assert_array_equal(c, G.counts(name, r))
                assert (el >= 1).all()


@pytest.mark.parametrize("name", [n for n in NAMES if G.level_cases(n)])
def test_level_contract_and_inconsistent_inputs(name):
    g = ograph(name)
    for arr, level, per_kernel in G.level_cases(name):
        for k, (want, cnt) in enumerate(per_kernel):
            for v in range(3):
                d = arr.copy()
                c, _ = oracle.run_level(g, d, level, k, v, threads=2)
                np.testing.assert_array_equal(d, want, err_msg=f"{name} L{level} k{k}")
                assert c == cnt


@pytest.mark.parametrize("name", NAMES)
def test_adaptive_traces(name):
    g = ograph(name)
    n, m, _ = G.graph_arrays(name)
    st = G.static24(G.stats(name), n, m)
    tr = G.traces()["small"][name]
    for r in G.roots(name):
        for key, fname in G.trees_for(name):
            d, recs = oracle.adaptive_bfs(g, r, otree(G.tree_path(fname)), st)
            np.testing.assert_array_equal(d, G.depth(name, r))
            got = [[k, v, int(fb), fr] for (_, k, v, fb, fr, *_rest) in recs]
            assert got == tr[str(r)][key], (name, r, key)


def test_aggregate_count_variants():
    rng = np.random.default_rng(7)
    for size in [0, 1, 31, 32, 33, 1023, 1024, 1025, 5000]:
        c = rng.integers(0, 5, size=size)
        for v in range(3):
            assert oracle.aggregate_count(c, v) == int(c.sum())
    with pytest.raises(ValueError):
        oracle.aggregate_count([1], 3)


def test_bad_arguments():
    g = ograph("hand1")
    with pytest.raises(ValueError):
        oracle.reference_bfs(g, 6)
    d = np.full(6, G.INF, np.int32)
    with pytest.raises(ValueError):
        oracle.run_level(g, d, 0, 5, 0)
    with pytest.raises(ValueError):
        oracle.run_level(g, d, 0, 4, 0, chunk_size=0)


@pytest.fixture(scope="module")
def k16():
    meta = G.traces()["k16"]
    src, dst = oracle.generate_rmat_pairs(16, 16 << 16, 1)
    g = oracle.build_combined(1 << 16, np.concatenate([src, dst]), np.concatenate([dst, src]))
    return g, meta


def test_k16_generator_and_build_bit_exact(k16):
    g, meta = k16
    assert (g.n, g.m) == (meta["V"], meta["E"])
    for a in G.ARRAYS:
        assert sha(getattr(g, a)) == meta["sha256"][a], a


def test_k16_64_roots_depths_and_t1_traces(k16):
    g, meta = k16
    st = G.static24(meta["stats"], meta["V"], meta["E"])
    t1 = otree(G.tree_path("t1"))
    t4 = otree(G.tree_path("t4_k16"))
    for r in meta["roots"]:
        run = meta["runs"][str(r)]
        d = oracle.reference_bfs(g, r)
        assert sha(d) == run["depth_sha256"]
        d2, recs = oracle.adaptive_bfs(g, r, t1, st, threads=4)
        assert sha(d2) == run["depth_sha256"]
        assert [[k, v, int(fb), fr] for (_, k, v, fb, fr, *_x) in recs] == run["t1"]
        _, recs = oracle.adaptive_bfs(g, r, t4, st, threads=4)
        assert [[k, v, int(fb), fr] for (_, k, v, fb, fr, *_x) in recs] == run["t4"]


@pytest.mark.parametrize("label", ["rmat_s8", "rmat_s12_sym", "uniform_n1024", "uniform_n2p16"])
def test_generator_pins(label):
    spec = G.meta()["generators"][label]
    p = spec["params"]
    if spec["model"] == "rmat-like":
        src, dst = oracle.generate_rmat_pairs(p["scale"], p["edges"], spec["seed"])
        n = 1 << p["scale"]
    else:
        src, dst = oracle.generate_uniform_pairs(p["n"], p["edges"], spec["seed"])
        n = p["n"]
    if spec["sym"]:
        src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
    g = oracle.build_combined(n, src, dst)
    for a in G.ARRAYS:
        assert sha(getattr(g, a)) == spec["sha256"][a], a
