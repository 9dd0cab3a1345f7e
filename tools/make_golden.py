"""Freeze golden vectors from the UNMODIFIED reference.

Run in the build container (the reference exists only here):

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden.py

It imports `adaptive_bfs` from /root/reference/pkg/src and the acceptance
fixture helpers from /root/reference/pkg/tests, and writes:

  tests/golden/graphs.npz      small graphs (combined arrays), roots,
                               reference_bfs depths, per-level counts,
                               compute_stats, level-contract cases
  tests/golden/traces.json     adaptive_bfs traces (pairs, fallback flags,
                               frontier sizes) under the parity tree set
                               T1..T4, plus the config-1 (K16) 64-root set
  tests/golden/trees/*.tree    the parity trees in the reference ADBT format
  tests/golden/meta.json       numpy / python versions and recipes

Nothing at test time reads /root/reference: the GPU box only sees these files.
"""

from __future__ import annotations

import hashlib
import json
import os
import platform
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.dont_write_bytecode = True
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

import adaptive_bfs as ab  # noqa: E402
from adaptive_bfs import kernels as K  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden")
INF = int(K.INF_DEPTH)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def symmetrised_rmat(scale, factor, seed):
    """Config 1-3 recipe: rmat-like + concat reversed pairs."""
    g = ab.generate_graph("rmat-like", {"scale": scale, "edges": factor << scale}, seed)
    p = g.edge_pairs().astype(np.int64)
    return ab.build_combined(np.concatenate([p, p[:, ::-1]]), g.vertex_count)


def mesh(rows, cols):
    """4-neighbour grid, both directions, through build_combined."""
    idx = np.arange(rows * cols, dtype=np.int64).reshape(rows, cols)
    right = np.stack([idx[:, :-1].ravel(), idx[:, 1:].ravel()], axis=1)
    down = np.stack([idx[:-1, :].ravel(), idx[1:, :].ravel()], axis=1)
    p = np.concatenate([right, down])
    return ab.build_combined(np.concatenate([p, p[:, ::-1]]), rows * cols)


def make_graph(pairs, n):
    return ab.build_combined(np.array(pairs, dtype=np.int64).reshape(-1, 2), n)


def small_graphs():
    return {
        "hand1": make_graph([(0, 1), (1, 2), (0, 3), (3, 4), (4, 1)], 6),
        "dup": make_graph([(0, 1)] * 5 + [(1, 2)] * 3, 3),
        "selfloop": make_graph([(0, 0), (0, 1), (1, 1), (1, 2)], 3),
        "unreach": make_graph([(0, 1), (2, 3)], 4),
        "single": make_graph([], 1),
        "star7": ab.generate_graph("star", {"leaves": 7}, 1),
        "path9": ab.generate_graph("path", {"n": 9}, 1),
        "bip3x4": ab.generate_graph("complete-bipartite", {"a": 3, "b": 4}, 1),
        "u60": ab.generate_graph("uniform-random", {"n": 60, "edges": 240}, 5),
        "u1000": ab.generate_graph("uniform-random", {"n": 1000, "edges": 7000}, 11),
        "rmat5": ab.generate_graph("rmat-like", {"scale": 5, "edges": 120}, 2),
        "rmat9": ab.generate_graph("rmat-like", {"scale": 9, "edges": 6000}, 26),
        "kron10": symmetrised_rmat(10, 16, 1),
        "kron12": symmetrised_rmat(12, 16, 1),
        "er12": ab.generate_graph("uniform-random", {"n": 4096, "edges": 131072}, 1),
        "mesh7x13": mesh(7, 13),
        "mesh64": mesh(64, 64),
    }


def pick_roots(g, k, seed):
    deg = g.out_degrees()
    cand = np.flatnonzero(deg > 0)
    if cand.size == 0:
        return [0]
    rng = np.random.default_rng(seed)
    k = min(k, cand.size)
    return sorted(int(v) for v in rng.choice(cand, size=k, replace=False))


def stats_vec(st):
    out = []
    for s in (st.out_degree_summary, st.in_degree_summary, st.abs_degree_summary):
        out += [s.min, s.q1, s.median, s.q3, s.max, s.stddev]
    return out


# --- parity tree set (SURVEY §8c ii) ---------------------------------------

def tree_t1():
    """Acceptance fixture tests/test_acceptance.py:174-257 (synthetic labels)."""
    import test_acceptance as ta
    samples = []
    for index, graph in enumerate(ta._training_corpus()):
        stats = ab.compute_stats(graph)
        for root in ab.select_roots(graph, 3, seed=500 + index):
            depths, _ = ab.bfs_full(graph, root, ab.KernelId.EDGE_LIST,
                                    ab.CountVariant.DIRECT_ATOMIC)
            finite = depths[depths != INF]
            hist = np.bincount(finite)
            cum = np.cumsum(hist)
            for level in range(len(hist)):
                v = ab.extract_runtime_features(stats, int(hist[level]), int(cum[level]))
                samples.append((v, ta._synthetic_best_pair(v)))
    train, _ = ab.split_train_test(samples, 0.7, seed=0)
    x = np.stack([v.as_array(ab.DEFAULT_MODEL_FEATURES) for v, _ in train])
    y = np.array([lab for _, lab in train], dtype=np.int64)
    tree = ab.fit(x, y, ab.DEFAULT_MODEL_FEATURES, ta._TRAIN_CONFIG)
    return ab.flatten(tree)


def tree_unknown():
    """tests/test_adaptive.py:49-53."""
    cfg = ab.TrainConfig(max_depth=1, min_samples_leaf=1, min_samples_split=2)
    return ab.flatten(ab.fit(np.array([[0.0], [0.0]]), np.array([0, 9]),
                             ["frontier_abs"], cfg))


def tree_leaf(k):
    """tests/test_adaptive.py:43-46."""
    return ab.flatten(ab.fit(np.array([[0.0]]), np.array([k]), ["frontier_abs"]))


def tree_t4(g, stats, seed):
    """Leaf-limited random tree over DEFAULT_MODEL_FEATURES."""
    rng = np.random.default_rng(seed)
    names = ab.DEFAULT_MODEL_FEATURES
    base = ab.extract_runtime_features(stats, 1, 1)
    rows = []
    n = g.vertex_count
    for _ in range(40):
        fr = int(round(np.exp(rng.uniform(0, np.log(max(n, 2))))))
        dpct = rng.uniform(0, 1)
        row = []
        for name in names:
            if name == "discovered_pct":
                row.append(dpct)
            elif name == "frontier_abs":
                row.append(float(fr))
            else:
                row.append(base.scalar(name))
        rows.append(row)
    y = rng.integers(0, 15, size=40)
    cfg = ab.TrainConfig(max_depth=3, min_samples_leaf=4, min_samples_split=8)
    return ab.flatten(ab.fit(np.array(rows), y, names, cfg))


def trace_of(tr):
    return [[int(r.kernel), int(r.variant), int(r.fallback_used), int(r.frontier_size)]
            for r in tr.records]


def shortcut_trace(flat, stats, depths):
    """Trace implied by the depth histogram (adaptive.py:101-129 semantics)."""
    finite = depths[depths != INF]
    hist = np.bincount(finite) if finite.size else np.zeros(1, np.int64)
    out = []
    prev = (0, 0)
    frontier, discovered = 1, 1
    level = 0
    while True:
        fv = ab.extract_runtime_features(stats, frontier, discovered)
        cls = flat.predict_one(fv)
        fb = cls == 254
        pair = prev if fb else (cls // 3, cls % 3)
        out.append([pair[0], pair[1], int(fb), frontier])
        prev = pair
        new = int(hist[level + 1]) if level + 1 < hist.size else 0
        if new == 0:
            return out
        frontier = new
        discovered += new
        level += 1


def level_cases(g, root, rng, n_random=4):
    """Level-contract inputs/outputs (tests/test_kernels.py:209-236) plus
    inconsistent arrays run through the reference."""
    ref = ab.reference_bfs(g, root)
    finite = ref[ref != INF]
    maxl = int(finite.max())
    cases = []
    for level in range(0, maxl + 1):
        partial = np.where(ref <= level, ref, INF).astype(np.int32)
        cases.append((partial, level))
    for _ in range(n_random):
        level = int(rng.integers(0, maxl + 2))
        arr = rng.integers(0, maxl + 4, size=g.vertex_count).astype(np.int32)
        arr[rng.random(g.vertex_count) < 0.5] = INF
        cases.append((arr, level))
    out = []
    for arr, level in cases:
        per_kernel = []
        for k in ab.KernelId:
            got = None
            for v in ab.CountVariant:
                d = arr.copy()
                o = ab.run_level(g, d, level, k, v, 32)
                if got is None:
                    got = (d, o.new_frontier_count)
                else:
                    assert np.array_equal(got[0], d) and got[1] == o.new_frontier_count
            per_kernel.append(got)
        out.append((arr, level, per_kernel))
    return out


def main():
    os.makedirs(os.path.join(OUT, "trees"), exist_ok=True)
    ab.set_worker_count(4)
    arrays = {}
    traces = {"small": {}, "k16": {}}
    t1 = tree_t1()
    t2 = tree_unknown()
    ab.serialize(t1, os.path.join(OUT, "trees", "t1.tree"))
    ab.serialize(t2, os.path.join(OUT, "trees", "t2_unknown.tree"))
    for k in range(15):
        ab.serialize(tree_leaf(k), os.path.join(OUT, "trees", f"t3_leaf{k:02d}.tree"))
    rng = np.random.default_rng(20260819)
    graphs = small_graphs()
    for name, g in graphs.items():
        p = f"g/{name}/"
        arrays[p + "n"] = np.array([g.vertex_count, g.edge_count], dtype=np.int64)
        for a in ("out_offsets", "destinations", "origins", "in_offsets", "sources"):
            arrays[p + a] = getattr(g, a)
        arrays[p + "rev_owner"] = g.rev_owner()
        stats = ab.compute_stats(g)
        arrays[p + "stats"] = np.array(stats_vec(stats), dtype=np.float64)
        roots = sorted({0, g.vertex_count - 1, *pick_roots(g, 4, 7)})
        arrays[p + "roots"] = np.array(roots, dtype=np.int64)
        t4 = tree_t4(g, stats, 0)
        ab.serialize(t4, os.path.join(OUT, "trees", f"t4_{name}.tree"))
        traces["small"][name] = {}
        for root in roots:
            ref = ab.reference_bfs(g, root)
            arrays[p + f"depth/{root}"] = ref
            counts = None
            for kk, vv in ab.ALL_PAIRS:
                d, outs = ab.bfs_full(g, root, kk, vv)
                assert np.array_equal(d, ref)
                c = [o.new_frontier_count for o in outs]
                counts = c if counts is None else counts
                assert c == counts
            arrays[p + f"counts/{root}"] = np.array(counts, dtype=np.int64)
            tr = {}
            for tname, flat in (("t1", t1), ("t2_unknown", t2), ("t4", t4),
                                ("t3_leaf03", tree_leaf(3)), ("t3_leaf09", tree_leaf(9)),
                                ("t3_leaf14", tree_leaf(14))):
                d, trace = ab.adaptive_bfs(g, root, flat, stats)
                assert np.array_equal(d, ref)
                tr[tname] = trace_of(trace)
                assert tr[tname] == shortcut_trace(flat, stats, ref), (name, root, tname)
            traces["small"][name][str(root)] = tr
        if g.edge_count > 0:
            cases = level_cases(g, roots[len(roots) // 2], rng,
                                n_random=4 if g.vertex_count < 5000 else 2)
            for i, (arr, level, per_kernel) in enumerate(cases):
                arrays[p + f"lc/{i}/in"] = arr
                arrays[p + f"lc/{i}/level"] = np.array([level], dtype=np.int64)
                for k, (d, cnt) in enumerate(per_kernel):
                    arrays[p + f"lc/{i}/out{k}"] = d
                    arrays[p + f"lc/{i}/cnt{k}"] = np.array([cnt], dtype=np.int64)
        print(f"{name}: V={g.vertex_count} E={g.edge_count} roots={roots}", flush=True)

    # --- config 1 at full size: Kronecker scale 16, 64 roots ----------------
    g = symmetrised_rmat(16, 16, 1)
    stats = ab.compute_stats(g)
    roots = pick_roots(g, 64, 1)
    k16 = {"V": g.vertex_count, "E": g.edge_count,
           "stats": stats_vec(stats), "roots": roots,
           "sha256": {a: sha(getattr(g, a)) for a in
                      ("out_offsets", "destinations", "origins", "in_offsets", "sources")},
           "runs": {}}
    t4k = tree_t4(g, stats, 0)
    ab.serialize(t4k, os.path.join(OUT, "trees", "t4_k16.tree"))
    for i, root in enumerate(roots):
        ref = ab.reference_bfs(g, root)
        finite = ref[ref != INF]
        run = {"depth_sha256": sha(ref), "hist": np.bincount(finite).tolist(),
               "t1": shortcut_trace(t1, stats, ref),
               "t4": shortcut_trace(t4k, stats, ref)}
        if i < 3:   # pin the shortcut against real reference adaptive runs
            for tname, flat in (("t1", t1), ("t4", t4k)):
                d, trace = ab.adaptive_bfs(g, root, flat, stats)
                assert np.array_equal(d, ref)
                assert trace_of(trace) == run[tname], (root, tname)
            d, outs = ab.bfs_full(g, root, ab.KernelId.REV_EDGE_LIST,
                                  ab.CountVariant.DIRECT_ATOMIC)
            assert np.array_equal(d, ref)
        k16["runs"][str(root)] = run
        print(f"k16 root {root}: levels={len(run['hist'])}", flush=True)
    traces["k16"] = k16

    # --- generator pins (config recipes at reduced size) ---------------------
    gens = {}
    for label, model, params, seed, sym in (
            ("rmat_s8", "rmat-like", {"scale": 8, "edges": 4096}, 3, False),
            ("rmat_s12_sym", "rmat-like", {"scale": 12, "edges": 16 << 12}, 1, True),
            ("uniform_n1024", "uniform-random", {"n": 1024, "edges": 9999}, 4, False),
            ("uniform_n2p16", "uniform-random", {"n": 65536, "edges": 1 << 20}, 1, False)):
        gg = symmetrised_rmat(params["scale"], params["edges"] >> params["scale"], seed) \
            if sym else ab.generate_graph(model, params, seed)
        gens[label] = {"model": model, "params": params, "seed": seed, "sym": sym,
                       "V": gg.vertex_count, "E": gg.edge_count,
                       "sha256": {a: sha(getattr(gg, a)) for a in
                                  ("out_offsets", "destinations", "origins",
                                   "in_offsets", "sources")}}
    m = mesh(4096, 4096)
    gens["mesh4096"] = {"V": m.vertex_count, "E": m.edge_count,
                        "sha256": {a: sha(getattr(m, a)) for a in
                                   ("out_offsets", "destinations", "origins",
                                    "in_offsets", "sources")}}
    del m
    np.savez_compressed(os.path.join(OUT, "graphs.npz"), **arrays)
    with open(os.path.join(OUT, "traces.json"), "w") as fh:
        json.dump(traces, fh)
    meta = {"numpy": np.__version__, "python": platform.python_version(),
            "reference": REF_SRC, "generators": gens,
            "script": "tools/make_golden.py"}
    with open(os.path.join(OUT, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print("done")


if __name__ == "__main__":
    main()
