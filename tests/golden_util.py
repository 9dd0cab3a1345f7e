"""Loader for tests/golden/ (frozen from the reference by tools/make_golden.py)."""

from __future__ import annotations

import functools
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ARRAYS = ("out_offsets", "destinations", "origins", "in_offsets", "sources")
INF = 2**31 - 1


@functools.lru_cache(maxsize=1)
def npz():
    with np.load(os.path.join(GOLDEN, "graphs.npz")) as z:
        return {k: z[k] for k in z.files}


@functools.lru_cache(maxsize=1)
def traces():
    with open(os.path.join(GOLDEN, "traces.json")) as fh:
        return json.load(fh)


@functools.lru_cache(maxsize=1)
def meta():
    with open(os.path.join(GOLDEN, "meta.json")) as fh:
        return json.load(fh)


def graph_names():
    return sorted({k.split("/")[1] for k in npz() if k.startswith("g/")})


def graph_arrays(name):
    z = npz()
    p = f"g/{name}/"
    n, m = (int(x) for x in z[p + "n"])
    return n, m, {a: z[p + a] for a in ARRAYS + ("rev_owner",)}


def roots(name):
    return [int(r) for r in npz()[f"g/{name}/roots"]]


def depth(name, root):
    return npz()[f"g/{name}/depth/{root}"]


def counts(name, root):
    return npz()[f"g/{name}/counts/{root}"]


def stats(name):
    return npz()[f"g/{name}/stats"]


def level_cases(name):
    z = npz()
    out = []
    i = 0
    while f"g/{name}/lc/{i}/in" in z:
        p = f"g/{name}/lc/{i}/"
        out.append((z[p + "in"], int(z[p + "level"][0]),
                    [(z[p + f"out{k}"], int(z[p + f"cnt{k}"][0])) for k in range(5)]))
        i += 1
    return out


def tree_path(name):
    return os.path.join(GOLDEN, "trees", name + ".tree")


def trees_for(name):
    """(trace key, tree file) pairs recorded for a small golden graph."""
    return [("t1", "t1"), ("t2_unknown", "t2_unknown"), ("t4", f"t4_{name}"),
            ("t3_leaf03", "t3_leaf03"), ("t3_leaf09", "t3_leaf09"), ("t3_leaf14", "t3_leaf14")]


def static24(stats18, n, m):
    return np.array([float(n), float(m), 0, 0, 0, 0, *stats18], dtype=np.float64)
