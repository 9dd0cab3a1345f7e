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
