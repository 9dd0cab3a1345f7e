"""FlatTree predictor and the ADBT model format (tree.py:24-56, 223-242,
303-447 of the reference).

The runtime structure is the reference's preorder flat array (u2 feature,
f8 threshold, u4 left/right, u1 class); `FlatTree.as_abfs()` hands the same
arrays to the engine, whose C descent (abfs_adaptive_bfs / abfs_tree_predict)
applies the identical strict `<` rule on the identical float64 values.
CART training stays offline (out of scope); models trained by the
reference's `fit` load here byte-for-byte.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib as L
from .features import canonical_indices
from .kernels import ALL_PAIRS, CountVariant, KernelId, pair_from_index

N_CLASSES = len(ALL_PAIRS)
LEAF_UNKNOWN = 254
NOT_A_LEAF = 255

TREE_MAGIC = b"ADBT"
TREE_FORMAT_VERSION = 1
_NODE_DTYPE = np.dtype([("feature", "<u2"), ("threshold", "<f8"), ("left", "<u4"),
                        ("right", "<u4"), ("leaf_class", "u1")])


class _UnknownType:
    """Singleton: a leaf with no unique majority label (tree.py:41-56)."""

    __slots__ = ()
    _instance = None

    def __new__(cls):
        if cls._instance is None:
            cls._instance = super().__new__(cls)
        return cls._instance

    def __repr__(self) -> str:
        return "UNKNOWN"


UNKNOWN = _UnknownType()


def _class_to_result(ordinal: int):
    if ordinal == LEAF_UNKNOWN:
        return UNKNOWN
    return pair_from_index(ordinal)


def _project(vector, selection: tuple[str, ...]) -> np.ndarray:
    if hasattr(vector, "as_array"):
        return vector.as_array(selection)
    vec = np.asarray(vector, dtype=np.float64)
    if vec.shape != (len(selection),):
        raise ValueError(f"expected a vector of {len(selection)} features, got {vec.shape}")
    return vec


@dataclass(eq=False)
class FlatTree:
    """Preorder array form of a decision tree (tree.py:303-359)."""

    selection: tuple[str, ...]
    features: np.ndarray
    thresholds: np.ndarray
    lefts: np.ndarray
    rights: np.ndarray
    leaf_classes: np.ndarray
    _fast: tuple | None = field(default=None, repr=False)
    _abfs: tuple | None = field(default=None, repr=False)

    @property
    def node_count(self) -> int:
        return len(self.leaf_classes)

    def _lists(self) -> tuple:
        if self._fast is None:
            object.__setattr__(self, "_fast", (
                self.features.tolist(), self.thresholds.tolist(), self.lefts.tolist(),
                self.rights.tolist(), self.leaf_classes.tolist()))
        return self._fast

    def predict_one(self, vector) -> int:
        """Class ordinal (or LEAF_UNKNOWN); `vec[f] < thr` goes left."""
        feats, thrs, lefts, rights, classes = self._lists()
        vec = _project(vector, self.selection).tolist()
        node = 0
        while classes[node] == NOT_A_LEAF:
            node = lefts[node] if vec[feats[node]] < thrs[node] else rights[node]
        return classes[node]

    def predict_batch(self, x: np.ndarray) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        if x.ndim != 2 or x.shape[1] != len(self.selection):
            raise ValueError(f"expected (n, {len(self.selection)}) feature matrix, got {x.shape}")
        cur = np.zeros(x.shape[0], dtype=np.int64)
        rows = np.arange(x.shape[0])
        while True:
            at_leaf = self.leaf_classes[cur] != NOT_A_LEAF
            if at_leaf.all():
                return self.leaf_classes[cur].astype(np.int64)
            go_left = x[rows, self.features[cur]] < self.thresholds[cur]
            cur = np.where(at_leaf, cur, np.where(go_left, self.lefts[cur], self.rights[cur]))

    def predict_pairs(self, x: np.ndarray) -> list:
        return [_class_to_result(int(c)) for c in self.predict_batch(x)]

    def as_abfs(self) -> L.AbfsTree:
        """ctypes view for the engine (arrays kept alive on the object)."""
        if self._abfs is None:
            arrs = (canonical_indices(self.selection),
                    np.ascontiguousarray(self.features, dtype=np.uint16),
                    np.ascontiguousarray(self.thresholds, dtype=np.float64),
                    np.ascontiguousarray(self.lefts, dtype=np.uint32),
                    np.ascontiguousarray(self.rights, dtype=np.uint32),
                    np.ascontiguousarray(self.leaf_classes, dtype=np.uint8))
            t = L.AbfsTree(self.node_count, len(self.selection), L.ptr(arrs[0], L.u16p),
                           L.ptr(arrs[1], L.u16p), L.ptr(arrs[2], L.f64p),
                           L.ptr(arrs[3], L.u32p), L.ptr(arrs[4], L.u32p),
                           L.ptr(arrs[5], L.u8p))
            object.__setattr__(self, "_abfs", (t, arrs))
        return self._abfs[0]


def predict(model: FlatTree, vector):
    """Descend to a leaf (tree.py:223-231); FlatTree models only."""
    if not isinstance(model, FlatTree):
        raise TypeError("predict expects a FlatTree (CART training is offline)")
    return _class_to_result(model.predict_one(vector))


def serialize(flat: FlatTree, path: str) -> None:
    """ADBT writer (tree.py:389-406): header, selection names, 19-byte records."""
    with open(path, "wb") as fh:
        fh.write(TREE_MAGIC)
        fh.write(struct.pack("<II", TREE_FORMAT_VERSION, flat.node_count))
        fh.write(struct.pack("<H", len(flat.selection)))
        for name in flat.selection:
            raw = name.encode("utf-8")
            fh.write(struct.pack("<H", len(raw)))
            fh.write(raw)
        rec = np.empty(flat.node_count, dtype=_NODE_DTYPE)
        rec["feature"] = flat.features
        rec["threshold"] = flat.thresholds
        rec["left"] = flat.lefts
        rec["right"] = flat.rights
        rec["leaf_class"] = flat.leaf_classes
        fh.write(rec.tobytes())


def deserialize(path: str) -> FlatTree:
    """ADBT reader (tree.py:409-447) with the reference's ValueErrors."""
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != TREE_MAGIC:
            raise ValueError(f"bad magic {magic!r} in model file {path}")
        header = fh.read(8)
        if len(header) != 8:
            raise ValueError(f"truncated model header in {path}")
        version, node_count = struct.unpack("<II", header)
        if version != TREE_FORMAT_VERSION:
            raise ValueError(f"unsupported model format version {version}")
        raw = fh.read(2)
        if len(raw) != 2:
            raise ValueError(f"truncated selection header in {path}")
        (n_names,) = struct.unpack("<H", raw)
        names = []
        for _ in range(n_names):
            raw = fh.read(2)
            if len(raw) != 2:
                raise ValueError(f"truncated selection name in {path}")
            (length,) = struct.unpack("<H", raw)
            name = fh.read(length)
            if len(name) != length:
                raise ValueError(f"truncated selection name in {path}")
            names.append(name.decode("utf-8"))
        body = fh.read(node_count * _NODE_DTYPE.itemsize)
        if len(body) != node_count * _NODE_DTYPE.itemsize:
            raise ValueError(f"truncated node records in {path}")
        if fh.read(1):
            raise ValueError(f"trailing bytes in model file {path}")
    rec = np.frombuffer(body, dtype=_NODE_DTYPE)
    return FlatTree(selection=tuple(names), features=rec["feature"].copy(),
                    thresholds=rec["threshold"].copy(), lefts=rec["left"].copy(),
                    rights=rec["right"].copy(), leaf_classes=rec["leaf_class"].copy())


def leaf_tree(label_ordinal: int, selection: Sequence[str] = ("frontier_abs",)) -> FlatTree:
    """Single-leaf model always predicting one pair (or LEAF_UNKNOWN)."""
    return FlatTree(selection=tuple(selection), features=np.zeros(1, np.uint16),
                    thresholds=np.zeros(1, np.float64), lefts=np.zeros(1, np.uint32),
                    rights=np.zeros(1, np.uint32),
                    leaf_classes=np.array([label_ordinal], dtype=np.uint8))
