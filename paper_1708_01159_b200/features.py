"""Per-level runtime features (features.py:22-121 of the reference).

24 float64 scalars: graph size (2), frontier/discovery state (4), three
6-value degree summaries.  Only frontier_abs and discovered_abs change per
level; both are integers the device produces with one readback per level
(the new-count of the previous level), so the tree sees exactly the values
the reference computes.  The native adaptive loop (abfs_adaptive_bfs) builds
the same vector in C with IEEE float64 true division.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .graph import DegreeSummary, GraphStats

_SUMMARY_FIELDS = ("min", "q1", "median", "q3", "max", "stddev")

FEATURE_NAMES: tuple[str, ...] = (
    "vertex_count",
    "edge_count",
    "frontier_abs",
    "frontier_pct",
    "discovered_abs",
    "discovered_pct",
    *(f"out_deg.{f}" for f in _SUMMARY_FIELDS),
    *(f"in_deg.{f}" for f in _SUMMARY_FIELDS),
    *(f"abs_deg.{f}" for f in _SUMMARY_FIELDS),
)

DEFAULT_MODEL_FEATURES: tuple[str, ...] = (
    "vertex_count",
    "edge_count",
    "discovered_pct",
    "out_deg.min",
    "out_deg.q1",
    "out_deg.median",
    "out_deg.q3",
    "out_deg.max",
    "out_deg.stddev",
    "frontier_abs",
)


def validate_selection(selection: Sequence[str]) -> tuple[str, ...]:
    """Non-empty, no duplicates, known names (features.py:53-63)."""
    names = tuple(selection)
    if not names:
        raise ValueError("feature selection must be non-empty")
    if len(set(names)) != len(names):
        raise ValueError("feature selection has duplicate names")
    unknown = [n for n in names if n not in FEATURE_NAMES]
    if unknown:
        raise ValueError(f"unknown feature names: {unknown}")
    return names


@dataclass(frozen=True)
class FeatureVector:
    vertex_count: int
    edge_count: int
    frontier_abs: int
    frontier_pct: float
    discovered_abs: int
    discovered_pct: float
    out_deg: DegreeSummary
    in_deg: DegreeSummary
    abs_deg: DegreeSummary

    def scalar(self, name: str) -> float:
        if "." in name:
            summary_name, fld = name.split(".", 1)
            return float(getattr(getattr(self, summary_name), fld))
        return float(getattr(self, name))

    def as_array(self, selection: Sequence[str] | None = None) -> np.ndarray:
        names = FEATURE_NAMES if selection is None else selection
        return np.array([self.scalar(n) for n in names], dtype=np.float64)


def extract_runtime_features(stats: GraphStats, frontier_abs: int,
                             discovered_abs: int) -> FeatureVector:
    """Static stats + traversal state (features.py:98-121), same checks."""
    n = stats.vertex_count
    if n < 1:
        raise ValueError("stats must describe a non-empty graph")
    if frontier_abs < 0 or discovered_abs < frontier_abs:
        raise ValueError(f"need 0 <= frontier_abs <= discovered_abs, got "
                         f"{frontier_abs} and {discovered_abs}")
    if discovered_abs > n:
        raise ValueError(f"discovered_abs {discovered_abs} exceeds |V|={n}")
    return FeatureVector(vertex_count=n, edge_count=stats.edge_count,
                         frontier_abs=frontier_abs, frontier_pct=frontier_abs / n,
                         discovered_abs=discovered_abs, discovered_pct=discovered_abs / n,
                         out_deg=stats.out_degree_summary, in_deg=stats.in_degree_summary,
                         abs_deg=stats.abs_degree_summary)


def static_vector(stats: GraphStats) -> np.ndarray:
    """The 24 canonical features with the 4 dynamic slots zeroed: the
    `static24` argument of abfs_adaptive_bfs."""
    out = [float(stats.vertex_count), float(stats.edge_count), 0.0, 0.0, 0.0, 0.0]
    for s in (stats.out_degree_summary, stats.in_degree_summary, stats.abs_degree_summary):
        out += [float(getattr(s, f)) for f in _SUMMARY_FIELDS]
    return np.array(out, dtype=np.float64)


def canonical_indices(selection: Sequence[str]) -> np.ndarray:
    return np.array([FEATURE_NAMES.index(n) for n in validate_selection(selection)],
                    dtype=np.uint16)
