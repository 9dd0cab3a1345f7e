"""GPU benchmark harness (reference bench.py:102-165 schema).

Times every (kernel, variant) pair level by level on the device (CUDA events
around each level, same accounting as LevelOutcome.elapsed_ns) and writes the
reference's levels.csv schema (bench.py:40-46), so the reference's own
`training_samples_from` / `fit` can train a GPU tree from it unchanged.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass

import numpy as np

from .engine import Traversal
from .kernels import ALL_PAIRS

LEVELS_HEADER = ("graph_id", "root", "kernel", "variant", "level", "mean_ns", "min_ns",
                 "frontier_size", "discovered_before", "new_count")


@dataclass(frozen=True)
class LevelRow:
    graph_id: str
    root: int
    kernel: str
    variant: str
    level: int
    mean_ns: float
    min_ns: int
    frontier_size: int
    discovered_before: int
    new_count: int


def benchmark_graph_gpu(dgraph, roots, graph_id: str, repetitions: int = 3,
                        warmup_runs: int = 1, chunk_size: int = 32, pairs=ALL_PAIRS,
                        traversal: Traversal | None = None) -> list[LevelRow]:
    """All `pairs` from every root; per-level mean/min over `repetitions`
    after `warmup_runs`; the level structure must repeat exactly."""
    t = traversal or Traversal(dgraph)
    rows: list[LevelRow] = []
    for root in roots:
        for kernel, variant in pairs:
            per_level: list[list[int]] = []
            structure = None
            for rep in range(warmup_runs + repetitions):
                counts, el = t.bfs_full(int(root), int(kernel), int(variant), chunk_size,
                                        cap=1 << 20)
                if structure is None:
                    structure = counts.tolist()
                elif counts.tolist() != structure:
                    raise RuntimeError(f"nondeterministic level structure at root {root}")
                if rep >= warmup_runs:
                    per_level.append(el.tolist())
            times = np.array(per_level, dtype=np.int64)
            discovered = 1
            for lvl, new in enumerate(structure):
                frontier = 1 if lvl == 0 else int(structure[lvl - 1])
                rows.append(LevelRow(graph_id, int(root), kernel.name, variant.name, lvl,
                                     float(times[:, lvl].mean()), int(times[:, lvl].min()),
                                     frontier, discovered, int(new)))
                discovered += int(new)
    return rows


def export_levels(rows, path: str, append: bool = False) -> None:
    with open(path, "a" if append else "w", newline="") as fh:
        w = csv.writer(fh)
        if not append:
            w.writerow(LEVELS_HEADER)
        for r in rows:
            w.writerow([r.graph_id, r.root, r.kernel, r.variant, r.level, repr(r.mean_ns),
                        r.min_ns, r.frontier_size, r.discovered_before, r.new_count])
