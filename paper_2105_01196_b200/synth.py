"""Synthetic benchmark inputs: planted-trend expression matrices and random
candidate populations (vectorised numpy; the bench must not depend on the
reference generator, which only exists in the build container).

planted_trend_matrix follows the reference's trend implant recipe
(datagen.cpp:72-130 `PatternKind::trend`: a shared random column order per
bicluster, each member row gets sorted N(0,1) values along it) on an N(0,1)
background (datagen.cpp:64-70), generated directly in float32 so the device
store is exact.  random_population follows init_population's shape
(evolution.cpp:117-126: length uniform in [len_min, len_max], distinct
columns in random order).
"""
from __future__ import annotations

import numpy as np

from .trend import Population


def planted_trend_matrix(rows: int, cols: int, n_bics: int = 3, bic_rows: int = 50, bic_cols: int = 8,
                         seed: int = 1) -> tuple[np.ndarray, list[tuple[np.ndarray, np.ndarray]]]:
    rng = np.random.default_rng(seed)
    m = rng.standard_normal((rows, cols), dtype=np.float32)
    truth = []
    used_cells = np.zeros((rows, cols), dtype=bool) if rows * cols <= 50_000_000 else None
    for _ in range(n_bics):
        for _attempt in range(1000):
            r = np.sort(rng.choice(rows, size=min(bic_rows, rows), replace=False))
            c = np.sort(rng.choice(cols, size=min(bic_cols, cols), replace=False))
            if used_cells is None or not used_cells[np.ix_(r, c)].any():
                break
        order = rng.permutation(c)
        vals = np.sort(rng.standard_normal((r.size, c.size), dtype=np.float32), axis=1)
        m[np.ix_(r, order)] = vals
        if used_cells is not None:
            used_cells[np.ix_(r, c)] = True
        truth.append((r, c))
    return m, truth


def random_population(n: int, n_cols: int, len_min: int = 3, len_max: int = 5, seed: int = 42) -> Population:
    if n_cols < len_max:
        raise ValueError("random_population: len_max exceeds column count")
    rng = np.random.default_rng(seed)
    lens = rng.integers(len_min, len_max + 1, size=n).astype(np.int64)
    draw = rng.integers(0, n_cols, size=(n, len_max))
    # redraw rows that contain a duplicate within their first `len` entries
    idx = np.arange(len_max)
    while True:
        s = np.sort(np.where(idx[None, :] < lens[:, None], draw, -1 - idx[None, :]), axis=1)
        dup = (s[:, 1:] == s[:, :-1]).any(axis=1)
        if not dup.any():
            break
        draw[dup] = rng.integers(0, n_cols, size=(int(dup.sum()), len_max))
    mask = idx[None, :] < lens[:, None]
    cols = draw[mask].astype(np.uint32)
    offs = np.zeros(n + 1, dtype=np.uint32)
    offs[1:] = np.cumsum(lens)
    return Population(cols, offs)


def exact_len_population(n: int, n_cols: int, length: int, seed: int = 42) -> Population:
    """Microbench populations: exactly `length` distinct random columns each."""
    rng = np.random.default_rng(seed)
    keys = rng.random((n, n_cols), dtype=np.float32) if n * n_cols <= 64_000_000 else None
    if keys is not None:
        cols = np.argpartition(keys, length - 1, axis=1)[:, :length]
        # random order within the sequence
        perm = rng.permuted(np.tile(np.arange(length), (n, 1)), axis=1)
        cols = np.take_along_axis(cols, perm, axis=1)
    else:
        cols = np.stack([rng.choice(n_cols, size=length, replace=False) for _ in range(n)])
    offs = (np.arange(n + 1) * length).astype(np.uint32)
    return Population(cols.reshape(-1).astype(np.uint32), offs)
