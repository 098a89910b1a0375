"""Independent brute-force pins (test-only).  No code shared with oracle/ or the product.

These re-derive what the method must produce from plain geometry, not from the
staged algorithm: every image inside a rank's import zone is present (X2), every
pair within the cutoff is co-resident with the right relative shift (X3),
per-atom force totals (F1), conservation (F2), shift forces (F3), virial (F4).
"""
from __future__ import annotations

import itertools
import math

import numpy as np


def cell_bounds(L, grid, cell):
    """Exact-real cell bounds [lo, hi) per dim (float64 of the float32 box length)."""
    lo, hi = [], []
    for d in range(3):
        Ld = float(np.float32(L[d]))
        lo.append(Ld * cell[d] / grid[d])
        hi.append(Ld * (cell[d] + 1) / grid[d])
    return lo, hi


def rank_cell(r, grid):
    return (r // (grid[1] * grid[2]), (r // grid[2]) % grid[1], r % grid[2])


def direct_gather(X, L, rc, grid, r, eps):
    """(inner, outer) sets of (gid, s) images for rank r.

    inner: images whose exact-real position lies in prod[lo, hi + rc - eps) over the
    decomposed dims (must be present); outer: prod[lo - eps, hi + rc + eps) (may be present).
    """
    X64 = np.asarray(X, dtype=np.float64)
    Lf = np.array([float(np.float32(v)) for v in L])
    rc = float(np.float32(rc))
    lo, hi = cell_bounds(L, grid, rank_cell(r, grid))
    dec = [d for d in range(3) if grid[d] > 1]
    inner, outer = set(), set()
    for s in itertools.product(*[(0, 1) if d in dec else (0,) for d in range(3)]):
        sv = np.array(s, dtype=np.float64)
        Y = X64 + sv * Lf
        m_in = np.ones(X.shape[0], bool)
        m_out = np.ones(X.shape[0], bool)
        for d in dec:
            m_in &= (Y[:, d] >= lo[d]) & (Y[:, d] < hi[d] + rc - eps)
            m_out &= (Y[:, d] >= lo[d] - eps) & (Y[:, d] < hi[d] + rc + eps)
        for g in np.nonzero(m_in)[0]:
            inner.add((int(g), s))
        for g in np.nonzero(m_out)[0]:
            outer.add((int(g), s))
    return inner, outer


def direct_gather_rounded(X, L, rc, grid, r, eps):
    """As direct_gather for the rounded zones (R31): an image belongs to rank r's
    import zone iff it lies at or above the cell's lower corner in every decomposed
    dim and its Euclidean distance to the cell box is < rc (inner: < rc - eps,
    outer: < rc + eps, lower faces widened by eps)."""
    X64 = np.asarray(X, dtype=np.float64)
    Lf = np.array([float(np.float32(v)) for v in L])
    rc = float(np.float32(rc))
    lo, hi = cell_bounds(L, grid, rank_cell(r, grid))
    dec = [d for d in range(3) if grid[d] > 1]
    inner, outer = set(), set()
    for s in itertools.product(*[(0, 1) if d in dec else (0,) for d in range(3)]):
        Y = X64 + np.array(s, dtype=np.float64) * Lf
        above_in = np.ones(X.shape[0], bool)
        above_out = np.ones(X.shape[0], bool)
        dist2 = np.zeros(X.shape[0])
        for d in dec:
            above_in &= Y[:, d] >= lo[d]
            above_out &= Y[:, d] >= lo[d] - eps
            ex = np.maximum(Y[:, d] - hi[d], 0.0)
            dist2 += ex * ex
        dist = np.sqrt(dist2)
        for g in np.nonzero(above_in & (dist < rc - eps))[0]:
            inner.add((int(g), s))
        for g in np.nonzero(above_out & (dist < rc + eps))[0]:
            outer.add((int(g), s))
    return inner, outer


def close_pairs(X, L, rc, eps):
    """All pairs (i, j, n) with minimum-image distance < rc - eps, n = integer shift of j."""
    X64 = np.asarray(X, dtype=np.float64)
    Lf = np.array([float(np.float32(v)) for v in L])
    out = []
    N = X64.shape[0]
    for i in range(N):
        d = X64[i + 1:] - X64[i]
        n = -np.round(d / Lf)
        dm = d + n * Lf
        dist = np.sqrt((dm * dm).sum(axis=1))
        for jj in np.nonzero(dist < rc - eps)[0]:
            out.append((i, i + 1 + int(jj), tuple(int(v) for v in n[jj])))
    return out


def scatter_totals(gids_per_rank, F_per_rank, n_atoms):
    """F1: per-gid total over all rows of all ranks, exact with fsum."""
    acc = [[[] for _ in range(3)] for _ in range(n_atoms)]
    for gids, F in zip(gids_per_rank, F_per_rank):
        for row, g in enumerate(gids):
            for c in range(3):
                acc[int(g)][c].append(float(F[row, c]))
    return np.array([[math.fsum(acc[g][c]) for c in range(3)] for g in range(n_atoms)])
