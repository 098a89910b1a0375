"""Seeded random geometries for the fuzz parity tests (test infrastructure; no halo
arithmetic): random grids (1-4 cells per dim), box lengths, cutoffs (1 or 2
pulses per dim where valid), layouts, atom counts, and uniform or clustered
positions (clustered boxes give DD ranks with no home atoms and empty maps)."""
from __future__ import annotations

import math

import numpy as np

from synth.water import wrap_f32


def random_case(seed: int):
    rng = np.random.Generator(np.random.PCG64(10_000 + seed))
    for _ in range(1000):
        grid = tuple(int(v) for v in rng.integers(1, 5, size=3))
        if grid[0] * grid[1] * grid[2] < 2 or grid[0] * grid[1] * grid[2] > 32:
            continue
        L = tuple(float(np.float32(v)) for v in rng.uniform(1.5, 6.0, size=3))
        rc = float(np.float32(rng.uniform(0.3, 0.49 * min(L))))
        pulses = []
        ok = True
        for d in range(3):
            if grid[d] == 1:
                pulses.append(0)
                continue
            w = float(np.float32(L[d])) / grid[d]
            p = max(1, math.ceil(float(np.float32(rc)) / w))
            if p * w < float(np.float32(rc)):
                p += 1
            if p > min(2, grid[d] - 1):
                ok = False
                break
            pulses.append(p)
        if not ok:
            continue
        n = int(rng.integers(50, 1500))
        if rng.random() < 0.3:  # clustered: empty ranks and empty maps
            lo = rng.uniform(0.0, 0.5, size=3) * np.asarray(L)
            X64 = lo + rng.random((n, 3)) * 0.4 * np.asarray(L)
        else:
            X64 = rng.random((n, 3)) * np.asarray(L)
        X = wrap_f32(X64, L)
        layout = 4 if rng.random() < 0.3 else 3
        return L, rc, grid, tuple(pulses), X, layout
    raise RuntimeError("no valid geometry drawn")
