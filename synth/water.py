"""SPC-water-like synthetic boxes (recipe: SURVEY.md §8(d)).

The paper benchmarks homogeneous water-ethanol "grappa" inputs (PAPER.md:473,
"more homogeneous"), so a uniform water box at liquid density is a faithful
stand-in for halo volumes.  Recipe:

* 3 atoms / molecule (O, H, H), O-H 0.1 nm, H-O-H 109.47 deg (SPC geometry).
* O placed on a jittered lattice with >= n_mol sites, sites drawn without
  replacement, jitter uniform +-0.05 nm, uniformly random orientation.
* molecules numbered in spatially binned order (0.5 nm bins, z-major, then y,
  then x) so that a rank's home atoms (ascending gid) are spatially coherent,
  like GROMACS's grid-sorted local atoms; ``shuffle_ids`` gives random order.
* positions wrapped in float64, cast to float32, ``x == L`` mapped to 0.0 and
  -0.0 normalised to +0.0 (reading R25).
* RNG: numpy PCG64 seeded by the caller.

No halo arithmetic lives here.
"""
from __future__ import annotations

import numpy as np

OH = 0.1
HOH_DEG = 109.47


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def wrap_f32(pos64: np.ndarray, L) -> np.ndarray:
    """Wrap float64 positions into [0, L) and cast to float32 with no -0.0 and no x == L."""
    L64 = np.asarray(L, dtype=np.float64)
    w = np.mod(pos64, L64)
    out = w.astype(np.float32)
    L32 = np.asarray(L, dtype=np.float32)
    out = np.where(out >= L32, np.float32(0.0), out)
    out = out + np.float32(0.0)  # -0.0 + 0.0 = +0.0
    return np.ascontiguousarray(out, dtype=np.float32)


def _random_rotations(rng: np.random.Generator, n: int) -> np.ndarray:
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    R = np.empty((n, 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - z * w)
    R[:, 0, 2] = 2 * (x * z + y * w)
    R[:, 1, 0] = 2 * (x * y + z * w)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - x * w)
    R[:, 2, 0] = 2 * (x * z - y * w)
    R[:, 2, 1] = 2 * (y * z + x * w)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def water_box(n_atoms: int, L, seed: int, shuffle_ids: bool = False,
              slab: tuple | None = None) -> np.ndarray:
    """Return float32 positions [n_atoms, 3] of an SPC-like water box of size L (nm).

    ``slab=(z_lo, z_hi)`` halves the molecule density for O with z in
    [z_lo, z_hi) (optional membrane-like slab for the C3 config).  The returned
    atom count is then smaller than ``n_atoms``.
    """
    if n_atoms % 3 != 0:
        raise ValueError("n_atoms must be a multiple of 3 (3-site water)")
    L = np.asarray(L, dtype=np.float64)
    n_mol = n_atoms // 3
    rng = _rng(seed)
    if n_mol == 0:
        return np.zeros((0, 3), dtype=np.float32)
    # lattice with >= n_mol sites, spacing as uniform as possible
    dens = n_mol / float(np.prod(L))
    a = dens ** (-1.0 / 3.0)
    nd = np.maximum(1, np.ceil(L / a).astype(np.int64))
    while int(np.prod(nd)) < n_mol:  # grow the coarsest dim until enough sites
        nd[np.argmax(L / nd)] += 1
    n_sites = int(np.prod(nd))
    sites = rng.choice(n_sites, size=n_mol, replace=False)
    ix = sites // (nd[1] * nd[2])
    iy = (sites // nd[2]) % nd[1]
    iz = sites % nd[2]
    idx = np.stack([ix, iy, iz], axis=1).astype(np.float64)
    O = (idx + 0.5) * (L / nd) + rng.uniform(-0.05, 0.05, size=(n_mol, 3))
    half = np.deg2rad(HOH_DEG) / 2.0
    local = np.array([[0.0, 0.0, 0.0],
                      [OH * np.sin(half), 0.0, OH * np.cos(half)],
                      [-OH * np.sin(half), 0.0, OH * np.cos(half)]])
    R = _random_rotations(rng, n_mol)
    mol = O[:, None, :] + np.einsum("mij,aj->mai", R, local)  # [n_mol, 3, 3]
    if slab is not None:
        z = np.mod(O[:, 2], L[2])
        in_slab = (z >= slab[0]) & (z < slab[1])
        drop = in_slab & (rng.uniform(size=n_mol) < 0.5)
        mol = mol[~drop]
        O = O[~drop]
        n_mol = mol.shape[0]
    # spatially binned molecule order: 0.5 nm bins, z-major, then y, then x
    Ow = np.mod(O, L)
    nb = np.maximum(1, np.floor(L / 0.5).astype(np.int64))
    b = np.minimum((Ow / (L / nb)).astype(np.int64), nb - 1)
    if shuffle_ids:
        order = rng.permutation(n_mol)
    else:
        order = np.lexsort((b[:, 0], b[:, 1], b[:, 2]))
    mol = mol[order]
    pos = mol.reshape(-1, 3)
    return wrap_f32(pos, L)


def forces_int(n_rows: int, seed: int, width: int = 3) -> np.ndarray:
    """Parity set A: integer-valued float32 forces, uniform in [-1024, 1024]."""
    rng = _rng(seed)
    return rng.integers(-1024, 1025, size=(n_rows, width)).astype(np.float32)


def forces_normal(n_rows: int, seed: int, width: int = 3, sigma: float = 300.0) -> np.ndarray:
    """Parity/timing set B: float32 normal(0, 300) kJ mol^-1 nm^-1."""
    rng = _rng(seed)
    f = rng.normal(0.0, sigma, size=(n_rows, width)).astype(np.float32)
    return f + np.float32(0.0)


def charges(n_atoms: int) -> np.ndarray:
    """SPC charges (O -0.82, H +0.41), used as the float4 ``w`` component."""
    q = np.tile(np.array([-0.82, 0.41, 0.41], dtype=np.float32), n_atoms // 3 + 1)
    return q[:n_atoms].copy()


def displacements(X: np.ndarray, L, seed: int, sigma: float = 0.05, n_far: int = 16, far: float = 0.6) -> np.ndarray:
    """Moved positions between two NS steps (input of halo_migrate tests/bench): every
    atom moves by normal(0, sigma) nm per component (nstlist steps of thermal motion;
    SPC water diffuses ~0.05 nm per 200 x 2 fs), and `n_far` random atoms move by
    +-`far` nm in every component (diagonal cell crossings).  Positions are NOT
    wrapped (atoms near a face leave the box): the wrap is the method's (R29).
    float32 [N, 3]."""
    rng = _rng(seed)
    Xm = np.asarray(X, np.float64) + rng.normal(0.0, sigma, size=(X.shape[0], 3))
    if n_far:
        idx = rng.choice(X.shape[0], size=min(n_far, X.shape[0]), replace=False)
        Xm[idx] += far * rng.choice([-1.0, 1.0], size=(idx.size, 3))
    return Xm.astype(np.float32)


def velocities(n_rows: int, seed: int, width: int = 3) -> np.ndarray:
    """Per-atom payload carried by halo_migrate (velocities, nm/ps), float32 [n, width]."""
    return _rng(seed).normal(0.0, 0.5, size=(n_rows, width)).astype(np.float32)
