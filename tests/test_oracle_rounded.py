"""Pins of the oracle's rounded zones (R31, SURVEY §8(f) f2 variant), CPU.

  Z1  brute force: every image within rc - eps of a rank's cell box (Euclidean,
      from above) is present, none beyond rc + eps (tests/pins.py, plain geometry);
  Z2  brute force: every pair within the cutoff is co-resident on some rank with
      the right relative shift (the property the halo exists for);
  Z3  rounded zones are a subset of the slab zones, identical in 1D (no edges or
      corners to round), strictly smaller with 2 or 3 decomposed dims.
A plausible slip (a squared term of the pulse dim twice, the lower instead of
the upper face, a dim skipped, <= for <) fails Z1 or Z2.
"""
import numpy as np
import pytest

from oracle import decompose
from synth import get_config, water_box
from tests import pins


def _sys(name, seed):
    c = get_config(name)
    return c, water_box(c.n_atoms, c.L, seed)


def _images(s):
    return [(int(g), tuple(int(v) for v in sv)) for g, sv in zip(s.gid, s.s)]


@pytest.mark.parametrize("name", ["C1", "T3D", "T2P", "T2D", "T4x2"])
def test_z1_rounded_import_zone_brute_force(name):
    c, X = _sys(name, 3)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses, rounded=True)
    for s in st:
        inner, outer = pins.direct_gather_rounded(X, c.L, c.rc, c.grid, s.rank, eps=1e-5)
        have = _images(s)
        assert len(have) == len(set(have)), "duplicate image on a rank"
        hs = set(have)
        assert inner <= hs, f"rank {s.rank}: missing {sorted(inner - hs)[:5]}"
        assert hs <= outer, f"rank {s.rank}: extra {sorted(hs - outer)[:5]}"


@pytest.mark.parametrize("name", ["T3D", "T2P", "T2D"])
def test_z2_rounded_pair_coverage(name):
    c, X = _sys(name, 4)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses, rounded=True)
    dec = [d for d in range(3) if c.grid[d] > 1]
    index = []
    for s in st:
        m = {}
        for g, sv in _images(s):
            m.setdefault(g, set()).add(sv)
        index.append(m)
    pairs = pins.close_pairs(X, c.L, c.rc, eps=1e-5)
    assert len(pairs) > 1000
    for i, j, n in pairs:
        ok = any(
            any(all(bb[d] - a[d] == n[d] for d in dec) for a in m.get(i, ()) for bb in m.get(j, ()))
            for m in index)
        assert ok, f"pair {i},{j} shift {n} not co-resident"


@pytest.mark.parametrize("name", ["C1", "C5", "T3D", "C2", "T2P"])
def test_z3_rounded_subset_of_slab(name):
    c, X = _sys(name, 5)
    slab = decompose(X, c.L, c.rc, c.grid, c.pulses)
    rnd = decompose(X, c.L, c.rc, c.grid, c.pulses, rounded=True)
    n_dec = sum(1 for g in c.grid if g > 1)
    tot_s = tot_r = 0
    for a, b in zip(slab, rnd):
        sa, sb = set(_images(a)), set(_images(b))
        assert sb <= sa
        assert a.n_home == b.n_home
        np.testing.assert_array_equal(a.x[: a.n_home].view(np.int32), b.x[: b.n_home].view(np.int32))
        tot_s += len(sa) - a.n_home
        tot_r += len(sb) - b.n_home
    if n_dec == 1:
        assert tot_r == tot_s
    else:
        assert tot_r < tot_s
