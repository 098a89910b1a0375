"""Pins of the oracle's NS-step redistribution (R29, R30), CPU.

oracle.migrate is pinned against things other than itself:
  M1  wrap_coord closed forms: identity inside the box, fl32(x - L) / fl32(x + L)
      outside, the two special cases that must become +0.0 (-tiny + L rounding to
      L, and -0.0), and rejection beyond a box length;
  M2  brute force: every output row lies in its rank's cell (plane inequalities
      written out here in float64), gids ascend, every gid appears exactly once and
      its row is the bit-exact wrapped input row (x, w, payload);
  M3  migrate(homes of X) == the home rows of a FRESH decomposition of the wrapped
      moved positions (decompose is pinned by X0-X5), rank by rank, bit-exact;
  M4  an atom moved by two cells (or a box length) is rejected (R30).
A plausible mistake (wrapping with fmod in float64, the lower cell on a tie, a
forgotten w / payload column, an unsorted merge, a missing diagonal neighbour)
fails one of them.
"""
import numpy as np
import pytest

from oracle import decompose, migrate, wrap_coord
from synth import displacements, get_config, velocities, water_box
from synth.water import charges


def test_wrap_closed_forms():
    L = np.float32(3.104)
    rng = np.random.default_rng(5)
    for x in rng.uniform(0, float(L), 200).astype(np.float32):
        w, ok = wrap_coord(x, L)
        assert ok and w.view(np.int32) == x.view(np.int32) or (x == 0 and w == 0)
    for x in rng.uniform(float(L), 2 * float(L), 200).astype(np.float32):
        w, ok = wrap_coord(x, L)
        exp = np.float32(x - L)
        assert ok and w == exp and 0 <= w < L
    for x in rng.uniform(-float(L), 0, 200).astype(np.float32):
        w, ok = wrap_coord(x, L)
        exp = np.float32(x + L)
        if exp == L:
            exp = np.float32(0.0)
        assert ok and w == exp and 0 <= w < L
    # -tiny + L rounds to L in float32 -> +0.0 (never L)
    w, ok = wrap_coord(np.float32(-1e-9), L)
    assert ok and w.view(np.int32) == 0
    # -0.0 -> +0.0
    w, ok = wrap_coord(np.float32(-0.0), L)
    assert ok and w.view(np.int32) == 0
    # exactly L -> 0.0
    w, ok = wrap_coord(L, L)
    assert ok and w.view(np.int32) == 0
    # more than one box length: rejected
    assert not wrap_coord(np.float32(2.5) * L, L)[1]
    assert not wrap_coord(np.float32(-1.5) * L, L)[1]


def _homes(states, X_moved, V=None, W=None):
    out = []
    for st in states:
        g = st.gid[: st.n_home]
        x = np.zeros((g.size, 3 if W is None else 4), np.float32)
        x[:, :3] = X_moved[g]
        if W is not None:
            x[:, 3] = W[g]
        out.append((g, x, None if V is None else V[g]))
    return out


def _wrap_all(Xm, L):
    Xw = Xm.copy()
    for i in range(Xm.shape[0]):
        for d in range(3):
            Xw[i, d], ok = wrap_coord(Xm[i, d], L[d])
            assert ok
    return Xw


@pytest.mark.parametrize("name,layout", [("C1", 3), ("T3D", 4), ("T2P", 3), ("C5", 4)])
def test_migrate_matches_fresh_decomposition(name, layout):
    c = get_config(name)
    X = water_box(c.n_atoms, c.L, 11)
    W = charges(X.shape[0]) if layout == 4 else None
    states = decompose(X, c.L, c.rc, c.grid, c.pulses, W=W)
    Xm = displacements(X, c.L, 12)
    V = velocities(X.shape[0], 13, width=layout)
    new = migrate(_homes(states, Xm, V, W), c.L, c.grid)
    Xw = _wrap_all(Xm, c.L)
    fresh = decompose(Xw, c.L, c.rc, c.grid, c.pulses, W=W)
    seen = np.zeros(X.shape[0], np.int64)
    moved = 0
    for r, ((g, x, v), st) in enumerate(zip(new, fresh)):
        # M3: same atoms, same order, same bits as a fresh decomposition
        np.testing.assert_array_equal(g, st.gid[: st.n_home])
        np.testing.assert_array_equal(x.view(np.int32), st.x[: st.n_home].view(np.int32))
        # M2: brute force
        assert np.all(np.diff(g) > 0)
        seen[g] += 1
        np.testing.assert_array_equal(x[:, :3].view(np.int32), Xw[g].view(np.int32))
        if W is not None:
            np.testing.assert_array_equal(x[:, 3].view(np.int32), W[g].view(np.int32))
        np.testing.assert_array_equal(v.view(np.int32), V[g].view(np.int32))
        cz = r % c.grid[2]
        cy = (r // c.grid[2]) % c.grid[1]
        cx = r // (c.grid[1] * c.grid[2])
        for d, cd in zip(range(3), (cx, cy, cz)):
            lo = float(np.float32(c.L[d])) * cd / c.grid[d]
            hi = float(np.float32(c.L[d])) * (cd + 1) / c.grid[d]
            xd = x[:, d].astype(np.float64)
            assert np.all(xd >= lo) and (cd == c.grid[d] - 1 or np.all(xd < hi))
        moved += int(np.sum(~np.isin(g, states[r].gid[: states[r].n_home])))
    assert np.all(seen == 1)
    assert moved > 0  # the case exercises redistribution


def test_migrate_rejects_two_cell_moves():
    c = get_config("C5")  # 8 cells of 0.957 nm along z
    X = water_box(c.n_atoms, c.L, 11)
    states = decompose(X, c.L, c.rc, c.grid, c.pulses)
    Xm = X.copy()
    g0 = states[3].gid[0]
    Xm[g0, 2] += np.float32(2.1)  # two cells up
    with pytest.raises(ValueError):
        migrate(_homes(states, Xm), c.L, c.grid)
    Xm = X.copy()
    Xm[g0, 0] += np.float32(2.5 * c.L[0])  # more than a box length beyond one wrap
    with pytest.raises(ValueError):
        migrate(_homes(states, Xm), c.L, c.grid)
    # one cell (periodically, across the box face) is fine
    Xm = X.copy()
    g7 = states[7].gid[0]
    Xm[g7, 2] += np.float32(1.0)
    new = migrate(_homes(states, Xm), c.L, c.grid)
    assert g7 in new[0][0]


def test_pme_gather_return_pins():
    """P1: the PME buffer holds every atom exactly once, row = its global position
    (the rank-order concatenation of the home rows, pinned against X through the
    home assignment); P2: with integer forces the returned increments sum to the
    PME forces exactly and each rank's rows get exactly its slice."""
    from oracle import pme_gather, pme_return
    from synth import forces_int
    c = get_config("T3D")
    X = water_box(c.n_atoms, c.L, 21)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses)
    pme_x, off = pme_gather([s.x[: s.n_home] for s in st])
    gids = np.concatenate([s.gid[: s.n_home] for s in st])
    assert pme_x.shape[0] == X.shape[0] and np.array_equal(np.sort(gids), np.arange(X.shape[0]))
    np.testing.assert_array_equal(pme_x.view(np.int32), X[gids].view(np.int32))
    assert off[-1] == X.shape[0] and all(off[r + 1] - off[r] == st[r].n_home for r in range(len(st)))
    F = [forces_int(s.n_home, 50 + s.rank) for s in st]
    pf = forces_int(X.shape[0], 99)
    out = pme_return(F, pf, off)
    tot = sum((o.astype(np.float64) - f.astype(np.float64)).sum(axis=0) for o, f in zip(out, F))
    np.testing.assert_array_equal(tot, pf.astype(np.float64).sum(axis=0))
    for r, o in enumerate(out):
        np.testing.assert_array_equal(o - F[r], pf[off[r]: off[r + 1]])
    ov = pme_return(F, pf, off, accumulate=False)
    np.testing.assert_array_equal(np.concatenate(ov).view(np.int32), pf.view(np.int32))
