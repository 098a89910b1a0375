"""Oracle pins (-m "not gpu"): the oracle checked against things other than itself.

Pins: golden hand-derived examples W1-W3, closed-form
halo values (X1), brute-force import zones (X2), brute-force pair coverage (X3),
structural invariants (X4), special cases (X5), brute-force per-atom force
totals (F1), conservation (F2), shift-force closed form (F3), virial identity
(F4) and the rounding bound for real-valued forces (F5).
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import decompose, force_halo, pulse_list, planes, home_cell, rank_of, check_geometry
from synth import water_box, forces_int, forces_normal, get_config
from tests import pins

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def run(cfg_or_dict, X, W=None):
    c = cfg_or_dict
    return decompose(X, tuple(c["L"]), c["rc"], tuple(c["grid"]), tuple(c["pulses"]), W=W)


# ---------------------------------------------------------------- golden W1-W3
def test_w1_golden():
    g = load("W1.json")
    X = np.array(g["X"], np.float32)
    st = run(g, X)
    for er, s in zip(g["expect"]["ranks"], st):
        assert s.n_home == er["n_home"]
        assert s.gid.tolist() == er["gid"]
        assert s.s.tolist() == er["s"]
        np.testing.assert_array_equal(s.x, np.array(er["x"], np.float32))
        for ep, p in zip(er["pulses"], s.pulses):
            assert p.map.tolist() == ep["map"]
            assert (p.send_rank, p.recv_rank, p.send_size, p.recv_size, p.atom_offset, p.remote_offset) == \
                (ep["send_rank"], ep["recv_rank"], ep["send_size"], ep["recv_size"], ep["atom_offset"], ep["remote_offset"])
            assert p.shift == ep["shift"] and sorted(p.dep) == ep["dep"]
    F = [np.array(f, np.float32) for f in g["expect"]["F_before"]]
    Fo, fs = force_halo(st, F)
    for r, s in enumerate(st):
        np.testing.assert_array_equal(Fo[r][:s.n_home], np.array(g["expect"]["F_after_home"][r], np.float32))
        np.testing.assert_array_equal(fs[r], np.array(g["expect"]["fshift"][r]))
    vir = sum(float((s.x[:, 2].astype(np.float64) * F[r][:, 0]).sum()) for r, s in enumerate(st))
    assert vir == g["expect"]["virial_zx_total"]


def test_w2_golden_dependency_witness():
    g = load("W2.json")
    st = run(g, np.array(g["X"], np.float32))
    e = g["expect"]
    r0 = st[0]
    assert r0.n_home == e["rank0"]["n_home"]
    assert [p.map.tolist() for p in r0.pulses] == e["rank0"]["maps"]
    assert sorted(r0.pulses[2].dep) == e["rank0"]["dep_x0"]  # x0 waits on z0, not (only) y0
    assert r0.gid[0] == e["rank0"]["row0_gid"]
    for key, rr in (("rank4", 4), ("rank5", 5)):
        s = st[rr]
        np.testing.assert_array_equal(s.x, np.array(e[key]["rows"], np.float32))
        assert s.s.tolist() == e[key]["s"]
        assert st[e[key]["x0_recv_from"]].pulses[2].send_rank == rr


def test_w3_golden_two_pulses():
    g = load("W3.json")
    X = np.array(g["X"], np.float32)
    st = run(g, X)
    e = g["expect"]
    for r, s in enumerate(st):
        assert [p.map.tolist() for p in s.pulses] == e["maps"][r]
        assert [[p.atom_offset, p.recv_size] for p in s.pulses] == e["offsets"][r]
        assert s.gid.tolist() == e["gids"][r]
        assert s.s[:, 2].tolist() == e["s_z"][r]
    assert [p.shift for p in st[0].pulses] == e["shift_applied_by_rank0"]
    F = [np.zeros((s.x.shape[0], 3), np.float32) for s in st]
    for r, row, v in e["forces_nonzero"]:
        F[r][row] = v
    Fo, fs = force_halo(st, F)
    home = {}
    for r, s in enumerate(st):
        for i in range(s.n_home):
            home["abcd"[s.gid[i]]] = Fo[r][i].tolist()
    assert home == {k: [float(x) for x in v] for k, v in e["home_after"].items()}
    assert fs[0][2].tolist() == e["fshift_rank0_z"]


# ---------------------------------------------------------------- generic pins
SMALL = ["C1", "T3D", "T2P", "T2D", "T4x2"]


def system(name, seed):
    c = get_config(name)
    X = water_box(c.n_atoms, c.L, seed)
    return c, X


def as_dict(c):
    return dict(L=c.L, grid=c.grid, pulses=c.pulses, rc=c.rc)


@pytest.mark.parametrize("name", SMALL)
def test_x0_home_cell_exact_rationals(name):
    """X0 pinned without the oracle's plane formula: the home cell of every atom is
    floor(x * grid / L) in exact rational arithmetic (fractions.Fraction of the float32
    values).  Where an atom lies within 1e-12 * L of a plane (the only place where the
    double-precision planes of R3 can round differently) the oracle must put it in a
    neighbouring cell, the higher one if it is exactly on the double plane (R4)."""
    from fractions import Fraction
    c, X = system(name, 1)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses)
    home = {}
    for s in st:
        for g in s.gid[: s.n_home]:
            home[int(g)] = pins.rank_cell(s.rank, c.grid)
    assert len(home) == X.shape[0]
    for g in range(X.shape[0]):
        for d in range(3):
            if c.grid[d] == 1:
                continue
            L = Fraction(float(np.float32(c.L[d])))
            x = Fraction(float(X[g, d]))
            q = x * c.grid[d] / L
            exact = int(q)  # x >= 0: floor
            near = abs(q - round(q)) * L / c.grid[d] < Fraction(1, 10 ** 12) * L
            if near:
                assert home[g][d] in (exact - 1, exact, min(exact, c.grid[d] - 1)), (g, d)
            else:
                assert home[g][d] == min(exact, c.grid[d] - 1), (g, d, float(q))


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("seed", [1, 2])
def test_x0_x1_x4_structure_and_closed_form(name, seed):
    c, X = system(name, seed)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses)
    b = planes(c.L, c.grid)
    L32 = np.array(c.L, np.float32)
    P = len(pulse_list(c.grid, c.pulses))
    assert P == sum(c.pulses)  # X4 pulse count
    seen = np.zeros(X.shape[0], int)
    for s in st:
        # X0: home rows lie in the rank's cell (planes recomputed independently)
        lo, hi = pins.cell_bounds(c.L, c.grid, pins.rank_cell(s.rank, c.grid))
        for d in range(3):
            xd = X[s.gid[:s.n_home], d].astype(np.float64)
            assert np.all(xd >= lo[d]) and (np.all(xd < hi[d]) or c.grid[d] == 1)
        seen[s.gid[:s.n_home]] += 1
        assert np.all(np.diff(s.gid[:s.n_home]) > 0)  # ascending gid
        # X1: every row equals fl32(X[gid] + s*L), one float32 add per shifted component
        exp = X[s.gid].copy()
        for d in range(3):
            m = s.s[:, d] == 1
            exp[m, d] = (exp[m, d] + L32[d]).astype(np.float32)
        np.testing.assert_array_equal(s.x[:, :3], exp)
        # X4: maps ascending, home entries first, disjoint contiguous tiling
        off = s.n_home
        for p, pi in enumerate(s.pulses):
            assert np.all(np.diff(pi.map) > 0)
            assert pi.atom_offset == off
            off += pi.recv_size
            peer = st[pi.send_rank].pulses[p]
            assert st[pi.recv_rank].pulses[p].send_size == pi.recv_size
            assert peer.recv_size == pi.send_size and peer.atom_offset == pi.remote_offset
            if pi.k > 0:  # a k>0 pulse has only dependent entries (X5)
                assert np.all(pi.map >= s.n_home)
            if p == 0:
                assert not pi.dep and np.all(pi.map < s.n_home)  # first pulse never waits
        assert off == s.x.shape[0]
    assert np.all(seen == 1)  # every atom home exactly once


@pytest.mark.parametrize("name", SMALL)
def test_x2_import_zone_brute_force(name):
    c, X = system(name, 3)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses)
    for s in st:
        inner, outer = pins.direct_gather(X, c.L, c.rc, c.grid, s.rank, eps=1e-5)
        have = [(int(g), tuple(int(v) for v in sv)) for g, sv in zip(s.gid, s.s)]
        assert len(have) == len(set(have)), "duplicate image on a rank"
        hs = set(have)
        assert inner <= hs, f"rank {s.rank}: missing {sorted(inner - hs)[:5]}"
        assert hs <= outer, f"rank {s.rank}: extra {sorted(hs - outer)[:5]}"


@pytest.mark.parametrize("name", ["C1", "T3D", "T2P", "T2D"])
def test_x3_pair_coverage_brute_force(name):
    c, X = system(name, 4)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses)
    dec = [d for d in range(3) if c.grid[d] > 1]
    index = []
    for s in st:
        m = {}
        for g, sv in zip(s.gid, s.s):
            m.setdefault(int(g), set()).add(tuple(int(v) for v in sv))
        index.append(m)
    pairs = pins.close_pairs(X, c.L, c.rc, eps=1e-5)
    assert len(pairs) > 1000
    for i, j, n in pairs:
        ok = False
        for m in index:
            si, sj = m.get(i), m.get(j)
            if not si or not sj:
                continue
            for a in si:
                for bb in sj:
                    if all(bb[d] - a[d] == n[d] for d in dec):
                        ok = True
                        break
                if ok:
                    break
            if ok:
                break
        assert ok, f"pair {i},{j} shift {n} not co-resident"


def test_x4_distinct_sources_q10():
    # 2x2x2 with 1 pulse each: 3 steps reach 7 ranks (P:147 read as R10)
    c, X = system("T3D", 5)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses)
    homes = {}
    for s in st:
        for g in s.gid[:s.n_home]:
            homes[int(g)] = s.rank
    for s in st:
        src = {homes[int(g)] for g in s.gid[s.n_home:]}
        assert len(src) == 7 and s.rank not in src


def test_x5_special_cases():
    X = water_box(300, (2.2, 2.2, 2.2), 1)
    st = decompose(X, (2.2, 2.2, 2.2), 1.0, (1, 1, 1), (0, 0, 0))
    assert len(st) == 1 and st[0].pulses == [] and st[0].n_home == 300
    F = [forces_int(300, 1)]
    Fo, fs = force_halo(st, F)
    np.testing.assert_array_equal(Fo[0], F[0])
    assert not fs[0].any()
    # grid[d]=2: lower and upper neighbour coincide
    c, X = system("C1", 1)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses)
    assert st[0].pulses[0].send_rank == st[0].pulses[0].recv_rank == 1
    # empty rank: W2 rank 0 has no home atoms yet forwards; all-empty system
    st = decompose(np.zeros((0, 3), np.float32), (4, 4, 4), 1.0, (2, 2, 2), (1, 1, 1))
    assert all(s.x.shape[0] == 0 for s in st)
    for bad in [((1, 1, 2), (0, 0, 0)), ((1, 1, 2), (0, 0, 2)), ((1, 1, 1), (0, 0, 1))]:
        with pytest.raises(ValueError):
            check_geometry((4, 4, 4), 1.0, *bad)
    with pytest.raises(ValueError):  # not enough pulses: w = 0.8 < rc
        check_geometry((4, 4, 4), 1.0, (1, 1, 5), (0, 0, 1))
    with pytest.raises(ValueError):  # rc >= L/2
        check_geometry((4, 4, 1.8), 1.0, (1, 1, 2), (0, 0, 1))


def test_planes_and_home_cell_tie():
    b = planes((4, 4, 4), (1, 1, 2))
    assert b[2] == [0.0, 2.0, 4.0]
    assert home_cell(np.array([0.25, 2.0, 2.0], np.float32), b, (1, 1, 2)) == (0, 0, 1)  # tie -> higher
    assert rank_of((1, 0, 1), (2, 2, 2)) == 5


@pytest.mark.parametrize("name", SMALL + ["C5"])
@pytest.mark.parametrize("seed", [1, 2])
def test_f1_f2_f3_integer_forces(name, seed):
    c, X = system(name, seed)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses)
    F = [forces_int(s.x.shape[0], 100 * seed + s.rank) for s in st]
    Fo, fs = force_halo(st, F)
    # F1: per-atom totals = sum over every image (brute force, exact)
    tot = pins.scatter_totals([s.gid for s in st], F, X.shape[0])
    got = np.zeros((X.shape[0], 3))
    for s, f in zip(st, Fo):
        got[s.gid[:s.n_home]] = f[:s.n_home]
    np.testing.assert_array_equal(got, tot)
    # F2: conservation
    before = sum(f.astype(np.float64).sum(axis=0) for f in F)
    after = sum(f[:s.n_home].astype(np.float64).sum(axis=0) for s, f in zip(st, Fo))
    np.testing.assert_array_equal(before, after)
    # F3: sum_r fshift_r[d] = sum of F_before over rows with s_d = 1
    fs_tot = sum(fs)
    for d in range(3):
        exp = sum(f[s.s[:, d] == 1].astype(np.float64).sum(axis=0) for s, f in zip(st, F))
        np.testing.assert_array_equal(fs_tot[d], exp)
    # halo rows keep their (possibly accumulated) values: never zeroed, home rows exact


@pytest.mark.parametrize("name", ["T3D", "T2P", "W1"])
def test_f4_virial_identity_dyadic(name):
    if name == "W1":
        g = load("W1.json")
        L, rc, grid, pulses = tuple(g["L"]), g["rc"], tuple(g["grid"]), tuple(g["pulses"])
        X = np.array(g["X"], np.float32)
    else:
        c = get_config(name)
        L = tuple(float(np.round(v * 64) / 64) for v in c.L)
        rc, grid, pulses = c.rc, c.grid, c.pulses
        X = (np.round(water_box(c.n_atoms, c.L, 7).astype(np.float64) * 64) / 64)
        X = np.mod(X, np.array(L)).astype(np.float32)  # dyadic, in [0, L)
    st = decompose(X, L, rc, grid, pulses)
    F = [forces_int(s.x.shape[0], 11 + s.rank) for s in st]
    Fo, fs = force_halo(st, F)
    lhs = sum(s.x[:, :3].astype(np.float64).T @ f.astype(np.float64) for s, f in zip(st, F))
    rhs = sum(s.x[:s.n_home, :3].astype(np.float64).T @ f[:s.n_home].astype(np.float64) for s, f in zip(st, Fo))
    for s, f3 in zip(st, fs):
        for d in range(3):
            rhs[d, :] += float(np.float32(L[d])) * f3[d]
    np.testing.assert_array_equal(lhs, rhs)


@pytest.mark.parametrize("name", ["T3D", "T2P", "C1"])
def test_f5_real_forces_within_rounding_bound(name):
    c, X = system(name, 2)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses)
    F = [forces_normal(s.x.shape[0], 40 + s.rank) for s in st]
    Fo, fs = force_halo(st, F)
    exact = pins.scatter_totals([s.gid for s in st], F, X.shape[0])
    absum = pins.scatter_totals([s.gid for s in st], [np.abs(f) for f in F], X.shape[0])
    nimg = np.bincount(np.concatenate([s.gid for s in st]), minlength=X.shape[0])
    u = 2.0 ** -24
    for s, f in zip(st, Fo):
        g = s.gid[:s.n_home]
        err = np.abs(f[:s.n_home].astype(np.float64) - exact[g])
        bound = (nimg[g][:, None] - 1) * u * absum[g] * 1.0000001
        assert np.all(err <= bound)
    # F3 with real forces: the wrapping slices carry float32-accumulated forwarded
    # forces, so sum_r fshift_r[d] equals the exact image sum up to <= P float32
    # roundings per image (P = pulse count)
    tot = sum(fs)
    P = len(st[0].pulses)
    for d in range(3):
        rows = [f[s.s[:, d] == 1, :3] for s, f in zip(st, F)]
        for comp in range(3):
            vals = np.concatenate([r[:, comp] for r in rows]).astype(np.float64)
            exp = math.fsum(vals.tolist())
            assert abs(tot[d, comp] - exp) <= P * u * (np.abs(vals).sum() + 1e-300)


def test_accumulate_false_single_pulse_overwrites():
    g = load("W1.json")
    st = run(g, np.array(g["X"], np.float32))
    F = [np.array(f, np.float32) for f in g["expect"]["F_before"]]
    Fo, _ = force_halo(st, F, accumulate=False)
    np.testing.assert_array_equal(Fo[0][0], F[1][3])  # g0 <- its image's force verbatim
    np.testing.assert_array_equal(Fo[1][0], F[0][2])
    c, X = system("T3D", 1)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses)
    with pytest.raises(ValueError):
        force_halo(st, [np.zeros((s.x.shape[0], 3), np.float32) for s in st], accumulate=False)


def test_float4_w_copied_unshifted():
    c, X = system("T3D", 1)
    W = np.arange(X.shape[0], dtype=np.float32) * np.float32(0.25) - np.float32(3.0)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses, W=W)
    for s in st:
        np.testing.assert_array_equal(s.x[:, 3], W[s.gid])


@pytest.mark.parametrize("name", ["T3D", "T2P", "C2", "T4x2"])
def test_coord_halo_step_fixed_maps(name):
    """Per-step x halo with fixed maps: reproduces the NS-step halo, and for moved
    home coordinates every halo row equals fl32(X'[gid] + s*L) (closed form X1)."""
    from oracle import coord_halo_step
    c, X = system(name, 3)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses)
    xs = coord_halo_step(st, [s.x[: s.n_home] for s in st])
    for s, x in zip(st, xs):
        np.testing.assert_array_equal(x, s.x)
    rng = np.random.default_rng(9)
    Xm = (X + rng.uniform(-0.02, 0.02, size=X.shape).astype(np.float32)).astype(np.float32)
    xs = coord_halo_step(st, [Xm[s.gid[: s.n_home]] for s in st])
    L32 = np.array(c.L, np.float32)
    for s, x in zip(st, xs):
        exp = Xm[s.gid].copy()
        for d in range(3):
            m = s.s[:, d] == 1
            exp[m, d] = (exp[m, d] + L32[d]).astype(np.float32)
        np.testing.assert_array_equal(x, exp)


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_geometries_pinned(seed):
    """The oracle on random geometries (tests/fuzz_cases.py: 1-4 cells per dim, 1-2
    pulses, uniform or clustered atoms, empty ranks): X1 closed form, X2 import
    zone by brute force, F1 per-atom totals, F2 conservation, F3 shift forces."""
    from tests.fuzz_cases import random_case
    L, rc, grid, pulses, X, _ = random_case(seed)
    st = decompose(X, L, rc, grid, pulses)
    L32 = np.array(L, np.float32)
    for s in st:
        exp = X[s.gid].copy()
        for d in range(3):
            m = s.s[:, d] == 1
            exp[m, d] = (exp[m, d] + L32[d]).astype(np.float32)
        np.testing.assert_array_equal(s.x[:, :3], exp)
        inner, outer = pins.direct_gather(X, L, rc, grid, s.rank, eps=1e-5)
        have = [(int(g), tuple(int(v) for v in sv)) for g, sv in zip(s.gid, s.s)]
        assert len(have) == len(set(have))
        assert inner <= set(have) <= outer
    F = [forces_int(s.x.shape[0], 7 * seed + s.rank) for s in st]
    Fo, fs = force_halo(st, F)
    tot = pins.scatter_totals([s.gid for s in st], F, X.shape[0])
    got = np.zeros((X.shape[0], 3))
    for s, f in zip(st, Fo):
        got[s.gid[:s.n_home]] = f[:s.n_home]
    np.testing.assert_array_equal(got, tot)
    fs_tot = sum(fs) if fs else np.zeros((3, 3))
    for d in range(3):
        exp = sum(f[s.s[:, d] == 1].astype(np.float64).sum(axis=0) for s, f in zip(st, F))
        np.testing.assert_array_equal(fs_tot[d], exp)


# ---------------------------------------------------------------- fshift tolerance
@pytest.mark.parametrize("name", ["T3D", "T2P", "W3"])
def test_fshift_abs_closed_form_nonnegative_forces(name):
    """sum|terms| (the fp64 tolerance basis) with every force >= 0 equals fshift itself
    (no cancellation), and in general |fshift| <= sum|terms| (triangle inequality)."""
    if name == "W3":
        g = load("W3.json")
        L, rc, grid, pulses = tuple(g["L"]), g["rc"], tuple(g["grid"]), tuple(g["pulses"])
        st = decompose(np.array(g["X"], np.float32), L, rc, grid, pulses)
    else:
        c, X = system(name, 3)
        st = decompose(X, c.L, c.rc, c.grid, c.pulses)
    F = [np.abs(forces_int(s.x.shape[0], 5 + s.rank)).astype(np.float32) for s in st]
    _, fs, fa = force_halo(st, F, with_abs=True)
    for a, b in zip(fs, fa):
        np.testing.assert_array_equal(a, b)
    Fn = [forces_normal(s.x.shape[0], 9 + s.rank) for s in st]
    _, fs, fa = force_halo(st, Fn, with_abs=True)
    for a, b in zip(fs, fa):
        assert np.all(np.abs(a) <= b)


@pytest.mark.parametrize("name", ["T3D", "T2P", "C1"])
def test_fshift_tolerance_rejects_fp32(name):
    """The parity bound for fshift (1e-12 * sum|terms| per rank, dim, component) must
    tell an fp64 reduction from an fp32 one: re-summing the oracle's own terms in fp64
    in another order (blocked + pairwise, as a GPU reduction does) passes; the same
    terms accumulated in fp32 (sequential and pairwise) fail for every case."""
    from tests.parity_common import fshift_violation
    c, X = system(name, 2)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses)
    F = [forces_normal(s.x.shape[0], 40 + s.rank) for s in st]
    terms = []
    _, fs, fa = force_halo(st, F, with_abs=True, terms_out=terms)

    def pairwise(v, dt):
        v = v.astype(dt)
        while v.size > 1:
            if v.size % 2:
                v = np.append(v, dt(0))
            v = (v[0::2] + v[1::2]).astype(dt)
        return dt(v[0]) if v.size else dt(0)

    worst64, worst32s, worst32p = 0.0, [], []
    for q in range(len(st)):
        g64 = np.zeros((3, 3))
        g32s = np.zeros((3, 3))
        g32p = np.zeros((3, 3))
        for d in range(3):
            for comp in range(3):
                t = terms[q][d][comp]
                if t.size == 0:
                    continue
                blocks = [pairwise(t[i:i + 64], np.float64) for i in range(0, t.size, 64)]
                g64[d, comp] = sum(blocks)
                acc = np.float32(0)
                for v in t.astype(np.float32):
                    acc = np.float32(acc + v)
                g32s[d, comp] = acc
                g32p[d, comp] = pairwise(t, np.float32)
        if np.any(fa[q] > 0):
            worst64 = max(worst64, fshift_violation(g64, fs[q], fa[q]))
            worst32s.append(fshift_violation(g32s, fs[q], fa[q]))
            worst32p.append(fshift_violation(g32p, fs[q], fa[q]))
    assert worst64 <= 1.0
    assert worst32s and min(worst32s) > 10.0, worst32s
    assert min(worst32p) > 10.0, worst32p
