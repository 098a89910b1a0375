"""GPU-vs-oracle parity harness (test-only).  Runs the CUDA path through the C ABI
(via the Python binding) and compares with oracle/ element by element.

Tolerances:
  maps, layout, dep masks, halo x, f (deterministic mode): bit-exact
  f (HALO_F_ATOMIC_UNPACK): per component |g - o| <= P * 2^-24 * sum|terms|  (R16)
  fshift (fp64 reduction, any order): per (rank, dim, component)
      |g - o| <= 1e-12 * sum|terms|, the terms being the float32 forces that
      component sums (oracle ``force_halo(with_abs=True)``); an fp32 accumulation
      misses this by orders of magnitude (test_oracle_pins::test_fshift_tolerance_rejects_fp32)
"""
from __future__ import annotations

import json
import os

import numpy as np
import torch

from oracle import decompose, force_halo
from synth import forces_int, forces_normal, get_config, water_box
from synth.water import charges

GOLD = os.path.join(os.path.dirname(__file__), "golden")

# fp64 shift-force bound: a sum of n fp64-rounded partial sums errs by at most
# (n-1) * 2^-53 * sum|terms| (< 1e-12 * sum|terms| for n < 9000 terms per slot
# chain; the kernels reduce per work item, then per item slot)
FSHIFT_RTOL = 1e-12


def fshift_violation(got, exp, absum, rtol=FSHIFT_RTOL):
    """max over (dim, component) of |got - exp| / (rtol * sum|terms|); <= 1 passes.
    A component with no terms must match exactly (0 / 0 -> 0, x / 0 -> inf)."""
    got = np.asarray(got, np.float64).reshape(3, 3)
    exp = np.asarray(exp, np.float64).reshape(3, 3)
    err = np.abs(got - exp)
    lim = rtol * np.asarray(absum, np.float64).reshape(3, 3)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(err == 0, 0.0, err / lim)
    return float(np.max(r))


def assert_fshift(got, exp, absum, where=""):
    v = fshift_violation(got, exp, absum)
    assert v <= 1.0, (where, v, np.asarray(got).tolist(), np.asarray(exp).tolist())


def load_system(name, seed, layout=3):
    """(L, rc, grid, pulses, X, W) for a config name or a golden W* example."""
    if name.startswith("W"):
        with open(os.path.join(GOLD, name + ".json")) as f:
            g = json.load(f)
        X = np.array(g["X"], np.float32)
        L, rc, grid, pulses = tuple(g["L"]), g["rc"], tuple(g["grid"]), tuple(g["pulses"])
    else:
        c = get_config(name)
        X = water_box(c.n_atoms, c.L, seed)
        L, rc, grid, pulses = c.L, c.rc, c.grid, c.pulses
    W = charges(X.shape[0]) if layout == 4 else None
    return L, rc, grid, pulses, X, W


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.int32)


class Case:
    """Oracle side of one parity case."""

    def __init__(self, name, seed=1, layout=3, force_kind="int", rounded=False):
        self.name, self.seed, self.layout, self.rounded = name, seed, layout, rounded
        self.L, self.rc, self.grid, self.pulses, self.X, self.W = load_system(name, seed, layout)
        self.states = decompose(self.X, self.L, self.rc, self.grid, self.pulses, W=self.W, rounded=rounded)
        self.nranks = len(self.states)
        self.capacity = max(max(s.x.shape[0] for s in self.states), 1) + 64
        mk = forces_int if force_kind == "int" else forces_normal
        self.F = [mk(s.x.shape[0], 1000 * seed + 7 * s.rank + 3, width=layout) for s in self.states]
        self.Fo, self.fshift, self.fshift_abs = force_halo(self.states, [f.copy() for f in self.F], with_abs=True)

    def absum_gid(self):
        if not hasattr(self, "_absum"):
            acc = np.zeros((self.X.shape[0], 3))
            for s, f in zip(self.states, self.F):
                np.add.at(acc, s.gid, np.abs(f[:, :3].astype(np.float64)))
            self._absum = acc
        return self._absum

    def home_rows(self, r):
        s = self.states[r]
        return s.x[: s.n_home]


def run_gpu_case(case: Case, sess, check_forces=True, atomic=False, use_explicit=False, steps=1, barrier=None,
                 fused=False):
    """Drive the CUDA path for the local ranks of `sess` and compare with the oracle.
    fused: each step is one halo_exchange_xf launch (f loaded before it) instead of
    exchange_x, check, exchange_f.  Returns True (asserts on the way)."""
    first, nl = sess.first_rank, sess.n_local
    sess.load_home([case.home_rows(first + l) for l in range(nl)])
    if use_explicit:
        maps = [[case.states[first + l].pulses[p].map for p in range(sess.npulse)] for l in range(nl)]
        sess.set_maps_explicit(maps)
    else:
        sess.set_maps()
    torch.cuda.synchronize()
    for l in range(nl):
        r = first + l
        st = case.states[r]
        lay = sess.layout_of(l)
        assert lay["n_home"] == st.n_home, (r, lay, st.n_home)
        assert lay["n_total"] == st.x.shape[0], (r, lay["n_total"], st.x.shape[0])
        for p, pi in enumerate(st.pulses):
            got = (lay["send_size"][p], lay["recv_size"][p], lay["recv_off"][p], lay["remote_off"][p])
            exp = (pi.send_size, pi.recv_size, pi.atom_offset, pi.remote_offset)
            assert got == exp, (r, p, got, exp)
            assert lay["dep_mask"][p] == sum(1 << q for q in pi.dep), (r, p, lay["dep_mask"][p], pi.dep)
            np.testing.assert_array_equal(sess.halo.get_map(l, p), pi.map)
    for step in range(steps):
        # poison halo rows (sentinel NaN payload): exchange_x must overwrite every one (G3)
        for l in range(nl):
            st = case.states[first + l]
            sess.x[l][st.n_home: st.x.shape[0]] = float("nan")
        if fused:
            for l in range(nl):
                r = first + l
                sess.f[l][: case.F[r].shape[0]] = torch.from_numpy(case.F[r]).to(sess.device)
            fshift = torch.zeros(nl, 3, 3, dtype=torch.float64, device=sess.device)
        if barrier is not None:
            # the poison is written outside the protocol: every process must have
            # poisoned before any peer stores this step's halo (R17)
            torch.cuda.synchronize()
            barrier()
        if fused:
            sess.exchange_xf(fshift=fshift)
        else:
            sess.exchange_x()
        torch.cuda.synchronize()
        for l in range(nl):
            st = case.states[first + l]
            got = sess.x[l][: st.x.shape[0]].cpu().numpy()
            np.testing.assert_array_equal(bits(got), bits(st.x), err_msg=f"halo x rank {first + l} step {step}")
        if not check_forces:
            continue
        if not fused:
            for l in range(nl):
                r = first + l
                n = case.F[r].shape[0]
                sess.f[l][:n] = torch.from_numpy(case.F[r]).to(sess.device)
            fshift = torch.zeros(nl, 3, 3, dtype=torch.float64, device=sess.device)
            sess.exchange_f(fshift=fshift)
            torch.cuda.synchronize()
        fs = fshift.cpu().numpy()
        for l in range(nl):
            r = first + l
            n = case.F[r].shape[0]
            got = sess.f[l][:n].cpu().numpy()
            exp = case.Fo[r]
            if not atomic:
                np.testing.assert_array_equal(bits(got), bits(exp), err_msg=f"f rank {r} step {step}")
            else:
                # unordered adds (R16): home rows within P * 2^-24 * sum|terms| of the ordered result
                st = case.states[r]
                P = max(1, sess.npulse)
                bound = 2 * P * 2.0 ** -24 * case.absum_gid()[st.gid[: st.n_home]] * 1.0000001
                err = np.abs(got[: st.n_home, :3].astype(np.float64) - exp[: st.n_home, :3].astype(np.float64))
                assert np.all(err <= bound), (r, float(err.max()))
            assert_fshift(fs[l], case.fshift[r], case.fshift_abs[r], where=f"fshift rank {r} step {step}")
    return True


def moved_case(case: Case, seed: int):
    """The second NS step of `case`: atoms displaced (synth.displacements), the
    oracle's wrapped positions (R29) and a Case over them.  Returns (Xm, V, case2)."""
    from oracle import wrap_coord
    from synth import displacements, velocities
    # moves stay well inside one cell (R30): thermal sigma and a few diagonal jumps
    cell = min(float(case.L[d]) / case.grid[d] for d in range(3))
    Xm = displacements(case.X, case.L, 100 + seed, sigma=min(0.05, cell / 12), far=min(0.6, cell / 3))
    V = velocities(case.X.shape[0], 200 + seed, width=case.layout)
    Xw = Xm.copy()
    for i in range(Xm.shape[0]):
        for d in range(3):
            Xw[i, d] = wrap_coord(Xm[i, d], case.L[d])[0]
    c2 = Case.__new__(Case)
    c2.__dict__.update(case.__dict__)
    c2.__dict__.pop("_absum", None)
    c2.X = Xw
    c2.states = decompose(Xw, case.L, case.rc, case.grid, case.pulses, W=case.W, rounded=case.rounded)
    c2.capacity = max(max(s.x.shape[0] for s in c2.states), 1) + 64
    c2.F = [forces_int(s.x.shape[0], 77 + s.rank, width=case.layout) for s in c2.states]
    c2.Fo, c2.fshift, c2.fshift_abs = force_halo(c2.states, [f.copy() for f in c2.F], with_abs=True)
    return Xm, V, c2


def run_gpu_migrate(case: Case, c2: Case, Xm, V, sess, with_v=True, barrier=None, steps=2):
    """NS step 1 + one exchange step on `case`; the home rows move to Xm; halo_migrate
    vs oracle.migrate (bit-exact x, gid, payload, counts); then NS step 2 on the
    migrated rows (maps, x halo, force halo vs the oracle of the moved system)."""
    from oracle import migrate
    run_gpu_case(case, sess, barrier=barrier)
    layout, cap = case.layout, sess.capacity
    homes = [None] * case.nranks
    gid_t, v_t = [], []
    for r, st in enumerate(case.states):
        g = st.gid[: st.n_home]
        rows = np.zeros((g.size, layout), np.float32)
        rows[:, :3] = Xm[g]
        if layout == 4:
            rows[:, 3] = case.W[g]
        homes[r] = (g, rows, V[g] if with_v else None)
    for l in range(sess.n_local):
        g, rows, _ = homes[sess.first_rank + l]
        sess.x[l][: g.size] = torch.from_numpy(rows).to(sess.device)
        gt = torch.zeros(cap, dtype=torch.int32, device=sess.device)
        gt[: g.size] = torch.from_numpy(g.astype(np.int32)).to(sess.device)
        gid_t.append(gt)
        vt = torch.zeros(cap, layout, dtype=torch.float32, device=sess.device)
        vt[: g.size] = torch.from_numpy(V[g]).to(sess.device)
        v_t.append(vt)
    torch.cuda.synchronize()
    if barrier is not None:
        barrier()
    n_new = sess.migrate(gid_t, v_t if with_v else None)
    torch.cuda.synchronize()
    exp = migrate(homes, case.L, case.grid)
    for l in range(sess.n_local):
        r = sess.first_rank + l
        g, x, v = exp[r]
        assert n_new[l] == g.size, (r, n_new[l], g.size)
        np.testing.assert_array_equal(gid_t[l][: g.size].cpu().numpy(), g.astype(np.int32))
        np.testing.assert_array_equal(bits(sess.x[l][: g.size].cpu().numpy()), bits(x), err_msg=f"x rank {r}")
        if with_v:
            np.testing.assert_array_equal(bits(v_t[l][: g.size].cpu().numpy()), bits(v), err_msg=f"v rank {r}")
        st2 = c2.states[r]
        np.testing.assert_array_equal(g, st2.gid[: st2.n_home])  # = a fresh decomposition
    run_gpu_case(c2, sess, steps=steps, barrier=barrier)
    return True


def run_gpu_pme(case: Case, sess, steps=3, barrier=None):
    """PP <-> PME redistribution vs oracle.pme_gather / pme_return,
    bit-exact; `sess` was created with pme_rank.  Several steps (sequence numbers,
    acks); the PME forces change every step."""
    from oracle import pme_gather, pme_return
    run_gpu_case(case, sess, check_forces=False, barrier=barrier)
    n_total, off = sess.pme_setup()
    exp_x, exp_off = pme_gather([s.x[: s.n_home] for s in case.states])
    assert n_total == exp_x.shape[0] and list(off) == list(exp_off), (n_total, off[:4], exp_off[:4])
    px, pf = sess.pme_buffers()
    hosts = px is not None
    for step in range(steps):
        F = [forces_int(s.n_home, 300 + 10 * step + s.rank, width=case.layout) for s in case.states]
        PF = forces_int(n_total, 900 + step, width=case.layout)
        for l in range(sess.n_local):
            r = sess.first_rank + l
            sess.f[l][: case.states[r].n_home] = torch.from_numpy(F[r]).to(sess.device)
        if hosts:
            px[:n_total] = float("nan")  # every row must be overwritten
        torch.cuda.synchronize()
        if barrier is not None:
            barrier()
        sess.pme_send_x()
        torch.cuda.synchronize()
        if hosts:
            np.testing.assert_array_equal(bits(px[:n_total].cpu().numpy()), bits(exp_x), err_msg=f"pme_x step {step}")
            pf[:n_total] = torch.from_numpy(PF).to(sess.device)  # the PME task's forces
            torch.cuda.synchronize()
        acc = step != 1
        sess.pme_recv_f(accumulate=acc)
        torch.cuda.synchronize()
        exp_f = pme_return(F, PF, exp_off, accumulate=acc)
        for l in range(sess.n_local):
            r = sess.first_rank + l
            n = case.states[r].n_home
            np.testing.assert_array_equal(bits(sess.f[l][:n].cpu().numpy()), bits(exp_f[r]),
                                          err_msg=f"pme f rank {r} step {step}")
        if barrier is not None:
            barrier()
    return True
