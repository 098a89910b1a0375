"""CPU ORACLE for the eighth-shell DD halo exchange — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this module.  The product path
(``paper_2509_21527_b200``, ``libhalo.so``) never imports, links or calls it;
the two share no code (only the seeded input generators in ``synth/``).

What it computes (PAPER.md = P:<line>; readings R<n> are listed in DESIGN.md):

* decomposition: planes b_d[k] = float64(L_d) * k / grid[d]; home cell c_d =
  largest k with b_d[k] <= float64(x_d) (R4: ties go to the higher cell);
  rank = (cx*np_y + cy)*np_z + cz (R5).  P:139-141 "divides the simulation box
  into spatial regions (domains)".
* pulse list: z, then y, then x, skipping undecomposed dims; pulses k = 0..p_d-1
  within a dim ("first np(z) pulses in the z-direction, then np(y) ..."
  and P:320 "[z0, y0, x0]").
* coordinate halo (staged forwarding, "boundary data is forwarded through
  intermediate ranks"; Alg. 3; Alg. 4): for each pulse in
  global order, every rank selects, among its candidate rows, those with
  float64(x_d) - b_d[c_d] < float64(rc) (R2/R3, slab criterion, strict), in
  ascending local row order (R11); sends them to the lower neighbour (R1); the
  sender at c_d = 0 adds +L_d e_d as a float32 add of the full 3-vector (R25);
  the receiver appends them contiguously after home rows, pulses in global order
  (R12; "remoteCoordDst + atomOffset").  Candidates: for k = 0 every row
  present before the first pulse of dim d; for k > 0 the rows received in pulse
  (d, k-1).
* force halo (Alg. 6, "begins with the last pulse's computed forces ...
  and works backwards through the dependency chain" P:412): pulses descending;
  the x-receiver's halo slice of pulse p (read after all pulses > p were applied)
  is added into the x-sender's rows map_p[i], one float32 RNE add per (entry,
  pulse), entries ascending (R15).  Shift forces (R13, paper silent; north_star
  requirement): fshift[d] of the rank that applied +L_d receives the exact sum of
  the received forces of its wrapping pulses, rounded once to float64
  (``math.fsum``).

Plain numpy; loops over pulses and ranks in the paper's order; no blocking,
fusion or reordering.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

DIM_ORDER = (2, 1, 0)  # z, y, x


def planes(L, grid):
    """b[d][k] = float64(L_d) * k / grid[d], k = 0..grid[d] (R3: multiply then divide)."""
    out = []
    for d in range(3):
        Ld = float(np.float32(L[d]))
        out.append([Ld * k / grid[d] for k in range(grid[d] + 1)])
    return out


def home_cell(x3, b, grid):
    """c_d = the largest k in [0, grid[d]-1] with b_d[k] <= float64(x_d) (R4)."""
    c = []
    for d in range(3):
        xd = float(x3[d])
        k = 0
        for kk in range(grid[d]):
            if b[d][kk] <= xd:
                k = kk
        c.append(k)
    return tuple(c)


def rank_of(c, grid):
    """rank = (cx*np_y + cy)*np_z + cz (R5)."""
    return (c[0] * grid[1] + c[1]) * grid[2] + c[2]


def cell_of(r, grid):
    cz = r % grid[2]
    cy = (r // grid[2]) % grid[1]
    cx = r // (grid[1] * grid[2])
    return (cx, cy, cz)


def pulse_list(grid, pulses):
    """Global pulse order [(d, k)], z -> y -> x, undecomposed dims omitted."""
    out = []
    for d in DIM_ORDER:
        if grid[d] > 1:
            for k in range(pulses[d]):
                out.append((d, k))
    return out


def check_geometry(L, rc, grid, pulses):
    """Geometry validity; raises ValueError."""
    for d in range(3):
        if grid[d] < 1:
            raise ValueError("grid[d] must be >= 1")
        if (grid[d] > 1) != (pulses[d] >= 1):
            raise ValueError("pulses[d] >= 1 iff grid[d] > 1")
        if pulses[d] > max(grid[d] - 1, 0):
            raise ValueError("pulses[d] must be <= grid[d]-1")
        if grid[d] > 1 and pulses[d] * (float(np.float32(L[d])) / grid[d]) < float(np.float32(rc)):
            raise ValueError("not enough pulses: pulses[d]*L_d/grid[d] < rc")
    if not (0.0 < float(np.float32(rc)) < min(float(np.float32(v)) for v in L) / 2.0):
        raise ValueError("need 0 < rc < min(L)/2")


@dataclass
class PulseInfo:
    dim: int
    k: int
    send_rank: int = -1       # rank this rank sends coordinates to (lower neighbour)
    recv_rank: int = -1       # rank this rank receives coordinates from (upper neighbour)
    send_size: int = 0
    recv_size: int = 0
    atom_offset: int = 0      # where this pulse's received rows start locally
    remote_offset: int = 0    # where this rank's sent rows land on send_rank
    shift: bool = False       # this rank applied +L_dim when sending
    map: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    dep: frozenset = frozenset()  # earlier pulses whose receive ranges map touches (R9)
    shift_vec: np.ndarray = field(default_factory=lambda: np.zeros(3, np.float32))  # +L_dim e_dim if shift


@dataclass
class RankState:
    rank: int
    cell: tuple
    n_home: int
    x: np.ndarray            # [n_rows, width] float32
    gid: np.ndarray          # [n_rows] int64
    s: np.ndarray            # [n_rows, 3] int64 shift vector (0/1 per dim)
    pulses: list


def decompose(X, L, rc, grid, pulses, W=None, rounded=False):
    """Home assignment + coordinate halo (maps built on the way), serial.

    X: [N, 3] float32 global positions in [0, L).  W: optional [N] float32 w
    component (float4 layout; copied, never shifted, R25).
    rounded: GROMACS-style rounded zones (R31, SURVEY §8(f) f2 variant): a
    candidate that passes the slab test and lies beyond this rank's upper face
    in some other dim d' is sent only if its squared distance to the RECEIVER's
    cell, dd^2 + sum_{d' != d} max(0, x_d' - b_d'[c_d'+1])^2 (float64, dims
    ascending), is < rc^2 (the eighth-shell zone with rounded edges/corners,
    Hess2008 via P:143).
    Returns the list of RankState, one per rank.
    """
    check_geometry(L, rc, grid, pulses)
    X = np.asarray(X, dtype=np.float32)
    width = 3 if W is None else 4
    nr = grid[0] * grid[1] * grid[2]
    b = planes(L, grid)
    rc64 = float(np.float32(rc))
    L32 = np.asarray(L, dtype=np.float32)

    # 1. home assignment (ascending gid per rank)
    # c_d = number of interior planes b_d[1..grid-1] that are <= float64(x_d)
    # (= the largest k with b_d[k] <= x_d, the rule of home_cell)
    cidx = np.zeros((X.shape[0], 3), dtype=np.int64)
    for d in range(3):
        inner = np.asarray(b[d][1:grid[d]], dtype=np.float64)
        cidx[:, d] = np.searchsorted(inner, X[:, d].astype(np.float64), side="right")
    ranks_of_atom = (cidx[:, 0] * grid[1] + cidx[:, 1]) * grid[2] + cidx[:, 2]
    states = []
    for r in range(nr):
        ids = np.nonzero(ranks_of_atom == r)[0].astype(np.int64)
        x = np.zeros((ids.size, width), dtype=np.float32)
        x[:, :3] = X[ids]
        if W is not None:
            x[:, 3] = np.asarray(W, dtype=np.float32)[ids]
        states.append(RankState(r, cell_of(r, grid), int(ids.size), x, ids.copy(),
                                np.zeros((ids.size, 3), dtype=np.int64), []))

    # 2./3. pulses in global order; every rank reads only pre-pulse state
    plist = pulse_list(grid, pulses)
    dim_start = {}
    for p, (d, k) in enumerate(plist):
        if k == 0:
            for st in states:
                dim_start[st.rank] = st.x.shape[0]
        sends = []
        for st in states:
            c = st.cell
            if k == 0:
                cand = np.arange(dim_start[st.rank], dtype=np.int64)
            else:
                prev = st.pulses[p - 1]
                cand = np.arange(prev.atom_offset, prev.atom_offset + prev.recv_size, dtype=np.int64)
            # selection: float64(x_d) - b_d[c_d] < float64(rc), strict (R2, R3)
            dd = st.x[cand, d].astype(np.float64) - b[d][c[d]]
            sel = dd < rc64
            if rounded:  # R31: distance to the receiver's cell box
                r2 = dd * dd
                beyond = np.zeros(cand.size, dtype=bool)
                for d2 in range(3):
                    if d2 == d:
                        continue
                    t = st.x[cand, d2].astype(np.float64) - b[d2][c[d2] + 1]
                    pos = t > 0.0
                    r2 = np.where(pos, r2 + t * t, r2)
                    beyond |= pos
                sel &= ~beyond | (r2 < rc64 * rc64)
            mp = cand[sel].astype(np.int32)  # ascending local row order (R11)
            lower = list(c)
            lower[d] = (c[d] - 1) % grid[d]
            upper = list(c)
            upper[d] = (c[d] + 1) % grid[d]
            shift = c[d] == 0
            payload = st.x[mp].copy()
            if shift:
                sv = np.zeros(3, dtype=np.float32)
                sv[d] = L32[d]
                payload[:, :3] = payload[:, :3] + sv  # float32 add of the full 3-vector (R25)
            # dep set: earlier pulses whose receive ranges contain entries of the map (R9)
            dep = set()
            for q in range(p):
                pq = st.pulses[q]
                if pq.recv_size and np.any((mp >= pq.atom_offset) & (mp < pq.atom_offset + pq.recv_size)):
                    dep.add(q)
            info = PulseInfo(dim=d, k=k, send_rank=rank_of(lower, grid), recv_rank=rank_of(upper, grid),
                             send_size=int(mp.size), shift=bool(shift), map=mp, dep=frozenset(dep))
            if shift:
                info.shift_vec = sv.copy()
            st.pulses.append(info)
            sends.append((info.send_rank, payload, st.gid[mp].copy(), st.s[mp].copy(), shift, st.rank))
        # receivers append (receiver = sender's lower neighbour)
        for (dst, payload, g, s, shift, src) in sends:
            rs = states[dst]
            info = rs.pulses[p]
            info.atom_offset = rs.x.shape[0]
            info.recv_size = payload.shape[0]
            states[src].pulses[p].remote_offset = info.atom_offset
            if shift:
                s = s.copy()
                s[:, d] += 1
            rs.x = np.concatenate([rs.x, payload], axis=0)
            rs.gid = np.concatenate([rs.gid, g])
            rs.s = np.concatenate([rs.s, s], axis=0)
    return states


def wrap_coord(x, L):
    """R29 (paper silent; GROMACS puts atoms back in the box at NS steps): ONE
    periodic wrap in float32 — x >= L -> fl32(x - L); x < 0 -> fl32(x + L) — then
    a result equal to L (a tiny negative x) or to zero (incl. -0.0) becomes +0.0.
    Returns (wrapped float32, ok) with ok = 0 <= wrapped < L (else the atom moved
    more than a box length)."""
    L = np.float32(L)
    x = np.float32(x)
    if x >= L:
        x = np.float32(x - L)
    elif x < np.float32(0.0):
        x = np.float32(x + L)
    if x == L or x == np.float32(0.0):
        x = np.float32(0.0)
    return x, bool(np.float32(0.0) <= x < L)


def migrate(homes, L, grid):
    """NS-step home-atom redistribution: the domains own the
    atoms inside their region, re-established at every
    neighbour-search step.  Plain definition, atom by atom:

    homes[r] = (gid [n] int, x [n, W] float32, v [n, W] float32 or None): rank r's
    home rows before the step (positions possibly moved out of the cell/box).
    Every row is wrapped (``wrap_coord`` per component; a float4 w is copied),
    assigned to the rank of its cell (``home_cell``, R3/R4) and collected there;
    each rank's new rows are sorted by gid.  R30: an atom may move at most one
    cell per dimension (periodically) from its old rank's cell; else ValueError.
    Returns the new homes in the same form."""
    b = planes(L, grid)
    nr = grid[0] * grid[1] * grid[2]
    got = [[] for _ in range(nr)]
    for r, (gid, x, v) in enumerate(homes):
        c_old = cell_of(r, grid)
        for i in range(len(gid)):
            row = np.array(x[i], dtype=np.float32).copy()
            for d in range(3):
                row[d], ok = wrap_coord(row[d], L[d])
                if not ok:
                    raise ValueError(f"atom {gid[i]} moved more than a box length")
            c_new = home_cell(row[:3], b, grid)
            for d in range(3):
                if (c_new[d] - c_old[d]) % grid[d] not in (0, 1 % grid[d], (grid[d] - 1) % grid[d]):
                    raise ValueError(f"atom {gid[i]} moved more than one cell in dim {d} (R30)")
            got[rank_of(c_new, grid)].append((int(gid[i]), row, None if v is None else np.asarray(v[i], np.float32)))
    out = []
    for r in range(nr):
        rows = sorted(got[r], key=lambda t: t[0])
        W = homes[0][1].shape[1]
        g = np.array([t[0] for t in rows], dtype=np.int64)
        x = np.array([t[1] for t in rows], dtype=np.float32).reshape(-1, W)
        v = None
        if homes[0][2] is not None:
            v = np.array([t[2] for t in rows], dtype=np.float32).reshape(-1, W)
        out.append((g, x, v))
    return out


def pme_gather(homes_x):
    """PP -> PME coordinate redistribution ("the
    communication of coordinates and forces to and from the PME tasks"): the PME
    task receives the home rows of every DD rank, concatenated in rank order.
    homes_x[r]: [n_r, W] float32.  Returns (pme_x [sum n_r, W], row_off [nranks+1])."""
    off = [0]
    for h in homes_x:
        off.append(off[-1] + h.shape[0])
    return np.concatenate(homes_x, axis=0).astype(np.float32), off


def pme_return(f_home, pme_f, row_off, accumulate=True):
    """PME -> PP force redistribution: rank r's home forces += its slice of pme_f
    (rows [row_off[r], row_off[r+1])), one float32 RNE add per component
    (accumulate=False: overwrite).  f_home[r]: [n_r, W] float32; returns new arrays."""
    out = []
    for r, f in enumerate(f_home):
        sl = np.asarray(pme_f[row_off[r]: row_off[r + 1]], dtype=np.float32)
        out.append((np.asarray(f, np.float32) + sl).astype(np.float32) if accumulate else sl.copy())
    return out


def coord_halo_step(states, x_home):
    """Per-step coordinate halo with the maps of the last neighbour-search step
    fixed (Alg. 3 P:252-262 with Alg. 4's forwarding, run serially pulse by
    pulse): returns new per-rank x arrays whose rows [0, n_home) are x_home[r]
    and whose halo rows are re-gathered through the stored maps, shifted by
    +L_d (float32 add of the full 3-vector, R25) on wrapping sends.

    x_home: list of [n_home_r, width] float32 arrays.  The box lengths are taken
    from the shift the rank recorded: states carry them in ``pulse.shift_vec``.
    """
    xs = []
    for st, xh in zip(states, x_home):
        x = np.zeros_like(st.x)
        x[: st.n_home] = xh
        xs.append(x)
    P = len(states[0].pulses) if states else 0
    for p in range(P):
        sends = []
        for st in states:
            pi = st.pulses[p]
            payload = xs[st.rank][pi.map].copy()
            if pi.shift:
                payload[:, :3] = payload[:, :3] + pi.shift_vec
            sends.append((pi.send_rank, st.pulses[p].remote_offset, payload))
        for dst, off, payload in sends:
            xs[dst][off: off + payload.shape[0]] = payload
    return xs


def force_halo(states, F, fshift_in=None, accumulate=True, with_abs=False, terms_out=None):
    """Serial force halo (R15 order): returns (F_after list, fshift list [3][3] float64).
    ``with_abs=True`` also returns, per rank, [3][3] float64 sums of |term| over the
    same shift-force terms (the basis of the fp64 parity tolerance, R13).
    ``terms_out`` (a list): receives, per rank, [dim][component] lists of the
    float64 terms that fshift sums (tests of the tolerance's resolution).

    F: list of [n_rows_r, width] float32 arrays, the forces on every local row
    of every rank before the exchange (as a non-bonded kernel leaves them).
    Halo rows keep their values (they are not zeroed).  ``accumulate=False`` is
    only defined for a single pulse (R14): the received forces overwrite.
    """
    nr = len(states)
    P = len(states[0].pulses) if nr else 0
    if not accumulate and P != 1:
        raise ValueError("accumulate=False is defined only for a single pulse (R14)")
    Fo = [np.array(f, dtype=np.float32, copy=True) for f in F]
    terms = [[[[] for _ in range(3)] for _ in range(3)] for _ in range(nr)]
    for p in range(P - 1, -1, -1):
        # every rank q receives back its pulse-p send from the rank it sent to
        bufs = []
        for q in range(nr):
            info = states[q].pulses[p]
            u = info.send_rank  # the x-receiver of q's pulse p
            ui = states[u].pulses[p]
            buf = Fo[u][ui.atom_offset: ui.atom_offset + ui.recv_size].copy()
            bufs.append(buf)
        for q in range(nr):
            info = states[q].pulses[p]
            buf = bufs[q]
            assert buf.shape[0] == info.send_size
            tgt = info.map.astype(np.int64)
            if accumulate:
                Fo[q][tgt] = Fo[q][tgt] + buf  # one float32 add per (entry, pulse)
            else:
                Fo[q][tgt] = buf
            if info.shift:
                for c in range(3):
                    terms[q][info.dim][c].append(buf[:, c].astype(np.float64))
    fshift, fabs = [], []
    for q in range(nr):
        fs = np.zeros((3, 3), dtype=np.float64) if fshift_in is None else np.array(fshift_in[q], dtype=np.float64)
        fa = np.abs(fs)
        for d in range(3):
            for c in range(3):
                if terms[q][d][c]:
                    vals = np.concatenate(terms[q][d][c]).tolist()
                    fs[d, c] = math.fsum([float(fs[d, c])] + vals)
                    fa[d, c] = math.fsum([float(fa[d, c])] + [abs(v) for v in vals])
        fshift.append(fs)
        fabs.append(fa)
    if terms_out is not None:
        terms_out.extend([[[np.concatenate(t) if t else np.zeros(0) for t in td] for td in tq] for tq in terms])
    if with_abs:
        return Fo, fshift, fabs
    return Fo, fshift


def layout_summary(states):
    """(n_home, n_total, per-pulse (send_size, recv_size, atom_offset, remote_offset))."""
    out = []
    for st in states:
        out.append(dict(n_home=st.n_home, n_total=int(st.x.shape[0]),
                        pulses=[(pi.send_size, pi.recv_size, pi.atom_offset, pi.remote_offset)
                                for pi in st.pulses]))
    return out
