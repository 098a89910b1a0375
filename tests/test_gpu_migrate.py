"""GPU parity of halo_migrate (NS-step home-atom redistribution)
vs oracle.migrate, through the C ABI; then the new decomposition's maps and both
halos vs the oracle built from scratch on the moved system.  Bit-exact."""
import numpy as np
import pytest
import torch

from tests.parity_common import Case, moved_case, run_gpu_case, run_gpu_migrate

pytestmark = pytest.mark.gpu

PAPER, CE = 1 << 4, 1 << 5


def _run(name, layout, flags, with_v, seed=1):
    from paper_2509_21527_b200.session import HaloSession
    case = Case(name, seed=seed, layout=layout, force_kind="int")
    Xm, V, c2 = moved_case(case, seed)
    cap = max(case.capacity, c2.capacity) + 64
    sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=layout, capacity=cap, device=0,
                       flags=flags, timeout_s=5.0)
    run_gpu_migrate(case, c2, Xm, V, sess, with_v=with_v)
    sess.destroy()


@pytest.mark.parametrize("name,layout,with_v", [("C1", 3, True), ("T3D", 4, True), ("T2P", 3, False),
                                                ("C2", 3, True), ("C5", 4, True), ("C3", 3, True)])
def test_migrate_then_exchange(name, layout, with_v):
    _run(name, layout, 0, with_v)


@pytest.mark.parametrize("flags", [PAPER, CE], ids=["paper", "ce"])
def test_migrate_other_protocols(flags):
    _run("T3D", 3, flags, True, seed=2)


def test_migrate_errors():
    from paper_2509_21527_b200 import HaloError
    from paper_2509_21527_b200.session import HaloSession
    case = Case("C5", seed=1)
    sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=3, capacity=case.capacity, device=0,
                       timeout_s=5.0)
    run_gpu_case(case, sess, check_forces=False)
    gid_t = []
    for l in range(sess.n_local):
        st = case.states[l]
        gt = torch.zeros(case.capacity, dtype=torch.int32, device=sess.device)
        gt[: st.n_home] = torch.from_numpy(st.gid[: st.n_home].astype(np.int32)).to(sess.device)
        gid_t.append(gt)
    # two cells along z on one rank: GEOMETRY on every rank
    sess.x[3][0, 2] += 2.1
    with pytest.raises(HaloError) as e:
        sess.migrate(gid_t)
    assert e.value.status == 2
    sess.x[3][0, 2] -= 2.1
    # gids not ascending: ARG
    g = gid_t[2][:2].clone()
    gid_t[2][0], gid_t[2][1] = g[1], g[0]
    with pytest.raises(HaloError) as e:
        sess.migrate(gid_t)
    assert e.value.status == 1
    gid_t[2][:2] = g
    # exchanges need set_maps again after a migrate
    with pytest.raises(HaloError) as e:
        sess.exchange_x()
    assert e.value.status == 4
    sess.destroy()


def test_migrate_capacity_overflow_is_agreed():
    """A rank that would receive more home rows than `capacity` fails the call on
    every rank (HALO_ERR_CAPACITY) and no row moves anywhere (x, gid unchanged)."""
    from paper_2509_21527_b200 import HaloError
    from paper_2509_21527_b200.session import HaloSession
    case = Case("C1", seed=1)
    cap = max(s.x.shape[0] for s in case.states) + 16
    sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=3, capacity=cap, device=0, timeout_s=5.0)
    run_gpu_case(case, sess, check_forces=False)
    gid_t = []
    for l in range(sess.n_local):
        st = case.states[l]
        gt = torch.zeros(cap, dtype=torch.int32, device=sess.device)
        gt[: st.n_home] = torch.from_numpy(st.gid[: st.n_home].astype(np.int32)).to(sess.device)
        gid_t.append(gt)
    # move every atom of rank 1 (upper z cell) down into rank 0's cell: one cell, but too many rows
    n1 = case.states[1].n_home
    lo = float(np.float32(case.L[2])) / 2
    sess.x[1][:n1, 2] = sess.x[1][:n1, 2] - lo
    before = [sess.x[l][: case.states[l].n_home].clone() for l in range(2)]
    with pytest.raises(HaloError) as e:
        sess.migrate(gid_t)
    assert e.value.status == 3
    for l in range(2):
        n = case.states[l].n_home
        assert torch.equal(sess.x[l][:n], before[l])
        assert torch.equal(gid_t[l][:n].cpu(), torch.from_numpy(case.states[l].gid[:n].astype(np.int32)))
    sess.destroy()
