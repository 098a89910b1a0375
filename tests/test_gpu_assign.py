"""halo_assign_home (the initial domain assignment, R3/R4) on the GPU
vs the oracle's decomposition: identical home atom sets per rank, ascending."""
import numpy as np
import pytest

from oracle import decompose
from synth import get_config, water_box

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,seed", [("C1", 1), ("T3D", 2), ("C3", 2509), ("C5", 3), ("T4x2", 1)])
def test_assign_home_matches_oracle(name, seed):
    from paper_2509_21527_b200.session import assign_home
    c = get_config(name)
    X = water_box(c.n_atoms, c.L, seed, slab=c.slab)
    homes = assign_home(X, c.L, c.grid, c.rc, c.pulses)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses)
    assert len(homes) == len(st)
    for h, s in zip(homes, st):
        np.testing.assert_array_equal(h, s.gid[: s.n_home])


def test_assign_home_plane_ties_and_errors():
    import torch
    from paper_2509_21527_b200.halo import Halo, HaloError
    from paper_2509_21527_b200.session import assign_home
    L = (4.0, 4.0, 4.0)
    # exactly on the interior plane 2.0: the upper cell (R4); 0.0 -> lower cell
    X = np.array([[0.5, 0.5, 2.0], [0.5, 0.5, 1.9999999], [0.0, 0.0, 0.0], [3.9999998, 2.0, 3.0]], np.float32)
    homes = assign_home(X, L, (2, 2, 2), 1.0, (1, 1, 1))
    rank = {int(i): r for r, h in enumerate(homes) for i in h}
    assert rank == {0: 1, 1: 0, 2: 0, 3: 7}
    # empty input
    assert [len(h) for h in assign_home(np.zeros((0, 3), np.float32), L, (2, 2, 2), 1.0, (1, 1, 1))] == [0] * 8
    # a coordinate outside [0, L): HALO_ERR_GEOMETRY
    h = Halo((1, 1, 2), L, 1.0, (0, 0, 1), capacity=1, device=0)
    x = torch.tensor([[0.5, 0.5, 4.0]], dtype=torch.float32, device="cuda")
    ids = torch.empty(1, dtype=torch.int32, device="cuda")
    with pytest.raises(HaloError):
        h.assign_home(x.data_ptr(), 1, 3, ids.data_ptr())
    h.destroy()
