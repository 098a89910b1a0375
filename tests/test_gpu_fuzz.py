"""Fuzz parity (-m gpu): random grids, boxes, cutoffs, 1-2 pulses per dim, float3 /
float4, uniform or clustered atoms (ranks with no home atoms, empty maps), all
three transports; every case bit-exact vs the oracle (maps, layout, halo x, f),
fshift within the fp64 bound."""
import numpy as np
import pytest

from oracle import decompose, force_halo
from synth import forces_int, forces_normal
from synth.water import charges
from tests.fuzz_cases import random_case
from tests.parity_common import run_gpu_case

pytestmark = pytest.mark.gpu


class FuzzCase:
    def __init__(self, seed, rounded=False):
        self.name = f"fuzz{seed}"
        self.seed, self.rounded = seed, rounded
        self.L, self.rc, self.grid, self.pulses, self.X, self.layout = random_case(seed)
        W = charges(self.X.shape[0]) if self.layout == 4 else None
        self.W = W
        self.states = decompose(self.X, self.L, self.rc, self.grid, self.pulses, W=W, rounded=rounded)
        self.nranks = len(self.states)
        self.capacity = max(max(s.x.shape[0] for s in self.states), 1) + 64
        mk = forces_int if seed % 2 == 0 else forces_normal
        self.F = [mk(s.x.shape[0], 31 * seed + s.rank, width=self.layout) for s in self.states]
        self.Fo, self.fshift, self.fshift_abs = force_halo(self.states, [f.copy() for f in self.F], with_abs=True)

    def home_rows(self, r):
        s = self.states[r]
        return s.x[: s.n_home]


@pytest.mark.parametrize("proto", [0, 1 << 4, (1 << 4) | (1 << 7) | (1 << 8), 1 << 5], ids=["ll", "paper", "paper_tma", "ce"])
@pytest.mark.parametrize("seed", range(24))
def test_fuzz_parity(seed, proto):
    from paper_2509_21527_b200.session import HaloSession
    case = FuzzCase(seed)
    sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=case.layout, capacity=case.capacity,
                       device=0, flags=proto, timeout_s=5.0)
    run_gpu_case(case, sess, steps=2)
    sess.destroy()


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_rounded_zones(seed):
    """Rounded zones (R31) on the random geometries, LL protocol, bit-exact."""
    from paper_2509_21527_b200.session import HaloSession
    case = FuzzCase(seed, rounded=True)
    sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=case.layout, capacity=case.capacity,
                       device=0, flags=1 << 9, timeout_s=5.0)
    run_gpu_case(case, sess, steps=2)
    sess.destroy()


@pytest.mark.parametrize("seed", range(0, 24, 2))
def test_fuzz_migrate(seed):
    """halo_migrate on the random geometries (clustered atoms, empty ranks, 1-4
    cells per dim): moves of up to a third of the smallest cell (R30 holds), then
    the new maps and both halos, bit-exact vs the oracle."""
    from paper_2509_21527_b200.session import HaloSession
    from tests.parity_common import moved_case, run_gpu_migrate
    case = FuzzCase(seed)
    case.layout = case.layout
    Xm, V, c2 = moved_case(case, seed)
    cap = max(case.capacity, c2.capacity) + 64
    sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=case.layout, capacity=cap, device=0,
                       timeout_s=5.0)
    run_gpu_migrate(case, c2, Xm, V, sess)
    sess.destroy()
