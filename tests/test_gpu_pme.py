"""GPU parity of the PP <-> PME redistribution: halo_pme_send_x /
halo_pme_recv_f through the C ABI vs oracle.pme_gather / pme_return, bit-exact."""
import pytest

from tests.parity_common import Case, run_gpu_pme

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,layout,pme_rank", [("C1", 3, 0), ("T3D", 4, 7), ("C2", 3, 2), ("C3", 3, 5),
                                                  ("C5", 4, 0)])
def test_pme_roundtrip(name, layout, pme_rank):
    from paper_2509_21527_b200.session import HaloSession
    case = Case(name, seed=1, layout=layout, force_kind="int")
    sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=layout, capacity=case.capacity, device=0,
                       timeout_s=5.0, pme_rank=pme_rank)
    run_gpu_pme(case, sess)
    # a new NS epoch: set_maps invalidates the PME layout until pme_setup
    from paper_2509_21527_b200 import HaloError
    sess.set_maps()
    with pytest.raises(HaloError) as e:
        sess.pme_send_x()
    assert e.value.status == 4
    run_gpu_pme(case, sess, steps=2)
    sess.destroy()
