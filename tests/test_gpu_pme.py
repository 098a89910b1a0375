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


def test_pme_cuda_graph_replay():
    """halo_pme_send_x / halo_pme_recv_f captured once into a CUDA graph and replayed:
    the sequence numbers live in device memory, so every replay is a fresh step."""
    import numpy as np
    import torch
    from oracle import pme_gather, pme_return
    from paper_2509_21527_b200.session import HaloSession
    from synth import forces_int
    from tests.parity_common import bits, run_gpu_case
    case = Case("T3D", seed=2, layout=3, force_kind="int")
    sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=3, capacity=case.capacity, device=0,
                       timeout_s=5.0, pme_rank=3)
    run_gpu_case(case, sess, check_forces=False)
    n_total, off = sess.pme_setup()
    exp_x, _ = pme_gather([s.x[: s.n_home] for s in case.states])
    px, pf = sess.pme_buffers()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    sess.pme_send_x(stream=s)  # warm-up outside the capture
    sess.pme_recv_f(stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        sess.pme_send_x(stream=s)
        sess.pme_recv_f(stream=s)
    torch.cuda.synchronize()
    for step in range(3):
        F = [forces_int(st.n_home, 700 + 10 * step + st.rank) for st in case.states]
        PF = forces_int(n_total, 800 + step)
        for l in range(sess.n_local):
            sess.f[l][: case.states[l].n_home] = torch.from_numpy(F[l]).to(sess.device)
        px[:n_total] = float("nan")
        pf[:n_total] = torch.from_numpy(PF).to(sess.device)  # the "PME task" wrote its forces before replay
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        np.testing.assert_array_equal(bits(px[:n_total].cpu().numpy()), bits(exp_x))
        exp_f = pme_return(F, PF, off)
        for l in range(sess.n_local):
            n = case.states[l].n_home
            np.testing.assert_array_equal(bits(sess.f[l][:n].cpu().numpy()), bits(exp_f[l]))
    sess.destroy()


def test_pme_call_order_errors():
    from paper_2509_21527_b200 import HaloError
    from paper_2509_21527_b200.session import HaloSession
    case = Case("C1", seed=1)
    sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=3, capacity=case.capacity, device=0,
                       timeout_s=5.0)
    with pytest.raises(HaloError) as e:  # no halo_pme_reserve
        sess.pme_setup()
    assert e.value.status == 4
    sess.destroy()
    sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=3, capacity=case.capacity, device=0,
                       timeout_s=5.0, pme_rank=1)
    with pytest.raises(HaloError) as e:  # reserve after registration
        sess.halo.pme_reserve(0)
    assert e.value.status == 4
    with pytest.raises(HaloError) as e:  # send before setup
        sess.pme_send_x()
    assert e.value.status == 4
    sess.destroy()
