"""GPU parity (-m gpu): CUDA path through the C ABI vs the oracle, one process,
all DD ranks of a config hosted by one GPU (one kernel launch covers them all).

Bar: maps, layout, dependency masks, halo x and forces
bit-exact (deterministic unpack); fshift within the fp64 reduction bound.
"""
import numpy as np
import pytest
import torch

from tests.parity_common import Case, assert_fshift, bits, run_gpu_case

pytestmark = pytest.mark.gpu

PAPER = 1 << 4  # HALO_F_PAPER_FLAGS: the paper's per-pulse flag protocol; 0 = LL protocol (default)
CE = 1 << 5  # HALO_F_CE_PATH: copy-engine path
TMA_STORE, TMA_GET = 1 << 7, 1 << 8  # the paper's TMA put of x (Alg. 3) / receiver-driven TMA get of f (Alg. 6)
TMA = PAPER | TMA_STORE | TMA_GET
# LL with HALO_COLLAPSE=0: every DD rank its own hop group (the staged per-pulse schedule
# with LL transport, receive items and force pushes on every pulse: the code paths a
# pulse between two GPUs takes); "ll" = the default, one hop group per process
STAGED = 1 << 30  # test-side marker, stripped before halo_init
# ll_staged + HALO_BULK_ROWS=1: every last pulse is a bulk pulse (the
# x-sender stores into the receiver's x, one wait item counts the rows)
BULK = 1 << 29
PROTOS = [pytest.param(0, id="ll"), pytest.param(STAGED, id="ll_staged"), pytest.param(BULK, id="ll_bulk"),
          pytest.param(PAPER, id="paper"), pytest.param(TMA, id="paper_tma"), pytest.param(CE, id="ce")]


def session_for(case, flags=0, layout=None, capacity=None):
    import os
    from paper_2509_21527_b200.session import HaloSession
    env = {}
    if flags & (STAGED | BULK):
        env["HALO_COLLAPSE"] = "0"  # read at halo_init
    if flags & BULK:
        env["HALO_BULK_ROWS"] = "1"
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return HaloSession(case.grid, case.L, case.rc, case.pulses, layout=layout or case.layout,
                           capacity=capacity or case.capacity, device=0, flags=flags & ~(STAGED | BULK),
                           timeout_s=5.0)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("proto", PROTOS)
@pytest.mark.parametrize("name", ["W1", "W2", "W3", "C1", "T3D", "T2P", "T2D", "T4x2", "C2", "C5", "C3"])
def test_parity_int_forces(name, proto):
    case = Case(name, seed=1, force_kind="int")
    sess = session_for(case, flags=proto)
    run_gpu_case(case, sess, steps=2)
    sess.destroy()


@pytest.mark.parametrize("proto", PROTOS)
@pytest.mark.parametrize("name", ["C1", "T3D", "T2P", "C2", "C5", "C3"])
@pytest.mark.parametrize("seed", [2, 3])
def test_parity_real_forces(name, seed, proto):
    case = Case(name, seed=seed, force_kind="normal")
    sess = session_for(case, flags=proto)
    run_gpu_case(case, sess)
    sess.destroy()


@pytest.mark.parametrize("proto", PROTOS)
@pytest.mark.parametrize("name", ["W2", "T3D", "T2P", "C2"])
def test_parity_float4(name, proto):
    case = Case(name, seed=1, layout=4, force_kind="normal")
    sess = session_for(case, flags=proto)
    run_gpu_case(case, sess)
    sess.destroy()


@pytest.mark.parametrize("proto", PROTOS)
@pytest.mark.parametrize("name", ["T3D", "T2P", "C3"])
def test_parity_explicit_maps(name, proto):
    case = Case(name, seed=2, force_kind="int")
    sess = session_for(case, flags=proto)
    run_gpu_case(case, sess, use_explicit=True)
    sess.destroy()


@pytest.mark.parametrize("name,kind", [("T3D", "int"), ("C2", "int"), ("C3", "normal"), ("C5", "normal")])
def test_parity_atomic_unpack(name, kind):
    from paper_2509_21527_b200 import HALO_F_ATOMIC_UNPACK
    case = Case(name, seed=1, force_kind=kind)
    sess = session_for(case, flags=HALO_F_ATOMIC_UNPACK | PAPER)
    run_gpu_case(case, sess, atomic=(kind != "int"))
    sess.destroy()


@pytest.mark.parametrize("name", ["T3D", "C3"])
def test_parity_paper_fence_variant(name):
    from paper_2509_21527_b200 import HALO_F_GPU_FENCE
    case = Case(name, seed=3, force_kind="int")
    sess = session_for(case, flags=HALO_F_GPU_FENCE | PAPER)
    run_gpu_case(case, sess, steps=3)
    sess.destroy()


def test_moved_coordinates_between_ns_steps():
    """Hot-path exchange_x with maps fixed and home coordinates moved: every halo
    row equals fl32(X'[gid] + s*L) (closed form X1 on the moved positions)."""
    case = Case("C3", seed=1)
    sess = session_for(case)
    run_gpu_case(case, sess, check_forces=False)
    rng = np.random.default_rng(5)
    Xm = (case.X + rng.uniform(-0.01, 0.01, size=case.X.shape).astype(np.float32)).astype(np.float32)
    L32 = np.array(case.L, np.float32)
    for l in range(sess.n_local):
        st = case.states[l]
        sess.x[l][: st.n_home] = torch.from_numpy(Xm[st.gid[: st.n_home]]).to(sess.device)
    sess.exchange_x()
    torch.cuda.synchronize()
    for l in range(sess.n_local):
        st = case.states[l]
        exp = Xm[st.gid].copy()
        for d in range(3):
            m = st.s[:, d] == 1
            exp[m, d] = (exp[m, d] + L32[d]).astype(np.float32)
        got = sess.x[l][: st.x.shape[0]].cpu().numpy()
        np.testing.assert_array_equal(bits(got), bits(exp))
    sess.destroy()


@pytest.mark.parametrize("proto", PROTOS)
def test_cuda_graph_replay(proto):
    """x+f captured once into a CUDA graph and replayed: the device-resident
    sequence numbers keep every replay correct."""
    case = Case("C3", seed=2, force_kind="int")
    sess = session_for(case, flags=proto)
    run_gpu_case(case, sess)
    s = torch.cuda.Stream()
    fshift = torch.zeros(sess.n_local, 3, 3, dtype=torch.float64, device=sess.device)
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        sess.exchange_x(stream=s)
        sess.exchange_f(fshift=fshift, stream=s)
    for rep in range(5):
        for l in range(sess.n_local):
            st = case.states[l]
            sess.x[l][st.n_home: st.x.shape[0]] = float("nan")
            sess.f[l][: case.F[l].shape[0]] = torch.from_numpy(case.F[l]).to(sess.device)
        fshift.zero_()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        for l in range(sess.n_local):
            st = case.states[l]
            np.testing.assert_array_equal(bits(sess.x[l][: st.x.shape[0]].cpu().numpy()), bits(st.x))
            np.testing.assert_array_equal(bits(sess.f[l][: case.F[l].shape[0]].cpu().numpy()), bits(case.Fo[l]))
            np.testing.assert_array_equal(fshift[l].cpu().numpy(), case.fshift[l])
    sess.destroy()


@pytest.mark.parametrize("proto", [pytest.param(0, id="ll"), pytest.param(STAGED, id="ll_staged")])
def test_long_run_stays_exact(proto):
    """50,000 exchange steps on one NS epoch (100,000 launches: sequence numbers, LL tags,
    completion counters cycling), then one step on fresh inputs without a set_maps in
    between: still bit-exact (x, f) and exact fshift (integer forces)."""
    case = Case("C3", seed=1, force_kind="int")
    sess = session_for(case, flags=proto)
    run_gpu_case(case, sess)
    fshift = torch.zeros(sess.n_local, 3, 3, dtype=torch.float64, device=sess.device)
    for _ in range(50000):
        sess.exchange_x()
        sess.exchange_f(fshift=fshift)
    torch.cuda.synchronize()
    sess.halo.sync()
    for l in range(sess.n_local):
        st = case.states[l]
        sess.x[l][st.n_home: st.x.shape[0]] = float("nan")
        sess.f[l][: case.F[l].shape[0]] = torch.from_numpy(case.F[l]).to(sess.device)
    fshift.zero_()
    sess.exchange_x()
    sess.exchange_f(fshift=fshift)
    torch.cuda.synchronize()
    for l in range(sess.n_local):
        st = case.states[l]
        np.testing.assert_array_equal(bits(sess.x[l][: st.x.shape[0]].cpu().numpy()), bits(st.x))
        np.testing.assert_array_equal(bits(sess.f[l][: case.F[l].shape[0]].cpu().numpy()), bits(case.Fo[l]))
        np.testing.assert_array_equal(fshift[l].cpu().numpy(), case.fshift[l])
    sess.destroy()


@pytest.mark.parametrize("proto", [pytest.param(0, id="ll"), pytest.param(BULK, id="ll_bulk")])
@pytest.mark.parametrize("renew", ["set_maps", "migrate"])
def test_stale_graph_replay_refused(renew, proto):
    """A graph captured before an NS step (set_maps / migrate) and replayed after it:
    every item of the new plan carries the new epoch, so the replay touches nothing
    and the next call reports HALO_ERR_STATE (ADVICE: captured launches freeze the plan)."""
    from paper_2509_21527_b200.halo import HaloError
    case = Case("T3D", seed=2, force_kind="int")
    sess = session_for(case, flags=proto)
    run_gpu_case(case, sess)
    s = torch.cuda.Stream()
    fshift = torch.zeros(sess.n_local, 3, 3, dtype=torch.float64, device=sess.device)
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        sess.exchange_x(stream=s)
        sess.exchange_f(fshift=fshift, stream=s)
    g.replay()  # the current epoch: fine
    torch.cuda.synchronize()
    sess.halo.sync()
    if renew == "set_maps":
        sess.set_maps()
    else:
        gid = [torch.zeros(sess.capacity, dtype=torch.int32, device=sess.device) for _ in range(sess.n_local)]
        for l in range(sess.n_local):
            gid[l][: sess.n_home[l]] = torch.from_numpy(case.states[l].gid[: sess.n_home[l]].astype(np.int32))
        sess.migrate(gid)
    torch.cuda.synchronize()
    for l in range(sess.n_local):
        sess.x[l][sess.n_home[l]:] = float("nan")
    g.replay()
    torch.cuda.synchronize()
    for l in range(sess.n_local):
        assert torch.isnan(sess.x[l][sess.n_home[l]: sess.n_home[l] + 8]).all(), "a stale replay wrote x"
    with pytest.raises(HaloError, match="HALO_ERR_STATE"):
        sess.halo.sync()
    del g
    sess.halo.destroy()


@pytest.mark.parametrize("proto", [pytest.param(0, id="ll"), pytest.param(STAGED, id="ll_staged"),
                                   pytest.param(BULK, id="ll_bulk")])
@pytest.mark.parametrize("name", ["T3D", "T2P", "T4x2", "C2", "C5", "C3"])
def test_gpu_plan_equals_host_plan(name, proto, monkeypatch):
    """The LL plan built on the device (kernels_plan.cu) == the host builder's plan of the
    same maps, item by item and field by field (HALO_PLAN_CHECK: set_maps fails on any
    difference; the shift-force bucket numbering differs by design), and parity holds."""
    monkeypatch.setenv("HALO_PLAN_CHECK", "1")
    case = Case(name, seed=1, force_kind="normal")
    sess = session_for(case, flags=proto)
    run_gpu_case(case, sess)
    sess.destroy()


@pytest.mark.parametrize("proto", [pytest.param(0, id="ll"), pytest.param(STAGED, id="ll_staged"),
                                   pytest.param(BULK, id="ll_bulk")])
@pytest.mark.parametrize("fused", [False, True])
def test_ll_tag_wrap(proto, fused, monkeypatch):
    """LL units carry the low 32 bits of the launch's sequence number: starting 3 below
    2^32, the steps cross the wrap (tag 0 is skipped) and stay bit-exact."""
    monkeypatch.setenv("HALO_SEQ_BASE", str((1 << 32) - 3))
    case = Case("T3D", seed=1, force_kind="int")
    sess = session_for(case, flags=proto)
    run_gpu_case(case, sess, steps=6, fused=fused)
    sess.destroy()


def test_step_host_e2e():
    case = Case("C2", seed=1, force_kind="int")
    sess = session_for(case)
    run_gpu_case(case, sess, check_forces=False)
    nl = sess.n_local
    xh = [torch.from_numpy(np.ascontiguousarray(case.home_rows(l))).pin_memory() for l in range(nl)]
    fa = [torch.from_numpy(case.F[l]).pin_memory() for l in range(nl)]
    xo = [torch.empty(case.states[l].x.shape[0] - case.states[l].n_home, 3).pin_memory() for l in range(nl)]
    fo = [torch.empty(case.states[l].n_home, 3).pin_memory() for l in range(nl)]
    fs = torch.zeros(nl, 3, 3, dtype=torch.float64).pin_memory()
    sess.halo.step_host([t.data_ptr() for t in xh], [t.data_ptr() for t in fa], [t.data_ptr() for t in xo],
                        [t.data_ptr() for t in fo], fs.data_ptr(), stream=torch.cuda.current_stream().cuda_stream)
    for l in range(nl):
        st = case.states[l]
        np.testing.assert_array_equal(bits(xo[l].numpy()), bits(st.x[st.n_home:]))
        np.testing.assert_array_equal(bits(fo[l].numpy()), bits(case.Fo[l][: st.n_home]))
        np.testing.assert_array_equal(fs[l].numpy(), case.fshift[l])
    sess.destroy()


@pytest.mark.parametrize("mode", ["graph", "eager", "direct"])
@pytest.mark.parametrize("cfg", ["C2", "C3", "T2P"])
def test_step_host_packed_e2e(cfg, mode, monkeypatch):
    """halo_step_host_packed (one host block in, one out) == the oracle, twice in a row:
    as one cached CUDA graph (default), eagerly, or with the forces written by the last
    kernel straight into the mapped output block; then a two-launch eager step."""
    if mode == "eager":
        monkeypatch.setenv("HALO_PACKED_GRAPH", "0")
    if mode == "direct":
        monkeypatch.setenv("HALO_PACKED_DIRECT", "1")
    case = Case(cfg, seed=2, force_kind="int")
    sess = session_for(case)
    run_gpu_case(case, sess, check_forces=False)
    nl = sess.n_local
    in_b, out_b = sess.halo.packed_sizes()
    xs = [np.ascontiguousarray(case.home_rows(l)) for l in range(nl)]
    fs_ = [case.F[l] for l in range(nl)]
    blk = np.concatenate([a.reshape(-1) for a in xs] + [a.reshape(-1) for a in fs_]).astype(np.float32)
    assert blk.nbytes == in_b
    hin = torch.from_numpy(blk).pin_memory()
    hout = torch.empty(out_b, dtype=torch.uint8).pin_memory()
    for _ in range(2):
        hout.fill_(0xFF)
        sess.halo.step_host_packed(hin.data_ptr(), hout.data_ptr(), stream=torch.cuda.current_stream().cuda_stream)
        raw = hout.numpy()
        o = 0
        for l in range(nl):
            st = case.states[l]
            n = (st.x.shape[0] - st.n_home) * st.x.shape[1] * 4
            np.testing.assert_array_equal(raw[o:o + n].view(np.int32), bits(st.x[st.n_home:]).reshape(-1))
            o += n
        for l in range(nl):
            st = case.states[l]
            n = st.n_home * case.Fo[l].shape[1] * 4
            np.testing.assert_array_equal(raw[o:o + n].view(np.int32), bits(case.Fo[l][: st.n_home]).reshape(-1))
            o += n
        o = (o + 7) // 8 * 8
        fsh = raw[o:o + nl * 72].view(np.float64).reshape(nl, 3, 3)
        for l in range(nl):
            np.testing.assert_array_equal(fsh[l], case.fshift[l])
    run_gpu_case(case, sess)  # eager launches after the graph replays (host sequence mirror in step)
    sess.destroy()


def test_baseline_pack_unpack_kernels():
    """Per-pulse pack/unpack kernels of the NCCL schedule reproduce the oracle when
    driven serially on one GPU (transfers done with torch copies)."""
    case = Case("T3D", seed=1, force_kind="int")
    sess = session_for(case)
    run_gpu_case(case, sess, check_forces=False)
    nl, P = sess.n_local, sess.npulse
    lays = [sess.layout_of(l) for l in range(nl)]
    for l in range(nl):
        st = case.states[l]
        sess.x[l][st.n_home: st.x.shape[0]] = 0.0
    for p in range(P):  # serialized pulses
        for l in range(nl):
            pi = case.states[l].pulses[p]
            buf = torch.empty(max(pi.send_size, 1), 3, device=sess.device)
            sess.halo.pack_x_pulse(l, p, buf.data_ptr())
            dst = pi.send_rank
            off = case.states[dst].pulses[p].atom_offset
            if pi.send_size:
                sess.x[dst][off: off + pi.send_size] = buf[: pi.send_size]
        torch.cuda.synchronize()
    for l in range(nl):
        st = case.states[l]
        np.testing.assert_array_equal(bits(sess.x[l][: st.x.shape[0]].cpu().numpy()), bits(st.x))
    for l in range(nl):
        sess.f[l][: case.F[l].shape[0]] = torch.from_numpy(case.F[l]).to(sess.device)
    fshift = torch.zeros(nl, 3, 3, dtype=torch.float64, device=sess.device)
    for p in range(P - 1, -1, -1):
        bufs = []
        for l in range(nl):
            pi = case.states[l].pulses[p]
            u = pi.send_rank
            ui = case.states[u].pulses[p]
            bufs.append(sess.f[u][ui.atom_offset: ui.atom_offset + ui.recv_size].clone())
        for l in range(nl):
            sess.halo.unpack_f_pulse(l, p, bufs[l].data_ptr(), fshift.data_ptr() + 0)
        torch.cuda.synchronize()
    for l in range(nl):
        np.testing.assert_array_equal(bits(sess.f[l][: case.F[l].shape[0]].cpu().numpy()), bits(case.Fo[l]))
        np.testing.assert_array_equal(fshift[l].cpu().numpy(), case.fshift[l])
    sess.destroy()


def test_errors():
    from paper_2509_21527_b200 import HaloError
    case = Case("C1", seed=1)
    # exchange before set_maps -> STATE
    sess = session_for(case)
    with pytest.raises(HaloError) as e:
        sess.exchange_x()
    assert e.value.status == 4
    sess.destroy()
    # capacity overflow agreed on all ranks
    small = max(s.n_home for s in case.states) + 10
    sess = session_for(case, capacity=small)
    sess.load_home([case.home_rows(l) for l in range(sess.n_local)])
    with pytest.raises(HaloError) as e:
        sess.set_maps()
    assert e.value.status == 3
    with pytest.raises(HaloError):
        sess.exchange_x()
    sess.destroy()
    # home atom outside its cell -> GEOMETRY
    sess = session_for(case)
    rows = [case.home_rows(l).copy() for l in range(sess.n_local)]
    rows[0][0, 2] = 3.0  # rank 0 owns z in [0, L/2)
    sess.load_home(rows)
    with pytest.raises(HaloError) as e:
        sess.set_maps()
    assert e.value.status == 2
    sess.destroy()
    # accumulate=0 with more than one pulse -> UNSUPPORTED
    case3 = Case("T3D", seed=1)
    sess = session_for(case3)
    run_gpu_case(case3, sess, check_forces=False)
    with pytest.raises(HaloError) as e:
        sess.exchange_f(accumulate=False)
    assert e.value.status == 8
    sess.destroy()


@pytest.mark.parametrize("flags", [PAPER | TMA_STORE, PAPER | TMA_GET, PAPER | TMA_GET | 1],
                         ids=["tma_put", "tma_get", "tma_get_atomic"])
@pytest.mark.parametrize("name", ["W3", "T3D", "T2P", "C5", "C3"])
def test_parity_tma_variants(name, flags):
    """The paper's NVLink transports one at a time: TMA put of x only,
    TMA get of f only (deterministic and atomic unpack; integer forces make the
    atomic sums exact), float3 rows whose 12-B pitch leaves chunk ends unaligned."""
    case = Case(name, seed=1, force_kind="int")
    sess = session_for(case, flags=flags)
    run_gpu_case(case, sess, steps=3)
    sess.destroy()
    case4 = Case(name, seed=2, layout=4, force_kind="int")
    sess = session_for(case4, flags=flags, layout=4)
    run_gpu_case(case4, sess, steps=2)
    sess.destroy()


ROUNDED = 1 << 9  # HALO_F_ROUNDED_ZONES (R31)


@pytest.mark.parametrize("proto", PROTOS)
@pytest.mark.parametrize("name,layout", [("W2", 3), ("T3D", 3), ("T2P", 4), ("T2D", 3), ("C2", 3), ("C5", 3),
                                         ("C3", 4)])
def test_parity_rounded_zones(name, layout, proto):
    """GROMACS-style rounded zones (SURVEY f2 variant): maps, halo x and forces
    bit-exact vs the oracle's rounded decomposition (pinned by Z1-Z3)."""
    case = Case(name, seed=2, layout=layout, force_kind="int", rounded=True)
    sess = session_for(case, flags=proto | ROUNDED, layout=layout)
    run_gpu_case(case, sess, steps=2)
    sess.destroy()


def test_tma_flags_need_paper_protocol():
    from paper_2509_21527_b200 import HaloError
    case = Case("C1", seed=1)
    for flags in (TMA_STORE, TMA_GET, CE | PAPER | TMA_GET):
        with pytest.raises(HaloError) as e:
            session_for(case, flags=flags)
        assert e.value.status == 8


@pytest.mark.parametrize("proto", PROTOS)
def test_accumulate_false_single_pulse(proto):
    case = Case("C1", seed=1, force_kind="int")
    sess = session_for(case, flags=proto)
    run_gpu_case(case, sess, check_forces=False)
    from oracle import force_halo
    Fo, _ = force_halo(case.states, [f.copy() for f in case.F], accumulate=False)
    for l in range(sess.n_local):
        sess.f[l][: case.F[l].shape[0]] = torch.from_numpy(case.F[l]).to(sess.device)
    sess.exchange_f(accumulate=False)
    torch.cuda.synchronize()
    for l in range(sess.n_local):
        np.testing.assert_array_equal(bits(sess.f[l][: case.F[l].shape[0]].cpu().numpy()), bits(Fo[l]))
    sess.destroy()


@pytest.mark.parametrize("proto", PROTOS)
def test_timers_and_many_steps(proto):
    from paper_2509_21527_b200 import HALO_F_TIMERS
    case = Case("C2", seed=1, force_kind="int")
    sess = session_for(case, flags=HALO_F_TIMERS | proto)
    run_gpu_case(case, sess, check_forces=True)
    for _ in range(200):
        sess.exchange_x()
        sess.exchange_f()
    sess.halo.sync()
    if proto != CE:  # the copy-engine path has no fused kernel to time (several launches per pulse)
        tx, tf = sess.halo.get_timers()
        assert 0 < tx < 10_000_000 and 0 < tf < 10_000_000
    run_gpu_case(case, sess, check_forces=True)  # still bit-exact after 200 unchecked steps
    sess.destroy()


@pytest.mark.parametrize("name", ["C4-1D", "C4-2D", "C4-3D"])
def test_parity_full_size_c4(name):
    """BASELINE configs[3] at full size (1.07M atoms), every element compared."""
    case = Case(name, seed=1, force_kind="normal")
    sess = session_for(case)
    run_gpu_case(case, sess)
    sess.destroy()


@pytest.mark.parametrize("rows", ["32", "512"])
def test_parity_item_size_bounds(rows, monkeypatch):
    """Smallest and largest work items (HALO_ITEM_ROWS is read at halo_init)."""
    monkeypatch.setenv("HALO_ITEM_ROWS", rows)
    case = Case("C3", seed=2, force_kind="normal")
    sess = session_for(case)
    run_gpu_case(case, sess, steps=2)
    sess.destroy()


@pytest.mark.parametrize("mut", [16, 32])
def test_mutation_is_caught(mut, monkeypatch):
    """Dependency safety (G3): with a protocol mutation (16: forward x rows without
    waiting for their arrival; 32: add force contributions without checking their
    sequence tag) the poisoned/bit-exact parity check must fail on a 3D grid with
    forwarding.  Proves the parity tests can see a protocol race.  HALO_COLLAPSE=0:
    every rank its own hop group, so every pulse waits (one group has no waits)."""
    monkeypatch.setenv("HALO_DEBUG", str(mut))
    monkeypatch.setenv("HALO_COLLAPSE", "0")
    case = Case("C3", seed=1, force_kind="int")
    sess = session_for(case, capacity=case.capacity)
    failed = False
    try:
        for _ in range(3):
            run_gpu_case(case, sess, steps=2)
    except AssertionError:
        failed = True
    sess.destroy()
    assert failed, "mutation not detected"


def test_two_neighbour_search_epochs():
    """set_maps twice on one context with different systems (atoms migrate, home
    counts change): the second epoch's maps, halo and forces are bit-exact."""
    case1 = Case("C2", seed=1, force_kind="int")
    case2 = Case("C2", seed=5, force_kind="normal")
    cap = max(case1.capacity, case2.capacity)
    sess = session_for(case1, capacity=cap)
    run_gpu_case(case1, sess, steps=2)
    run_gpu_case(case2, sess, steps=2)
    run_gpu_case(case1, sess, steps=1)
    sess.destroy()


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_notification_minimality_paper_protocol(name, monkeypatch):
    """Pin G4: the paper protocol emits exactly ONE system-scope flag
    store per (rank, pulse) per exchange, from the last CTA of the pulse."""
    monkeypatch.setenv("HALO_DEBUG", "64")
    case = Case(name, seed=1, force_kind="int")
    sess = session_for(case, flags=PAPER)
    run_gpu_case(case, sess)  # set_maps + one checked step
    x0, f0 = sess.halo.get_notify_counts(0), sess.halo.get_notify_counts(1)
    K = 7
    for _ in range(K):
        sess.exchange_x()
        sess.exchange_f()
    sess.halo.sync()
    dx, df = sess.halo.get_notify_counts(0) - x0, sess.halo.get_notify_counts(1) - f0
    for l in range(sess.n_local):
        lay = sess.layout_of(l)
        for p in range(sess.npulse):
            assert dx[l, p] == K * (lay["send_size"][p] > 0), (l, p, dx[l, p])
            assert df[l, p] == K * (lay["recv_size"][p] > 0), (l, p, df[l, p])
    sess.destroy()


@pytest.mark.parametrize("proto", PROTOS)
def test_parity_under_concurrent_compute(proto):
    """Alg. 2 schedule: the exchanges run on a high-priority stream while
    a GEMM that fills every SM runs on another stream; results stay bit-exact and the
    co-resident grids make progress."""
    case = Case("C3", seed=2, force_kind="int")
    sess = session_for(case, flags=proto)
    run_gpu_case(case, sess)  # set_maps + one checked step
    s_nl = torch.cuda.Stream(priority=-1)
    s_loc = torch.cuda.Stream()
    A = torch.randn(4096, 4096, device=sess.device, dtype=torch.bfloat16)
    for _ in range(3):
        for l in range(sess.n_local):
            st = case.states[l]
            sess.x[l][st.n_home: st.x.shape[0]] = float("nan")
        torch.cuda.synchronize()
        with torch.cuda.stream(s_loc):
            for _ in range(4):
                torch.mm(A, A)
        sess.exchange_x(stream=s_nl)
        with torch.cuda.stream(s_loc):
            torch.mm(A, A)
        torch.cuda.synchronize()
        for l in range(sess.n_local):
            st = case.states[l]
            np.testing.assert_array_equal(bits(sess.x[l][: st.x.shape[0]].cpu().numpy()), bits(st.x))
            sess.f[l][: case.F[l].shape[0]] = torch.from_numpy(case.F[l]).to(sess.device)
        fshift = torch.zeros(sess.n_local, 3, 3, dtype=torch.float64, device=sess.device)
        torch.cuda.synchronize()
        with torch.cuda.stream(s_loc):
            for _ in range(4):
                torch.mm(A, A)
        sess.exchange_f(fshift=fshift, stream=s_nl)
        torch.cuda.synchronize()
        fs = fshift.cpu().numpy()
        for l in range(sess.n_local):
            n = case.F[l].shape[0]
            np.testing.assert_array_equal(bits(sess.f[l][:n].cpu().numpy()), bits(case.Fo[l]))
            assert_fshift(fs[l], case.fshift[l], case.fshift_abs[l], where=f"rank {l}")
    sess.destroy()


def test_auto_transport_switches_per_epoch(monkeypatch):
    """HALO_F_AUTO_TRANSPORT: set_maps votes LL or copy engine by pulse
    size (threshold HALO_AUTO_CE_BYTES, read at every set_maps); switching between
    NS epochs in both directions keeps the results bit-exact (sequence numbers
    stay consistent across transports)."""
    AUTO = 1 << 10
    case = Case("T3D", seed=3, force_kind="int")
    sess = session_for(case, flags=AUTO)
    for thr, expect in (("1000000000", "ll"), ("1", "ce"), ("1000000000", "ll"), ("1", "ce")):
        monkeypatch.setenv("HALO_AUTO_CE_BYTES", thr)
        run_gpu_case(case, sess, steps=2)
        assert sess.halo.transport() == expect
    sess.destroy()
    monkeypatch.delenv("HALO_AUTO_CE_BYTES")
    big = Case("C3", seed=1, force_kind="int")  # pulses of ~2.5k rows: far below 4 MiB -> LL
    sess = session_for(big, flags=AUTO)
    run_gpu_case(big, sess)
    assert sess.halo.transport() == "ll"
    sess.destroy()
    from paper_2509_21527_b200 import HaloError
    with pytest.raises(HaloError) as e:
        session_for(case, flags=AUTO | CE)
    assert e.value.status == 8


# ------------------------------------------------ fused x+f launch (halo_exchange_xf)
@pytest.mark.parametrize("kind", ["int", "normal"])
@pytest.mark.parametrize("name", ["W1", "W2", "W3", "C1", "T3D", "T2P", "T2D", "T4x2", "C2", "C5", "C3"])
def test_parity_fused_xf(name, kind):
    """One launch per step: x halo and forces bit-exact, fshift
    within the fp64 bound, several steps (sequence numbers, per-rank halo counters)."""
    case = Case(name, seed=1 if kind == "int" else 2, force_kind=kind)
    sess = session_for(case)
    run_gpu_case(case, sess, steps=3, fused=True)
    run_gpu_case(case, sess, steps=1)  # the two-launch path in the same NS epoch
    run_gpu_case(case, sess, steps=2, fused=True)
    sess.destroy()


@pytest.mark.parametrize("name", ["T2P", "C3"])
def test_parity_fused_xf_float4_and_large_items(name, monkeypatch):
    monkeypatch.setenv("HALO_ITEM_ROWS", "256")  # batched (wide) variants
    case = Case(name, seed=3, layout=4, force_kind="normal")
    sess = session_for(case, layout=4)
    run_gpu_case(case, sess, steps=2, fused=True)
    sess.destroy()


def test_parity_fused_xf_receive_path(monkeypatch):
    """Fused launch with every halo row through receive items (the cross-GPU path)."""
    monkeypatch.setenv("HALO_DIRECT_X", "0")
    case = Case("C3", seed=1, force_kind="normal")
    sess = session_for(case)
    run_gpu_case(case, sess, steps=3, fused=True)
    sess.destroy()


def test_fused_xf_cuda_graph_replay():
    """exchange_xf captured once and replayed: device-resident sequence numbers and
    halo counters keep every replay bit-exact; mixed with eager two-launch steps."""
    case = Case("C3", seed=2, force_kind="int")
    sess = session_for(case)
    run_gpu_case(case, sess, fused=True)
    s = torch.cuda.Stream()
    fshift = torch.zeros(sess.n_local, 3, 3, dtype=torch.float64, device=sess.device)
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        sess.exchange_xf(fshift=fshift, stream=s)
    for rep in range(4):
        for l in range(sess.n_local):
            st = case.states[l]
            sess.x[l][st.n_home: st.x.shape[0]] = float("nan")
            sess.f[l][: case.F[l].shape[0]] = torch.from_numpy(case.F[l]).to(sess.device)
        fshift.zero_()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        for l in range(sess.n_local):
            st = case.states[l]
            np.testing.assert_array_equal(bits(sess.x[l][: st.x.shape[0]].cpu().numpy()), bits(st.x))
            np.testing.assert_array_equal(bits(sess.f[l][: case.F[l].shape[0]].cpu().numpy()), bits(case.Fo[l]))
            np.testing.assert_array_equal(fshift[l].cpu().numpy(), case.fshift[l])
        if rep == 1:
            sess.exchange_x()
            sess.exchange_f()
    sess.destroy()
