"""Multi-GPU parity (-m gpu, needs >= 2 devices): one process per GPU, DD ranks
spread over the processes, peers mapped with CUDA IPC, flags over NVLink.
Same bar as test_gpu_parity.py (bit-exact x and f, fshift within bound)."""
import os
import socket
import traceback

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _ndev():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, out):
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dev = rank % torch.cuda.device_count()  # world 8 on 4 GPUs: two processes per GPU
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2509_21527_b200 import _lib
        from paper_2509_21527_b200.session import HaloSession
        from tests.parity_common import Case, run_gpu_case
        assert _lib.LIB_PATH == os.environ.get("HALO_LIB_PATH", _lib.LIB_PATH)  # (the checked build when set)
        for (name, seed, kind, flags, layout, steps) in cases:
            case = Case(name, seed=seed, force_kind=kind, layout=layout, rounded=bool(flags & ROUNDED))
            if case.nranks % world:
                continue
            if flags & BULK:
                os.environ["HALO_BULK_ROWS"] = "1"  # read at halo_init (every process sets it)
            else:
                os.environ.pop("HALO_BULK_ROWS", None)
            sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=layout, capacity=case.capacity,
                               device=dev, flags=flags & ~(BULK | FUSED), nprocs=world, proc=rank, timeout_s=30.0)
            run_gpu_case(case, sess, steps=steps, atomic=bool(flags & 1) and kind != "int", barrier=dist.barrier,
                         fused=bool(flags & FUSED))
            sess.halo.sync()  # (the checked build: raises if a bounds check fired)
            dist.barrier()
            sess.destroy()
            dist.barrier()
        out[rank] = "ok"
        dist.destroy_process_group()
    except Exception:
        out[rank] = traceback.format_exc()


PAPER = 1 << 4
CE = 1 << 5
TMA = (1 << 7) | (1 << 8)  # HALO_F_TMA_STORE | HALO_F_TMA_GET
ROUNDED = 1 << 9  # HALO_F_ROUNDED_ZONES
# test-side markers, stripped before halo_init: BULK = HALO_BULK_ROWS=1 (every last pulse
# between processes is a bulk pulse); FUSED = one halo_exchange_xf per step
BULK, FUSED = 1 << 28, 1 << 29
CASES = [  # (config, seed, forces, flags, layout, steps); flags 0 = LL protocol
    ("C1", 1, "int", 0, 3, 2),
    ("W3", 1, "int", 0, 3, 1),
    ("T3D", 2, "normal", 0, 3, 2),
    ("C2", 1, "normal", 0, 3, 2),
    ("C3", 1, "int", 0, 3, 3),
    ("C5", 1, "normal", 0, 3, 2),
    ("T2P", 1, "int", 0, 4, 2),
    ("C1", 2, "int", PAPER, 3, 2),
    ("C3", 2, "normal", PAPER, 3, 2),
    ("C3", 2, "normal", PAPER | 4, 3, 2),   # + HALO_F_GPU_FENCE (paper's exact fence scheme)
    ("C5", 1, "normal", PAPER, 3, 2),
    ("C3", 3, "int", PAPER | 1, 3, 2),      # + HALO_F_ATOMIC_UNPACK, integer forces: exact
    ("C3", 1, "normal", PAPER | TMA, 3, 2),  # + TMA put of x / TMA get of f over NVLink (Alg. 3, Alg. 6)
    ("T2P", 2, "int", PAPER | TMA, 4, 2),
    ("C3", 2, "int", ROUNDED, 3, 2),          # rounded zones (R31), LL protocol
    ("C2", 1, "normal", PAPER | ROUNDED, 4, 2),
    ("C3", 1, "normal", BULK, 3, 3),         # bulk x pulses over NVLink (last pulse stored straight into x)
    ("T2P", 1, "int", BULK, 4, 2),
    ("C1", 2, "normal", BULK | FUSED, 3, 3),
    ("C5", 2, "normal", BULK | FUSED, 3, 2),
    ("C1", 1, "int", CE, 3, 2),             # copy-engine path
    ("C3", 1, "normal", CE, 3, 3),
    ("C5", 2, "int", CE, 3, 2),
    ("T2P", 1, "normal", CE, 4, 2),
]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_multiprocess_parity(world):
    # world 8 = one DD rank per process (the 8-GPU layout of C3/C5); with 4 GPUs two
    # processes share a GPU (time-sliced: slow but a full functional check)
    if _ndev() < min(world, 4):
        pytest.skip(f"needs {min(world, 4)} GPUs")
    cases = CASES if world < 8 else [c for c in CASES if c[0] in ("C3", "C5") and c[3] in (0, PAPER)][:3]
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, cases, out), nprocs=world, join=True)
        out = dict(out)
    for r in range(world):
        assert out.get(r) == "ok", out.get(r)


BOUNDS_CASES = [("C3", 1, "normal", 0, 3, 2), ("T2P", 1, "int", 0, 4, 2), ("C1", 2, "normal", BULK, 3, 2),
                ("C5", 1, "normal", BULK | FUSED, 3, 2)]


@pytest.mark.parametrize("world", [2])
def test_multiprocess_bounds_checked(world):
    """The cross-process LL paths through the bounds-checked build (DESIGN.md §7,
    tests/test_gpu_bounds.py): the spawned processes load libhalo_checked.so."""
    if _ndev() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2509_21527_b200.build import build_checked
    lib = build_checked()
    old = os.environ.get("HALO_LIB_PATH")
    os.environ["HALO_LIB_PATH"] = lib  # read at import by every spawned process
    try:
        port = _free_port()
        with mp.Manager() as mgr:
            out = mgr.dict()
            mp.spawn(_worker, args=(world, port, BOUNDS_CASES, out), nprocs=world, join=True)
            out = dict(out)
    finally:
        if old is None:
            os.environ.pop("HALO_LIB_PATH")
        else:
            os.environ["HALO_LIB_PATH"] = old
    for r in range(world):
        assert out.get(r) == "ok", out.get(r)


def _worker_g2(rank, world, port, cases, out):
    """G2: the NCCL send/recv schedule, the fused kernels and the
    copy-engine path on identical maps all reproduce the oracle bit-exactly."""
    try:
        import numpy as np
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
        from paper_2509_21527_b200.nccl_baseline import NcclSchedule
        from paper_2509_21527_b200.session import HaloSession
        from tests.parity_common import Case, assert_fshift, bits, run_gpu_case
        for (name, seed, kind) in cases:
            case = Case(name, seed=seed, force_kind=kind)
            if case.nranks != world:
                continue
            for flags in (0, CE):
                sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=3, capacity=case.capacity,
                                   device=rank, flags=flags, nprocs=world, proc=rank, timeout_s=10.0)
                run_gpu_case(case, sess, steps=1, barrier=dist.barrier)  # fused / CE vs oracle
                st = case.states[rank]
                n, nh = st.x.shape[0], st.n_home
                sched = NcclSchedule(sess)
                torch.cuda.synchronize()
                dist.barrier()
                sess.x[0][nh:n] = float("nan")
                torch.cuda.synchronize()
                dist.barrier()
                sched.exchange_x()
                torch.cuda.synchronize()
                np.testing.assert_array_equal(bits(sess.x[0][:n].cpu().numpy()), bits(st.x),
                                              err_msg=f"NCCL schedule halo x rank {rank}")
                sess.f[0][:n] = torch.from_numpy(case.F[rank]).to(sess.device)
                fshift = torch.zeros(1, 3, 3, dtype=torch.float64, device=sess.device)
                sched.exchange_f(fshift)
                torch.cuda.synchronize()
                np.testing.assert_array_equal(bits(sess.f[0][:n].cpu().numpy()), bits(case.Fo[rank]),
                                              err_msg=f"NCCL schedule f rank {rank}")
                assert_fshift(fshift[0].cpu().numpy(), case.fshift[rank], case.fshift_abs[rank], where="nccl")
                dist.barrier()
                # the same schedule captured into a CUDA graph (NCCL in the same graph)
                gs = torch.cuda.Stream()
                g = torch.cuda.CUDAGraph()
                torch.cuda.synchronize()
                dist.barrier()
                with torch.cuda.graph(g, stream=gs):
                    sched.step(fshift, stream=gs)
                for _ in range(2):
                    sess.x[0][nh:n] = float("nan")
                    sess.f[0][:n] = torch.from_numpy(case.F[rank]).to(sess.device)
                    fshift.zero_()
                    torch.cuda.synchronize()
                    dist.barrier()
                    g.replay()
                    torch.cuda.synchronize()
                    np.testing.assert_array_equal(bits(sess.x[0][:n].cpu().numpy()), bits(st.x),
                                                  err_msg=f"NCCL graph halo x rank {rank}")
                    np.testing.assert_array_equal(bits(sess.f[0][:n].cpu().numpy()), bits(case.Fo[rank]),
                                                  err_msg=f"NCCL graph f rank {rank}")
                    assert_fshift(fshift[0].cpu().numpy(), case.fshift[rank], case.fshift_abs[rank], where="nccl g")
                dist.barrier()
                del g
                # the fused / CE path still runs after the baseline touched the buffers
                run_gpu_case(case, sess, steps=1, barrier=dist.barrier)
                dist.barrier()
                sess.destroy()
                dist.barrier()
        out[rank] = "ok"
        dist.destroy_process_group()
    except Exception:
        out[rank] = traceback.format_exc()


G2_CASES = [("C1", 1, "normal"), ("W1", 1, "int"), ("C2", 2, "normal"), ("T2D", 1, "int")]


@pytest.mark.parametrize("world", [2, 4])
def test_schedule_equivalence_nccl_fused_ce(world):
    if _ndev() < world:
        pytest.skip(f"needs {world} GPUs")
    cases = [c for c in G2_CASES if _nranks(c[0]) == world]
    if not cases:
        pytest.skip(f"no G2 case with {world} DD ranks")
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker_g2, args=(world, port, cases, out), nprocs=world, join=True)
        out = dict(out)
    for r in range(world):
        assert out.get(r) == "ok", out.get(r)


def _nranks(name):
    from tests.parity_common import load_system
    g = load_system(name, 1)[2]
    return g[0] * g[1] * g[2]


def _worker_migrate(rank, world, port, cases, out):
    """halo_migrate across processes (f2): rows leave through the peers' staging
    areas over NVLink; then the new maps and both halos vs the oracle."""
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2509_21527_b200.session import HaloSession
        from tests.parity_common import Case, moved_case, run_gpu_migrate
        for (name, seed, flags, layout) in cases:
            case = Case(name, seed=seed, force_kind="int", layout=layout)
            if case.nranks % world:
                continue
            Xm, V, c2 = moved_case(case, seed)
            cap = max(case.capacity, c2.capacity) + 64
            sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=layout, capacity=cap,
                               device=rank, flags=flags, nprocs=world, proc=rank, timeout_s=10.0)
            run_gpu_migrate(case, c2, Xm, V, sess, barrier=dist.barrier)
            dist.barrier()
            sess.destroy()
            dist.barrier()
        out[rank] = "ok"
        dist.destroy_process_group()
    except Exception:
        out[rank] = traceback.format_exc()


MIGRATE_CASES = [("C1", 1, 0, 3), ("C3", 2, 0, 4), ("T2P", 1, 0, 3), ("C2", 3, PAPER, 3)]


@pytest.mark.parametrize("world", [2, 4])
def test_multiprocess_migrate(world):
    if _ndev() < world:
        pytest.skip(f"needs {world} GPUs")
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker_migrate, args=(world, port, MIGRATE_CASES, out), nprocs=world, join=True)
        out = dict(out)
    for r in range(world):
        assert out.get(r) == "ok", out.get(r)


def _worker_pme(rank, world, port, cases, out):
    """PP <-> PME across processes (f4): every rank's home rows to the PME rank's
    buffer over NVLink and its force slice back."""
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2509_21527_b200.session import HaloSession
        from tests.parity_common import Case, run_gpu_pme
        for (name, seed, layout, pme_rank) in cases:
            case = Case(name, seed=seed, force_kind="int", layout=layout)
            if case.nranks % world:
                continue
            sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=layout, capacity=case.capacity,
                               device=rank, nprocs=world, proc=rank, timeout_s=10.0, pme_rank=pme_rank)
            run_gpu_pme(case, sess, barrier=dist.barrier)
            dist.barrier()
            sess.destroy()
            dist.barrier()
        out[rank] = "ok"
        dist.destroy_process_group()
    except Exception:
        out[rank] = traceback.format_exc()


PME_CASES = [("C1", 1, 3, 1), ("C3", 2, 4, 0), ("C2", 1, 3, 3)]


@pytest.mark.parametrize("world", [2, 4])
def test_multiprocess_pme(world):
    if _ndev() < world:
        pytest.skip(f"needs {world} GPUs")
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker_pme, args=(world, port, PME_CASES, out), nprocs=world, join=True)
        out = dict(out)
    for r in range(world):
        assert out.get(r) == "ok", out.get(r)
