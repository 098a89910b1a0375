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
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2509_21527_b200.session import HaloSession
        from tests.parity_common import Case, run_gpu_case
        for (name, seed, kind, flags, layout, steps) in cases:
            case = Case(name, seed=seed, force_kind=kind, layout=layout)
            if case.nranks % world:
                continue
            sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=layout, capacity=case.capacity,
                               device=rank, flags=flags, nprocs=world, proc=rank, timeout_s=10.0)
            run_gpu_case(case, sess, steps=steps, atomic=bool(flags & 1) and kind != "int", barrier=dist.barrier)
            dist.barrier()
            sess.destroy()
            dist.barrier()
        out[rank] = "ok"
        dist.destroy_process_group()
    except Exception:
        out[rank] = traceback.format_exc()


PAPER = 1 << 4
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
]


@pytest.mark.parametrize("world", [2, 4])
def test_multiprocess_parity(world):
    if _ndev() < world:
        pytest.skip(f"needs {world} GPUs")
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, CASES, out), nprocs=world, join=True)
        out = dict(out)
    for r in range(world):
        assert out.get(r) == "ok", out.get(r)
