"""N>1 host logic on CPU (world_size 2, gloo): the DD-rank -> process partition
from halo_query_config, the blob all-gather ordering the IPC import relies on,
and bench.py's max-over-ranks timing reduction."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_21527_b200.halo import query_config
    from synth import get_config
    res = {}
    for name in ["C3", "C2", "C5", "T4x2"]:
        c = get_config(name)
        q = query_config(c.grid, c.L, c.rc, c.pulses, capacity=1000, nprocs=world, proc=rank)
        got = [None] * world
        dist.all_gather_object(got, (rank, q["first_rank"], q["n_local"], q["dims"], q["scratch_bytes"]))
        res[name] = got
    # blob all-gather keeps process order (halo_ipc_import expects rank order)
    blobs = [None] * world
    dist.all_gather_object(blobs, bytes([rank]) * 16)
    res["blobs"] = [b[0] for b in blobs]
    # max-over-ranks reduction used by bench.py
    import bench
    res["max"] = bench.max_over_ranks(float(rank + 1) * 2.5)
    out[rank] = res
    dist.destroy_process_group()


def test_two_process_partition_and_reductions():
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        out = dict(out)
    for rank in range(2):
        r = out[rank]
        assert r["blobs"] == [0, 1]
        assert r["max"] == 5.0
        for name in ["C3", "C2", "C5", "T4x2"]:
            rows = r[name]
            covered = []
            for (pr, first, nl, dims, sb) in rows:
                covered += list(range(first, first + nl))
            from synth import get_config
            c = get_config(name)
            assert sorted(covered) == list(range(c.nranks))  # every DD rank hosted exactly once
            assert len({tuple(x[3]) for x in rows}) == 1 and len({x[4] for x in rows}) == 1
            assert len(rows[0][3]) == sum(c.pulses)
            assert rows[0][3] == sorted(rows[0][3], reverse=True)  # z -> y -> x
