"""Debug: 2-process C1 force halo — dump fbuf vs expected slice and mismatch pattern."""
import os
import socket
import sys

import numpy as np
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, name):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_21527_b200.session import HaloSession
    from tests.parity_common import Case
    case = Case(name, seed=1, force_kind="int")
    sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=3, capacity=case.capacity, device=rank,
                       nprocs=world, proc=rank, timeout_s=10.0)
    first, nl = sess.first_rank, sess.n_local
    print(f"[{rank}] ptrs x={sess.x[0].data_ptr():#x} f={sess.f[0].data_ptr():#x} s={sess.scratch[0].data_ptr():#x}",
          flush=True)
    sess.load_home([case.home_rows(first + l) for l in range(nl)])
    sess.set_maps()
    sess.exchange_x()
    torch.cuda.synchronize()
    for l in range(nl):
        r = first + l
        n = case.F[r].shape[0]
        sess.f[l][:n] = torch.from_numpy(case.F[r]).to(sess.device)
    torch.cuda.synchronize()
    dist.barrier()
    fshift = torch.zeros(nl, 3, 3, dtype=torch.float64, device=sess.device)
    sess.exchange_f(fshift=fshift)
    torch.cuda.synchronize()
    try:
        sess.halo.sync()
        print(f"[{rank}] sync ok", flush=True)
    except Exception as e:
        print(f"[{rank}] sync error {e}", flush=True)
    P = sess.npulse
    cap = sess.capacity
    import math
    map_stride = (cap + 63) // 64 * 64
    fb_off = 4096 + P * map_stride * 4
    for l in range(nl):
        r = first + l
        st = case.states[r]
        n = case.F[r].shape[0]
        got = sess.f[l][:n].cpu().numpy()
        exp = case.Fo[r]
        bad = np.nonzero(np.any(got != exp, axis=1))[0]
        print(f"[{rank}] rank {r}: n_home {st.n_home} n_total {n} bad rows {bad.size} first {bad[:8]}", flush=True)
        for p in range(P):
            pi = st.pulses[p]
            u = pi.send_rank
            ui = case.states[u].pulses[p]
            exp_slice = case.F[u][ui.atom_offset: ui.atom_offset + ui.recv_size]
            raw = sess.scratch[l].cpu().numpy()
            fb = raw[fb_off: fb_off + pi.send_size * 12].view(np.float32).reshape(-1, 3)
            nbad = np.count_nonzero(np.any(fb != exp_slice, axis=1))
            print(f"[{rank}]  pulse {p}: send {pi.send_size} fbuf mismatches {nbad}; fbuf[:2]={fb[:2].tolist()} "
                  f"exp[:2]={exp_slice[:2].tolist()}", flush=True)
            hdr = raw[:4096].view(np.uint64)
            print(f"[{rank}]  flags x={hdr[0:2].tolist()} f={hdr[16:18].tolist()}", flush=True)
        if bad.size:
            i = bad[0]
            print(f"[{rank}]  row {i}: got {got[i].tolist()} exp {exp[i].tolist()} F {case.F[r][i].tolist()}",
                  flush=True)
    dist.barrier()
    sess.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    name = sys.argv[1] if len(sys.argv) > 1 else "C1"
    mp.spawn(worker, args=(2, port, name), nprocs=2, join=True)
