"""Variant sweep of the fused x+f step (timing only; parity is covered by tests/).

    python scripts/sweep.py --config C3 --steps 300 [--flush]
    torchrun --nproc-per-node 2 scripts/sweep.py ...

Each variant = (env overrides, flags).  Prints one JSON line per variant with
eager x/f/step µs (mean, max over ranks) and device-side kernel spans.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

VARIANTS = {
    "base": ({}, 0),
    "poll32": ({"HALO_POLL_NS": "32"}, 0),
    "poll64": ({"HALO_POLL_NS": "64"}, 0),
    "poll128": ({"HALO_POLL_NS": "128"}, 0),
    "poll256": ({"HALO_POLL_NS": "256"}, 0),
    "poll512": ({"HALO_POLL_NS": "512"}, 0),
    "rows32": ({"HALO_ITEM_ROWS": "32"}, 0),
    "rows64": ({"HALO_ITEM_ROWS": "64"}, 0),
    "rows128": ({"HALO_ITEM_ROWS": "128"}, 0),
    "rows256": ({"HALO_ITEM_ROWS": "256"}, 0),
    "rows96": ({"HALO_ITEM_ROWS": "96"}, 0),
    "rows192": ({"HALO_ITEM_ROWS": "192"}, 0),
    "paper": ({}, 16),
    "paper_gpufence": ({}, 16 | 4),
    "rows1024": ({"HALO_ITEM_ROWS": "1024"}, 0),
    "rows2048": ({"HALO_ITEM_ROWS": "2048"}, 0),
    "gpufence": ({}, 4),
    "atomic": ({}, 1),
    "nocoop": ({"HALO_COOP": "0"}, 0),
    "nocoop_gpufence": ({"HALO_COOP": "0"}, 4),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--flush", action="store_true")
    ap.add_argument("--variants", default=",".join(VARIANTS))
    ap.add_argument("--layout", type=int, default=3)
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
    import bench
    from paper_2509_21527_b200 import HALO_F_TIMERS
    from paper_2509_21527_b200.session import HaloSession, assign_home
    from synth import forces_normal
    c, X = bench.build_workload(args.config)
    homes = assign_home(X, c.L, c.grid, c.rc, c.pulses)
    cap = int(max(len(h) for h in homes) * 2.2) + 4096
    dev = torch.device("cuda", local)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    # reference: back-to-back tiny torch kernels (launch floor of a plain launch)
    tiny = torch.zeros(1, device=dev)
    st0 = torch.cuda.current_stream()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(200)]
    for k in range(220):
        kk = k - 20
        if kk >= 0:
            evs[kk][0].record(st0)
        tiny.add_(1.0)
        if kk >= 0:
            evs[kk][1].record(st0)
        tiny.add_(1.0)
        if kk >= 0:
            evs[kk][2].record(st0)
    torch.cuda.synchronize()
    if rank == 0:
        print(json.dumps({"variant": "torch_tiny_kernel", "us": round(float(np.mean(
            [e[0].elapsed_time(e[1]) * 1e3 for e in evs])), 2), "us2": round(float(np.mean(
            [e[1].elapsed_time(e[2]) * 1e3 for e in evs])), 2)}), flush=True)
    for name in args.variants.split(","):
        env, flags = VARIANTS[name]
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        sess = HaloSession(c.grid, c.L, c.rc, c.pulses, layout=args.layout, capacity=cap, device=local,
                           flags=flags | HALO_F_TIMERS, nprocs=world, proc=rank, timeout_s=20.0)
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        first, nl = sess.first_rank, sess.n_local
        sess.load_home([X[homes[first + l]] for l in range(nl)])
        sess.set_maps()
        F0 = [torch.from_numpy(forces_normal(sess.layout_of(l)["n_total"], 1 + l, width=args.layout)).to(dev)
              for l in range(nl)]
        st = torch.cuda.current_stream()
        fshift = torch.zeros(nl, 3, 3, dtype=torch.float64, device=dev)
        K = args.steps
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
        spans = []
        F0_all = torch.zeros_like(sess.f_all)
        for l in range(nl):
            F0_all[l, : F0[l].shape[0]] = F0[l]
        for k in range(K + 20):
            sess.f_all.copy_(F0_all)
            if args.flush:
                flush.fill_(1.0)
            kk = k - 20
            if kk >= 0:
                ev[kk][0].record(st)
            sess.exchange_x()
            if kk >= 0:
                ev[kk][1].record(st)
            sess.exchange_f(fshift=fshift)
            if kk >= 0:
                ev[kk][2].record(st)
            if kk >= 0 and kk % 50 == 0:
                torch.cuda.synchronize()
                spans.append(sess.halo.get_timers())
        torch.cuda.synchronize()
        xs = float(np.mean([e[0].elapsed_time(e[1]) * 1e3 for e in ev]))
        fs = float(np.mean([e[1].elapsed_time(e[2]) * 1e3 for e in ev]))
        sx = float(np.mean([s[0] for s in spans])) / 1e3
        sf = float(np.mean([s[1] for s in spans])) / 1e3
        res = {k: bench.max_over_ranks(v) for k, v in dict(x=xs, f=fs, span_x=sx, span_f=sf).items()}
        if rank == 0:
            print(json.dumps({"variant": name, "config": c.name, "n_gpus": world, "flush": args.flush,
                              **{k: round(v, 2) for k, v in res.items()}}), flush=True)
        sess.destroy()
        bench.barrier()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
