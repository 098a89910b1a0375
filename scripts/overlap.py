"""Overlap of the halo exchange with compute (paper Alg. 2 P:229-243,
device-side timing P:537-541).

The GPU-resident time-step skeleton of Alg. 2 with synthetic non-bonded work:

    update stream : [step start] ........................ wait(L) wait(N) -> integrate
    local stream  : Local NB (synthetic GEMM, ns_per_atom x home atoms)
    non-local (high priority): exchange_x -> Non-local NB (ns_per_atom x halo atoms) -> exchange_f

The synthetic NB kernels are bf16 cuBLAS GEMMs sized (calibrated once) to take
``ns_per_atom`` (default 1.85 ns, the paper's 1.7-2.0 ns/atom) times the
atoms: a load that occupies every SM, so the halo kernels run under SM
contention.  No L2 flush (steady state: the GEMMs evict L2 anyway).

Reports the paper's device-side metrics, max over ranks:
  local      Local work: start -> end of the local NB kernel
  nonlocal   Non-local work: start of exchange_x -> end of exchange_f
  nonoverlap end of local NB -> end of exchange_f, clamped at 0
  step       time per step (step start -> next step start)
for the fused LL kernels, the paper-flag protocol, the copy-engine path and
(one DD rank per GPU) the NCCL send/recv schedule; plus the same step with no
exchange (compute only) — the exchange's cost is step - compute-only step.

    python scripts/overlap.py --config C3
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/overlap.py --config C1
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PROTOS = {"ll": 0, "paper": 1 << 4, "ce": 1 << 5}


def calibrate_gemm(dev, target_us):
    """Square bf16 GEMM size whose duration is ~target_us (>= 64)."""
    if target_us <= 0:
        return 0
    sizes = [256, 384, 512, 768, 1024, 1536, 2048, 3072, 4096, 6144, 8192]
    best, times = 0, {}
    for n in sizes:
        a = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
        b = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
        for _ in range(3):
            torch.mm(a, b)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            torch.mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        times[n] = e0.elapsed_time(e1) * 1e3 / 10
        if times[n] >= target_us:
            break
    # interpolate on n^3
    ns = sorted(times)
    for lo, hi in zip(ns, ns[1:]):
        if times[lo] <= target_us <= times[hi]:
            f = (target_us - times[lo]) / max(times[hi] - times[lo], 1e-9)
            n3 = lo ** 3 + f * (hi ** 3 - lo ** 3)
            return max(64, int(round(n3 ** (1 / 3) / 64)) * 64)
    return ns[-1] if target_us > times[ns[-1]] else ns[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--ns-per-atom", type=float, default=1.85)
    ap.add_argument("--protos", default="ll,paper,ce,nccl")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    import bench
    from paper_2509_21527_b200.nccl_baseline import NcclSchedule
    from paper_2509_21527_b200.session import HaloSession, assign_home
    from synth import forces_normal

    c, X = bench.build_workload(args.config)
    homes = assign_home(X, c.L, c.grid)
    cap = int(max(len(h) for h in homes) * 2.2) + 4096
    nl_ranks = c.nranks // world
    first = rank * nl_ranks
    n_home = sum(len(homes[first + l]) for l in range(nl_ranks))

    def mx(v):
        return bench.max_over_ranks(v)

    results = []
    sizes = None
    for proto in args.protos.split(","):
        if proto == "nccl" and (world == 1 or nl_ranks != 1):
            continue
        flags = PROTOS.get(proto, 0)
        sess = HaloSession(c.grid, c.L, c.rc, c.pulses, capacity=cap, device=local, flags=flags, nprocs=world,
                           proc=rank, timeout_s=20.0)
        sess.load_home([X[homes[first + l]] for l in range(nl_ranks)])
        sess.set_maps()
        lay = [sess.layout_of(l) for l in range(nl_ranks)]
        n_halo = sum(l_["n_total"] - l_["n_home"] for l_ in lay)
        if sizes is None:  # calibrate once (same for every protocol)
            sizes = (calibrate_gemm(dev, args.ns_per_atom * n_home / 1e3),
                     calibrate_gemm(dev, args.ns_per_atom * n_halo / 1e3))
        nloc, nnl = sizes
        A = torch.randn(max(nloc, 64), max(nloc, 64), device=dev, dtype=torch.bfloat16)
        B = torch.randn(max(nnl, 64), max(nnl, 64), device=dev, dtype=torch.bfloat16)
        F0 = torch.zeros_like(sess.f_all)
        for l in range(nl_ranks):
            n = lay[l]["n_total"]
            F0[l, :n] = torch.from_numpy(forces_normal(n, 900 + first + l)).to(dev)
        fshift = torch.zeros(nl_ranks, 3, 3, dtype=torch.float64, device=dev)
        s_upd = torch.cuda.current_stream()
        s_loc = torch.cuda.Stream(device=dev, priority=0)
        s_nl = torch.cuda.Stream(device=dev, priority=-1)
        sched = NcclSchedule(sess) if proto == "nccl" else None

        def step(k, ev, exchange=True):
            ev["start"][k].record(s_upd)
            s_loc.wait_event(ev["start"][k])
            s_nl.wait_event(ev["start"][k])
            with torch.cuda.stream(s_loc):
                ev["l0"][k].record(s_loc)
                if nloc:
                    torch.mm(A, A)
                ev["l1"][k].record(s_loc)
            with torch.cuda.stream(s_nl):
                ev["n0"][k].record(s_nl)
                if exchange:
                    if sched is not None:
                        sched.exchange_x(stream=s_nl)
                    else:
                        sess.exchange_x(stream=s_nl)
                if nnl:
                    torch.mm(B, B)
                if exchange:
                    if sched is not None:
                        sched.exchange_f(fshift, stream=s_nl)
                    else:
                        sess.exchange_f(fshift=fshift, stream=s_nl)
                ev["n1"][k].record(s_nl)
            s_upd.wait_event(ev["l1"][k])
            s_upd.wait_event(ev["n1"][k])
            sess.f_all.copy_(F0)  # "integration": consumes the forces, resets them for the next step

        out = {}
        for exchange in (True, False):
            K = args.steps
            ev = {k: [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)] for k in ("start", "l0", "l1", "n0", "n1")}
            for k in range(args.warmup):
                step(0, ev, exchange)
            torch.cuda.synchronize()
            bench.barrier()
            for k in range(K):
                step(k, ev, exchange)
            ev["start"][K].record(s_upd)
            torch.cuda.synchronize()
            bench.barrier()
            loc = np.mean([ev["l0"][k].elapsed_time(ev["l1"][k]) * 1e3 for k in range(K)])
            non = np.mean([ev["n0"][k].elapsed_time(ev["n1"][k]) * 1e3 for k in range(K)])
            nov = np.mean([max(0.0, ev["l1"][k].elapsed_time(ev["n1"][k]) * 1e3) for k in range(K)])
            stp = np.mean([ev["start"][k].elapsed_time(ev["start"][k + 1]) * 1e3 for k in range(K)])
            key = "" if exchange else "compute_only_"
            out.update({key + "local_us": round(mx(loc), 2), key + "nonlocal_us": round(mx(non), 2),
                        key + "nonoverlap_us": round(mx(nov), 2), key + "step_us": round(mx(stp), 2)})
        out["exchange_cost_us"] = round(out["step_us"] - out["compute_only_step_us"], 2)
        res = {"config": c.name, "gpus": world, "proto": proto, "ns_per_atom": args.ns_per_atom,
               "home_atoms_per_gpu": n_home, "halo_atoms_per_gpu": n_halo, "gemm_local": nloc, "gemm_nonlocal": nnl,
               **out}
        results.append(res)
        sess.destroy()
        bench.barrier()
    if rank == 0:
        for r in results:
            print(json.dumps(r), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
