"""Per-CTA device timeline of one x+f step (HALO_F_TIMERS trace), after W warm-up steps.

    python scripts/trace.py --config C3 [--flush]
    torchrun --nproc-per-node 2 scripts/trace.py --config C1 --flush

Prints, per kernel, quantiles (µs, relative to the x kernel's first CTA start)
of CTA start / plan-record loaded / items done / exit, and the gap between the
x kernel's last exit and the f kernel's first start.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def q(a):
    return [round(float(v), 2) for v in np.quantile(a, [0.0, 0.5, 0.9, 1.0])]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--flush", action="store_true")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--no-fshift", action="store_true")
    ap.add_argument("--no-mid-event", action="store_true", help="no event between x and f (keeps PDL)")
    ap.add_argument("--queue", type=int, default=0, help="queue this many un-synchronised steps before the traced one")
    ap.add_argument("--fused", action="store_true", help="trace the fused x+f launch (halo_exchange_xf)")
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
    sess = HaloSession(c.grid, c.L, c.rc, c.pulses, capacity=cap, device=local, flags=HALO_F_TIMERS | args.flags,
                       nprocs=world, proc=rank, timeout_s=20.0)
    first, nl = sess.first_rank, sess.n_local
    sess.load_home([X[homes[first + l]] for l in range(nl)])
    sess.set_maps()
    F0 = [torch.from_numpy(forces_normal(sess.layout_of(l)["n_total"], 1 + l)).to(dev) for l in range(nl)]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    fshift = torch.zeros(nl, 3, 3, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream()
    out = []
    F0_all = torch.zeros_like(sess.f_all)
    for l in range(nl):
        F0_all[l, : F0[l].shape[0]] = F0[l]
    def one_step():
        if args.fused:
            sess.exchange_xf(fshift=None if args.no_fshift else fshift)
        else:
            sess.exchange_x()
            sess.exchange_f(fshift=None if args.no_fshift else fshift)

    for k in range(args.steps):
        if world > 1:
            torch.cuda.synchronize()
            dist.barrier()  # start every traced step together (host skew is not kernel time)
        for _ in range(args.queue):  # steady state: the host runs ahead of the GPU
            if args.flush:
                flush.fill_(1.0)
            sess.f_all.copy_(F0_all)
            one_step()
        if args.flush:
            flush.fill_(1.0)
        sess.f_all.copy_(F0_all)
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(st)
        if args.fused:
            sess.exchange_xf(fshift=None if args.no_fshift else fshift)
        else:
            sess.exchange_x()
            if not args.no_mid_event:
                e1.record(st)
            sess.exchange_f(fshift=None if args.no_fshift else fshift)
        e2.record(st)
        torch.cuda.synchronize()
        tx = sess.halo.get_trace(0).astype(np.int64)
        tf = tx if args.fused else sess.halo.get_trace(1).astype(np.int64)
        t0 = tx[:, 0].min()
        mid = not (args.no_mid_event or args.fused)
        res = {
            "step": k, "rank": rank, "fused": args.fused,
            "x_event_us": round(e0.elapsed_time(e1) * 1e3, 2) if mid else None,
            "f_event_us": round(e1.elapsed_time(e2) * 1e3, 2) if mid else None,
            "step_event_us": round(e0.elapsed_time(e2) * 1e3, 2), "x_ctas": int(tx.shape[0]), "f_ctas": int(tf.shape[0]),
            "x_start": q((tx[:, 0] - t0) / 1e3), "x_rec": q((tx[:, 1] - t0) / 1e3),
            "x_done": q((tx[:, 2] - t0) / 1e3), "x_exit": q((tx[:, 3] - t0) / 1e3),
        }
        if not args.fused:
            res.update({"gap_x_exit_to_f_start": round(float((tf[:, 0].min() - tx[:, 3].max()) / 1e3), 2),
                        "f_start": q((tf[:, 0] - t0) / 1e3), "f_rec": q((tf[:, 1] - t0) / 1e3),
                        "f_done": q((tf[:, 2] - t0) / 1e3), "f_exit": q((tf[:, 3] - t0) / 1e3)})
        if os.environ.get("HALO_DEBUG") == "8192":  # kTraceDetail: stamps inside the first tree item
            for nm, tr in (("x", tx), ("f", tf)):  # griddepcontrol.wait released / prologue done (slots 14, 15)
                if (tr[:, 14] > 0).all():
                    res[nm + "_wait_released"] = q((tr[:, 14] - t0) / 1e3)
                    res[nm + "_prologue_done"] = q((tr[:, 15] - t0) / 1e3)
            tr = tf
            m = (tr[:, 10] > 0) & (tr[:, 13] >= tr[:, 10])
            if m.any():
                d = tr[m]
                res["detail_rec_to_records"] = q((d[:, 10] - d[:, 1]) / 1e3)
                res["detail_records_to_loads"] = q((d[:, 11] - d[:, 10]) / 1e3)
                res["detail_loads_to_fold"] = q((d[:, 12] - d[:, 11]) / 1e3)
                res["detail_fold_to_flushed"] = q((d[:, 13] - d[:, 12]) / 1e3)
                res["detail_flush_to_itemend"] = q((d[:, 5] - d[:, 13]) / 1e3)
        # per (kind, level) item end quantiles [min, median, p90, max, count], µs relative
        # to the first CTA start of the (x or fused) launch
        kinds = {4: "xrecv", 6: "fshift", 7: "xsend", 8: "tree"}
        for nm, tr in ((("xf", tx),) if args.fused else (("x", tx), ("f", tf))):
            groups = {}
            for row in tr:
                for sl in range((tr.shape[1] - 4) // 2):
                    tag, end = int(row[4 + 2 * sl]), int(row[5 + 2 * sl])
                    if end == 0 or end < tr[:, 0].min():
                        continue
                    lev = tag & 0xff
                    key = f"{kinds.get(tag >> 16, tag >> 16)}_p{'home' if lev == 255 else lev}"
                    groups.setdefault(key, []).append((end - t0) / 1e3)
            res[nm + "_items"] = {k: q(np.array(v)) + [len(v)] for k, v in sorted(groups.items())}
        out.append(res)
    if world > 1:
        allres = [None] * world
        dist.all_gather_object(allres, out[-1])
    else:
        allres = [out[-1]]
    if rank == 0:
        for r in allres:
            print(json.dumps(r), flush=True)
    sess.destroy()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
