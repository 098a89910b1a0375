#!/usr/bin/env python
"""bench.py — x+f halo exchange µs/step on 1/2/4/8 B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl fused|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU)

A step = one exchange_x + one exchange_f of the whole DD grid (every §8(a)
row).  The workload's DD ranks are spread over the N GPUs (nranks/N per GPU,
all of a GPU's ranks in one kernel launch); the system is fixed as N grows
(strong scaling).  Timing: W warm-up steps, then K steps, each preceded by
an L2 flush (256 MiB write) and the reset of f to this step's non-bonded
forces (both outside the timed spans); CUDA events on the launching stream;
max over ranks.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

if "--cpu-child" in sys.argv or "reference" in sys.argv:
    # the oracle legs run single-threaded (OMP/MKL/OPENBLAS_NUM_THREADS=1, one pinned core)
    for _v in ("OMP_NUM_THREADS", "MKL_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        os.environ[_v] = "1"

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# HALO_F_PAPER_FLAGS (+ HALO_F_TMA_STORE | HALO_F_TMA_GET: the paper's TMA put / get), HALO_F_CE_PATH
PROTO_FLAGS = {"ll": 0, "paper": 1 << 4, "paper_tma": (1 << 4) | (1 << 7) | (1 << 8), "ce": 1 << 5,
               "auto": 1 << 10}  # HALO_F_AUTO_TRANSPORT: LL or copy engine by pulse size, per NS epoch
METRIC = "x+f halo exchange us/step (max over ranks); achieved NVLink GB/s vs 900"
UNIT = "us/step"
SEED = 2509


# ------------------------------------------------------------------ dist utils
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def max_over_ranks(v: float) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(v)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(v: float) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(v)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


# ------------------------------------------------------------------ workload
def build_workload(cfg_name):
    from synth import get_config, water_box
    c = get_config(cfg_name)
    X = water_box(c.n_atoms, c.L, SEED, slab=c.slab)
    return c, X


def workload_desc(c, n_gpus, layout):
    return {"workload": f"{c.name}: {c.desc}", "n_atoms": int(c.n_atoms), "grid": list(c.grid),
            "pulses": list(c.pulses), "rc_nm": c.rc, "box_nm": list(c.L), "dd_ranks": c.nranks,
            "dd_ranks_per_gpu": c.nranks // n_gpus, "layout": f"float{layout}", "seed": SEED,
            "l2": "flushed: 256 MiB write before every timed step (then f is reset, so the forces are "
                  "L2-resident as the non-bonded kernel leaves them; x, plan, maps, LL buffers are flushed)",
            "forces": "normal(0,300) float32, reset before every step"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clocks and throttle reasons of the GPUs in use during the timed region (NVML)."""

    def __init__(self, devices, period_s=0.005):
        self.devices, self.period = devices, period_s
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.handles = [pynvml.nvmlDeviceGetHandleByIndex(d) for d in devices]
            self.max_mhz = max(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM) for h in self.handles)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4): "sw_power_cap",
            getattr(nv, "nvmlClocksThrottleReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake_slowdown",
        }
        while not self._stop.is_set():
            for h in self.handles:
                try:
                    self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    for bit, name in names.items():
                        if r & bit:
                            self.reasons.add(name)
                except Exception:
                    pass
            time.sleep(self.period)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "NVML unavailable"}
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


class NvlCounters:
    """This GPU's NVLink data counters (NVML field values NVLINK_THROUGHPUT_DATA_TX/RX: user
    payload bytes, KiB units, summed over every link with scopeId = UINT_MAX; per link if the
    aggregate is not supported).  Read on both sides of the timed region: the hardware's own
    count of the bytes the exchanges moved over NVLink, beside the algorithmic figure."""

    def __init__(self, device):
        self.ok, self.err = False, None
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(device)
            self.links = [0xFFFFFFFF]
            if self._read_raw(self.links) is None:
                self.links = list(range(18))
                if self._read_raw(self.links) is None:
                    raise RuntimeError("NVLink throughput field values not supported")
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML / no NVLink here
            self.err = str(e)[:200]

    def _read_raw(self, links):
        nv = self.nv
        ids = []
        for l in links:
            ids += [(nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, l), (nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, l)]
        vals = nv.nvmlDeviceGetFieldValues(self.h, ids)
        tx = rx = 0
        seen = False
        for i, v in enumerate(vals):
            if v.nvmlReturn != 0:
                continue
            seen = True
            x = int(v.value.ullVal)
            if i % 2 == 0:
                tx += x
            else:
                rx += x
        return (tx * 1024, rx * 1024) if seen else None

    def read(self):
        if not self.ok:
            return None
        try:
            return self._read_raw(self.links)
        except Exception:  # pragma: no cover
            return None


# ------------------------------------------------------------------ cpu legs
def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def pin_one_core():
    """Pin this process to one allowed core (taskset -c <first allowed>); returns it."""
    try:
        cpu = min(os.sched_getaffinity(0))
        os.sched_setaffinity(0, {cpu})
        return cpu
    except (AttributeError, OSError):
        return None


def oracle_step_timing(c, X, budget_s=15.0, max_steps=None, warmup=1):
    """The oracle (as it stands) per step: fixed-map x halo + force halo, all DD
    ranks serially, on this host; maps built once outside the timed region.
    Returns (mean us/step, steps, best-of-5 us/step)."""
    from oracle import coord_halo_step, decompose, force_halo  # cpu_baseline leg only
    from synth import forces_normal
    states = decompose(X, c.L, c.rc, c.grid, c.pulses)
    F = [forces_normal(s.x.shape[0], 77 + s.rank) for s in states]
    xh = [s.x[: s.n_home].copy() for s in states]
    for _ in range(warmup):
        coord_halo_step(states, xh)
        force_halo(states, F)
    n, ts, t0 = 0, [], time.perf_counter()
    while True:
        a = time.perf_counter()
        coord_halo_step(states, xh)
        force_halo(states, F)
        ts.append(time.perf_counter() - a)
        n += 1
        el = time.perf_counter() - t0
        if el >= budget_s or (max_steps is not None and n >= max_steps):
            break
    best5 = min(float(np.mean(ts[i:i + max(1, n // 5)])) for i in range(0, n, max(1, n // 5)))
    return el / n * 1e6, n, best5 * 1e6


def oracle_c1_pipeline():
    """BASELINE.json configs[0] ("CPU oracle in seconds"): the whole C1 oracle pipeline —
    generate the 3,000-atom box, decomposition + maps, x halo + force halo, and the
    brute-force pins X2 (import zones), X3 (pair coverage), F1-F3 (integer forces: totals,
    conservation, shift forces) — wall seconds on this core."""
    from oracle import decompose, force_halo  # cpu_baseline leg only
    from synth import forces_int, get_config, water_box
    from tests import pins  # test-only brute-force checks
    t0 = time.perf_counter()
    c = get_config("C1")
    X = water_box(c.n_atoms, c.L, 1)
    st = decompose(X, c.L, c.rc, c.grid, c.pulses)
    F = [forces_int(s.x.shape[0], 100 + s.rank) for s in st]
    Fo, fs = force_halo(st, [f.copy() for f in F])
    t_core = time.perf_counter() - t0
    ok = True
    for s in st:  # X2
        inner, outer = pins.direct_gather(X, c.L, c.rc, c.grid, s.rank, eps=1e-5)
        hs = {(int(g), tuple(int(v) for v in sv)) for g, sv in zip(s.gid, s.s)}
        ok &= inner <= hs <= outer
    index = []
    for s in st:  # X3
        m = {}
        for g, sv in zip(s.gid, s.s):
            m.setdefault(int(g), set()).add(tuple(int(v) for v in sv))
        index.append(m)
    dec = [d for d in range(3) if c.grid[d] > 1]
    pairs = pins.close_pairs(X, c.L, c.rc, eps=1e-5)
    for i, j, n in pairs:
        ok &= any(any(all(b[d] - a[d] == n[d] for d in dec) for a in m.get(i, ()) for b in m.get(j, ()))
                  for m in index)
    tot = pins.scatter_totals([s.gid for s in st], F, X.shape[0])  # F1
    got = np.zeros((X.shape[0], 3))
    for s, f in zip(st, Fo):
        got[s.gid[:s.n_home]] = f[:s.n_home]
    ok &= bool(np.array_equal(got, tot))
    before = sum(f.astype(np.float64).sum(axis=0) for f in F)  # F2
    after = sum(f[:s.n_home].astype(np.float64).sum(axis=0) for s, f in zip(st, Fo))
    ok &= bool(np.array_equal(before, after))
    fs_tot = sum(fs)  # F3
    for d in range(3):
        exp = sum(f[s.s[:, d] == 1].astype(np.float64).sum(axis=0) for s, f in zip(st, F))
        ok &= bool(np.array_equal(fs_tot[d], exp))
    return {"seconds": round(time.perf_counter() - t0, 2), "core_seconds": round(t_core, 3),
            "pairs_checked": len(pairs), "pins_ok": bool(ok),
            "what": "C1: generate 3,000 atoms + decomposition/maps + x halo + force halo (core_seconds), "
                    "then brute-force pins X2, X3 (every pair within rc co-resident), F1-F3"}


def cpu_child(args):
    """--cpu-child: the cpu_baseline leg in its own pinned, single-threaded process."""
    cpu = pin_one_core()
    c, X = build_workload(args.config)
    us, n, best = oracle_step_timing(c, X, budget_s=args.cpu_budget)
    out = {"us": us, "n": n, "best5_us": best, "cpu": cpu}
    if not args.no_c1_pipeline:
        out["c1_pipeline"] = oracle_c1_pipeline()
    print(json.dumps(out), flush=True)


def cpu_baseline_leg(args, P, c):
    import subprocess
    env = dict(os.environ, OMP_NUM_THREADS="1", MKL_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1")
    cmd = [sys.executable, os.path.abspath(__file__), "--cpu-child", "--config", args.config,
           "--cpu-budget", str(args.cpu_budget)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    if r.returncode != 0:
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "oracle", "error": r.stderr[-400:]}
    d = json.loads(r.stdout.strip().splitlines()[-1])
    out = {"value": round(d["us"], 1), "unit": UNIT, "cores": 1, "kind": "oracle",
           "best_of_5_us": round(d["best5_us"], 1),
           "sample": f"{c.name} full workload ({c.nranks} DD ranks, {P} pulses), {d['n']} oracle steps "
                     f"(fixed-map x halo + force halo, all ranks serially), numpy, one thread pinned to "
                     f"core {d['cpu']} (OMP/MKL/OPENBLAS_NUM_THREADS=1)",
           **host_info()}
    if "c1_pipeline" in d:
        out["c1_pipeline"] = d["c1_pipeline"]
    return out


# ------------------------------------------------------------------ main arm
def run_fused(args, rank, world, local):
    import torch
    import torch.distributed as dist

    from paper_2509_21527_b200 import HALO_F_TIMERS
    from paper_2509_21527_b200.session import HaloSession, assign_home
    from synth import forces_normal

    c, X = build_workload(args.config)
    if c.nranks % world != 0:
        raise SystemExit(f"config {c.name} has {c.nranks} DD ranks, not divisible by {world} GPUs")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    homes = assign_home(X, c.L, c.grid, c.rc, c.pulses, device=local)
    cap = int(max(len(h) for h in homes) * 2.2) + 4096
    flags = (HALO_F_TIMERS if args.timers else 0) | PROTO_FLAGS[args.proto] | ((1 << 6) if args.l2_persist else 0)
    flags |= (1 << 9) if args.zones == "rounded" else 0  # HALO_F_ROUNDED_ZONES (R31)
    sess = HaloSession(c.grid, c.L, c.rc, c.pulses, layout=args.layout, capacity=cap, device=local, flags=flags,
                       nprocs=world, proc=rank, timeout_s=20.0, pme_rank=0 if args.pme else None,
                       probe_bytes=(64 << 20) if (world > 1 and not args.no_floors) else None)
    first, nl = sess.first_rank, sess.n_local
    sess.load_home([X[homes[first + l]] for l in range(nl)])
    sess.set_maps()
    transport = sess.halo.transport()  # --proto auto: the one set_maps chose
    lay = [sess.layout_of(l) for l in range(nl)]
    P = sess.npulse
    W = args.layout
    F0 = []
    F0_all = torch.zeros_like(sess.f_all)  # this step's non-bonded forces, all local ranks
    for l in range(nl):
        n = lay[l]["n_total"]
        F0.append(torch.from_numpy(forces_normal(n, 5000 + first + l, width=W)).to(dev))
        F0_all[l, :n] = F0[l]
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    fshift = torch.zeros(nl, 3, 3, dtype=torch.float64, device=dev)

    def reset_f():
        sess.f_all.copy_(F0_all)  # one op: keeps the host ahead of the GPU

    def step():
        sess.exchange_x()
        sess.exchange_f(fshift=fshift)

    for _ in range(args.warmup):
        flush.fill_(1.0)
        reset_f()
        step()
    torch.cuda.synchronize()
    barrier()

    sampler = ClockSampler([local])
    sampler.start()
    nvc = NvlCounters(local) if world > 1 else None
    K = args.steps
    # main timed loop: events only at the step boundaries, so exchange_f is
    # launched right behind exchange_x (programmatic dependent launch)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    torch.cuda.synchronize()
    barrier()
    nv0 = nvc.read() if nvc else None
    t_wall0 = time.perf_counter()
    for k in range(K):
        flush.fill_(float(k))
        reset_f()
        ev[k][0].record(stream)
        sess.exchange_x()
        sess.exchange_f(fshift=fshift)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall0
    nv1 = nvc.read() if nvc else None
    barrier()
    tot = [ev[k][0].elapsed_time(ev[k][1]) * 1e3 for k in range(K)]
    nvl_counted = None
    if nvc is not None:  # every rank takes part in the reductions (collectives)
        have = nv0 is not None and nv1 is not None
        per = [(nv1[i] - nv0[i]) / K for i in range(2)] if have else [-1.0, -1.0]
        tx_max, rx_max = max_over_ranks(per[0]), max_over_ranks(per[1])
        tx_min = -max_over_ranks(-per[0])
        if tx_min >= 0:
            nvl_counted = {"tx_bytes_per_step": round(tx_max, 1), "rx_bytes_per_step": round(rx_max, 1),
                           "source": "NVML NVLINK_THROUGHPUT_DATA_TX/RX (user payload, KiB counters) read around the "
                                     "K timed steps, max over ranks; the flush and reset in that loop are local",
                           "wall_s": round(t_wall, 4)}
        else:
            nvl_counted = {"unavailable": (nvc.err or "NVML NVLink field read failed") + " (on some rank)"}
    # the same steps as ONE fused launch each (halo_exchange_xf, LL protocol)
    fused = None  # timed last (fused_timing): a failure there cannot take the other numbers with it
    sampler.stop()
    # per-kernel split (roofline): isolated steps (device idle, ranks released together by a
    # host barrier), events around each kernel, same flush discipline
    Kx = min(K, 200)
    ev3 = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(Kx)]
    for k in range(Kx):
        flush.fill_(float(k))
        reset_f()
        torch.cuda.synchronize()
        barrier()
        # ~40 us of GPU sleep: the host enqueues x and f behind it, so the events time
        # device execution, not the host's launch submission
        torch.cuda._sleep(80000)
        ev3[k][0].record(stream)
        sess.exchange_x()
        ev3[k][1].record(stream)
        sess.exchange_f(fshift=fshift)
        ev3[k][2].record(stream)
    torch.cuda.synchronize()
    barrier()
    xs = [ev3[k][0].elapsed_time(ev3[k][1]) * 1e3 for k in range(Kx)]
    fs = [ev3[k][1].elapsed_time(ev3[k][2]) * 1e3 for k in range(Kx)]
    my = {"step": float(np.mean(tot)), "x": float(np.mean(xs)), "f": float(np.mean(fs)),
          "step_median": float(np.median(tot)), "step_p90": float(np.percentile(tot, 90)),
          "step_p99": float(np.percentile(tot, 99)), "step_max": float(np.max(tot)),
          "x_median": float(np.median(xs)), "f_median": float(np.median(fs))}
    res = {k: max_over_ranks(v) for k, v in my.items()}
    dev_spans = None
    if args.timers:
        tx, tf = sess.halo.get_timers()
        dev_spans = {"x_us": max_over_ranks(tx / 1e3), "f_us": max_over_ranks(tf / 1e3)}

    # CUDA-graph mode: one captured x+f step, replayed (flush between replays)
    graph_us = None
    if not args.no_graph:
        gs = torch.cuda.Stream(device=dev)
        g = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        barrier()
        with torch.cuda.graph(g, stream=gs):
            sess.exchange_x(stream=gs)
            sess.exchange_f(fshift=fshift, stream=gs)
        torch.cuda.synchronize()
        barrier()
        gev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
        for k in range(min(K, 2000) + args.warmup):
            flush.fill_(1.0)
            reset_f()
            kk = k - args.warmup
            if kk >= 0:
                gev[kk][0].record(stream)
            g.replay()
            if kk >= 0:
                gev[kk][1].record(stream)
        torch.cuda.synchronize()
        nk = min(K, 2000)
        graph_us = max_over_ranks(float(np.mean([gev[k][0].elapsed_time(gev[k][1]) * 1e3 for k in range(nk)])))
        barrier()
        del g

    # e2e through the C-ABI host-buffer call (halo_step_host_packed: one pinned host block
    # in, one out; the H2D of the inputs and the D2H of the results inside the timed span)
    e2e_us = h2d = d2h = e2e_med = None
    if not args.no_e2e:
        e2e_us, h2d, d2h, e2e_med = e2e_timing(sess, X, homes, F0, first, nl, W, flush, stream, K, args.warmup)

    # NCCL send/recv baseline on the same maps (one DD rank per GPU only)
    nccl = None
    if world > 1 and nl == 1 and not args.no_nccl:
        if world > torch.cuda.device_count():  # oversubscribed functional runs: NCCL allows one rank per GPU
            nccl = {"skipped": "more processes than GPUs (NCCL needs one rank per device)"}
        else:
            err = None
            try:
                nccl = run_nccl_baseline(sess, lay[0], F0[0], flush, K, args.warmup, W)
            except Exception as e:  # noqa: BLE001 - reported in the line, the rest still measured
                err = str(e)[:200]
            if -max_over_ranks(-(1.0 if err is None else 0.0)) < 1.0:
                nccl = {"error": err or "failed on another rank"}

    # latency floor: peer flag ping-pong between process 0 and process 1; bandwidth
    # floor: one-directional SM peer stores and copy-engine copies 0 -> 1
    floor = None
    if world > 1 and not args.no_floors:
        t0 = t0r = None
        bw = {}
        if rank in (0, 1):
            peer = sess.first_rank + sess.n_local if rank == 0 else 0
            t0 = sess.halo.floor_pingpong(peer, iters=10000, relaxed=False)
            t0r = sess.halo.floor_pingpong(peer, iters=10000, relaxed=True)
        barrier()
        # t(B): payload + signal one-way latency, process 0 <-> process 1 (collective between them)
        curve = []
        for nb in (4 << 10, 16 << 10, 64 << 10, 256 << 10, 1 << 20, 4 << 20, 16 << 20, 64 << 20):
            v = None
            if rank in (0, 1):
                peer = sess.first_rank + sess.n_local if rank == 0 else 0
                v = sess.halo.floor_payload(peer, nb, iters=200 if nb <= (1 << 20) else 40)
            barrier()
            if rank == 0:
                curve.append({"bytes": nb, "one_way_us": round(v, 3), "gbs": round(nb / (v * 1e-6) / 1e9, 1)})
        if rank == 0:
            # bandwidth (64 MiB per peer, back-to-back): one pair, then every other process's first rank at once
            per = sess.n_local
            others = [q * per for q in range(1, world)]
            for name, peers in (("1_peer", others[:1]), (f"{len(others)}_peers", others) if len(others) > 1 else (None, None)):
                if name is None:
                    continue
                bw[name] = {"bytes_per_peer": 64 << 20, "peers": peers,
                            "sm_gbs_total": round(sess.halo.floor_bandwidth_multi(peers, 64 << 20, mode=0, iters=20), 1),
                            "ce_gbs_total": round(sess.halo.floor_bandwidth_multi(peers, 64 << 20, mode=1, iters=20), 1)}
            peer = sess.first_rank + sess.n_local
            for name, nb in (("8MiB", 8 << 20), ("1MiB", 1 << 20), ("64KiB", 64 << 10)):
                bw[name] = {"bytes": nb,
                            "sm_gbs": round(sess.halo.floor_bandwidth(peer, nb, mode=0, iters=50), 1),
                            "ce_gbs": round(sess.halo.floor_bandwidth(peer, nb, mode=1, iters=50), 1)}
            bw["t_of_B"] = curve
        barrier()
        t0 = max_over_ranks(t0 or 0.0)
        t0r = max_over_ranks(t0r or 0.0)
        floor = {"t0_one_way_us": t0r, "t0_release_acquire_us": t0, "bandwidth": bw or None,
                 "note": "t0 = relaxed 8-B peer store seen by a relaxed poll (the LL unit); median of 1e4 "
                         "round trips / 2.  bandwidth: back-to-back transfers GPU0 -> GPU1, SM 16-B stores "
                         "(8 CTAs/SM) and cudaMemcpyAsync (copy engine), measured on rank 0"}

    # algorithmic bytes per launch (this GPU), DESIGN.md "Roofline"
    rows_x = sum(sum(lay[l]["send_size"]) for l in range(nl))
    rows_f = sum(sum(lay[l]["recv_size"]) for l in range(nl))
    bx = (4 + 8 * W) * rows_x            # map + gather read + peer write
    bf = (4 + 20 * W) * rows_f           # slice read + peer write + buf read + map + RMW f
    # rows that cross NVLink (receiver on another GPU), both directions
    per_gpu = c.nranks // world
    remote_rows = 0
    for l in range(nl):
        r = first + l
        for p in range(P):
            dst = _neighbour(c.grid, r, sess.halo.pulse_order()[p], -1)
            if dst // per_gpu != r // per_gpu:
                remote_rows += lay[l]["send_size"][p]
    nvl_bytes = remote_rows * 4 * W * 2  # x out + f back (per direction)

    peaks = load_peaks()
    dom = "x" if res["x"] >= res["f"] else "f"
    dom_bytes = bx if dom == "x" else bf
    dom_us = res[dom]
    achieved = dom_bytes / (dom_us * 1e-6) / 1e9
    traffic = load_traffic(c.name, world, dom)
    roof = {"bound": "hbm", "kernel": f"k_exchange_{dom}", "achieved": round(achieved, 3),
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 6),
            "traffic": traffic, "algorithmic_bytes_per_launch": int(dom_bytes),
            "note": "latency-bound path: the HBM bytes of every config take < 1 us; see latency_floor / DESIGN.md"}
    out = {
        "metric": METRIC, "value": round(res["step"], 3), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": round(res["step"] / 1e3, 6), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": dict(workload_desc(c, world, W), parallelism=f"spatial DD {c.grid[0]}x{c.grid[1]}x{c.grid[2]}",
                       protocol=args.proto, transport=transport, zones=args.zones, plan_in_l2=("persisting (HALO_F_L2_PERSIST)" if args.l2_persist
                                                        else "flushed with everything else"),
                       mode=("eager, one exchange_x + one exchange_f launch per GPU per step" if transport != "ce"
                             else "eager, copy-engine path: per pulse pack + cudaMemcpyAsync + flag kernels")),
        "x_us": round(res["x"], 3), "f_us": round(res["f"], 3), "step_median_us": round(res["step_median"], 3),
        "step_percentiles_us": {"p90": round(res["step_p90"], 3), "p99": round(res["step_p99"], 3),
                                "max": round(res["step_max"], 3)},
        "x_median_us": round(res["x_median"], 3), "f_median_us": round(res["f_median"], 3),
        "x_f_split_note": "x_us / f_us: 200 isolated steps (synchronize + host barrier + a 40-us GPU sleep "
                          "before each, so both launches are queued; events around each launch, i.e. no "
                          "programmatic dependent launch across the middle event), so x_us + f_us > value",
        "graph_us_per_step": None if graph_us is None else round(graph_us, 3),
        "fused_xf": None,
        "clocks": sampler.summary(),
        "e2e": None if e2e_us is None else {"value": round(e2e_us, 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "median_us": round(e2e_med, 3),
                "path": "halo_step_host_packed (C ABI): one pinned host block in (x home rows + forces), one out "
                        "(halo x rows + home forces + fshift) per process; 2 uploads + 2 downloads on 3 streams; "
                        "the call returns with the results in host memory (it polls the stream); value = mean "
                        "over the K steps (host stalls included), median_us beside it"},
        "gpu_launches": (2 if transport != "ce" else 4 * P) * K * world,
        "roofline": roof,
        "nvlink": {"bytes_per_step_per_gpu_per_direction": int(nvl_bytes),
                   "achieved_gbs": round(nvl_bytes / (res["step"] * 1e-6) / 1e9, 3) if nvl_bytes else 0.0,
                   "peak_gbs": 900.0, "counters": nvl_counted},
        "latency_floor": floor or None,
        "nccl_baseline": nccl,
        "device_spans": dev_spans,
    }
    if world == 1 and nl > 1 and not args.no_floors:
        # all DD ranks on one GPU: the same-GPU flag round trip (two CTAs of one launch)
        t0 = sess.halo.floor_pingpong(first + 1, iters=10000, relaxed=False)
        t0r = sess.halo.floor_pingpong(first + 1, iters=10000, relaxed=True)
        floor = {"t0_one_way_us": t0r, "t0_release_acquire_us": t0, "bandwidth": None,
                 "note": "same-GPU floor: relaxed 8-B store seen by a relaxed poll from another CTA (L2 "
                         "round trip); median of 1e4 round trips / 2"}
        out["latency_floor"] = floor
    launch_eager = max_over_ranks(sess.halo.floor_launch(1000, graph=False)) if not args.no_floors else 0.0
    launch_graph = max_over_ranks(sess.halo.floor_launch(1000, graph=True)) if not args.no_floors else 0.0
    if floor is None:
        floor = {}
        out["latency_floor"] = floor
    floor["launch_us_eager"] = round(launch_eager, 3)
    floor["launch_us_graph"] = round(launch_graph, 3)
    if not args.no_floors:
        # the step's fixed cost: the same loop as the timed step (flush, reset, events)
        # around two EMPTY kernels with the x / f grids and launch attributes
        evp = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(min(K, 300))]
        for k in range(-args.warmup, len(evp)):
            flush.fill_(1.0)
            reset_f()
            if k >= 0:
                evp[k][0].record(stream)
            sess.halo.floor_empty_pair(stream.cuda_stream)
            if k >= 0:
                evp[k][1].record(stream)
        torch.cuda.synchronize()
        floor["empty_step_us"] = round(max_over_ranks(float(np.mean([a.elapsed_time(b) * 1e3 for a, b in evp]))), 3)
        floor["empty_step_note"] = ("two empty kernels with the x / f grids and PDL attributes, timed like the step "
                                    "(L2 flush + f reset before each, events around): the launch / drain / hand-off "
                                    "cost every two-launch step pays")
    if floor.get("t0_one_way_us"):
        t0 = floor["t0_one_way_us"]
        bwd = floor.get("bandwidth") or {}
        bw_peer = (bwd.get("1_peer") or {}).get("sm_gbs_total") or (bwd.get("8MiB") or {}).get("sm_gbs")
        bw_src = "measured SM peer stores, 64 MiB, one pair" if (bwd.get("1_peer") or {}).get("sm_gbs_total") else \
            ("measured SM peer stores, 8 MiB" if bw_peer else None)
        if not bw_peer:  # N=1: no NVLink bytes; the guide's measured peer copy (B200_PROFILING.md), labelled
            bw_peer, bw_src = 770.0, "not measured here (N=1, no NVLink traffic): B200_PROFILING.md peer copy 770 GB/s"
        # nvl_bytes already holds x out + f back (one direction): x and f are serial, so their
        # bandwidth terms add once each
        fl = 2 * P * t0 + nvl_bytes / (bw_peer * 1e9) * 1e6
        out["nvlink"]["bw_peer_gbs"] = bw_peer
        out["nvlink"]["bw_peer_source"] = bw_src
        out["nvlink"]["frac_of_measured"] = round(out["nvlink"]["achieved_gbs"] / bw_peer, 4)
        floor["floor_step_us"] = round(fl, 3)
        floor["value_over_floor"] = round(res["step"] / fl, 3)
        fl2 = fl + 2 * launch_eager
        floor["floor_step_with_launch_us"] = round(fl2, 3)
        floor["value_over_floor_with_launch"] = round(res["step"] / fl2, 3)
        # the bound that actually limits this path: the measured latency floor
        roof["latency"] = {"floor_us": round(fl2, 3), "frac": round(fl2 / res["step"], 4),
                           "definition": "2*P*t0 + (x+f NVLink bytes per direction)/BW_peer (nvlink.bw_peer_source) "
                                         "+ 2 launches (eager)"}
    if args.pme:
        out["pme"] = pme_timing(sess, K, args.warmup, flush)
    if not args.no_ns:
        out["ns_step"] = ns_step_timing(sess, c, X, homes, dev)
    if transport == "ll" and not args.no_fused:
        out["fused_xf"] = fused_timing(sess, fshift, flush, reset_f, stream, K, args.warmup)
    if world == 1 and rank == 0 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline_leg(args, P, c)
    sess.destroy()
    return out


def fused_timing(sess, fshift, flush, reset_f, stream, K, warmup):
    """The same steps as ONE fused launch each (halo_exchange_xf, LL protocol; SURVEY §7
    step 9), timed like the two-launch step.  Run last; an error is reported in the line
    (every rank agrees on success before the reductions)."""
    import torch
    tf_, err = None, None
    try:
        for _ in range(warmup):
            flush.fill_(1.0)
            reset_f()
            sess.exchange_xf(fshift=fshift)
        torch.cuda.synchronize()
        barrier()
        evf = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
        for k in range(K):
            flush.fill_(float(k))
            reset_f()
            evf[k][0].record(stream)
            sess.exchange_xf(fshift=fshift)
            evf[k][1].record(stream)
        torch.cuda.synchronize()
        tf_ = [evf[k][0].elapsed_time(evf[k][1]) * 1e3 for k in range(K)]
    except Exception as e:  # noqa: BLE001 - reported, not raised
        err = str(e)[:200]
    ok = -max_over_ranks(-(1.0 if err is None else 0.0))  # min over ranks
    if ok < 1.0:
        return {"error": err or "failed on another rank"}
    return {"us_per_step": round(max_over_ranks(float(np.mean(tf_))), 3),
            "median_us": round(max_over_ranks(float(np.median(tf_))), 3),
            "p90_us": round(max_over_ranks(float(np.percentile(tf_, 90))), 3),
            "path": "halo_exchange_xf: x and f of the step in ONE launch; rank l's gather items start when "
                    "l's halo rows are complete (the non-bonded kernel's slot, Alg. 2)"}


def e2e_timing(sess, X, homes, F0, first, nl, W, flush, stream, K, warmup):
    """e2e through the C-ABI host-buffer call halo_step_host_packed: one pinned host block
    in (x home rows + this step's forces), one out (halo x rows + home forces + fshift) per
    process; the H2D of the inputs and the D2H of the results inside the timed span.
    Returns (us/step max over ranks, H2D bytes, D2H bytes summed over processes)."""
    import torch
    in_b, out_b = sess.halo.packed_sizes()
    blk = np.concatenate(
        [np.pad(X[homes[first + l]], ((0, 0), (0, W - 3))).astype(np.float32).reshape(-1) for l in range(nl)] +
        [F0[l].cpu().numpy().reshape(-1) for l in range(nl)]).astype(np.float32)
    assert blk.nbytes == in_b, (blk.nbytes, in_b)
    hin = torch.from_numpy(blk).pin_memory()
    hout = torch.empty(out_b, dtype=torch.uint8).pin_memory()

    def host_step():
        sess.halo.step_host_packed(hin.data_ptr(), hout.data_ptr(), stream=stream.cuda_stream)

    for _ in range(warmup):
        host_step()
    barrier()
    eev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    import gc
    gc.collect()
    gc.disable()  # a collector pause of this harness's Python objects is not the API's cost
    try:
        for k in range(K):
            flush.fill_(1.0)
            eev[k][0].record(stream)
            host_step()
            eev[k][1].record(stream)
        torch.cuda.synchronize()
    finally:
        gc.enable()
    per = [eev[k][0].elapsed_time(eev[k][1]) * 1e3 for k in range(K)]
    e2e_us = max_over_ranks(float(np.mean(per)))
    med_us = max_over_ranks(float(np.median(per)))
    h2d, d2h = sum_over_ranks(in_b), sum_over_ranks(out_b)  # every process's blocks
    barrier()
    return e2e_us, h2d, d2h, med_us


def pme_timing(sess, K, warmup, flush):
    """PP <-> PME redistribution, PME task on DD rank 0's GPU: per
    step halo_pme_send_x + halo_pme_recv_f (no PME compute in between), L2 flushed
    before each step, CUDA events on the stream, mean per rank, max over ranks."""
    import torch
    n_total, _ = sess.pme_setup()
    st = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for i in range(warmup + K):
        flush.zero_()
        if i >= warmup:
            ev[i - warmup][0].record(st)
        sess.pme_send_x()
        sess.pme_recv_f()
        if i >= warmup:
            ev[i - warmup][1].record(st)
    torch.cuda.synchronize()
    us = statistics.mean(a.elapsed_time(b) * 1e3 for a, b in ev)
    W = sess.layout
    return {"us_per_step": round(max_over_ranks(us), 3), "rows": int(n_total),
            "nvlink_bytes_per_step": int(n_total * W * 4 * 2), "pme_rank": 0,
            "note": "halo_pme_send_x + halo_pme_recv_f per step (every DD rank's home x to the PME GPU, "
                    "force slices back), L2 flushed before each step; not in value"}


def ns_step_timing(sess, c, X, homes, dev, reps=3):
    """The NS step that precedes the hot path every nstlist steps:
    halo_migrate (home-atom redistribution) + halo_set_maps (GPU map build + the
    coordinate exchange of every pulse), host wall time around each call (both
    host-synchronise), max over ranks, median of `reps` NS steps.  Atoms move by
    normal(0, 0.05 nm) per component between NS steps (synth.displacements, then
    torch normal draws on the device for later steps).  Not part of `value`."""
    import torch
    from synth import displacements
    first, nl, cap = sess.first_rank, sess.n_local, sess.capacity
    Xm = displacements(X, c.L, 4242, n_far=0)
    gid = []
    for l in range(nl):
        h = homes[first + l]
        sess.x[l][: h.size, :3] = torch.from_numpy(Xm[h]).to(dev)
        g = torch.zeros(cap, dtype=torch.int32, device=dev)
        g[: h.size] = torch.from_numpy(h.astype(np.int32)).to(dev)
        gid.append(g)
    gen = torch.Generator(device=dev)
    gen.manual_seed(4243 + first)
    t_mig, t_maps, moved = [], [], []
    for rep in range(reps + 1):
        if rep:
            for l in range(nl):
                n = sess.n_home[l]
                sess.x[l][:n, :3] += 0.05 * torch.randn(n, 3, generator=gen, device=dev)
        before = [set(gid[l][: sess.n_home[l]].tolist()) for l in range(nl)] if rep == 1 else None
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        sess.migrate(gid)
        t1 = time.perf_counter()
        barrier()
        t2 = time.perf_counter()
        sess.set_maps()
        t3 = time.perf_counter()
        if rep:
            t_mig.append(max_over_ranks((t1 - t0) * 1e6))
            t_maps.append(max_over_ranks((t3 - t2) * 1e6))
        if before is not None:
            moved.append(sum(len(set(gid[l][: sess.n_home[l]].tolist()) - before[l]) for l in range(nl)))
    return {"migrate_us": round(float(np.median(t_mig)), 1), "set_maps_us": round(float(np.median(t_maps)), 1),
            "rows_moved_between_ranks_local": int(moved[0]) if moved else 0, "reps": reps,
            "note": "NS step every nstlist steps (P:976: 200): halo_migrate + halo_set_maps, host wall "
                    "(both host-synchronise), max over ranks; not in value"}


def _neighbour(grid, r, d, delta):
    c = [r // (grid[1] * grid[2]), (r // grid[2]) % grid[1], r % grid[2]]
    c[d] = (c[d] + delta) % grid[d]
    return (c[0] * grid[1] + c[1]) * grid[2] + c[2]


def run_nccl_baseline(sess, lay, F0, flush, K, warmup, W):
    """Serialized per-pulse schedule (Fig. 1) with NCCL send/recv on the same maps
    (halo_nccl_*, csrc/nccl_baseline.cu, torch's libnccl): pack kernel -> ncclGroupStart/Send/
    Recv/GroupEnd per pulse ascending; forces: send/recv of the halo slice per pulse descending
    -> ordered scatter-add kernel.  Timed eager and as one captured CUDA graph per step (the
    same flush / f reset between steps as the fused arm), mean per rank, max over ranks."""
    import torch
    from paper_2509_21527_b200.nccl_baseline import NcclSchedule
    dev = sess.device
    sched = NcclSchedule(sess)
    fshift = torch.zeros(1, 3, 3, dtype=torch.float64, device=dev)
    f = sess.f[0]
    stream = torch.cuda.current_stream()

    def timed(run):
        for _ in range(warmup):
            f[: F0.shape[0]].copy_(F0)
            flush.fill_(1.0)
            run()
        torch.cuda.synchronize()
        barrier()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
        for k in range(K):
            f[: F0.shape[0]].copy_(F0)
            flush.fill_(1.0)
            ev[k][0].record(stream)
            run()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        us = max_over_ranks(float(np.mean([ev[k][0].elapsed_time(ev[k][1]) * 1e3 for k in range(K)])))
        barrier()
        return us

    eager = timed(lambda: sched.step(fshift))
    graph_us = None
    try:
        gs = torch.cuda.Stream(device=dev)
        g = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        barrier()
        with torch.cuda.graph(g, stream=gs):
            sched.step(fshift, stream=gs)
        torch.cuda.synchronize()
        barrier()
        graph_us = timed(g.replay)
        del g
    except Exception as e:  # pragma: no cover - recorded, not hidden
        graph_us = f"capture failed: {e}"
    return {"us_per_step": round(eager, 3), "graph_us_per_step": graph_us if isinstance(graph_us, str) or graph_us is None
            else round(graph_us, 3),
            "schedule": "per-pulse pack kernel -> ncclGroupStart/ncclSend/ncclRecv/ncclGroupEnd (C++, halo_nccl_*, "
                        "torch's libnccl) -> reverse send/recv + ordered scatter-add, same maps; eager and one "
                        "CUDA graph per step",
            "launches_per_step": 2 * sess.npulse}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback"}


def load_traffic(cfg, world, dom):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"{cfg}/n{world}/{dom}")
    except Exception:
        return None


def run_reference(args, rank, world):
    """--impl reference: the oracle as it stands, timed on the host cores (rank 0 only)."""
    if rank != 0:
        return None
    cpu = pin_one_core()
    c, X = build_workload(args.config)
    # warm-up steps W, then K timed steps, each step one full oracle x+f over all DD ranks
    from oracle import coord_halo_step, decompose, force_halo
    from synth import forces_normal
    states = decompose(X, c.L, c.rc, c.grid, c.pulses)
    F = [forces_normal(s.x.shape[0], 77 + s.rank) for s in states]
    xh = [s.x[: s.n_home].copy() for s in states]
    for _ in range(args.warmup):
        coord_halo_step(states, xh)
        force_halo(states, F)
    ts = []
    t_end = time.perf_counter() + args.cpu_budget * 8
    for k in range(args.steps):
        t0 = time.perf_counter()
        coord_halo_step(states, xh)
        force_halo(states, F)
        ts.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end:
            break
    us = float(np.mean(ts)) * 1e6
    P = len(states[0].pulses)
    samp = f"{c.name} full workload ({c.nranks} DD ranks, {P} pulses), {len(ts)} of {args.steps} steps"
    return {"impl": "reference", "metric": METRIC, "value": round(us, 1), "unit": UNIT, "n_gpus": world,
            "steps": len(ts), "warmup": args.warmup, "ms_per_step": round(us / 1e3, 4), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_desc(c, world, 3),
            "cpu_baseline": {"value": round(us, 1), "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": samp + f", one thread pinned to core {cpu}", **host_info()},
            "e2e": {"value": round(us, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--layout", type=int, default=3, choices=(3, 4))
    ap.add_argument("--impl", default="fused", choices=("fused", "reference"))
    ap.add_argument("--proto", default="ll", choices=sorted(PROTO_FLAGS),
                    help="ll: default LL protocol; paper: per-pulse flags (Alg. 5); paper_tma: the same with the "
                         "x put as warp-leader TMA bulk stores (Alg. 3) and the force halo as a receiver-driven "
                         "TMA get (Alg. 6); ce: copy-engine path")
    ap.add_argument("--timers", action="store_true")
    ap.add_argument("--l2-persist", action="store_true", help="HALO_F_L2_PERSIST: static plan in persisting L2")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-fused", action="store_true", help="skip the fused x+f launch (halo_exchange_xf) timing")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-floors", action="store_true", help="skip the latency/bandwidth/launch floor probes")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--cpu-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--no-c1-pipeline", action="store_true", help="cpu leg: skip the C1 whole-pipeline timing")
    ap.add_argument("--zones", default="slab", choices=("slab", "rounded"),
                    help="import zones: slab (box-shaped, default) or GROMACS-style rounded (HALO_F_ROUNDED_ZONES)")
    ap.add_argument("--pme", action="store_true", help="also time the PP<->PME redistribution (halo_pme_*)")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e timing")
    ap.add_argument("--no-ns", action="store_true", help="skip the NS-step (halo_migrate + halo_set_maps) timing")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.cpu_child:
        cpu_child(args)
        return
    rank, world, local = dist_env()
    if args.gpus is not None and args.gpus != world and world != 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    import torch
    import torch.distributed as dist
    # one process per GPU (LOCAL_RANK = device).  HALO_BENCH_PG=gloo + more processes than GPUs
    # (device = LOCAL_RANK mod GPUs) only checks the N-process path on a smaller box: not a bench value
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        torch.cuda.set_device(local)
        if os.environ.get("HALO_BENCH_PG", "nccl") == "gloo":
            dist.init_process_group("gloo", rank=rank, world_size=world)
        else:
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
    out = run_fused(args, rank, world, local)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
