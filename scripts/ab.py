"""A/B timing of library builds on one box (alternating runs cancel drift).

    python scripts/ab.py --libs new=paper_2509_21527_b200/libhalo.so,base=ab/libhalo_r568.so \
        --config C3 --gpus 1 --reps 3 [--proto ll] [--steps 300]

Each run is `bench.py --no-graph --no-cpu --no-nccl` with HALO_LIB_PATH set to
the build; prints per build the median value / x_us / f_us over the reps.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(lib, args, port):
    lib, _, extra = lib.partition("+")
    lib, *kvs = lib.split("@")  # path@KEY=VAL@KEY2=VAL2: environment of this variant only
    env = dict(os.environ, HALO_LIB_PATH=os.path.join(ROOT, lib))
    for kv in kvs:
        k, v = kv.split("=", 1)
        env[k] = v
    if args.env:
        for kv in args.env.split(","):
            k, v = kv.split("=", 1)
            env[k] = v
    bench = [os.path.join(ROOT, "bench.py"), "--steps", str(args.steps), "--warmup", "20", "--config", args.config,
             "--no-graph", "--no-cpu", "--no-nccl", "--no-floors", "--no-ns", "--no-e2e", "--proto", args.proto, *args.bench_args.split(), *[a for a in extra.split("+") if a]]
    if args.gpus > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), *bench, "--gpus", str(args.gpus)]
    else:
        cmd = [sys.executable, *bench]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    for line in r.stdout.splitlines()[::-1]:
        if line.startswith("{"):
            return json.loads(line)
    raise RuntimeError(r.stderr[-2000:])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", required=True)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--proto", default="ll")
    ap.add_argument("--env", default="")
    ap.add_argument("--bench-args", default="", help="extra bench.py arguments, e.g. '--l2-persist'")
    args = ap.parse_args()
    libs = [kv.split("=", 1) for kv in args.libs.split(",")]
    # name=path[@K=V...][+ARG...]: per-variant environment and bench arguments
    # (e.g. fence=lib.so@HALO_DEBUG=128, l2=lib.so+--l2-persist)
    res = {n: [] for n, _ in libs}
    port = 29600
    for _ in range(args.reps):
        for n, lib in libs:
            port += 1
            try:
                d = run(lib, args, port)
                res[n].append((d["value"], d["x_us"], d["f_us"], (d.get("fused_xf") or {}).get("us_per_step") or 0.0))
            except Exception as e:  # keep going: one failed run must not hide the others
                print(json.dumps({"lib": n, "error": str(e)[-500:]}), flush=True)
    for n, v in res.items():
        if v:
            med = [statistics.median(c) for c in zip(*v)]
            print(json.dumps({"config": args.config, "gpus": args.gpus, "lib": n, "value": med[0], "x_us": med[1],
                              "f_us": med[2], "fused_us": med[3], "runs": v}), flush=True)


if __name__ == "__main__":
    main()
