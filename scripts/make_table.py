"""Markdown rows of the round's bench table from gpurun_out/t_*.json (scripts/gpu_table.sh)."""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
rows = []
for f in sorted(glob.glob(os.path.join(src, "t_*_n*_*.json"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        print(f"<!-- {os.path.basename(f)}: no JSON line -->")
        continue
    c = d["config"]
    fl = d.get("latency_floor") or {}
    nccl = (d.get("nccl_baseline") or {}).get("us_per_step")
    pme = (d.get("pme") or {}).get("us_per_step")
    ns = d.get("ns_step") or {}
    rows.append((c["workload"].split(":")[0], d["n_gpus"], c.get("dd_ranks_per_gpu"),
                 (c.get("protocol") if c.get("transport") in (None, c.get("protocol")) or c.get("protocol") != "auto"
                  else f"auto → {c.get('transport')}") + ("" if c.get("zones", "slab") == "slab" else ", rounded"),
                 d["value"], d.get("step_median_us"), d.get("graph_us_per_step"), d.get("x_us"), d.get("f_us"),
                 (d.get("e2e") or {}).get("value"), nccl, fl.get("t0_one_way_us"), fl.get("floor_step_with_launch_us"),
                 fl.get("value_over_floor_with_launch"), (d.get("nvlink") or {}).get("achieved_gbs"),
                 ns.get("migrate_us"), ns.get("set_maps_us"), pme, (d.get("clocks") or {}).get("sm_mhz"),
                 (d.get("clocks") or {}).get("reasons")))
rows.sort(key=lambda r: (r[1], r[0], r[3]))
hdr = ["config", "GPUs", "DD ranks/GPU", "transport", "value µs/step", "median", "CUDA graph", "x_us / f_us",
       "e2e", "NCCL send/recv", "t0 µs", "floor+launch µs", "value / floor", "NVLink GB/s",
       "NS: migrate / set_maps µs", "PME µs", "SM MHz", "throttle"]
print("| " + " | ".join(hdr) + " |")
print("|" + "---|" * len(hdr))
fmt = lambda v: "—" if v is None else (f"{v:.1f}" if isinstance(v, float) else str(v))
for r in rows:
    nccl = "—" if r[10] is None else f"{r[10]:.0f} ({r[10] / r[4]:.1f}×)"
    print("| " + " | ".join([r[0], str(r[1]), str(r[2]), r[3], fmt(r[4]), fmt(r[5]), fmt(r[6]),
                             f"{fmt(r[7])} / {fmt(r[8])}", fmt(r[9]), nccl, fmt(r[11]), fmt(r[12]), fmt(r[13]),
                             fmt(r[14]), f"{fmt(r[15])} / {fmt(r[16])}", fmt(r[17]), fmt(r[18]), str(r[19])]) + " |")
