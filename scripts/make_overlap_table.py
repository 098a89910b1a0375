"""Markdown rows of the f1 overlap study from gpurun_out/<prefix>_overlap_*.txt (scripts/gpu_overlap.sh)."""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
prefix = sys.argv[1] if len(sys.argv) > 1 else "o2"
rows = []
for f in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", f"{prefix}_overlap_*.txt"))):
    for line in open(f):
        if line.startswith("{"):
            rows.append(json.loads(line))
rows.sort(key=lambda d: (d["gpus"], d["config"], ["ll", "paper", "ce", "nccl"].index(d["proto"])
                         if d["proto"] in ("ll", "paper", "ce", "nccl") else 9))
print("| config | GPUs | protocol | NB local alone µs | Local work | Non-local work | Non-overlap | step (eager) | "
      "compute-only step (eager) | exchange cost (eager) | step (CUDA graph) | compute-only (graph) | exchange cost (graph) |")
print("|" + "---|" * 13)
f = lambda v: "—" if v is None else f"{v:.1f}"
for d in rows:
    print(f"| {d['config']} | {d['gpus']} | {d['proto']} | {d['nb_local_alone_us']:.0f} | {f(d['local_us'])} | "
          f"{f(d['nonlocal_us'])} | {f(d['nonoverlap_us'])} | {f(d['step_us'])} | {f(d['compute_only_step_us'])} | "
          f"{f(d['exchange_cost_us'])} | {f(d.get('graph_step_us'))} | {f(d.get('graph_compute_only_step_us'))} | "
          f"{f(d.get('graph_exchange_cost_us'))} |")
