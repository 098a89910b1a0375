"""Build libhalo.so in-tree with nvcc for sm_100a (no torch JIT cache).

    python -m paper_2509_21527_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libhalo.so")
# the checked build (-DHALO_BOUNDS_CHECK, tests/bounds_check_run.py, tests/test_gpu_bounds.py)
CHECKED = os.path.join(HERE, "libhalo_checked.so")
SOURCES = ["runtime.cu", "kernels.cu", "kernels_ll.cu", "kernels_ce.cu", "kernels_ns.cu", "kernels_pme.cu", "kernels_plan.cu",
           "nccl_baseline.cu",
           "kernels_floor.cu"]
HEADERS = ["halo_internal.h", "ptx.cuh", os.path.join("..", "..", "include", "halo.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-cudart", "static",
    "-Xptxas", "-v",
]


def _newest_input() -> float:
    paths = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, h) for h in HEADERS]
    return max(os.path.getmtime(p) for p in paths)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """defines: extra -D switches (A/B timing variants in scripts/, written to `out`)."""
    if not force and out in (LIB, CHECKED) and os.path.exists(out) and os.path.getmtime(out) >= _newest_input():
        return out
    tag = ".o" if out == LIB else ".checked.o" if out == CHECKED else ".ab.o"
    objs = [os.path.join(CSRC, src.replace(".cu", tag)) for src in SOURCES]

    def compile_one(k):
        cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-c",
               os.path.join(CSRC, SOURCES[k]), "-o", objs[k]]
        return subprocess.run(cmd, capture_output=True, text=True)

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, range(len(SOURCES))))
    logs = []
    for src, r in zip(SOURCES, results):
        logs.append(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    tmp = out + ".tmp"
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
           "-Xcompiler", "-fPIC", *objs, "-lpthread", "-ldl", "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, out)
    if out != LIB:
        return out
    with open(os.path.join(CSRC, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return out


def build_checked(force: bool = False) -> str:
    """The bounds-checked variant of the library (same sources, -DHALO_BOUNDS_CHECK)."""
    return build(force=force, out=CHECKED, defines=("HALO_BOUNDS_CHECK",))


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
    if "--checked" in sys.argv:
        print(build_checked(force="--force" in sys.argv))
