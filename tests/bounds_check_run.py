"""Test infrastructure (run by tests/test_gpu_bounds.py; it calls the oracle): parity
cases through the CHECKED build of the library (-DHALO_BOUNDS_CHECK: every global index the LL kernels derive from a plan record is checked against its buffer;
DESIGN.md §7).  compute-sanitizer is closed on this GPU pool (profiles/r02s4/
compute_sanitizer_closed.txt); this is the bounds-check substitute it recommends.

    HALO_LIB_PATH=paper_2509_21527_b200/libhalo_checked.so python tests/bounds_check_run.py [CASE ...]

A case is NAME[:mode[:fused]] with mode ll (one hop group), staged (every DD rank its
own group: the LL receive paths) or bulk (staged + every last pulse a bulk pulse).
Exits 0 with one "ok" line per case when every case matches the oracle and no check
fired; a failed check surfaces as HaloError("bounds check failed ...")."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

DEFAULT = ["T3D:ll", "T3D:staged", "T3D:bulk", "T2P:ll", "T2P:staged", "C2:staged", "C5:ll", "C5:bulk",
           "C3:ll", "C3:staged", "C3:ll:fused", "C3:staged:fused", "W2:staged", "T4x2:bulk"]


def run(spec):
    parts = spec.split(":")
    name, mode = parts[0], parts[1] if len(parts) > 1 else "ll"
    fused = len(parts) > 2 and parts[2] == "fused"
    env = {"HALO_COLLAPSE": "0" if mode in ("staged", "bulk") else "1", "HALO_BULK_ROWS": "1" if mode == "bulk" else "0"}
    os.environ.update(env)  # read at halo_init
    from paper_2509_21527_b200.session import HaloSession
    from tests.parity_common import Case, run_gpu_case
    case = Case(name, seed=1, force_kind="normal", layout=4 if name == "W2" else 3)
    sess = HaloSession(case.grid, case.L, case.rc, case.pulses, layout=case.layout, capacity=case.capacity,
                       device=0, timeout_s=20.0)
    try:
        run_gpu_case(case, sess, steps=2, fused=fused)
    except AssertionError:
        sess.halo.sync()  # a fired check (whose clamped access broke parity) surfaces here as a HaloError
        raise
    sess.halo.sync()  # raises if any check fired
    sess.destroy()
    print(f"bounds_check {spec}: ok", flush=True)


def main():
    lib = os.environ.get("HALO_LIB_PATH", "")
    if "checked" not in os.path.basename(lib):
        sys.exit("set HALO_LIB_PATH to the checked build (paper_2509_21527_b200/libhalo_checked.so)")
    for spec in sys.argv[1:] or DEFAULT:
        run(spec)


if __name__ == "__main__":
    main()
