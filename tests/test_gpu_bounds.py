"""Checked build (-DHALO_BOUNDS_CHECK): the parity cases of tests/bounds_check_run.py run
through libhalo_checked.so, where every global index the LL kernels derive from a plan
record is checked against its buffer (compute-sanitizer is closed on this GPU pool:
profiles/r02s4/compute_sanitizer_closed.txt).  Each run is a subprocess (one library
per process).  The self-test shrinks the bounds the kernels see (HALO_BC_CAP) and
expects the checks to fire."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _checked_lib():
    from paper_2509_21527_b200.build import build_checked
    return build_checked()  # no-op when up to date (build() of __graft_entry__ builds it)


def _run(args, extra_env=None, timeout=600):
    env = dict(os.environ, HALO_LIB_PATH=_checked_lib(), **(extra_env or {}))
    return subprocess.run([sys.executable, os.path.join(ROOT, "tests", "bounds_check_run.py"), *args], env=env,
                          capture_output=True, text=True, timeout=timeout, cwd=ROOT)


def test_bounds_checked_parity():
    r = _run([])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.count(": ok") >= 14, r.stdout


@pytest.mark.parametrize("spec,env", [("T3D:ll", "HALO_BC_CAP"), ("T3D:staged", "HALO_BC_CAP"),
                                      ("C3:ll:fused", "HALO_BC_CAP"), ("C3:ll", "HALO_BC_ITEMS"),
                                      ("T2P:staged", "HALO_BC_NS")])
def test_bounds_check_fires(spec, env):
    # HALO_BC_CAP: the exchange kernels see 8-row buffers; HALO_BC_ITEMS: the plan kernels
    # see one x item and one f item; HALO_BC_NS: the NS-step coordinate exchange sees 8 rows
    r = _run([spec], {env: "1" if env == "HALO_BC_ITEMS" else "8"})
    assert r.returncode != 0, r.stdout
    assert "bounds check failed" in r.stderr, r.stderr[-4000:]
