"""Dependency safety and parity resolution on the GPU (-m gpu, one process).

* G3: a protocol mutation must be
  caught by the poisoned, bit-exact parity check in >= 1 of N = 50 runs, with a
  slow producer (``kDelayPulse0``: pulse-0 send items sleep ~20 us) widening the
  race; the unmutated protocol with the same slow producer must pass all N runs.
  Mutations: (iv) the paper-literal firstDependentPulse (x0 waits for y0
  only; R9), (ii) the a4/a5 flags without release semantics, and the LL
  protocol's (i) forward-without-wait / tag-check-skipped variants.  Every
  mutation's catch count is appended to ``$HALO_G3_LOG`` (JSON lines) when set.
* fshift resolution: a build that rounds its shift-force partials to fp32 must
  violate the 1e-12 * sum|terms| bound (tests/parity_common.py).
* the cross-GPU receive path (``kItemXRecv``: LL units -> halo rows) on one GPU:
  ``HALO_DIRECT_X=0`` routes every same-process pulse through it.
"""
import json
import os

import numpy as np
import pytest
import torch

from tests.parity_common import Case, fshift_violation, run_gpu_case

pytestmark = pytest.mark.gpu

PAPER = 1 << 4
KX_NOWAIT, KF_NOWAIT = 16, 32
K_RELAXED, K_Q9, K_DELAY0, K_FS32 = 512, 1024, 2048, 4096
N_RUNS = 50


def session_for(case, flags=0):
    from paper_2509_21527_b200.session import HaloSession
    return HaloSession(case.grid, case.L, case.rc, case.pulses, layout=case.layout, capacity=case.capacity,
                       device=0, flags=flags, timeout_s=5.0)


def log_g3(rec):
    path = os.environ.get("HALO_G3_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def count_catches(case, flags, debug, monkeypatch, runs=N_RUNS):
    monkeypatch.setenv("HALO_DEBUG", str(debug))
    sess = session_for(case, flags=flags)
    caught = 0
    for _ in range(runs):
        try:
            run_gpu_case(case, sess, steps=1)
        except AssertionError:
            caught += 1
    sess.halo.sync()
    sess.destroy()
    return caught


@pytest.mark.parametrize("name", ["W2", "T3D", "C3"])
def test_g3_paper_literal_q9_caught(name, monkeypatch):
    """(iv): x0 forwards rows that arrived in z0 (witness W2); waiting only for y0
    (the paper-literal firstDependentPulse) forwards the poison of a slow z0."""
    case = Case(name, seed=1, force_kind="int")
    caught = count_catches(case, PAPER, K_Q9 | K_DELAY0, monkeypatch)
    log_g3({"mutation": "iv paper-literal firstDependentPulse", "case": name, "runs": N_RUNS, "caught": caught})
    assert caught >= 1, "paper-literal dependency set not detected"


@pytest.mark.parametrize("name", ["W2", "T3D", "C3"])
def test_g3_slow_producer_correct_protocol_passes(name, monkeypatch):
    """Control: the same slow producer with the R9 dependency sets is never caught."""
    case = Case(name, seed=1, force_kind="int")
    caught = count_catches(case, PAPER, K_DELAY0, monkeypatch)
    log_g3({"mutation": "none (control, slow pulse-0 producer)", "case": name, "runs": N_RUNS, "caught": caught})
    assert caught == 0


@pytest.mark.parametrize("name", ["T3D", "C3"])
def test_g3_relaxed_flags(name, monkeypatch):
    """(ii): flags without release (no per-CTA fence, relaxed counter and store).
    Logged; on one GPU the L2 is the coherence point, so the reordering may not
    be observable within N runs (the count is reported either way)."""
    case = Case(name, seed=1, force_kind="int")
    caught = count_catches(case, PAPER, K_RELAXED | K_DELAY0, monkeypatch)
    log_g3({"mutation": "ii relaxed a4/a5 flags", "case": name, "runs": N_RUNS, "caught": caught})


@pytest.mark.parametrize("mut", [KX_NOWAIT, KF_NOWAIT])
def test_g3_ll_mutations_50(mut, monkeypatch):
    """(i) on the LL protocol: forward x rows without waiting for their tag /
    add force contributions without checking theirs; caught in >= 1 of 50 runs.
    HALO_COLLAPSE=0: every rank its own hop group, every pulse waits."""
    monkeypatch.setenv("HALO_COLLAPSE", "0")
    case = Case("C3", seed=1, force_kind="int")
    caught = count_catches(case, 0, mut, monkeypatch)
    log_g3({"mutation": f"i LL debug {mut}", "case": "C3", "runs": N_RUNS, "caught": caught})
    assert caught >= 1


@pytest.mark.parametrize("proto", [0, PAPER])
def test_fshift_fp32_partials_violate_bound(proto, monkeypatch):
    """Resolution of the fshift tolerance on hardware: the kernels with their
    shift-force partials rounded to fp32 fail it; the fp64 build passes."""
    case = Case("C3", seed=2, force_kind="normal")
    worst = {}
    for debug in (0, K_FS32):
        monkeypatch.setenv("HALO_DEBUG", str(debug))
        sess = session_for(case, flags=proto)
        run_gpu_case(case, sess, check_forces=False)
        for l in range(sess.n_local):
            sess.f[l][: case.F[l].shape[0]] = torch.from_numpy(case.F[l]).to(sess.device)
        fs = torch.zeros(sess.n_local, 3, 3, dtype=torch.float64, device=sess.device)
        sess.exchange_f(fshift=fs)
        torch.cuda.synchronize()
        fs = fs.cpu().numpy()
        worst[debug] = max(fshift_violation(fs[l], case.fshift[l], case.fshift_abs[l]) for l in range(sess.n_local))
        sess.destroy()
    log_g3({"mutation": "fshift fp32 partials", "proto": proto, "violation_fp64": worst[0],
            "violation_fp32": worst[K_FS32]})
    assert worst[0] <= 1.0
    assert worst[K_FS32] > 1.0


@pytest.mark.parametrize("name,kind", [("C2", "int"), ("C3", "normal"), ("C5", "int"), ("T4x2", "normal"),
                                       ("C4-3D", "normal")])
def test_parity_receive_path_single_gpu(name, kind, monkeypatch):
    """HALO_DIRECT_X=0: every pulse's halo rows go through the receive items
    (LL units polled and copied into x), the path every cross-GPU pulse takes."""
    monkeypatch.setenv("HALO_DIRECT_X", "0")
    case = Case(name, seed=3, force_kind=kind)
    sess = session_for(case)
    run_gpu_case(case, sess, steps=2)
    sess.destroy()
