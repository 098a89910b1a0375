"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol
include/halo.h declares, and rejects invalid geometry before touching CUDA."""
import ctypes
import os
import re

import pytest

from paper_2509_21527_b200 import _lib
from paper_2509_21527_b200.halo import Halo, HaloError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "halo.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"HALO_API\s+[\w\s\*]+?\b(halo_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.EXPORTS) == syms


def test_strerror_names():
    lib = _lib.load()
    for code in range(9):
        assert lib.halo_strerror(code)


@pytest.mark.parametrize("grid,pulses,box,rc,status", [
    ((1, 1, 2), (0, 0, 0), (4, 4, 4), 1.0, 2),   # decomposed dim without pulses
    ((1, 1, 2), (0, 0, 2), (4, 4, 4), 1.0, 2),   # pulses > grid-1
    ((1, 1, 1), (0, 0, 1), (4, 4, 4), 1.0, 2),   # pulse on an undecomposed dim
    ((1, 1, 5), (0, 0, 1), (4, 4, 4), 1.0, 2),   # not enough pulses
    ((1, 1, 2), (0, 0, 1), (4, 4, 1.8), 1.0, 2), # rc >= L/2
    ((1, 1, 2), (0, 0, 1), (4, 4, 4), 0.0, 2),   # rc <= 0
    ((1, 1, 8), (0, 0, 3), (10, 10, 10), 1.0, 8),  # > 2 pulses per dim
    ((8, 8, 2), (1, 1, 1), (40, 40, 40), 1.0, 8),  # too many ranks for this build
])
def test_init_rejects_invalid_geometry_without_gpu(grid, pulses, box, rc, status):
    with pytest.raises(HaloError) as e:
        Halo(grid, box, rc, pulses, capacity=100)
    assert e.value.status == status


def test_init_rejects_bad_args():
    with pytest.raises(HaloError) as e:
        Halo((1, 1, 2), (4, 4, 4), 1.0, (0, 0, 1), layout=5, capacity=100)
    assert e.value.status == 1
    with pytest.raises(HaloError) as e:
        Halo((1, 1, 2), (4, 4, 4), 1.0, (0, 0, 1), capacity=100, nprocs=3)  # 2 ranks on 3 procs
    assert e.value.status == 1


def test_null_ctx_calls_are_errors():
    lib = _lib.load()
    assert lib.halo_exchange_x(None, None) == 1
    assert lib.halo_exchange_f(None, None, 1, None) == 1
    assert lib.halo_sync(None) == 1
    assert lib.halo_destroy(None) == 0


def test_flag_constants_match_header():
    """Every HALO_F_* flag of include/halo.h has the same value in the Python binding and
    in bench.py's protocol table (no drift between the ABI and its users)."""
    with open(os.path.join(ROOT, "include", "halo.h")) as f:
        src = f.read()
    flags = {m.group(1): 1 << int(m.group(2)) for m in re.finditer(r"#define (HALO_F_\w+)\s+\(1u << (\d+)\)", src)}
    assert len(flags) >= 11
    for name, val in flags.items():
        assert getattr(_lib, name) == val, name
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    assert bench.PROTO_FLAGS["paper"] == flags["HALO_F_PAPER_FLAGS"]
    assert bench.PROTO_FLAGS["ce"] == flags["HALO_F_CE_PATH"]
    assert bench.PROTO_FLAGS["auto"] == flags["HALO_F_AUTO_TRANSPORT"]
    assert bench.PROTO_FLAGS["paper_tma"] == (flags["HALO_F_PAPER_FLAGS"] | flags["HALO_F_TMA_STORE"]
                                              | flags["HALO_F_TMA_GET"])
