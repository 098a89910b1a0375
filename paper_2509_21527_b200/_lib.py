"""ctypes loader of libhalo.so (argument marshalling only; fails loudly if missing)."""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_size_t, c_uint, c_uint64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
# HALO_LIB_PATH: an alternative build of the same library (A/B timing of kernel variants in scripts/)
LIB_PATH = os.environ.get("HALO_LIB_PATH") or os.path.join(HERE, "libhalo.so")

HALO_OK = 0
STATUS_NAMES = {0: "HALO_OK", 1: "HALO_ERR_ARG", 2: "HALO_ERR_GEOMETRY", 3: "HALO_ERR_CAPACITY",
                4: "HALO_ERR_STATE", 5: "HALO_ERR_CUDA", 6: "HALO_ERR_PEER", 7: "HALO_ERR_TIMEOUT",
                8: "HALO_ERR_UNSUPPORTED"}

HALO_F_DETERMINISTIC = 0  # the default: the oracle's accumulation order, bit-exact (R15)
HALO_F_ATOMIC_UNPACK = 1 << 0
HALO_F_NO_HOME_CHECK = 1 << 1
HALO_F_GPU_FENCE = 1 << 2
HALO_F_TIMERS = 1 << 3
HALO_F_PAPER_FLAGS = 1 << 4
HALO_F_CE_PATH = 1 << 5
HALO_F_L2_PERSIST = 1 << 6
HALO_F_TMA_STORE = 1 << 7
HALO_F_TMA_GET = 1 << 8
HALO_F_ROUNDED_ZONES = 1 << 9
HALO_F_AUTO_TRANSPORT = 1 << 10
HALO_F_NCCL_BASELINE = 1 << 11
HALO_MAX_PULSES = 6

# every symbol include/halo.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "halo_init", "halo_query_config", "halo_local_ranks", "halo_pulse_order", "halo_scratch_bytes", "halo_register_buffers",
    "halo_ipc_export", "halo_ipc_import", "halo_set_maps", "halo_set_maps_explicit", "halo_get_layout",
    "halo_get_map", "halo_assign_home", "halo_migrate", "halo_transport", "halo_pme_reserve", "halo_pme_setup",
    "halo_pme_buffers", "halo_pme_send_x", "halo_pme_recv_f", "halo_exchange_x", "halo_exchange_f", "halo_exchange_xf", "halo_nccl_unique_id", "halo_nccl_init", "halo_nccl_version", "halo_nccl_exchange_x",
    "halo_nccl_exchange_f", "halo_step_host", "halo_packed_sizes", "halo_step_host_packed", "halo_pack_x_pulse",
    "halo_unpack_f_pulse", "halo_get_timers", "halo_get_trace", "halo_get_notify_counts", "halo_floor_pingpong", "halo_floor_launch", "halo_floor_empty_pair", "halo_floor_launch_remote", "halo_floor_bandwidth", "halo_probe_reserve", "halo_floor_payload", "halo_floor_bandwidth_multi", "halo_sync", "halo_strerror",
    "halo_last_error", "halo_destroy",
]


class halo_config(ctypes.Structure):
    _fields_ = [("grid", c_int * 3), ("box", c_float * 3), ("cutoff", c_float), ("pulses", c_int * 3),
                ("layout", c_int), ("capacity", c_int), ("device", c_int), ("flags", c_uint),
                ("nprocs", c_int), ("proc", c_int), ("timeout_s", c_double)]


_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libhalo.so; raises if it has not been built (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libhalo.so not found at {path}: run `python -m paper_2509_21527_b200.build` "
                           "(there is no CPU or PyTorch fallback)")
    lib = ctypes.CDLL(path)
    P = c_void_p
    IP = POINTER(c_int)
    sig = {
        "halo_init": ([POINTER(halo_config), POINTER(c_void_p)], c_int),
        "halo_query_config": ([POINTER(halo_config), IP, IP, IP, IP, POINTER(c_size_t)], c_int),
        "halo_local_ranks": ([P, IP, IP], c_int),
        "halo_pulse_order": ([P, IP, IP], c_int),
        "halo_scratch_bytes": ([P, POINTER(c_size_t)], c_int),
        "halo_register_buffers": ([P, c_int, P, P, P], c_int),
        "halo_ipc_export": ([P, P, POINTER(c_size_t)], c_int),
        "halo_ipc_import": ([P, P, c_size_t], c_int),
        "halo_set_maps": ([P, IP, P], c_int),
        "halo_set_maps_explicit": ([P, IP, IP, POINTER(IP), P], c_int),
        "halo_get_layout": ([P, c_int, IP, IP, IP, IP, IP, IP, IP, POINTER(c_uint)], c_int),
        "halo_get_map": ([P, c_int, c_int, IP, c_int], c_int),
        "halo_assign_home": ([P, P, c_int, c_int, P, IP, P], c_int),
        "halo_migrate": ([P, IP, POINTER(c_void_p), POINTER(c_void_p), IP, P], c_int),
        "halo_transport": ([P, IP], c_int),
        "halo_pme_reserve": ([P, c_int], c_int),
        "halo_pme_setup": ([P, P, IP], c_int),
        "halo_pme_buffers": ([P, POINTER(c_void_p), POINTER(c_void_p), IP], c_int),
        "halo_pme_send_x": ([P, P], c_int),
        "halo_pme_recv_f": ([P, c_int, P], c_int),
        "halo_exchange_x": ([P, P], c_int),
        "halo_exchange_f": ([P, P, c_int, P], c_int),
        "halo_exchange_xf": ([P, P, c_int, P], c_int),
        "halo_nccl_unique_id": ([P, POINTER(c_size_t)], c_int),
        "halo_nccl_init": ([P, P, c_size_t], c_int),
        "halo_nccl_version": ([IP], c_int),
        "halo_nccl_exchange_x": ([P, P], c_int),
        "halo_nccl_exchange_f": ([P, P, c_int, P], c_int),
        "halo_step_host": ([P, POINTER(c_void_p), POINTER(c_void_p), POINTER(c_void_p), POINTER(c_void_p), P, P], c_int),
        "halo_packed_sizes": ([P, POINTER(c_size_t), POINTER(c_size_t)], c_int),
        "halo_step_host_packed": ([P, P, P, P], c_int),
        "halo_pack_x_pulse": ([P, c_int, c_int, P, P], c_int),
        "halo_unpack_f_pulse": ([P, c_int, c_int, P, P, c_int, P], c_int),
        "halo_get_timers": ([P, POINTER(c_uint64), POINTER(c_uint64)], c_int),
        "halo_get_trace": ([P, c_int, POINTER(c_uint64), c_int, POINTER(c_int)], c_int),
        "halo_get_notify_counts": ([P, c_int, POINTER(c_uint), c_int], c_int),
        "halo_floor_pingpong": ([P, c_int, c_int, c_int, POINTER(c_double)], c_int),
        "halo_floor_launch": ([P, c_int, c_int, POINTER(c_double)], c_int),
        "halo_floor_empty_pair": ([P, P], c_int),
        "halo_floor_launch_remote": ([P, c_int, c_int, c_int, c_int, POINTER(c_double)], c_int),
        "halo_floor_bandwidth": ([P, c_int, c_size_t, c_int, c_int, POINTER(c_double)], c_int),
        "halo_probe_reserve": ([P, c_size_t], c_int),
        "halo_floor_payload": ([P, c_int, c_size_t, c_int, c_int, POINTER(c_double)], c_int),
        "halo_floor_bandwidth_multi": ([P, IP, c_int, c_size_t, c_int, c_int, POINTER(c_double)], c_int),
        "halo_sync": ([P], c_int),
        "halo_strerror": ([c_int], c_char_p),
        "halo_last_error": ([P], c_char_p),
        "halo_destroy": ([P], c_int),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("HALO_LIB_PATH") and not hasattr(lib, name):
            continue  # an older build under A/B timing may lack newer entry points
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib
