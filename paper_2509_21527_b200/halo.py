"""Thin Python binding of the libhalo C ABI (include/halo.h).

Same names as the C calls; argument marshalling only — every step of the halo
exchange runs in libhalo's CUDA kernels.  Pointers are plain integers (e.g.
``tensor.data_ptr()``); streams are ``torch.cuda.Stream.cuda_stream`` ints.
"""
from __future__ import annotations

import ctypes
from ctypes import c_double, c_int, c_size_t, c_uint, c_uint64, c_void_p

import numpy as np

from . import _lib
from ._lib import halo_config, STATUS_NAMES


class HaloError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def make_config(grid, box, cutoff, pulses, layout=3, capacity=1 << 16, device=0, flags=0, nprocs=1, proc=0,
                timeout_s=10.0) -> halo_config:
    cfg = halo_config()
    cfg.grid[:] = [int(v) for v in grid]
    cfg.box[:] = [float(v) for v in box]
    cfg.cutoff = float(cutoff)
    cfg.pulses[:] = [int(v) for v in pulses]
    cfg.layout = int(layout)
    cfg.capacity = int(capacity)
    cfg.device = int(device)
    cfg.flags = int(flags)
    cfg.nprocs = int(nprocs)
    cfg.proc = int(proc)
    cfg.timeout_s = float(timeout_s)
    return cfg


def query_config(grid, box, cutoff, pulses, layout=3, capacity=1 << 16, nprocs=1, proc=0):
    """halo_query_config: host-only plan (no CUDA).  Returns dict(first_rank, n_local, dims, scratch_bytes)."""
    lib = _lib.load()
    cfg = make_config(grid, box, cutoff, pulses, layout, capacity, 0, 0, nprocs, proc)
    a, b, n = c_int(), c_int(), c_int()
    dims = (c_int * _lib.HALO_MAX_PULSES)()
    sb = c_size_t()
    st = lib.halo_query_config(ctypes.byref(cfg), ctypes.byref(a), ctypes.byref(b), ctypes.byref(n), dims,
                               ctypes.byref(sb))
    if st != 0:
        raise HaloError(st, lib.halo_strerror(st).decode())
    return dict(first_rank=a.value, n_local=b.value, dims=[dims[i] for i in range(n.value)],
                scratch_bytes=sb.value)


class Halo:
    """One context per process (hosts nranks/nprocs DD ranks)."""

    def __init__(self, grid, box, cutoff, pulses, layout=3, capacity=1 << 16, device=0, flags=0,
                 nprocs=1, proc=0, timeout_s=10.0):
        self.lib = _lib.load()
        cfg = make_config(grid, box, cutoff, pulses, layout, capacity, device, flags, nprocs, proc, timeout_s)
        self.cfg = cfg
        self.layout = int(layout)
        self.nranks = int(grid[0]) * int(grid[1]) * int(grid[2])
        h = c_void_p()
        st = self.lib.halo_init(ctypes.byref(cfg), ctypes.byref(h))
        if st != 0:
            raise HaloError(st, self.lib.halo_strerror(st).decode())
        self.h = h

    # ---------------------------------------------------------------- helpers
    def _ck(self, st):
        if st != 0:
            msg = self.lib.halo_last_error(self.h).decode() if self.h else ""
            raise HaloError(st, msg or self.lib.halo_strerror(st).decode())

    def local_ranks(self):
        a, b = c_int(), c_int()
        self._ck(self.lib.halo_local_ranks(self.h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def pulse_order(self):
        n = c_int()
        dims = (c_int * _lib.HALO_MAX_PULSES)()
        self._ck(self.lib.halo_pulse_order(self.h, ctypes.byref(n), dims))
        return [dims[i] for i in range(n.value)]

    def scratch_bytes(self) -> int:
        b = c_size_t()
        self._ck(self.lib.halo_scratch_bytes(self.h, ctypes.byref(b)))
        return b.value

    def register_buffers(self, local, x_ptr, f_ptr, scratch_ptr):
        self._ck(self.lib.halo_register_buffers(self.h, int(local), c_void_p(x_ptr), c_void_p(f_ptr),
                                                c_void_p(scratch_ptr)))

    def ipc_export(self) -> bytes:
        n = c_size_t()
        self._ck(self.lib.halo_ipc_export(self.h, None, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        self._ck(self.lib.halo_ipc_export(self.h, buf, ctypes.byref(n)))
        return buf.raw[: n.value]

    def ipc_import(self, blobs):
        ln = len(blobs[0])
        assert all(len(b) == ln for b in blobs)
        buf = ctypes.create_string_buffer(b"".join(blobs), ln * len(blobs))
        self._ck(self.lib.halo_ipc_import(self.h, buf, c_size_t(ln)))

    def set_maps(self, n_home, stream=0):
        arr = (c_int * len(n_home))(*[int(v) for v in n_home])
        self._ck(self.lib.halo_set_maps(self.h, arr, c_void_p(stream)))

    def set_maps_explicit(self, n_home, maps, stream=0):
        """maps[local][pulse] = int array of ascending local row indices."""
        nl = len(n_home)
        P = len(self.pulse_order())
        arr = (c_int * nl)(*[int(v) for v in n_home])
        sizes = (c_int * max(1, nl * P))()
        ptrs = (ctypes.POINTER(c_int) * max(1, nl * P))()
        keep = []
        for l in range(nl):
            for p in range(P):
                m = np.ascontiguousarray(maps[l][p], dtype=np.int32)
                keep.append(m)
                sizes[l * P + p] = m.size
                ptrs[l * P + p] = m.ctypes.data_as(ctypes.POINTER(c_int))
        self._ck(self.lib.halo_set_maps_explicit(self.h, arr, sizes, ptrs, c_void_p(stream)))

    def get_layout(self, local):
        P = _lib.HALO_MAX_PULSES
        nh, nt, npl = c_int(), c_int(), c_int()
        ro, rs, ss, rm = (c_int * P)(), (c_int * P)(), (c_int * P)(), (c_int * P)()
        dm = (c_uint * P)()
        self._ck(self.lib.halo_get_layout(self.h, int(local), ctypes.byref(nh), ctypes.byref(nt), ctypes.byref(npl),
                                          ro, rs, ss, rm, dm))
        n = npl.value
        return dict(n_home=nh.value, n_total=nt.value, npulse=n, recv_off=list(ro[:n]), recv_size=list(rs[:n]),
                    send_size=list(ss[:n]), remote_off=list(rm[:n]), dep_mask=list(dm[:n]))

    def get_map(self, local, pulse) -> np.ndarray:
        lay = self.get_layout(local)
        n = lay["send_size"][pulse]
        out = np.zeros(max(n, 1), dtype=np.int32)
        self._ck(self.lib.halo_get_map(self.h, int(local), int(pulse),
                                       out.ctypes.data_as(ctypes.POINTER(c_int)), c_int(n)))
        return out[:n]

    def assign_home(self, x_ptr, n_atoms, stride, ids_ptr, stream=0):
        """Home rank of every row of a global DEVICE coordinate array (halo_assign_home);
        fills ids_ptr (device int32[n_atoms], grouped by rank, ascending) and returns the
        per-rank counts."""
        nr = self.nranks
        cnt = (c_int * nr)()
        self._ck(self.lib.halo_assign_home(self.h, c_void_p(x_ptr), int(n_atoms), int(stride), c_void_p(ids_ptr), cnt,
                                           c_void_p(stream)))
        return [int(cnt[r]) for r in range(nr)]

    def migrate(self, n_home, gid_ptrs, v_ptrs=None, stream=0):
        """NS-step home-atom redistribution (halo_migrate); returns the new n_home per local rank."""
        nl = len(n_home)
        arr = (c_int * nl)(*[int(v) for v in n_home])
        g = (c_void_p * nl)(*[c_void_p(p) for p in gid_ptrs])
        vv = (c_void_p * nl)(*[c_void_p(p) for p in v_ptrs]) if v_ptrs is not None else None
        out = (c_int * nl)()
        self._ck(self.lib.halo_migrate(self.h, arr, g, vv, out, c_void_p(stream)))
        return [int(out[l]) for l in range(nl)]

    # ---- PP <-> PME (halo_pme_*)
    def pme_reserve(self, pme_rank):
        self._ck(self.lib.halo_pme_reserve(self.h, int(pme_rank)))

    def pme_setup(self, stream=0):
        n = c_int()
        self._ck(self.lib.halo_pme_setup(self.h, c_void_p(stream), ctypes.byref(n)))
        return n.value

    def pme_buffers(self, nranks):
        x, f = c_void_p(), c_void_p()
        off = (c_int * (nranks + 1))()
        self._ck(self.lib.halo_pme_buffers(self.h, ctypes.byref(x), ctypes.byref(f), off))
        return x.value or 0, f.value or 0, [int(v) for v in off]

    def pme_send_x(self, stream=0):
        self._ck(self.lib.halo_pme_send_x(self.h, c_void_p(stream)))

    def pme_recv_f(self, accumulate=True, stream=0):
        self._ck(self.lib.halo_pme_recv_f(self.h, int(bool(accumulate)), c_void_p(stream)))

    def transport(self):
        """Transport of the current NS epoch: 'll', 'paper' or 'ce' (HALO_F_AUTO_TRANSPORT chooses per epoch)."""
        t = c_int()
        self._ck(self.lib.halo_transport(self.h, ctypes.byref(t)))
        return ("ll", "paper", "ce")[t.value]

    def exchange_x(self, stream=0):
        self._ck(self.lib.halo_exchange_x(self.h, c_void_p(stream)))

    def exchange_f(self, fshift_ptr=0, accumulate=True, stream=0):
        self._ck(self.lib.halo_exchange_f(self.h, c_void_p(fshift_ptr or None), int(bool(accumulate)),
                                          c_void_p(stream)))

    def exchange_xf(self, fshift_ptr=0, accumulate=True, stream=0):
        self._ck(self.lib.halo_exchange_xf(self.h, c_void_p(fshift_ptr or None), int(bool(accumulate)),
                                           c_void_p(stream)))

    # NCCL send/recv baseline (halo_nccl_*; the paper's serialized schedule, not the product)
    def nccl_unique_id(self) -> bytes:
        n = c_size_t(128)
        buf = ctypes.create_string_buffer(128)
        self._ck(self.lib.halo_nccl_unique_id(buf, ctypes.byref(n)))
        return buf.raw[: n.value]

    def nccl_init(self, uid: bytes):
        buf = ctypes.create_string_buffer(uid, len(uid))
        self._ck(self.lib.halo_nccl_init(self.h, buf, len(uid)))

    def nccl_exchange_x(self, stream=0):
        self._ck(self.lib.halo_nccl_exchange_x(self.h, c_void_p(stream)))

    def nccl_exchange_f(self, fshift_ptr=0, accumulate=True, stream=0):
        self._ck(self.lib.halo_nccl_exchange_f(self.h, c_void_p(fshift_ptr or None), int(bool(accumulate)),
                                               c_void_p(stream)))

    def step_host(self, x_home_ptrs, f_all_ptrs, x_halo_out_ptrs=None, f_home_out_ptrs=None, fshift_ptr=0,
                  stream=0):
        n = len(x_home_ptrs)

        def arr(ptrs):
            if ptrs is None:
                return None
            return (c_void_p * n)(*[c_void_p(p) for p in ptrs])

        self._ck(self.lib.halo_step_host(self.h, arr(x_home_ptrs), arr(f_all_ptrs), arr(x_halo_out_ptrs),
                                         arr(f_home_out_ptrs), c_void_p(fshift_ptr or None), c_void_p(stream)))

    def floor_empty_pair(self, stream=0):
        self._ck(self.lib.halo_floor_empty_pair(self.h, c_void_p(stream)))

    def packed_sizes(self):
        """(in_bytes, out_bytes) of halo_step_host_packed's host blocks for the current maps."""
        a, b = c_size_t(0), c_size_t(0)
        self._ck(self.lib.halo_packed_sizes(self.h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def step_host_packed(self, in_ptr, out_ptr=0, stream=0):
        self._ck(self.lib.halo_step_host_packed(self.h, c_void_p(in_ptr), c_void_p(out_ptr or None), c_void_p(stream)))

    def pack_x_pulse(self, local, pulse, sendbuf_ptr, stream=0):
        self._ck(self.lib.halo_pack_x_pulse(self.h, int(local), int(pulse), c_void_p(sendbuf_ptr), c_void_p(stream)))

    def unpack_f_pulse(self, local, pulse, recvbuf_ptr, fshift_ptr=0, accumulate=True, stream=0):
        self._ck(self.lib.halo_unpack_f_pulse(self.h, int(local), int(pulse), c_void_p(recvbuf_ptr),
                                              c_void_p(fshift_ptr or None), int(bool(accumulate)), c_void_p(stream)))

    def get_timers(self):
        a, b = c_uint64(), c_uint64()
        self._ck(self.lib.halo_get_timers(self.h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def get_notify_counts(self, which):
        """Cumulative system-scope flag stores per (local rank, pulse) (HALO_DEBUG=64, paper protocol)."""
        nl, P = self.local_ranks()[1], len(self.pulse_order())
        buf = (c_uint * max(1, nl * P))()
        self._ck(self.lib.halo_get_notify_counts(self.h, int(which), buf, len(buf)))
        return np.array(buf[: nl * P], dtype=np.int64).reshape(nl, P)

    def get_trace(self, which):
        """Per-CTA [start, record loaded, items done, exit, item0 tag, item0 end, item1 tag, item1 end]
        (ns; tag = kind << 16 | lrank << 8 | pulse) of the last x (0) / f (1) launch."""
        cap = 16 * 2048
        buf = (c_uint64 * cap)()
        n = c_int()
        self._ck(self.lib.halo_get_trace(self.h, int(which), buf, cap, ctypes.byref(n)))
        return np.array(buf[: 16 * n.value], dtype=np.uint64).reshape(-1, 16)

    def floor_pingpong(self, peer_rank, iters=10000, relaxed=False) -> float:
        v = c_double()
        self._ck(self.lib.halo_floor_pingpong(self.h, int(peer_rank), int(iters), int(bool(relaxed)), ctypes.byref(v)))
        return v.value

    def floor_launch(self, iters=1000, graph=False) -> float:
        v = c_double()
        self._ck(self.lib.halo_floor_launch(self.h, int(iters), int(bool(graph)), ctypes.byref(v)))
        return v.value

    def floor_launch_remote(self, peer_rank, words=1, iters=1000, graph=False) -> float:
        v = c_double()
        self._ck(self.lib.halo_floor_launch_remote(self.h, int(peer_rank), int(words), int(iters), int(bool(graph)),
                                                   ctypes.byref(v)))
        return v.value

    def floor_bandwidth(self, peer_rank, nbytes, mode=0, iters=20) -> float:
        """GB/s of SM peer stores (mode 0) or copy-engine copies (mode 1) into peer_rank's scratch."""
        v = c_double()
        self._ck(self.lib.halo_floor_bandwidth(self.h, int(peer_rank), c_size_t(int(nbytes)), int(mode), int(iters),
                                               ctypes.byref(v)))
        return v.value

    def probe_reserve(self, max_bytes):
        """Reserve the floor-probe area (before register_buffers; same size on every rank)."""
        self._ck(self.lib.halo_probe_reserve(self.h, c_size_t(int(max_bytes))))

    def floor_payload(self, peer_rank, nbytes, iters=200, ctas=592) -> float:
        """One-way latency (us) of an nbytes payload + its signal to peer_rank (collective with the peer)."""
        v = c_double()
        self._ck(self.lib.halo_floor_payload(self.h, int(peer_rank), c_size_t(int(nbytes)), int(iters), int(ctas),
                                             ctypes.byref(v)))
        return v.value

    def floor_bandwidth_multi(self, peers, nbytes, mode=0, iters=20) -> float:
        """Total GB/s from local rank 0 to len(peers) concurrent peers (SM stores / copy engine)."""
        arr = (c_int * len(peers))(*[int(p) for p in peers])
        v = c_double()
        self._ck(self.lib.halo_floor_bandwidth_multi(self.h, arr, len(peers), c_size_t(int(nbytes)), int(mode),
                                                     int(iters), ctypes.byref(v)))
        return v.value

    def sync(self):
        self._ck(self.lib.halo_sync(self.h))

    def destroy(self):
        if getattr(self, "h", None):
            self.lib.halo_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass
