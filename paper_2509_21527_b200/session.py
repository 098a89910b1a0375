"""PyTorch plumbing around the C ABI: device memory, streams and the process
group that swaps CUDA-IPC blobs (north_star: "PyTorch is used only for device
memory, streams and the process group").  No halo arithmetic here.
"""
from __future__ import annotations

import numpy as np
import torch

from .halo import Halo


def assign_home(X: np.ndarray, L, grid, cutoff, pulses, device=0):
    """Home DD rank of every atom at a neighbour-search step (input preparation,
    not a hot-path step), computed on the GPU by ``halo_assign_home`` (R3/R4
    planes, stable counting sort).  Returns a list, per rank, of atom ids in
    ascending order."""
    X = np.ascontiguousarray(np.asarray(X, dtype=np.float32))
    dev = torch.device("cuda", device)
    h = Halo(grid, L, cutoff, pulses, capacity=1, device=device)
    try:
        xd = torch.from_numpy(X).to(dev)
        ids = torch.empty(max(X.shape[0], 1), dtype=torch.int32, device=dev)
        counts = h.assign_home(xd.data_ptr(), X.shape[0], X.shape[1], ids.data_ptr(),
                               torch.cuda.current_stream(dev).cuda_stream)
        ids = ids[: X.shape[0]].cpu().numpy().astype(np.int64)
    finally:
        h.destroy()
    return np.split(ids, np.cumsum(counts)[:-1])


class HaloSession:
    """One per process: allocates (torch) x, f, scratch for every local DD rank,
    registers them, and imports the peers' IPC blobs over ``torch.distributed``."""

    def __init__(self, grid, box, cutoff, pulses, layout=3, capacity=1 << 16, device=0, flags=0,
                 nprocs=1, proc=0, timeout_s=10.0, group=None, pme_rank=None, probe_bytes=None):
        self.device = torch.device("cuda", device)
        torch.cuda.set_device(self.device)
        self.halo = Halo(grid, box, cutoff, pulses, layout=layout, capacity=capacity, device=device, flags=flags,
                         nprocs=nprocs, proc=proc, timeout_s=timeout_s)
        self.grid, self.box, self.cutoff, self.pulses = tuple(grid), tuple(box), cutoff, tuple(pulses)
        self.layout, self.capacity, self.nprocs, self.proc = layout, capacity, nprocs, proc
        self.first_rank, self.n_local = self.halo.local_ranks()
        self.npulse = len(self.halo.pulse_order())
        self.pme_rank = pme_rank
        if probe_bytes:  # floor-probe area (halo_probe_reserve), before PME and registration
            self.halo.probe_reserve(probe_bytes)
        if pme_rank is not None:  # PP <-> PME buffers in pme_rank's scratch (before registration)
            self.halo.pme_reserve(pme_rank)
        sb = self.halo.scratch_bytes()
        # one allocation per array kind for all local ranks (views per rank, 512-B aligned rows blocks):
        # one copy resets every local rank's forces, one IPC handle covers every local rank
        cap_pad = (capacity + 127) // 128 * 128
        sb_pad = (sb + 4095) // 4096 * 4096
        self.x_all = torch.zeros(self.n_local, cap_pad, layout, dtype=torch.float32, device=self.device)
        self.f_all = torch.zeros(self.n_local, cap_pad, layout, dtype=torch.float32, device=self.device)
        self.scratch_all = torch.zeros(self.n_local, sb_pad, dtype=torch.uint8, device=self.device)
        self.x = [self.x_all[l] for l in range(self.n_local)]
        self.f = [self.f_all[l] for l in range(self.n_local)]
        self.scratch = [self.scratch_all[l, :sb] for l in range(self.n_local)]
        for l in range(self.n_local):
            self.halo.register_buffers(l, self.x[l].data_ptr(), self.f[l].data_ptr(), self.scratch[l].data_ptr())
        if nprocs > 1:
            import torch.distributed as dist
            blob = self.halo.ipc_export()
            blobs = [None] * nprocs
            dist.all_gather_object(blobs, blob, group=group)
            self.halo.ipc_import(blobs)
        self.n_home = [0] * self.n_local

    # ------------------------------------------------------------- inputs
    def load_home(self, rows_per_local):
        """rows_per_local[l]: float32 [n_home, layout] (or [n_home, 3] + zero w) host array."""
        for l, rows in enumerate(rows_per_local):
            rows = np.asarray(rows, dtype=np.float32)
            n = rows.shape[0]
            if n > self.capacity:
                raise ValueError("n_home exceeds capacity")
            t = torch.zeros(n, self.layout, dtype=torch.float32)
            t[:, :rows.shape[1]] = torch.from_numpy(rows)
            self.x[l][:n].copy_(t.to(self.device))
            self.n_home[l] = n
        torch.cuda.synchronize(self.device)

    def set_maps(self, stream=None):
        self.halo.set_maps(self.n_home, stream=self._s(stream))

    def set_maps_explicit(self, maps, stream=None):
        self.halo.set_maps_explicit(self.n_home, maps, stream=self._s(stream))

    def migrate(self, gid, v=None, stream=None):
        """NS-step redistribution of the home rows (halo_migrate): gid[l] / v[l] are
        device tensors (int32 [capacity] / float32 [capacity, layout]) of local rank l,
        rewritten in place with x; returns and records the new n_home per local rank."""
        self.n_home = self.halo.migrate(self.n_home, [g.data_ptr() for g in gid],
                                        [t.data_ptr() for t in v] if v is not None else None, stream=self._s(stream))
        return list(self.n_home)

    # ---- PP <-> PME
    def pme_setup(self, stream=None):
        """After every set_maps: all-gather the home counts; returns (n_total, row_off)."""
        n = self.halo.pme_setup(stream=self._s(stream))
        nranks = self.grid[0] * self.grid[1] * self.grid[2]
        _, _, off = self.halo.pme_buffers(nranks)
        return n, off

    def pme_buffers(self):
        """(pme_x, pme_f) as float32 [nranks*capacity, layout] views of the scratch on the
        process hosting pme_rank (None elsewhere)."""
        nranks = self.grid[0] * self.grid[1] * self.grid[2]
        px, pf, _ = self.halo.pme_buffers(nranks)
        if not px:
            return None, None
        rows = nranks * self.capacity
        out = []
        for ptr in (px, pf):
            for l in range(self.n_local):
                base = self.scratch[l].data_ptr()
                if base <= ptr < base + self.scratch[l].numel():
                    o = ptr - base
                    out.append(self.scratch[l][o: o + rows * self.layout * 4].view(torch.float32).view(rows, self.layout))
                    break
        return out[0], out[1]

    def pme_send_x(self, stream=None):
        self.halo.pme_send_x(stream=self._s(stream))

    def pme_recv_f(self, accumulate=True, stream=None):
        self.halo.pme_recv_f(accumulate, stream=self._s(stream))

    def layout_of(self, l):
        return self.halo.get_layout(l)

    def exchange_x(self, stream=None):
        self.halo.exchange_x(stream=self._s(stream))

    def exchange_f(self, fshift=None, accumulate=True, stream=None):
        self.halo.exchange_f(fshift.data_ptr() if fshift is not None else 0, accumulate, stream=self._s(stream))

    def nccl_init(self, group=None):
        """NCCL communicator of the send/recv baseline (halo_nccl_init): process 0's
        unique id is broadcast over torch.distributed; one DD rank per process."""
        import torch.distributed as dist
        uid = [self.halo.nccl_unique_id() if self.proc == 0 else None]
        if self.nprocs > 1:
            dist.broadcast_object_list(uid, src=0, group=group)
        self.halo.nccl_init(uid[0])

    def exchange_xf(self, fshift=None, accumulate=True, stream=None):
        self.halo.exchange_xf(fshift.data_ptr() if fshift is not None else 0, accumulate, stream=self._s(stream))

    @staticmethod
    def _s(stream):
        if stream is None:
            return torch.cuda.current_stream().cuda_stream
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)

    def destroy(self):
        self.halo.sync()
        self.halo.destroy()
