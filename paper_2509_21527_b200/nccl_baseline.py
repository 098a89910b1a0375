"""The NCCL send/recv schedule of the halo exchange — the BASELINE, not the product.

This is the staged exchange the paper replaces (Fig. 1):
per pulse, a pack kernel (``halo_pack_x_pulse``), a grouped NCCL send/recv of
the packed rows into the receiver's halo range, and for forces the reverse
send/recv followed by a scatter-add kernel (``halo_unpack_f_pulse``), pulses
descending.  It runs on the maps the fused path built, so its results must be
bit-identical (SURVEY §8(c) pin G2) — used by ``bench.py`` for the baseline
timing and by the multi-process tests for schedule equivalence.

One DD rank per process (``sess.n_local == 1``); ``torch.distributed`` must be
initialised with the NCCL backend.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def neighbour(grid, r, d, delta):
    """DD rank of the cell at c + delta*e_d (periodic), rank = (cx*np_y + cy)*np_z + cz (R5)."""
    c = [r // (grid[1] * grid[2]), (r // grid[2]) % grid[1], r % grid[2]]
    c[d] = (c[d] + delta) % grid[d]
    return (c[0] * grid[1] + c[1]) * grid[2] + c[2]


class NcclSchedule:
    def __init__(self, sess):
        if sess.n_local != 1:
            raise ValueError("the NCCL baseline runs one DD rank per process")
        self.sess = sess
        self.lay = sess.layout_of(0)
        self.P = sess.npulse
        self.dims = sess.halo.pulse_order()
        self.me = sess.first_rank
        W = sess.layout
        dev = sess.device
        self.sendbuf = [torch.empty(max(self.lay["send_size"][p], 1), W, device=dev) for p in range(self.P)]
        self.fbuf = [torch.empty(max(self.lay["send_size"][p], 1), W, device=dev) for p in range(self.P)]

    def exchange_x(self, stream=None):
        s = self.sess
        st = (stream or torch.cuda.current_stream()).cuda_stream
        x, lay = s.x[0], self.lay
        for p in range(self.P):
            lo, up = neighbour(s.grid, self.me, self.dims[p], -1), neighbour(s.grid, self.me, self.dims[p], +1)
            n_s, n_r, off = lay["send_size"][p], lay["recv_size"][p], lay["recv_off"][p]
            s.halo.pack_x_pulse(0, p, self.sendbuf[p].data_ptr(), stream=st)
            ops = []
            if n_s:
                ops.append(dist.P2POp(dist.isend, self.sendbuf[p][:n_s], lo))
            if n_r:
                ops.append(dist.P2POp(dist.irecv, x[off: off + n_r], up))
            for w in dist.batch_isend_irecv(ops) if ops else []:
                w.wait()

    def exchange_f(self, fshift=None, stream=None):
        s = self.sess
        st = (stream or torch.cuda.current_stream()).cuda_stream
        f, lay = s.f[0], self.lay
        for p in range(self.P - 1, -1, -1):
            lo, up = neighbour(s.grid, self.me, self.dims[p], -1), neighbour(s.grid, self.me, self.dims[p], +1)
            n_s, n_r, off = lay["send_size"][p], lay["recv_size"][p], lay["recv_off"][p]
            ops = []
            if n_r:
                ops.append(dist.P2POp(dist.isend, f[off: off + n_r], up))
            if n_s:
                ops.append(dist.P2POp(dist.irecv, self.fbuf[p][:n_s], lo))
            for w in dist.batch_isend_irecv(ops) if ops else []:
                w.wait()
            s.halo.unpack_f_pulse(0, p, self.fbuf[p].data_ptr(), 0 if fshift is None else fshift.data_ptr(),
                                  stream=st)

    def step(self, fshift=None):
        self.exchange_x()
        self.exchange_f(fshift)
