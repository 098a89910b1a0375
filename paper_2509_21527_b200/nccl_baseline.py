"""The NCCL send/recv schedule of the halo exchange — the BASELINE, not the product.

Thin marshalling over the C ABI (``halo_nccl_*``, csrc/nccl_baseline.cu): the
paper's serialized per-pulse schedule (Fig. 1) — pack
kernel, ``ncclGroupStart/ncclSend/ncclRecv/ncclGroupEnd`` per pulse, and for
forces the reverse send/recv followed by the ordered scatter-add kernel, pulses
descending — enqueued by the library on the caller's stream (eager or inside a
CUDA graph).  It runs on the maps the fused path built, so its results must be
bit-identical (SURVEY §8(c) pin G2).  One DD rank per process.
"""
from __future__ import annotations

import torch


class NcclSchedule:
    def __init__(self, sess, group=None):
        if sess.n_local != 1:
            raise ValueError("the NCCL baseline runs one DD rank per process")
        self.sess = sess
        sess.nccl_init(group=group)

    def exchange_x(self, stream=None):
        self.sess.halo.nccl_exchange_x(stream=self.sess._s(stream))

    def exchange_f(self, fshift=None, stream=None):
        self.sess.halo.nccl_exchange_f(0 if fshift is None else fshift.data_ptr(), True, stream=self.sess._s(stream))

    def step(self, fshift=None, stream=None):
        self.exchange_x(stream)
        self.exchange_f(fshift, stream)
