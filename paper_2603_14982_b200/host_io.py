"""Host-owned state with pipelined PCIe transfers.

A drop-in caller of the reference keeps the particle arrays on the host and
lets ``CoupledSim.step()`` mutate them.  ``HostMirror`` keeps pinned host
copies of a set of device tensors and moves them in row chunks on two copy
streams: the download of step k and the upload of step k + 1 use the two
directions of the link at the same time (chunk c of the upload only waits for
chunk c of the download), so a round trip costs about one direction's
transfer time instead of two.
"""
from __future__ import annotations

import torch


class HostMirror:
    def __init__(self, tensors, chunks=8):
        self.dev = list(tensors)
        self.host = [torch.empty_like(t, device="cpu").pin_memory() for t in self.dev]
        for h, t in zip(self.host, self.dev):
            h.copy_(t)
        # chunk list: (tensor index, row slice)
        self.parts = []
        for k, t in enumerate(self.dev):
            rows = t.shape[0]
            step = max(1, rows // max(1, chunks // len(self.dev)))
            for r0 in range(0, rows, step):
                self.parts.append((k, slice(r0, min(rows, r0 + step))))
        dev = self.dev[0].device
        self.s_up = torch.cuda.Stream(device=dev)
        self.s_down = torch.cuda.Stream(device=dev)
        self.ev_down = [None] * len(self.parts)

    @property
    def nbytes(self):
        return sum(t.numel() * t.element_size() for t in self.dev)

    def upload(self):
        """host -> device; the current stream waits for every chunk."""
        main = torch.cuda.current_stream()
        done = []
        for i, (k, sl) in enumerate(self.parts):
            if self.ev_down[i] is not None:
                self.s_up.wait_event(self.ev_down[i])
            with torch.cuda.stream(self.s_up):
                self.dev[k][sl].copy_(self.host[k][sl], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.s_up)
            done.append(ev)
        for ev in done:
            main.wait_event(ev)

    def download(self):
        """device -> host after the work queued so far on the current stream;
        the next upload of a chunk waits only for that chunk."""
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream())
        self.s_down.wait_event(ready)
        for i, (k, sl) in enumerate(self.parts):
            with torch.cuda.stream(self.s_down):
                self.host[k][sl].copy_(self.dev[k][sl], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.s_down)
            self.ev_down[i] = ev
        # the device tensors must not be overwritten before the copies read them
        torch.cuda.current_stream().wait_stream(self.s_down)

    def synchronize(self):
        self.s_down.synchronize()
