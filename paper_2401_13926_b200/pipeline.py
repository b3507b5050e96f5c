"""Streamed batch driver: a sequence of same-pattern batches through one device handle with
the host traffic overlapped (the harness loop of harness._run_direct_family,
harness.py:217-269, for a batch of independent systems per barrier step).

Each batch (``values [B][nnz]``, ``rhs [B][n]`` in pinned host memory) goes through
``kkt_dev_refactor`` then ``kkt_dev_step_solve`` (lu_solve -> refine_fgmres) on the handle's
stream, while one copy stream uploads the NEXT batch's inputs and another downloads the
PREVIOUS batch's solution (both PCIe directions at once).  Values and rhs have their own events: the refactorization starts once the
values have landed, the rhs upload overlaps it.  Device buffers are double-buffered; events
order the copies against the step.  Nothing is computed on the host.
"""

from __future__ import annotations

import numpy as np

from .device import DeviceSystem


class BatchPipeline:
    """``run(batches)`` -> list of per-batch reports; solutions land in the caller's pinned
    ``x`` arrays.  ``batches`` yields ``(values, rhs, x_out, delta)`` with host tensors
    (torch, pinned) — ``delta`` a float or per-system sequence (barrier-tied tolerance)."""

    def __init__(self, dev: DeviceSystem, layout: int, m: int = 10, max_outer: int = 10):
        torch = dev.torch
        self.dev, self.layout, self.m, self.max_outer = dev, layout, m, max_outer
        import os
        self.split = os.environ.get("KKT_PIPE_SPLIT", "1") != "0"  # refactor on values arrival
        self.torch = torch
        self.copy = torch.cuda.Stream(device=dev.device)   # host -> device
        self.copy_out = torch.cuda.Stream(device=dev.device)  # device -> host (PCIe is duplex)
        self._v = [None, None]
        self._r = [None, None]
        self._x = [None, None]

    def _bufs(self, i, values, rhs):
        t = self.torch
        if self._v[i] is None or self._v[i].shape != values.shape:
            self._v[i] = t.empty(values.shape, dtype=t.float64, device=self.dev.device)
            self._r[i] = t.empty(rhs.shape, dtype=t.float64, device=self.dev.device)
            self._x[i] = t.empty(rhs.shape, dtype=t.float64, device=self.dev.device)
        return self._v[i], self._r[i], self._x[i]

    def run(self, batches):
        t = self.torch
        dev = self.dev
        items = list(batches)
        if not items:
            return []
        reps = []
        up_vals = [t.cuda.Event(), t.cuda.Event()]
        up_done = [t.cuda.Event(), t.cuda.Event()]
        down_done = [t.cuda.Event(), t.cuda.Event()]
        step_done = [t.cuda.Event(), t.cuda.Event()]
        for e in down_done:
            e.record(self.copy_out)

        def upload(i):
            v, r, _ = self._bufs(i % 2, items[i][0], items[i][1])
            with t.cuda.stream(self.copy):
                self.copy.wait_event(step_done[i % 2])  # step i-2 has consumed the buffer
                v.copy_(items[i][0], non_blocking=True)
                up_vals[i % 2].record(self.copy)
                r.copy_(items[i][1], non_blocking=True)
                up_done[i % 2].record(self.copy)

        def download(i):
            with t.cuda.stream(self.copy_out):
                self.copy_out.wait_event(step_done[i % 2])
                items[i][2].copy_(self._x[i % 2], non_blocking=True)
                down_done[i % 2].record(self.copy_out)

        for e in step_done:
            e.record(dev.stream)
        upload(0)
        for i in range(len(items)):
            slot = i % 2
            v, r, x = self._v[slot], self._r[slot], self._x[slot]
            if self.split:
                dev.stream.wait_event(up_vals[slot])
                dev.refactor_device(v, self.layout)      # async: overlaps this batch's rhs upload
            dev.stream.wait_event(up_done[slot])
            dev.stream.wait_event(down_done[slot])  # x of batch i-2 is on the host
            if i + 1 < len(items):
                upload(i + 1)
            if i >= 1:
                download(i - 1)
            if self.split:
                reps.append(dev.step_solve(r, x, True, self.m, self.max_outer, items[i][3]))
            else:
                reps.append(dev.step(v, self.layout, r, x, True, self.m, self.max_outer, items[i][3]))
            step_done[slot].record(dev.stream)
        download(len(items) - 1)
        self.copy.synchronize()
        self.copy_out.synchronize()
        return reps


def as_pinned(a: np.ndarray):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
