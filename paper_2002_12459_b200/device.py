"""Device-resident form of an ``IndexedRelation`` and small buffer helpers.

The upload converts the reference's int64 CSR arrays (relation.py:157-166)
to int32 (every dense id and offset of the path is < 2^31) and adds
``fwd_row`` (the left id of each tuple in forward order), which the
x-driven light expansion and the operand build read.  PyTorch is used only as
the device allocator and stream provider.
"""

from __future__ import annotations

import numpy as np

from . import _native as nat

INT32_MAX = np.iinfo(np.int32).max


def _torch():
    import torch
    return torch


class DeviceRelation:
    """int32 CSR of one relation in HBM (both directions + degrees)."""

    __slots__ = ("n", "dom_left", "dom_right", "fwd_ptr", "fwd_idx", "fwd_row", "rev_ptr", "rev_idx",
                 "left_deg", "right_deg", "fwd_ptr_host", "device", "h2d_bytes")

    @classmethod
    def from_indexed(cls, idx, device=None, pinned: bool = False) -> "DeviceRelation":
        torch = _torch()
        nat.require_cuda()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        n = int(idx.rel.n)
        dom_l = int(idx.rel.dom_left)
        dom_r = int(idx.rel.dom_right)
        if n > INT32_MAX or dom_l > INT32_MAX or dom_r > INT32_MAX:
            raise ValueError("relations with more than 2^31-1 tuples/values are not supported")
        host = {
            "fwd_ptr": np.asarray(idx.fwd_indptr),
            "fwd_idx": np.asarray(idx.fwd_indices),
            "rev_ptr": np.asarray(idx.rev_indptr),
            "rev_idx": np.asarray(idx.rev_indices),
            "left_deg": np.asarray(idx.left_deg),
            "right_deg": np.asarray(idx.right_deg),
        }
        host["fwd_row"] = np.repeat(np.arange(dom_l, dtype=np.int32), host["left_deg"])
        self = cls()
        self.n, self.dom_left, self.dom_right = n, dom_l, dom_r
        self.device = dev
        self.fwd_ptr_host = host["fwd_ptr"].astype(np.int64, copy=False)
        nbytes = 0
        for k, v in host.items():
            a = np.ascontiguousarray(v, dtype=np.int32)
            t = torch.from_numpy(a)
            if pinned:
                t = t.pin_memory()
            nbytes += a.nbytes
            setattr(self, k, t.to(dev, non_blocking=pinned))
        self.h2d_bytes = nbytes
        return self


def device_relation(idx) -> DeviceRelation:
    """Cached upload of an IndexedRelation (reference or local class)."""
    torch = _torch()
    nat.require_cuda()
    dev = torch.cuda.current_device()
    cache = getattr(idx, "_mmj_device_cache", None)
    if cache is None:
        cache = {}
        try:
            idx._mmj_device_cache = cache
        except AttributeError:
            return DeviceRelation.from_indexed(idx)
    dr = cache.get(dev)
    if dr is None or dr.n != idx.rel.n:
        dr = cache[dev] = DeviceRelation.from_indexed(idx)
    return dr


class Workspace:
    """Grow-only scratch buffers keyed by role (avoids per-call allocation)."""

    def __init__(self):
        self._bufs = {}

    def get(self, key, numel: int, dtype):
        torch = _torch()
        numel = max(int(numel), 1)
        t = self._bufs.get(key)
        if t is None or t.numel() < numel or t.dtype != dtype:
            t = torch.empty(max(numel, int(numel * 1.25) if t is not None else numel), dtype=dtype,
                            device="cuda")
            self._bufs[key] = t
        return t[:numel]

    def scan_ws(self, n: int):
        lib = nat.load()
        torch = _torch()
        return self.get("scan_ws", lib.mmj_scan_workspace_bytes(int(max(n, 1))), torch.uint8)
