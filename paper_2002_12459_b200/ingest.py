"""Device-side ingest: raw int64 pairs -> the
engines' input format, entirely in HBM.

Replaces the host preparation the reference runs before its operators:

* ``Relation.from_raw_pairs`` (relation.py:37-69): keep-first dedup of the
  tuples, dense ids in first-seen order  -> :func:`from_raw_pairs_device`
* ``semi_join_reduce_many`` (relation.py:119-140): common right values in
  ``repr`` order, kept tuples in input order, left ids re-assigned first-seen
  over the kept tuples  -> :func:`semi_join_reduce_device`
* ``_csr`` / ``IndexedRelation`` (relation.py:148-186): both CSR directions
  -> the :class:`DeviceIndexedRelation` these functions return.

A :class:`DeviceIndexedRelation` quacks like the reference's
``IndexedRelation`` (``rel.n``, ``rel.dom_left``, ``left_values``,
``fwd_indptr`` ...): the engines find its :class:`DeviceRelation` without an
upload, and the large host arrays are only copied back if something asks for
them.  Every dense id equals the one the reference assigns (checked against
``relation.py``'s host encoding in tests/test_gpu_ingest.py).
All compute is in libmmjoin_b200.so (csrc/ingest.cu: CUB radix sorts + flag /
scan / scatter kernels); PyTorch only allocates.
"""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from . import _native as nat
from .device import DeviceRelation
from .relation import ValueIndex

__all__ = ["DeviceIndexedRelation", "from_raw_pairs_device", "semi_join_reduce_device", "IngestWorkspace",
           "sorted_ids", "remap", "histogram", "distinct", "lookup", "csr"]


def _torch():
    import torch
    return torch


class IngestWorkspace:
    """One growable byte buffer shared by the ingest calls."""

    def __init__(self):
        self.buf = None

    def get(self, n: int):
        torch = _torch()
        need = int(nat.load().mmj_ingest_workspace_bytes(int(n)))
        if self.buf is None or self.buf.numel() < need:
            self.buf = torch.empty(need, dtype=torch.uint8, device="cuda")
        return self.buf, need


def _raw_tensor(raw):
    torch = _torch()
    if isinstance(raw, torch.Tensor):
        t = raw.to(device="cuda", dtype=torch.int64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(raw, dtype=np.int64))).to("cuda")
    t = t.reshape(-1, 2).contiguous()
    if t.shape[0] >= (1 << 31) - 1:
        raise ValueError("relations with 2^31 or more tuples are not supported")
    return t


def _scalar(t) -> int:
    return int(t.item())


def _dedup(t, ws: IngestWorkspace):
    torch = _torch()
    n = t.shape[0]
    out = torch.empty_like(t)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    buf, nb = ws.get(n)
    nat.call("mmj_ingest_dedup", nat.ptr(t), n, nat.ptr(out), nat.ptr(cnt), nat.ptr(buf), nb, nat.stream_handle())
    return out[:_scalar(cnt)]


def _first_seen(vals, stride: int, n: int, ws: IngestWorkspace):
    torch = _torch()
    ids = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    dct = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    buf, nb = ws.get(n)
    nat.call("mmj_ingest_first_seen", nat.ptr(vals), stride, n, nat.ptr(ids), nat.ptr(dct), nat.ptr(cnt),
             nat.ptr(buf), nb, nat.stream_handle())
    return ids[:n], dct[:_scalar(cnt)]


def _distinct(vals, stride: int, n: int, ws: IngestWorkspace):
    torch = _torch()
    out = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    buf, nb = ws.get(n)
    nat.call("mmj_ingest_distinct", nat.ptr(vals), stride, n, nat.ptr(out), nat.ptr(cnt), nat.ptr(buf), nb,
             nat.stream_handle())
    return out[:_scalar(cnt)]


def _intersect(a, b, ws: IngestWorkspace):
    torch = _torch()
    out = torch.empty(max(a.numel(), 1), dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    buf, nb = ws.get(a.numel())
    nat.call("mmj_ingest_intersect", nat.ptr(a), a.numel(), nat.ptr(b), b.numel(), nat.ptr(out), nat.ptr(cnt),
             nat.ptr(buf), nb, nat.stream_handle())
    return out[:_scalar(cnt)]


def _csr(rows, cols, n: int, dom_rows: int, dom_cols: int, ws: IngestWorkspace, want_rows: bool):
    torch = _torch()
    ptr = torch.empty(dom_rows + 1, dtype=torch.int32, device="cuda")
    idx = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    row_of = torch.empty(max(n, 1), dtype=torch.int32, device="cuda") if want_rows else None
    deg = torch.empty(max(dom_rows, 1), dtype=torch.int32, device="cuda")
    buf, nb = ws.get(max(n, dom_rows))
    nat.call("mmj_ingest_csr", nat.ptr(rows), nat.ptr(cols), n, dom_rows, dom_cols, nat.ptr(ptr), nat.ptr(idx),
             nat.ptr(row_of) if want_rows else 0, nat.ptr(deg), nat.ptr(buf), nb, nat.stream_handle())
    return ptr, idx[:n], (row_of[:n] if want_rows else None), deg[:dom_rows]


class _DeviceRel:
    """``Relation``-shaped view (relation.py:23-97) of a device-encoded relation."""

    def __init__(self, owner: "DeviceIndexedRelation", name: str, n: int, left_values, right_values, right_ids):
        self._owner = owner
        self.name = name
        self._n = n
        self.left_values = left_values          # numpy int64 (dom_left)
        self.right_values = right_values        # numpy int64 (dom_right), shared after a semi-join
        self._left_ids = None
        self._right_ids = right_ids               # ValueIndex or a zero-arg factory (built on first use)
        self._pairs = None

    @property
    def n(self) -> int:
        return self._n

    @property
    def dom_left(self) -> int:
        return len(self.left_values)

    @property
    def dom_right(self) -> int:
        return len(self.right_values)

    @property
    def right_ids(self):
        if callable(self._right_ids):
            self._right_ids = self._right_ids()
        return self._right_ids

    @property
    def left_ids(self):
        if self._left_ids is None:
            self._left_ids = ValueIndex(self.left_values)
        return self._left_ids

    @property
    def pairs(self) -> np.ndarray:
        """(n, 2) int64 dense pairs in the reference's tuple order (copied back on first use)."""
        if self._pairs is None:
            o = self._owner
            self._pairs = np.stack([o._lid.cpu().numpy(), o._rid.cpu().numpy()], axis=1).astype(np.int64)
        return self._pairs

    def raw_pairs(self):
        a = self.left_values[self.pairs[:, 0]].tolist()
        b = self.right_values[self.pairs[:, 1]].tolist()
        return iter(zip(a, b))

    def raw_pair_set(self) -> set:
        return set(self.raw_pairs())

    def raw_array(self) -> np.ndarray:
        return np.stack([self.left_values[self.pairs[:, 0]], self.right_values[self.pairs[:, 1]]], axis=1)

    def __repr__(self):
        return f"Relation({self.name!r}, n={self.n}, dom={self.dom_left}x{self.dom_right}, device)"


class DeviceIndexedRelation:
    """``IndexedRelation`` (relation.py:157-186) whose CSR lives in HBM.

    The engines read :attr:`device` (a :class:`DeviceRelation`, also seeded
    into the ``device_relation`` cache); the host attributes are materialised
    lazily, the degree vectors eagerly (they are small and the planners read
    them)."""

    def __init__(self, name, lid, rid, left_values_dev, right_values_host, right_ids, ws: IngestWorkspace,
                 right_values_dev=None):
        torch = _torch()
        self._right_values_dev = right_values_dev
        n = int(lid.numel())
        dom_l = int(left_values_dev.numel())
        dom_r = len(right_values_host)
        self._lid, self._rid = lid, rid
        self._left_values_dev = left_values_dev
        fwd_ptr, fwd_idx, fwd_row, ldeg = _csr(lid, rid, n, dom_l, dom_r, ws, True)
        rev_ptr, rev_idx, _, rdeg = _csr(rid, lid, n, dom_r, dom_l, ws, False)
        dr = DeviceRelation()
        dr.n, dr.dom_left, dr.dom_right = n, dom_l, dom_r
        dr.device = torch.device("cuda", torch.cuda.current_device())
        dr.fwd_ptr, dr.fwd_idx, dr.fwd_row = fwd_ptr, fwd_idx, fwd_row
        dr.rev_ptr, dr.rev_idx = rev_ptr, rev_idx
        dr.left_deg, dr.right_deg = ldeg, rdeg
        dr.fwd_ptr_host = fwd_ptr.cpu().numpy().astype(np.int64)
        dr.h2d_bytes = 0
        self.device = dr
        self._mmj_device_cache = {torch.cuda.current_device(): dr}
        self.left_deg = ldeg.cpu().numpy().astype(np.int64)
        self.right_deg = rdeg.cpu().numpy().astype(np.int64)
        self.left_deg.flags.writeable = False
        self.right_deg.flags.writeable = False
        self.rel = _DeviceRel(self, name, n, left_values_dev.cpu().numpy(), right_values_host, right_ids)
        self._host = {}

    # ---- lazily copied host CSR (relation.py:160-166 names, int64)
    def _h(self, key, t):
        if key not in self._host:
            self._host[key] = t.cpu().numpy().astype(np.int64)
        return self._host[key]

    @property
    def fwd_indptr(self):
        return self.device.fwd_ptr_host

    @property
    def fwd_indices(self):
        return self._h("fwd_idx", self.device.fwd_idx)

    @property
    def rev_indptr(self):
        return self._h("rev_ptr", self.device.rev_ptr)

    @property
    def rev_indices(self):
        return self._h("rev_idx", self.device.rev_idx)

    def fwd(self, a: int) -> np.ndarray:
        return self.fwd_indices[self.fwd_indptr[a]:self.fwd_indptr[a + 1]]

    def rev(self, b: int) -> np.ndarray:
        return self.rev_indices[self.rev_indptr[b]:self.rev_indptr[b + 1]]

    @property
    def n(self) -> int:
        return self.rel.n

    def shares_right_dict(self, other) -> bool:
        return self.rel.right_values is other.rel.right_values

    def out_join_with(self, other) -> int:
        if not self.shares_right_dict(other):
            raise ValueError("relations do not share a right dictionary; run semi_join_reduce first")
        return int(np.dot(self.right_deg, other.right_deg))

    def __repr__(self):
        return f"DeviceIndexedRelation({self.rel!r})"


def from_raw_pairs_device(name: str, raw, ws: Optional[IngestWorkspace] = None) -> DeviceIndexedRelation:
    """``build_indexed(Relation.from_raw_pairs(name, raw))`` on the device.

    ``raw``: (n, 2) int64 array or CUDA tensor of raw (left, right) values."""
    nat.require_cuda()
    ws = ws or IngestWorkspace()
    t = _dedup(_raw_tensor(raw), ws)
    n = t.shape[0]
    flat = t.reshape(-1)
    lid, lvals = _first_seen(flat, 2, n, ws)
    rid, rvals = _first_seen(flat[1:] if n else flat, 2, n, ws)
    rv = rvals.cpu().numpy()
    return DeviceIndexedRelation(name, lid, rid, lvals, rv, lambda: ValueIndex(rv), ws, right_values_dev=rvals)


def semi_join_reduce_device(raws: Sequence, names: Optional[Sequence[str]] = None,
                            ws: Optional[IngestWorkspace] = None) -> list:
    """``[build_indexed(r) for r in semi_join_reduce_many([Relation.from_raw_pairs(..) ..])]``
    on the device: every result shares one right dictionary (the common right
    values in ``repr`` order) and one host ``right_values`` object."""
    torch = _torch()
    nat.require_cuda()
    ws = ws or IngestWorkspace()
    names = list(names) if names is not None else [f"R{j}" for j in range(len(raws))]
    deduped = [_dedup(_raw_tensor(r), ws) for r in raws]
    common = None
    for t in deduped:
        d = _distinct(t.reshape(-1)[1:] if t.shape[0] else t.reshape(-1), 2, t.shape[0], ws)
        common = d if common is None else _intersect(common, d, ws)
    m = int(common.numel())
    right_sorted = torch.empty(max(m, 1), dtype=torch.int64, device="cuda")
    rank = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
    if m:
        buf, nb = ws.get(m)
        nat.call("mmj_ingest_repr_order", nat.ptr(common), m, nat.ptr(right_sorted), nat.ptr(rank), nat.ptr(buf), nb,
                 nat.stream_handle())
    rv = right_sorted[:m].cpu().numpy()
    shared_ids = []

    def rids():   # one ValueIndex for the whole group, built on first use
        if not shared_ids:
            shared_ids.append(ValueIndex(rv))
        return shared_ids[0]
    out = []
    for name, t in zip(names, deduped):
        n = t.shape[0]
        rid_all = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        if n:
            nat.call("mmj_ingest_lookup", nat.ptr(common), nat.ptr(rank), m, nat.ptr(t.reshape(-1)[1:]), 2, n,
                     nat.ptr(rid_all), nat.stream_handle())
        left_kept = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
        rid = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        buf, nb = ws.get(n)
        nat.call("mmj_ingest_filter", nat.ptr(t), nat.ptr(rid_all), n, nat.ptr(left_kept), nat.ptr(rid), nat.ptr(cnt),
                 nat.ptr(buf), nb, nat.stream_handle())
        k = _scalar(cnt)
        lid, lvals = _first_seen(left_kept, 1, k, ws)
        out.append(DeviceIndexedRelation(name, lid, rid[:k], lvals, rv, rids, ws, right_values_dev=right_sorted[:m]))
    return out


# ---- small device helpers reused by the BSI preparation (bsi.py)
def sorted_ids(vals, ws: Optional[IngestWorkspace] = None):
    """(ascending values, int32 position of each) of a device int64 vector."""
    torch = _torch()
    ws = ws or IngestWorkspace()
    n = int(vals.numel())
    srt = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    order = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    buf, nb = ws.get(n)
    nat.call("mmj_ingest_sort_ids", nat.ptr(vals), n, nat.ptr(srt), nat.ptr(order), nat.ptr(buf), nb,
             nat.stream_handle())
    return srt[:n], order[:n]


def remap(idx, table):
    torch = _torch()
    out = torch.empty_like(idx)
    nat.call("mmj_ingest_remap", nat.ptr(idx), int(idx.numel()), nat.ptr(table), nat.ptr(out), nat.stream_handle())
    return out


def histogram(idx, dom: int):
    torch = _torch()
    cnt = torch.empty(max(dom, 1), dtype=torch.int32, device="cuda")
    nat.call("mmj_ingest_histogram", nat.ptr(idx), int(idx.numel()), dom, nat.ptr(cnt), nat.stream_handle())
    return cnt[:dom]


def distinct(vals, ws: Optional[IngestWorkspace] = None):
    ws = ws or IngestWorkspace()
    return _distinct(vals, 1, int(vals.numel()), ws)


def lookup(sorted_vals, q, ids_of_sorted=None):
    torch = _torch()
    n = int(q.numel())
    out = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    nat.call("mmj_ingest_lookup", nat.ptr(sorted_vals), nat.ptr(ids_of_sorted) if ids_of_sorted is not None else 0,
             int(sorted_vals.numel()), nat.ptr(q), 1, n, nat.ptr(out), nat.stream_handle())
    return out[:n]


def csr(rows, cols, dom_rows: int, dom_cols: int, ws: Optional[IngestWorkspace] = None, want_rows: bool = True):
    ws = ws or IngestWorkspace()
    return _csr(rows, cols, int(rows.numel()), dom_rows, dom_cols, ws, want_rows)
