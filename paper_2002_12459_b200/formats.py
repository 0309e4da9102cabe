"""Result text formats of the reference CLI, produced on the device.

The reference's CLI prints each operator's result as sorted text lines of raw
dictionary values (cli.py:129-136 two-path, 154-161 star, 180-182 SSJ,
205-206 SCJ; 175-178 ordered SSJ keeps its own order):

    "\n".join(sorted(f"{left_values[a]} {right_values[c]}[ {count}]" ...))

Here the lines are built by format.cu from the device codes: each column's
dictionary becomes (rank of its string, string offsets, UTF-8 blob) tables
once per dictionary; every output tuple gets an int64 key of its columns'
ranks (the line order, see format.cu), the keys are radix-sorted on the
device, and the line bytes are written at scanned offsets.  The functions
return the text the CLI passes to ``click.echo`` (no trailing newline).
"""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from . import _native as nat


def _torch():
    import torch
    return torch


class Column:
    """Device string tables of one dictionary (or of the count values 0..m)."""

    def __init__(self, values: Sequence):
        torch = _torch()
        strs = [str(v) for v in values]
        n = len(strs)
        enc = [s.encode("utf-8") for s in strs]
        # Python's str order (code points) == UTF-8 byte order
        order = sorted(range(n), key=enc.__getitem__)
        rank = np.empty(max(n, 1), dtype=np.int32)
        rank[order] = np.arange(n, dtype=np.int32)
        lens = np.fromiter((len(b) for b in enc), dtype=np.int64, count=n)
        soff = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lens, out=soff[1:])
        blob = np.frombuffer(b"".join(enc) or b"\0", dtype=np.uint8)
        self.n = n
        self.rank = torch.from_numpy(rank).cuda()
        self.soff = torch.from_numpy(soff).cuda()
        self.blob = torch.from_numpy(blob.copy()).cuda()


def _column_cache(values) -> Column:
    """One Column per dictionary object (dictionaries are immutable lists),
    for the last _COLS_MAX dictionaries formatted."""
    key = id(values)
    hit = _COLS.pop(key, None)
    if hit is not None and hit[0] is values:
        _COLS[key] = hit                  # most recently used last
        return hit[1]
    col = Column(values)
    _COLS[key] = (values, col)
    while len(_COLS) > _COLS_MAX:
        _COLS.pop(next(iter(_COLS)))
    return col


_COLS: dict = {}
_COLS_MAX = 8


def _as_dev_i64(a):
    torch = _torch()
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.int64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.int64))).cuda()


def lines(codes, dims: Sequence[int], columns: Sequence[Column], counts=None, sort: bool = True) -> str:
    """Text of one line per code (columns decoded from the mixed-radix codes
    over ``dims``, then the count when given), sorted like Python's
    ``sorted()`` of the lines unless ``sort`` is False, joined by newlines."""
    import ctypes as C

    from .ingest import IngestWorkspace, sorted_ids
    torch = _torch()
    nat.require_cuda()
    codes = _as_dev_i64(codes)
    counts = _as_dev_i64(counts)
    n = int(codes.numel())
    if n == 0:
        return ""
    ncode = len(dims)
    cols = list(columns)
    if counts is not None:
        top = int(counts.max().item())
        if int(counts.min().item()) < 0:
            raise ValueError("counts must be non-negative")
        cols.append(Column(range(top + 1)))
    if len(cols) != ncode + (counts is not None) or len(cols) > 5:
        raise ValueError("one string column per code column (+ the count column), at most 5 in all")
    st = nat.stream_handle()
    dims_a = (C.c_int64 * 5)(*[int(d) for d in dims], *([1] * (5 - ncode)))
    rank_a = (C.c_void_p * 5)(*[nat.ptr(c.rank) for c in cols], *([None] * (5 - len(cols))))
    nrank_a = (C.c_int64 * 5)(*[max(c.n, 1) for c in cols], *([1] * (5 - len(cols))))
    soff_a = (C.c_void_p * 5)(*[nat.ptr(c.soff) for c in cols], *([None] * (5 - len(cols))))
    blob_a = (C.c_void_p * 5)(*[nat.ptr(c.blob) for c in cols], *([None] * (5 - len(cols))))
    cnt_p = nat.ptr(counts) if counts is not None else 0
    order_p = 0
    if sort:
        key = torch.empty(n, dtype=torch.int64, device="cuda")
        bad = torch.zeros(1, dtype=torch.int32, device="cuda")
        nat.call("mmj_format_keys", nat.ptr(codes), cnt_p, n, ncode, dims_a, rank_a, nrank_a, nat.ptr(key),
                 nat.ptr(bad), st)
        if int(bad.item()):
            raise ValueError("a decoded value lies outside its column's dictionary")
        _, order = sorted_ids(key, IngestWorkspace())
        order_p = nat.ptr(order)
    ln = torch.empty(n, dtype=torch.int32, device="cuda")
    nat.call("mmj_format_lengths", nat.ptr(codes), cnt_p, order_p, n, ncode, dims_a, soff_a, nat.ptr(ln), st)
    off = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    from .device import Workspace
    ws = Workspace()
    nat.call("mmj_exclusive_scan_i32", nat.ptr(ln), nat.ptr(off), n, nat.ptr(ws.scan_ws(n)), st)
    total = int(off[n].item()) if n else 0
    out = torch.empty(max(total, 1), dtype=torch.uint8, device="cuda")
    nat.call("mmj_format_write", nat.ptr(codes), cnt_p, order_p, n, ncode, dims_a, soff_a, blob_a, nat.ptr(off),
             nat.ptr(out), st)
    return bytes(out[:total].cpu().numpy()).decode("utf-8")


def twopath_lines(res, r, s, counts: Optional[bool] = None) -> str:
    """cli.py:129-136: ``{r.left_values[a]} {s.left_values[c]}[ {count}]``
    per output pair of ``res`` (an OutputSet of two_path_join(r, s)), sorted.
    ``r``/``s`` are the (reduced) relations or IndexedRelations joined."""
    rr, sr = getattr(r, "rel", r), getattr(s, "rel", s)
    with_counts = res.counts is not None if counts is None else counts
    return lines(res.codes, res.dims, [_column_cache(rr.left_values), _column_cache(sr.left_values)],
                 res.counts if with_counts else None)


def star_lines(res, rels, counts: Optional[bool] = None) -> str:
    """cli.py:154-161: one column per relation's left values (+ count)."""
    cols = [_column_cache(getattr(x, "rel", x).left_values) for x in rels]
    with_counts = res.counts is not None if counts is None else counts
    return lines(res.codes, res.dims, cols, res.counts if with_counts else None)


def ssj_lines(family, a, b, overlap, ordered: bool = False) -> str:
    """cli.py:180-182 (method mmjoin): ``{raw a} {raw b} {count}`` sorted;
    ``ordered`` (cli.py:175-178, ssj_ordered): the given order, unsorted."""
    dom = family.relation.dom_left
    codes = _as_dev_i64(a) * dom + _as_dev_i64(b)
    col = _column_cache(family.relation.left_values)
    return lines(codes, (dom, dom), [col, col], overlap, sort=not ordered)


def scj_lines(family, a, b) -> str:
    """cli.py:205-206: ``{raw small} {raw big}`` sorted."""
    dom = family.relation.dom_left
    codes = _as_dev_i64(a) * dom + _as_dev_i64(b)
    col = _column_cache(family.relation.left_values)
    return lines(codes, (dom, dom), [col, col])
