"""Applications on the B200 join-project engine (drop-in for ``mmjoin.apps``
on the hot path: apps.py:26-72, 291-351).

  SetFamily            apps.py:26-50
  ssj_mmjoin           apps.py:57-72   exact overlap counts on the tensor-core
                                       count path; the (a < b, count >= c)
                                       filter runs inside the emission kernel
  ssj_ordered          apps.py:291-294
  scj_join_project     apps.py:297-304
  bsi_batch_size       apps.py:307-311
  bsi_answer_batch     apps.py:314-351 per-query heavy-y bitset test plus a
                                       light-list merge intersection (bsi.cu)

``*_arrays`` variants return numpy arrays for outputs too large for Python
dicts/lists (cfg4: ~2.4e8 pairs; cfg5: 4M answers).
"""

from __future__ import annotations

import math
from typing import Optional, Sequence

import numpy as np

from .optimizer import PARTITIONED, ThresholdPlan
from .relation import IndexedRelation, Relation, ValueIndex, build_indexed

__all__ = ["SetFamily", "ssj_mmjoin", "ssj_mmjoin_arrays", "ssj_ordered", "scj_join_project",
           "bsi_batch_size", "bsi_answer_batch", "bsi_answer_batch_arrays"]


class SetFamily:
    """A family of non-empty sets stored as a (set-id, element-id) relation."""

    def __init__(self, relation: Relation):
        self.relation = relation
        self.indexed = build_indexed(relation)
        self._sizes = np.asarray(self.indexed.left_deg)

    @property
    def sets(self) -> dict:
        return {a: self.indexed.fwd(a) for a in range(self.relation.dom_left)}

    @classmethod
    def from_dict(cls, sets: dict) -> "SetFamily":
        pairs = [(a, e) for a, elems in sets.items() for e in elems]
        return cls(Relation.from_raw_pairs("sets", pairs))

    def __len__(self):
        return self.relation.dom_left

    def size(self, a: int) -> int:
        return int(self._sizes[a])

    def raw_id(self, a: int):
        return self.relation.left_values[a]

    def raw_pair(self, a: int, b: int) -> tuple:
        return (self.raw_id(a), self.raw_id(b))


def _ssj_plan(idx, plan: Optional[ThresholdPlan], c: int = 1, upper_only: bool = True) -> ThresholdPlan:
    from .optimizer import gpu_plan
    return plan if plan is not None else gpu_plan(idx, idx, counts=True, min_count=c, upper_only=upper_only)


def _device_pairs(eng):
    """Run a count-path engine; (codes, counts) concatenated on the device
    (each chunk is copied out of the engine's reused workspace)."""
    import torch
    codes, counts = [], []

    def sink(ch):
        codes.append(ch.codes.clone())
        counts.append(ch.counts.clone())

    eng.run(sink)
    if not codes:
        return (torch.empty(0, dtype=torch.int64, device="cuda"), torch.empty(0, dtype=torch.int32, device="cuda"))
    return torch.cat(codes), torch.cat(counts)


# compact the family when at most this share of its sets can reach overlap c
COMPACT_MAX_KEPT = 0.9


def _compact_host_plan(idx, c: int):
    """Host side of the compaction: (#kept sets, their CSR offsets, their
    degrees), all read-only.  A function of the family's (frozen) degree
    vector and c alone, so it is remembered on the index object: repeated
    joins over one family (batches, shards, bench steps) skip ~0.6 ms of numpy
    scans while the device compaction itself runs every time."""
    ldeg = np.asarray(idx.left_deg)
    memo = getattr(idx, "_mmj_compact_plan", None)
    if memo is not None and memo[0] == c and memo[1] is idx.left_deg and not ldeg.flags.writeable:
        return memo[2]
    keep = ldeg >= c
    nk = int(keep.sum())
    hdeg = np.ascontiguousarray(ldeg[keep])
    ptr = np.concatenate([[0], np.cumsum(hdeg, dtype=np.int64)])
    for arr in (hdeg, ptr):
        arr.flags.writeable = False      # engine._host_max memoises read-only degree vectors
    plan = (nk, ptr, hdeg)
    if not ldeg.flags.writeable:
        try:
            idx._mmj_compact_plan = (c, idx.left_deg, plan)
        except AttributeError:
            pass
    return plan


def _compact_family(idx, c: int, ws=None):
    """Sets with fewer than ``c`` elements reach no overlap >= c (the
    ``cnt >= c`` filter of apps.py:61-62), so their rows and columns of the
    count matrix are dead work: drop them on the device and renumber the kept
    sets 0..n'-1 in id order (``mmj_compact_rows``).  The renumbering is
    monotone, so the compact codes come out in the same ascending order and
    :func:`_decode_compact` maps them back one-to-one.  cfg4: 28.8k of 100k
    sets kept, 12x fewer count-matrix cells.  Returns (DeviceRelation,
    orig ids (device int32), host left degrees) or None when the saving is
    small."""
    import torch

    from . import _native as nat
    from .device import DeviceRelation, device_relation
    from .ingest import IngestWorkspace
    nk, fwd_ptr_host, hdeg = _compact_host_plan(idx, c)
    if nk == 0 or nk > COMPACT_MAX_KEPT * len(idx.left_deg):
        return None   # nothing to save (or nothing left: the plain engine handles empty outputs)
    dr = device_relation(idx)
    n, dom, dom_y = dr.n, dr.dom_left, dr.dom_right

    def buf(k, key):
        if ws is not None:
            return ws.get("cf_" + key, max(k, 1), torch.int32)
        return torch.empty(max(k, 1), dtype=torch.int32, device="cuda")
    new_id, orig = buf(dom, "new_id"), buf(dom, "orig")
    dc = DeviceRelation()
    dc.fwd_ptr, dc.fwd_idx, dc.fwd_row, dc.left_deg = (buf(dom + 1, "fptr"), buf(n, "fidx"), buf(n, "frow"),
                                                       buf(dom, "ldeg"))
    dc.rev_ptr, dc.rev_idx, dc.right_deg = buf(dom_y + 1, "rptr"), buf(n, "ridx"), buf(dom_y, "rdeg")
    sizes = (ws.get("cf_sizes", 2, torch.int64) if ws is not None
             else torch.empty(2, dtype=torch.int64, device="cuda"))   # written by mmj_compact_rows
    if ws is not None:
        nb = int(nat.load().mmj_ingest_workspace_bytes(int(max(n, dom, dom_y))))
        ws_buf = ws.get("cf_ingest", nb, torch.uint8)
    else:
        ws_buf, nb = IngestWorkspace().get(max(n, dom, dom_y))
    nat.call("mmj_compact_rows", nat.ptr(dr.fwd_ptr), nat.ptr(dr.fwd_idx), nat.ptr(dr.fwd_row), nat.ptr(dr.rev_ptr),
             nat.ptr(dr.rev_idx), nat.ptr(dr.left_deg), n, dom, dom_y, int(c), nat.ptr(new_id), nat.ptr(orig),
             nat.ptr(dc.fwd_ptr), nat.ptr(dc.fwd_idx), nat.ptr(dc.fwd_row), nat.ptr(dc.left_deg), nat.ptr(dc.rev_ptr),
             nat.ptr(dc.rev_idx), nat.ptr(dc.right_deg), nat.ptr(sizes), nat.ptr(ws_buf), nb, nat.stream_handle())
    # the compacted offsets follow from the host degrees (kept sets keep their
    # order and their whole rows): no device -> host copy, no sync
    dom_c = nk
    dc.fwd_ptr_host = fwd_ptr_host
    n_c = int(dc.fwd_ptr_host[-1])
    dc.n, dc.dom_left, dc.dom_right, dc.device, dc.h2d_bytes = n_c, dom_c, dom_y, dr.device, 0
    dc.fwd_ptr, dc.left_deg = dc.fwd_ptr[:dom_c + 1], dc.left_deg[:dom_c]
    dc.fwd_idx, dc.fwd_row, dc.rev_idx = dc.fwd_idx[:n_c], dc.fwd_row[:n_c], dc.rev_idx[:n_c]
    return dc, orig[:dom_c], hdeg


def _decode_compact(codes, dom_c: int, orig, dom: int):
    """compact codes a' * dom_c + b' -> orig[a'] * dom + orig[b'], in place"""
    from . import _native as nat
    if codes.numel():
        nat.call("mmj_decode_compact_codes", nat.ptr(codes), int(codes.numel()), dom_c, nat.ptr(orig),
                 nat.ptr(orig), dom, nat.ptr(codes), nat.stream_handle())
    return codes


def _ssj_engine(idx, c: int, plan: ThresholdPlan, chunk_rows: Optional[int] = None, compact: bool = True,
                ws=None):
    """(engine, decode) for the SSJ count join over ``idx``: the engine runs on
    the compacted family when sets below ``c`` are a large share, and
    ``decode(codes)`` maps its codes back to ``idx``'s dense ids.  ``ws``: a
    workspace reused across calls (the compacted family and the engine's
    buffers live in it; one call at a time)."""
    from .joinproject import _engine
    comp = _compact_family(idx, c, ws) if (compact and c > 1) else None
    if comp is None:
        return (_engine(idx, idx, plan, True, min_count=c, upper_only=True, chunk_rows=chunk_rows, ws=ws),
                (lambda x: x))
    from .engine import TwoPathEngine
    dc, orig, hdeg = comp
    if plan.strategy == PARTITIONED:
        d1, d2 = plan.delta1, plan.delta2
    else:
        d1 = d2 = max(dc.n, 1)
    eng = TwoPathEngine(dc, dc, plan.strategy, d1, d2, True, min_count=c, upper_only=True, chunk_rows=chunk_rows,
                        host_left_deg_r=hdeg, host_left_deg_s=hdeg, ws=ws)
    dom = int(idx.rel.dom_left)
    return eng, (lambda x: _decode_compact(x, dc.dom_left, orig, dom))


def _ssj_device(family: SetFamily, c: int, plan: Optional[ThresholdPlan], chunk_rows: Optional[int],
                compact: bool = True):
    if c < 1:
        raise ValueError("c must be >= 1")
    idx = family.indexed
    plan = _ssj_plan(idx, plan, int(c))
    plan.validate()
    eng, decode = _ssj_engine(idx, int(c), plan, chunk_rows, compact)
    codes, counts = _device_pairs(eng)
    return decode(codes), counts


def _split(codes: np.ndarray, dz: int):
    return codes // dz, codes % dz


def _split_device(codes, dz: int):
    """(codes // dz, codes % dz) computed on the device (mmj_split_codes) and
    copied back: the host would otherwise divide ~2e8 int64 codes in numpy."""
    import torch

    from . import _native as nat
    n = int(codes.numel())
    a = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    b = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    nat.call("mmj_split_codes", nat.ptr(codes), n, int(dz), nat.ptr(a), nat.ptr(b), nat.stream_handle())
    return a[:n].cpu().numpy(), b[:n].cpu().numpy()


def ssj_mmjoin_arrays(family: SetFamily, c: int, plan: Optional[ThresholdPlan] = None,
                      chunk_rows: Optional[int] = None):
    """(a, b, overlap) int64 arrays of every unordered pair a < b (dense set
    ids) with |a n b| >= c, in ascending (a, b) order."""
    cd, cn = _ssj_device(family, c, plan, chunk_rows)
    a, b = _split_device(cd, family.indexed.rel.dom_left)
    return a, b, cn.cpu().numpy().astype(np.int64)


def ssj_mmjoin(family: SetFamily, c: int, plan: Optional[ThresholdPlan] = None) -> dict:
    """apps.py:65-72: {(a, b): |a n b|} over dense set ids with a < b and
    overlap >= c; insertion order = ascending code (as the reference's)."""
    a, b, n = ssj_mmjoin_arrays(family, c, plan)
    return dict(zip(zip(a.tolist(), b.tolist()), n.tolist()))


def ssj_ordered_arrays(family: SetFamily, c: int, plan: Optional[ThresholdPlan] = None):
    """(a, b, overlap) sorted by overlap descending, then (a, b) ascending
    (apps.py:291-294), ordered on the device: the codes arrive ascending, so
    one stable radix sort by (max overlap - overlap) gives the order."""
    import torch

    from . import _native as nat
    from .ingest import IngestWorkspace, sorted_ids
    cd, cn = _ssj_device(family, c, plan, None)
    n = int(cd.numel())
    if n:
        top = int(cn.max().item())
        key = (top - cn).to(torch.int64)
        _, order = sorted_ids(key, IngestWorkspace())
        cd2 = torch.empty_like(cd)
        cn2 = torch.empty_like(cn)
        st = nat.stream_handle()
        nat.call("mmj_ingest_gather", nat.ptr(cd), 8, nat.ptr(order), n, nat.ptr(cd2), st)
        nat.call("mmj_ingest_gather", nat.ptr(cn), 4, nat.ptr(order), n, nat.ptr(cn2), st)
        cd, cn = cd2, cn2
    a, b = _split_device(cd, family.indexed.rel.dom_left)
    return a, b, cn.cpu().numpy().astype(np.int64)


def ssj_ordered(family: SetFamily, c: int) -> list:
    """apps.py:291-294: ssj_mmjoin sorted by overlap descending, pair ascending."""
    a, b, n = ssj_ordered_arrays(family, c)
    return [((x, y), k) for x, y, k in zip(a.tolist(), b.tolist(), n.tolist())]


def scj_join_project_arrays(family: SetFamily, plan: Optional[ThresholdPlan] = None):
    """(a, b) int64 arrays, ascending: every ordered pair a != b with a a
    subset of b, i.e. overlap(a, b) == |a| (apps.py:297-304).  Fused into the
    count path's emission: per-row threshold |a| (an overlap cannot exceed it)
    and the diagonal excluded, so nothing else leaves the device."""
    from .device import device_relation
    from .engine import TwoPathEngine
    idx = family.indexed
    plan = _ssj_plan(idx, plan, 1, upper_only=False)
    plan.validate()
    dr = device_relation(idx)
    d1, d2 = (plan.delta1, plan.delta2) if plan.strategy == PARTITIONED else (max(idx.n, 1),) * 2
    eng = TwoPathEngine(dr, dr, plan.strategy, d1, d2, True, off_diagonal=True, row_min=dr.left_deg,
                        host_left_deg_r=idx.left_deg, host_left_deg_s=idx.left_deg)
    cd, _ = _device_pairs(eng)
    return _split_device(cd, idx.rel.dom_left)


def scj_join_project(family: SetFamily) -> set:
    """apps.py:297-304: ordered containment pairs (a, b), a != b, a subset of b."""
    a, b = scj_join_project_arrays(family)
    return set(zip(a.tolist(), b.tolist()))


def bsi_batch_size(rate: float, n: int) -> int:
    """apps.py:307-311: latency-optimal batch size ceil((B*N)^(3/5))."""
    if rate < 1 or n < 1:
        raise ValueError("rate and n must be >= 1")
    return math.ceil((rate * n) ** 0.6)


def bsi_answer_batch_arrays(r, s, batch_a, batch_b, heavy_bits: int = 256, form: str = "auto") -> np.ndarray:
    """int8 answers per query: 1 = sets intersect, 0 = disjoint, -1 = an id
    unknown to the (unreduced) relation (apps.py:321-329).  `form` picks the
    device algorithm (bsi.BsiEngine: "records", "lists" or "auto"); the
    answers are the same."""
    from .bsi import answer_batch
    return answer_batch(r, s, batch_a, batch_b, heavy_bits=heavy_bits, form=form)


def bsi_answer_batch(r, s, batch: Sequence[tuple]) -> list:
    """apps.py:314-351: answer[i] True iff sets a_i (in R) and b_i (in S)
    intersect; unknown set ids yield None for that query."""
    if len(batch) == 0:
        return []
    ba = [a for a, _ in batch]
    bb = [b for _, b in batch]
    ans = bsi_answer_batch_arrays(r, s, ba, bb)
    return [None if v < 0 else bool(v) for v in ans.tolist()]
