"""Star join-project on the B200 (joinproject.py:281-378, star_join).

The output pi_{x1..xk} is evaluated as a two-path over composite rows
(x1..x_{k-1}) and column x_k (code = row * d_k + x_k, the reference's
mixed-radix _encode).  Join values y are split on the device by the product
of their k degrees: heavy y go through the tcgen05 product (A = row-wise AND
of the heavy rows of R_1..R_{k-1}, generated per x1 chunk; B = heavy rows of
R_k), light y are enumerated witness by witness.  The reference's own
heavy/light decomposition only decides its `heavy_dims` statistic and its
StarResourceError cap; both are reproduced from degrees on the host, so the
drop-in keeps the same results, stats and errors for every (delta1, delta2)
(the output itself is plan-independent).
"""

from __future__ import annotations

import ctypes as C
import math
import os
from typing import Optional, Sequence

import numpy as np

from . import _native as nat
from .device import Workspace, device_relation
from .errors import StarResourceError

BK = 128
# B200 rates of the star cost model, fitted to cfg3 sweeps (profiles/r3_star_sweep.txt:
# K = 128 / 256 / 384 / 512 heavy y -> product 16.1 / 21.5 / 25.1 / 31.6 ms, light
# expansion 22.1 / 5.4 / 3.9 / 3.9 ms for 1.85e9 / 2.6e8 / 8.1e7 / 3.5e7 witnesses)
LIGHT_RATE = 1.0e11          # light witnesses / s (bitmap atomics), marginal
MMA_RATE = 7.0e15            # int8 ops / s, marginal per heavy y (z-pair operand: two cells per accumulator)
CELL_RATE = 1.1e13           # output cells / s of the product's TMEM read-out + bitmap epilogue (K-independent part)
DEFAULT_CHUNK_BYTES = 256 << 20


def _rup(a: int, b: int) -> int:
    return -(-a // b) * b


def reference_heavy_dims(rels, delta1: int, delta2: int, cap: int) -> list:
    """joinproject.py:321-333, 360: the reference's heavy-part geometry
    (raises StarResourceError exactly when the reference does)."""
    k = len(rels)
    deg = np.stack([np.asarray(r.right_deg) for r in rels])
    nheavy = [int((np.asarray(r.left_deg) > delta2).sum()) for r in rels]
    ny = int(((deg > delta1).sum(axis=0) >= 2).sum())
    if not (ny and all(nheavy)):
        return []
    g1 = list(range(math.ceil(k / 2)))
    g2 = list(range(math.ceil(k / 2), k))
    rows = [math.prod(nheavy[i] for i in g) for g in (g1, g2)]
    for n in rows:
        if n > cap:
            raise StarResourceError(f"{n} heavy combinations exceed the cap; increase delta2")
    return [rows[0], rows[1], ny]


def choose_threshold(rels) -> float:
    """Product-degree threshold minimising modelled B200 time."""
    deg = np.stack([np.asarray(r.right_deg, dtype=np.float64) for r in rels])
    prod = deg.prod(axis=0)
    order = np.sort(prod)[::-1]
    order = order[order > 0]
    dims = [r.rel.dom_left for r in rels]
    cells = float(math.prod(dims))
    tail = np.concatenate([np.cumsum(order[::-1])[::-1], [0.0]])   # tail[k] = sum of order[k:]
    best_t, best_thr = tail[0] / LIGHT_RATE, math.inf                 # no heavy y
    for kk in range(BK, min(len(order), 8192) + BK, BK):
        ke = min(kk, len(order))
        t = tail[ke] / LIGHT_RATE + 2.0 * cells * _rup(ke, BK) / MMA_RATE + cells / CELL_RATE
        if t < best_t:
            best_t, best_thr = t, (float(order[ke]) if ke < len(order) else 0.0)
    return best_thr


def _ptr_array(vals, ctype=C.c_void_p):
    arr = (ctype * 4)()
    for i, v in enumerate(vals):
        arr[i] = v
    return arr


class StarEngine:
    def __init__(self, rels, want_counts: bool, threshold: Optional[float] = None,
                 chunk_bytes: int = DEFAULT_CHUNK_BYTES, ws: Optional[Workspace] = None):
        import torch
        self.torch = torch
        self.lib = nat.load()
        self.rels = rels
        self.k = len(rels)
        self.dev = [device_relation(r) for r in rels]
        self.dims = [r.rel.dom_left for r in rels]
        self.dom_y = rels[0].rel.dom_right
        self.counts = want_counts
        self.threshold = choose_threshold(rels) if threshold is None else float(threshold)
        self.ws = ws or Workspace()
        self.dk = self.dims[-1]
        self.wpr = _rup(max(self.dk, 1), 1024) // 32
        self.ldc = _rup(max(self.dk, 1), 1024)
        self.row_per_x1 = math.prod(self.dims[1:-1]) if self.k > 2 else 1
        row_bytes = self.ldc * 4 if want_counts else self.wpr * 4
        import os
        chunk_bytes = int(os.environ.get("MMJ_STAR_CHUNK_BYTES", chunk_bytes))
        self.x1_per_chunk = max(1, chunk_bytes // max(row_bytes * self.row_per_x1, 1))
        self.nnz = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.wit = torch.zeros(1, dtype=torch.int64, device="cuda")
        # projection tail: scan + look-back + emission in one kernel (MMJ_FUSED_EMIT=0: scan, then emission)
        self.one_kernel_tail = os.environ.get("MMJ_FUSED_EMIT", "1") != "0"
        self.timer = None          # optional PhaseTimer (bench instrumentation)
        self._tot_host = None      # pinned chunk sizes + events of the look-ahead projection path
        self._tot_evt = None

    def prepare(self):
        torch = self.torch
        st = nat.stream_handle()
        dom_y = self.dom_y
        self.nnz.zero_()       # per-run statistics (an engine may run many times)
        self.wit.zero_()
        rev_ptrs = _ptr_array([nat.ptr(d.rev_ptr) for d in self.dev])
        hflag = self.ws.get("s_hflag", dom_y, torch.uint8)
        lflag = self.ws.get("s_lflag", dom_y, torch.uint8)
        hscan = self.ws.get("s_hscan", dom_y + 1, torch.int32)
        lscan = self.ws.get("s_lscan", dom_y + 1, torch.int32)
        self.hpos = torch.empty(max(dom_y, 1), dtype=torch.int32, device="cuda")
        self.light_y = torch.empty(max(dom_y, 1), dtype=torch.int32, device="cuda")
        nat.call("mmj_star_split", self.k, rev_ptrs, dom_y, self.threshold, nat.ptr(hflag), nat.ptr(lflag),
                 nat.ptr(hscan), nat.ptr(lscan), nat.ptr(self.hpos), nat.ptr(self.light_y),
                 nat.ptr(self.ws.scan_ws(dom_y)), st)
        kk, nl = (int(v) for v in torch.stack([hscan[dom_y], lscan[dom_y]]).cpu())
        self.kh, self.n_light = kk, nl
        self.H = None
        self.pairs = False
        if kk > 0:
            self.kpad = _rup(kk, BK)
            self.H = []
            # z-pair B operand (two x_k per accumulator, c0 + 128*c1) when every
            # count is < 128: a composite row's heavy degree is at most the
            # smallest left degree among R_1..R_{k-1} rows, and x_k's its own
            import os
            maxdeg = [int(np.asarray(r.left_deg).max(initial=0)) for r in self.rels]
            self.pairs = (not self.counts and os.environ.get("MMJ_PAIR", "1") != "0"
                          and (kk <= 127 or min(maxdeg[:-1]) <= 127 or maxdeg[-1] <= 127))
            for j, d in enumerate(self.dev):
                pad = 1024 if j == self.k - 1 else 256
                rows = _rup(max(d.dom_left, 1), pad)
                if j == self.k - 1 and self.pairs:
                    h = torch.empty((rows // 2, self.kpad), dtype=torch.uint8, device="cuda")
                    nat.call("mmj_build_operand_pairs", nat.ptr(d.fwd_row), nat.ptr(d.fwd_idx), d.n,
                             nat.ptr(d.left_deg), 0, nat.ptr(self.hpos), nat.ptr(h), 0, rows, self.kpad, st)
                else:
                    h = torch.empty((rows, self.kpad), dtype=torch.uint8, device="cuda")
                    nat.call("mmj_build_operand", nat.ptr(d.fwd_row), nat.ptr(d.fwd_idx), d.n, nat.ptr(d.left_deg),
                             0, nat.ptr(self.hpos), nat.ptr(h), 0, rows, self.kpad, st)
                self.H.append(h)

    def _ph(self, name: str, start: bool):
        if self.timer is not None:
            (self.timer.start if start else self.timer.stop)(name)

    def run(self, sink=None, x1_range=None):
        """Evaluate every x1 chunk (of ``x1_range`` = [lo, hi) when given:
        x1-range sharding).  Without `sink` the codes (and counts) are
        collected to host numpy arrays; with `sink(x1_lo, x1_hi, codes_dev,
        counts_dev)` they stay on the device (valid during the call)."""
        torch = self.torch
        st = nat.stream_handle()
        self.prepare()
        dims_arr = (C.c_int64 * 4)(*(self.dims + [0] * (4 - self.k)))
        rev_ptrs = _ptr_array([nat.ptr(d.rev_ptr) for d in self.dev])
        rev_idxs = _ptr_array([nat.ptr(d.rev_idx) for d in self.dev])
        heavy_ptrs = _ptr_array([nat.ptr(h) for h in self.H]) if self.H else None
        codes_out, counts_out = [], []
        lo1, hi1 = (0, self.dims[0]) if x1_range is None else x1_range
        # projection with a device consumer: chunk i + 1 is issued before the
        # host reads chunk i's size (two sets of chunk buffers, sizes through
        # pinned memory + events), so the GPU never waits for the host between
        # chunks (61 chunks at cfg3, ~50 us of idle GPU per synchronous size
        # read: 185.3 -> see profiles/README.md)
        ahead = sink is not None and not self.counts and self.one_kernel_tail
        pending = None
        if ahead and self._tot_host is None:
            self._tot_host = torch.empty(2, dtype=torch.int64).pin_memory()
            self._tot_evt = [torch.cuda.Event(), torch.cuda.Event()]

        def deliver(p):
            par, pxa, pxb, pcodes = p
            self._tot_evt[par].synchronize()
            sink(pxa, pxb, pcodes[: int(self._tot_host[par])], None)
        for ci, xa in enumerate(range(lo1, hi1, self.x1_per_chunk)):
            par = (ci & 1) if ahead else 0
            sfx = f"_{par}" if par else ""
            xb = min(hi1, xa + self.x1_per_chunk)
            rows = (xb - xa) * self.row_per_x1
            ld = self.ldc if self.counts else self.wpr
            buf = self.ws.get("star_out" + sfx, rows * ld, torch.int32)
            self._ph("heavy_mma", True)
            if self.H is not None:
                arows = _rup(rows, 256)
                A = self.ws.get("star_A", arows * self.kpad, torch.uint8)
                nat.call("mmj_star_operand", self.k, dims_arr, heavy_ptrs, self.kpad, xa, rows, nat.ptr(A), st)
                B = self.H[-1]
                if self.counts:
                    mode = nat.MODE_COUNT32
                elif self.pairs:
                    mode = nat.MODE_BITMAP_PAIR
                else:
                    mode = nat.MODE_BITMAP_U8 if self.kh <= 255 else nat.MODE_BITMAP
                nat.call("mmj_heavy_mma", nat.ptr(A), arows, nat.ptr(B), B.shape[0], self.kpad, 0, self.kpad, 0, rows,
                         mode, 0, nat.ptr(buf), ld, nat.ptr(self.nnz), 0, st)
            else:
                buf.zero_()
            self._ph("heavy_mma", False)
            self._ph("light", True)
            lws = self.ws.get("star_lws", int(self.lib.mmj_star_light_workspace_bytes(self.n_light)), torch.uint8)
            nat.call("mmj_star_light", self.k, dims_arr, rev_ptrs, rev_idxs, nat.ptr(self.light_y), self.n_light, xa,
                     xb, 1 if self.counts else 0, nat.ptr(buf), ld, nat.ptr(self.wit), nat.ptr(lws), st)
            self._ph("light", False)
            x0 = xa * self.row_per_x1
            if self.counts:
                ncell = rows * self.ldc
                nseg = int(self.lib.mmj_count_segment_count(ncell))
                segcnt = self.ws.get("segcnt", nseg, torch.int32)
                segoff = self.ws.get("segoff", nseg + 1, torch.int64)
                nat.call("mmj_count_segments", nat.ptr(buf), 4, rows, self.ldc, self.dk, x0, 1, 0, 0, nat.ptr(segcnt),
                         nat.ptr(segoff), nat.ptr(self.ws.scan_ws(nseg)), st)
                total = int(segoff[nseg].item())
                codes = self.ws.get("codes", total, torch.int64)
                cnts = self.ws.get("counts", total, torch.int32)
                if total:
                    nat.call("mmj_count_emit", nat.ptr(buf), 4, rows, self.ldc, self.dk, x0, self.dk, 1, 0, 0,
                             nat.ptr(segoff), nat.ptr(codes), nat.ptr(cnts), st)
                if sink is not None:
                    sink(xa, xb, codes[:total], cnts[:total])
                else:
                    codes_out.append(codes[:total].cpu().numpy())
                    counts_out.append(cnts[:total].cpu().numpy().astype(np.int64))
            elif self.one_kernel_tail:
                # scan + look-back + emission in one kernel (mmj_merge_emit with
                # no light lists: mmj_star_light already OR-ed them in)
                wsb = int(self.lib.mmj_merge_emit_workspace_size(rows, self.wpr))
                fws = self.ws.get("fuse_ws" + sfx, wsb, torch.uint8)
                codes = self.ws.get("codes" + sfx, rows * self.dk, torch.int64)
                tot = self.ws.get("star_total" + sfx, 1, torch.int64)
                self._ph("merge_emit", True)
                nat.call("mmj_merge_emit", nat.ptr(buf), 1, x0, rows, self.wpr, self.dk, 0, 0, 0, 0, 0, 0, 0, 0, 0,
                         0, 0, nat.ptr(self.wit), 0, nat.ptr(codes), nat.ptr(tot), nat.ptr(fws), wsb, st)
                self._ph("merge_emit", False)
                if ahead:
                    self._tot_host[par:par + 1].copy_(tot, non_blocking=True)
                    self._tot_evt[par].record()
                    if pending is not None:
                        deliver(pending)
                    pending = (par, xa, xb, codes)
                    continue
                total = int(tot.item())
                if sink is not None:
                    sink(xa, xb, codes[:total], None)
                else:
                    codes_out.append(codes[:total].cpu().numpy())
            else:
                nwords = rows * self.wpr
                nseg = int(self.lib.mmj_bitmap_segment_count(nwords))
                segcnt = self.ws.get("segcnt", nseg, torch.int32)
                segoff = self.ws.get("segoff", nseg + 1, torch.int64)
                nat.call("mmj_bitmap_segments", nat.ptr(buf), nwords, nat.ptr(segcnt), nat.ptr(segoff),
                         nat.ptr(self.ws.scan_ws(nseg)), st)
                total = int(segoff[nseg].item())
                codes = self.ws.get("codes", total, torch.int64)
                if total:
                    nat.call("mmj_emit_codes", nat.ptr(buf), nat.ptr(segoff), rows, self.wpr, x0, self.dk,
                             nat.ptr(codes), st)
                if sink is not None:
                    sink(xa, xb, codes[:total], None)
                else:
                    codes_out.append(codes[:total].cpu().numpy())
        if pending is not None:
            deliver(pending)
        codes = np.concatenate(codes_out) if codes_out else np.empty(0, dtype=np.int64)
        counts = (np.concatenate(counts_out) if counts_out else np.empty(0, dtype=np.int64)) if self.counts else None
        return codes, counts


def star_join(relations: Sequence, delta1: int, delta2: int, want_counts: bool = False, cores: int = 1,
              heavy_rows_cap: int = 1 << 22, threshold: Optional[float] = None):
    """joinproject.py:281-378: pi_{x1..xk} of k relations joined on the
    shared right column, with exact witness counts on request."""
    from .joinproject import OutputSet, _check_code_space, _ensure_reduced_many
    k = len(relations)
    if not 2 <= k <= 4:
        raise ValueError("star_join supports 2 <= k <= 4 relations")
    if delta1 < 1 or delta2 < 1:
        raise ValueError("thresholds must be >= 1")
    rels = _ensure_reduced_many(relations)
    dims = [r.rel.dom_left for r in rels]
    _check_code_space(dims)
    hdims = reference_heavy_dims(rels, delta1, delta2, heavy_rows_cap)
    nat.require_cuda()
    eng = StarEngine(rels, want_counts, threshold=threshold)
    codes, counts = eng.run()
    return OutputSet(codes, dims, counts, {"heavy_dims": hdims})
