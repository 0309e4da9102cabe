"""Host orchestration of batched boolean set intersection on the B200
(apps.py:314-351).  See csrc/bsi.cu for the device algorithm.

Steps (all kernels of libmmjoin_b200.so), "records" form:
  1. degree split of y over both relations (mmj_heavy_y_positions) with
     delta1 chosen so that at most `heavy_bits` y are heavy;
  2. one record per left id of R and S: heavy-y bitset + light list header,
     light lists compacted in place (mmj_bsi_records);
  3. per query: raw id -> dense id through each relation's own (unreduced)
     dictionary, bitset test, light merge intersection (mmj_bsi_answer).
"lists" form (short lists, BsiEngine): no per-batch build.  Raw ids resolve
through span tables (one 8-byte entry per raw id: list offset / length and a
32-bit signature of the id's heaviest y, built once per relation pair); a
shared signature bit answers the query, the others intersect the two ids'
full forward lists (mmj_bsi_answer_spans; mmj_bsi_answer_lists without span
tables).
If R and S do not share a right dictionary, their y ids are first mapped to
a common raw-value space on the host (input preparation, as the reference's
semi_join_reduce does) -- left ids, hence "known" ids, stay those of the
unreduced relations.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .device import Workspace

BITS_BLOCK = 128     # bitset width granularity (4 words)
LIST_MAX_MEAN = 64   # "lists" form when both sides' mean list length is at most this
DIRECT_SPREAD = 4    # direct id table when max - min + 1 <= 4 x the number of ids
SIG_BITS = 32          # heavy y per span-table signature (0: no signatures)
SPAN_MAX_LEN_BITS = 16
SPAN_MIN_LEN_BITS = 4  # span table only when a 32-bit entry leaves >= 4 length bits ...
SPAN_MEAN_FRAC = 2     # ... and the mean list is at most half the largest length they hold


def _torch():
    import torch
    return torch


@dataclass
class BsiSide:
    """Device arrays of one relation in the shared y space."""
    n: int
    dom_left: int
    fwd_ptr: object
    fwd_idx: object
    fwd_row: object
    ydeg: object              # device int32 degrees over the shared y space
    sorted_vals: object       # device int64 sorted raw left values (or None)
    order: object             # device int32 dense id of each sorted value
    h2d_bytes: int = 0
    table: object = None      # (direct-address id table, vmin, range) or None
    span: object = None       # (span table, vmin, range, len_bits) or None


def _attach_table(sd: BsiSide, ends, hpos=None) -> None:
    """Direct-address raw id -> dense id table when the side's raw ids fill
    at most DIRECT_SPREAD x their count of a value range: each query id then
    resolves with one load instead of a binary search (cfg5: 4M ids in
    [0, 4M), a 16 MB table).  Part of the device form of the relation's
    left_ids dictionary, so it is built once with the sides."""
    if sd.sorted_vals is None or sd.dom_left == 0:
        return
    torch = _torch()
    lo, hi = next(ends), next(ends)
    vmin, rng = int(lo), int(hi) - int(lo) + 1
    if rng > DIRECT_SPREAD * sd.dom_left or rng >= (1 << 31) - 1:
        return
    table = torch.empty(rng, dtype=torch.int32, device="cuda")
    nat.call("mmj_bsi_direct_table", nat.ptr(sd.sorted_vals), nat.ptr(sd.order), sd.dom_left, vmin, rng,
             nat.ptr(table), nat.stream_handle())
    sd.table = (table, vmin, rng)
    # span table: raw id -> (list offset, length) in one 32-bit entry, when
    # the tuple count leaves enough length bits for the typical list (a
    # saturated length costs the query a binary search over fwd_ptr)
    len_bits = min(SPAN_MAX_LEN_BITS, 32 - (sd.n + 1).bit_length())
    if len_bits >= SPAN_MIN_LEN_BITS and sd.n * SPAN_MEAN_FRAC <= ((1 << len_bits) - 1) * sd.dom_left:
        # 8-byte entries: the span and the id's signature over the SIG_BITS
        # heaviest y (hpos), which answers most intersecting pairs by itself
        span = torch.empty(rng, dtype=torch.int64, device="cuda")
        nat.call("mmj_bsi_span_table", nat.ptr(sd.sorted_vals), nat.ptr(sd.order), sd.dom_left, vmin, rng,
                 nat.ptr(sd.fwd_ptr), nat.ptr(sd.fwd_idx), nat.ptr(hpos) if hpos is not None else 0, sd.n, len_bits,
                 nat.ptr(span), nat.stream_handle())
        sd.span = (span, vmin, rng, len_bits)


def _with_tables(sides):
    """Attach the direct id tables of both sides (one device -> host copy of
    their smallest / largest raw ids)."""
    torch = _torch()
    sR, sS, dom_y = sides
    have = [sd for sd in (sR, sS) if sd.sorted_vals is not None and sd.dom_left > 0]
    ends = iter(torch.cat([sd.sorted_vals[[0, sd.dom_left - 1]] for sd in have]).cpu().tolist()) if have else iter(())
    hpos = _signature_positions(sR, sS, dom_y) if len(have) == 2 else None
    for sd in have:
        _attach_table(sd, ends, hpos)
    return sides


def _signature_positions(sR: BsiSide, sS: BsiSide, dom_y: int):
    """hpos[y] = rank of y among the SIG_BITS join values shared by the most
    (a, b) pairs (largest degR(y) * degS(y) > 0), -1 for every other y: the
    heavy y of the span tables' signatures.  Which y are chosen never changes
    an answer (a signature bit is exact membership of one y)."""
    torch = _torch()
    if dom_y == 0 or SIG_BITS <= 0:
        return None
    w = sR.ydeg.to(torch.float64) * sS.ydeg.to(torch.float64)
    vals, idx = torch.topk(w, min(SIG_BITS, dom_y))
    idx = idx[vals > 0]
    hpos = torch.full((dom_y,), -1, dtype=torch.int32, device="cuda")
    hpos[idx] = torch.arange(idx.numel(), dtype=torch.int32, device="cuda")
    return hpos


def _int_values(vals):
    """int64 array of a dictionary's raw values when every value is an
    integer (an integer ndarray, or Python / numpy ints that are not bools),
    else None: floats, numeric strings and bools must keep Python equality
    semantics (1.5 != 1, '5' != 5), so they never go through an int cast."""
    if isinstance(vals, np.ndarray):
        if vals.dtype.kind in "iu":
            return vals.astype(np.int64)
        if vals.dtype.kind != "O":
            return None
    try:
        if not all(isinstance(v, (int, np.integer)) and not isinstance(v, (bool, np.bool_)) for v in vals):
            return None
        return np.asarray(vals, dtype=np.int64)
    except (OverflowError, TypeError, ValueError):
        return None


def _left_lookup_arrays(rel):
    """(sorted raw values, order) for int-valued dictionaries, else None."""
    vals = _int_values(rel.left_values)
    if vals is None:
        return None
    order = np.argsort(vals, kind="stable")
    return vals[order], order.astype(np.int32)


def _side(idx, y_map, dom_y, pinned=False) -> BsiSide:
    torch = _torch()
    fptr = np.asarray(idx.fwd_indptr, dtype=np.int64)
    fidx = np.asarray(idx.fwd_indices, dtype=np.int64)
    ldeg = np.diff(fptr)
    rows = np.repeat(np.arange(idx.rel.dom_left, dtype=np.int64), ldeg)
    if y_map is not None:
        fidx = y_map[fidx]
        order = np.lexsort((fidx, rows))          # keep each list sorted by shared y id
        fidx = fidx[order]
    ydeg = torch.from_numpy(np.bincount(fidx, minlength=dom_y).astype(np.int32)).to("cuda")
    lk = _left_lookup_arrays(idx.rel)
    dev = {}
    nbytes = 0
    for name, arr in (("fwd_ptr", fptr.astype(np.int32)), ("fwd_idx", fidx.astype(np.int32)),
                      ("fwd_row", rows.astype(np.int32))):
        t = torch.from_numpy(np.ascontiguousarray(arr))
        if pinned:
            t = t.pin_memory()
        nbytes += arr.nbytes
        dev[name] = t.to("cuda", non_blocking=pinned)
    sv = od = None
    if lk is not None:
        sv = torch.from_numpy(lk[0]).to("cuda")
        od = torch.from_numpy(lk[1]).to("cuda")
        nbytes += lk[0].nbytes + lk[1].nbytes
    return BsiSide(len(fidx), idx.rel.dom_left, dev["fwd_ptr"], dev["fwd_idx"], dev["fwd_row"], ydeg, sv, od, nbytes)


def _side_device(idx, y_map, dom_y, ws) -> BsiSide:
    """BsiSide of a device-ingested relation without any host round trip:
    y ids remapped into the shared space and each list re-sorted on the
    device (ingest.cu)."""
    from . import ingest
    d = idx.device
    if y_map is None:
        fptr, fidx, frow = d.fwd_ptr, d.fwd_idx, d.fwd_row
        ydeg = d.right_deg
    else:
        mapped = ingest.remap(d.fwd_idx, y_map)
        fptr, fidx, frow, _ = ingest.csr(d.fwd_row, mapped, d.dom_left, dom_y, ws)
        ydeg = ingest.histogram(mapped, dom_y)
    sv, od = ingest.sorted_ids(idx._left_values_dev, ws)
    return BsiSide(d.n, d.dom_left, fptr, fidx, frow, ydeg, sv, od, 0)


def _prepare_device(r, s):
    from . import ingest
    ws = ingest.IngestWorkspace()
    if r.rel.right_values is s.rel.right_values:
        dom_y = r.rel.dom_right
        return _side_device(r, None, dom_y, ws), _side_device(s, None, dom_y, ws), dom_y
    torch = _torch()
    rv, sv = r._right_values_dev, s._right_values_dev
    allv = ingest.distinct(torch.cat([rv, sv]), ws)
    dom_y = int(allv.numel())
    rmap, smap = ingest.lookup(allv, rv), ingest.lookup(allv, sv)
    return _side_device(r, rmap, dom_y, ws), _side_device(s, smap, dom_y, ws), dom_y


def prepare(r, s, pinned=False):
    """Device sides of R and S over one y id space (cached on the objects)."""
    key = (id(r), id(s))
    cache = getattr(r, "_mmj_bsi_cache", None)
    if cache is not None and cache[0] == key and not pinned:
        return cache[1]
    from .ingest import DeviceIndexedRelation
    if (isinstance(r, DeviceIndexedRelation) and isinstance(s, DeviceIndexedRelation) and not pinned
            and r._right_values_dev is not None and s._right_values_dev is not None):
        sides = _with_tables(_prepare_device(r, s))
        r._mmj_bsi_cache = (key, sides)
        return sides
    if r.rel.right_values is s.rel.right_values:
        dom_y = r.rel.dom_right
        sides = (_side(r, None, dom_y, pinned), _side(s, None, dom_y, pinned), dom_y)
    else:
        rv, sv = r.rel.right_values, s.rel.right_values
        ra, sa = _int_values(rv), _int_values(sv)
        if ra is not None and sa is not None:
            allv = np.union1d(ra, sa)
            rmap, smap = np.searchsorted(allv, ra), np.searchsorted(allv, sa)
        else:
            # any other values: one dictionary under Python equality, as the
            # reference's raw-value comparison (apps.py:332-350)
            allv = {}
            for v in list(rv) + list(sv):
                allv.setdefault(v, len(allv))
            rmap = np.array([allv[v] for v in rv], dtype=np.int64)
            smap = np.array([allv[v] for v in sv], dtype=np.int64)
        dom_y = len(allv)
        sides = (_side(r, rmap, dom_y, pinned), _side(s, smap, dom_y, pinned), dom_y)
    sides = _with_tables(sides)
    if not pinned:
        try:
            r._mmj_bsi_cache = (key, sides)
        except AttributeError:
            pass
    return sides


def _dense_queries(rel, q):
    """Host dictionary probe for non-integer raw ids (-1 when unknown)."""
    ids = rel.left_ids
    return np.array([ids.get(v, -1) if ids.get(v) is not None else -1 for v in q], dtype=np.int64)


class BsiEngine:
    """Index build + answering for one (R, S) pair (reusable across batches).

    Two exact forms of the same answers:
      "records"  heavy-y split + one record per left id (bitset of its heavy
                 y, then its light list): popc(bits_a & bits_b) decides any
                 query with a heavy witness, the light lists the rest -- the
                 heavy part of the reference's product restricted to the
                 queried cells (apps.py:332-350 -> joinproject.py:208-216);
      "lists"    no per-batch build: span-table signatures of the heaviest y
                 decide most intersecting pairs, the queried ids' forward
                 lists the rest (mmj_bsi_answer_spans / mmj_bsi_answer_lists).
    "auto" takes "lists" when both sides' mean list length is at most
    LIST_MAX_MEAN: a record is 64 B, as many DRAM sectors as a 16-entry list,
    so for short lists the records only add their build pass (cfg5: 16 y per
    id; the build was 1.34 of the 2.0 ms step, r2b)."""

    def __init__(self, sR: BsiSide, sS: BsiSide, dom_y: int, heavy_bits: int = 256, ws=None, form: str = "auto"):
        self.sR, self.sS, self.dom_y = sR, sS, dom_y
        self.lib = nat.load()
        if heavy_bits not in (128, 256, 512, 1024):
            raise ValueError("heavy_bits must be 128, 256, 512 or 1024")
        if form not in ("auto", "lists", "records", "walk"):
            raise ValueError("form must be 'auto', 'lists', 'records' or 'walk'")
        # "walk" = the lists form resolving ids through the id table and
        # fwd_ptr even where span tables exist (A/B and parity of the two)
        self.use_spans = form != "walk"
        if form == "walk":
            form = "lists"
        if form == "auto":
            short = all(sd.n <= LIST_MAX_MEAN * max(sd.dom_left, 1) for sd in (sR, sS))
            form = "lists" if short else "records"
        self.form = form
        self.heavy_bits = max(BITS_BLOCK, -(-heavy_bits // BITS_BLOCK) * BITS_BLOCK)
        self.ws = ws or Workspace()
        self.rdeg, self.sdeg = sR.ydeg, sS.ydeg
        self.delta1 = self._threshold() if form == "records" else None
        self.k = 0

    def _threshold(self) -> int:
        """Smallest delta1 >= 1 with #{y : max(degR, degS) > delta1} <=
        heavy_bits, from two device histograms (log2 buckets, then linear
        bins inside the crossing bucket).  Which y are heavy never changes the
        answers (bitsets and light lists are both exact), only the split."""
        torch = _torch()
        st = nat.stream_handle()
        hist = self.ws.get("bsi_hist", 1024, torch.int32)
        nat.call("mmj_bsi_degree_histogram", nat.ptr(self.rdeg), nat.ptr(self.sdeg), self.dom_y, 0, 1, 64, 1,
                 nat.ptr(hist), st)
        h = hist[:64].cpu().numpy().astype(np.int64)
        above = np.concatenate([np.cumsum(h[::-1])[::-1], [0]])     # above[b] = #{m >= 2^b}
        if above[0] <= self.heavy_bits:
            return 1
        b = int(np.nonzero(above > self.heavy_bits)[0].max())        # bucket holding the crossing
        lo, hi = 1 << b, 1 << (b + 1)
        nb = int(min(1024, hi - lo))
        nat.call("mmj_bsi_degree_histogram", nat.ptr(self.rdeg), nat.ptr(self.sdeg), self.dom_y, lo, hi, nb, 0,
                 nat.ptr(hist), st)
        g = hist[:nb].cpu().numpy().astype(np.int64)
        # count(m > t) for t = the last value of linear bin i: above[b+1] + sum of bins after i
        tail = above[b + 1] + np.concatenate([np.cumsum(g[::-1])[::-1][1:], [0]])
        ok = np.nonzero(tail <= self.heavy_bits)[0]
        i = int(ok.min())
        t = lo + ((i + 1) * (hi - lo) + nb - 1) // nb - 1              # largest m in bin i
        return max(1, t)

    def build(self):
        """Heavy-y split, then one record per left id on each side (heavy-y
        bit row + light list header; light lists compacted in place).  The
        "lists" form has nothing to build."""
        if self.form == "lists":
            return
        torch = _torch()
        st = nat.stream_handle()
        dom_y = self.dom_y
        flag = self.ws.get("yflag", dom_y, torch.uint8)
        scan = self.ws.get("yscan", dom_y + 1, torch.int32)
        self.hpos = self.ws.get("hpos", max(dom_y, 1), torch.int32)
        nat.call("mmj_heavy_y_positions", nat.ptr(self.rdeg), nat.ptr(self.sdeg), dom_y, self.delta1,
                 nat.ptr(flag), nat.ptr(scan), nat.ptr(self.hpos), nat.ptr(self.ws.scan_ws(dom_y)), st)
        self.words = self.heavy_bits // 32
        stride = int(self.lib.mmj_bsi_record_words(self.words))
        self.sides = []
        for tag, sd in (("r", self.sR), ("s", self.sS)):
            rec = self.ws.get(f"rec_{tag}", max(sd.dom_left, 1) * stride, torch.int32)
            ovf = self.ws.get(f"ovf_{tag}", max(sd.n, 1), torch.int32)
            nat.call("mmj_bsi_records", nat.ptr(sd.fwd_ptr), nat.ptr(sd.fwd_idx), sd.dom_left, nat.ptr(self.hpos),
                     self.words, nat.ptr(rec), nat.ptr(ovf), st)
            self.sides.append((rec, ovf))

    def answer(self, qa_dev, qb_dev, nq, dense_a=False, dense_b=False, out=None):
        torch = _torch()
        ans = out if out is not None else torch.empty(max(nq, 1), dtype=torch.int8, device="cuda")

        def idmap(side, dense):
            if dense:
                return 0, 0, 0, 0, 0, 0
            t = side.table
            if t is not None:
                return 0, 0, 0, nat.ptr(t[0]), t[1], t[2]
            return nat.ptr(side.sorted_vals), nat.ptr(side.order), side.dom_left, 0, 0, 0
        if self.form == "lists" and not (dense_a or dense_b) and self.sR.span and self.sS.span and self.use_spans:
            # raw id -> list span in one load per side (cfg5)
            def span(side):
                t = side.span
                return (nat.ptr(t[0]), t[1], t[2], t[3], nat.ptr(side.fwd_ptr), side.dom_left, nat.ptr(side.fwd_idx))
            nat.call("mmj_bsi_answer_spans", nat.ptr(qa_dev), nat.ptr(qb_dev), nq, *span(self.sR), *span(self.sS),
                     nat.ptr(ans), nat.stream_handle())
            return ans[:nq]
        if self.form == "lists":
            nat.call("mmj_bsi_answer_lists", nat.ptr(qa_dev), nat.ptr(qb_dev), nq, *idmap(self.sR, dense_a),
                     *idmap(self.sS, dense_b), nat.ptr(self.sR.fwd_ptr), nat.ptr(self.sR.fwd_idx),
                     nat.ptr(self.sS.fwd_ptr), nat.ptr(self.sS.fwd_idx), nat.ptr(ans), nat.stream_handle())
            return ans[:nq]
        (rrec, rovf), (srec, sovf) = self.sides
        nat.call("mmj_bsi_answer", nat.ptr(qa_dev), nat.ptr(qb_dev), nq, *idmap(self.sR, dense_a),
                 *idmap(self.sS, dense_b), nat.ptr(rrec), nat.ptr(rovf), nat.ptr(srec), nat.ptr(sovf), self.words,
                 nat.ptr(ans), nat.stream_handle())
        return ans[:nq]


def answer_batch(r, s, batch_a, batch_b, heavy_bits: int = 256, form: str = "auto") -> np.ndarray:
    """int8 answers (1 / 0 / -1 for None) for raw query ids."""
    torch = _torch()
    nat.require_cuda()
    qa = list(batch_a) if not isinstance(batch_a, np.ndarray) else batch_a
    qb = list(batch_b) if not isinstance(batch_b, np.ndarray) else batch_b
    nq = len(qa)
    if nq == 0:
        return np.empty(0, dtype=np.int8)
    sR, sS, dom_y = prepare(r, s)
    eng = BsiEngine(sR, sS, dom_y, heavy_bits, form=form)
    eng.build()

    def to_dev(rel, side, q):
        # raw ids go to the device only when the side's dictionary is
        # integer-valued AND every query id is an integer; anything else (5.5,
        # '5', True) is resolved by the dictionary itself, so an id the
        # relation does not hold answers None (apps.py:321-329)
        if side.sorted_vals is not None:
            arr = _int_values(q)
            if arr is not None:
                return torch.from_numpy(arr).to("cuda"), False
        return torch.from_numpy(_dense_queries(rel, q)).to("cuda"), True

    da, dense_a = to_dev(r.rel, sR, qa)
    db, dense_b = to_dev(s.rel, sS, qb)
    return eng.answer(da, db, nq, dense_a, dense_b).cpu().numpy()
