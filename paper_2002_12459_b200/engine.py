"""Device pipeline of the two-path join-project operator.

One call = degree split -> heavy operand build -> per x-chunk
{tcgen05 heavy product -> light expansion -> segment scan -> emission}.
Reference: joinproject.py:155-225 (two_path_join) and 228-248
(full_join_dedup); every step is a kernel of libmmjoin_b200.so.

Per x-chunk [x0, x1) the output lives in HBM as
  * a bitmap (rows x wpr uint32 words, wpr = ceil(dom_z/256)*8): bit (x, z)
    set iff the pair is in the projection; the heavy product writes every
    word of the chunk (light x / light z rows and columns of the operands are
    zero), the light witnesses are OR-ed in afterwards, or
  * an int32 count matrix (rows x ldc, ldc = ceil(dom_z/256)*256) when exact
    witness counts are requested (heavy counts stored, light counts added).
Both are compacted into strictly increasing int64 codes x*dom_z + z, which is
the reference's OutputSet.codes order (np.unique sorts), so no sort runs.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _native as nat
from .device import DeviceRelation, Workspace
from .optimizer import FULL_JOIN, PARTITIONED

BM = 128          # MMA tile rows
BN = 256          # MMA tile columns
BK = 128          # K block (bytes)

DEFAULT_BITMAP_CHUNK_BYTES = 1 << 30
DEFAULT_COUNT_CHUNK_BYTES = 4 << 30
FUSED_SMEM_LIMIT = 200 * 1024
SYNC_FUSED_CAP_BYTES = 4 << 30
OR_MAX_MEAN_DEG = 16       # engine._heavy_or: heavy y per heavy row up to which the OR path wins


_HOST_MAX = {}


def _host_max(arr) -> int:
    """max of a host degree array.  Read-only arrays (this package's
    IndexedRelation freezes its degree vectors) are remembered per array
    object, so engines for the same relations (one per batch / shard / step)
    do not rescan them (~0.3 ms per 500k entries); writeable arrays (e.g. a
    caller's own index) are rescanned on every call, so an in-place edit can
    never leave a stale maximum behind (that maximum gates the uint16 count
    cells and the z-pair operand)."""
    a = np.asarray(arr)
    if a.flags.writeable:
        return int(a.max(initial=0))
    hit = _HOST_MAX.get(id(arr))
    if hit is not None and hit[0] is arr:
        return hit[1]
    m = int(a.max(initial=0))
    if len(_HOST_MAX) >= 64:
        _HOST_MAX.clear()
    _HOST_MAX[id(arr)] = (arr, m)   # the reference keeps the id from being reused
    return m


def _rup(a: int, b: int) -> int:
    return -(-a // b) * b


@dataclass
class ChunkResult:
    x0: int
    x1: int
    n: int
    codes: object            # torch int64 view (device)
    counts: Optional[object]  # torch int32 view (device) or None
    light: int
    total_dev: Optional[object] = None   # async chunks: device int64[1] holding n


@dataclass
class EngineStats:
    light_intermediate: int = 0
    heavy_pairs: int = 0
    k_heavy: int = 0
    kpad: int = 0
    chunks: int = 0
    out_size: int = 0
    launches: int = 0
    extra: dict = field(default_factory=dict)


class TwoPathEngine:
    """Device state for one (R, S, plan) two-path evaluation."""

    def __init__(self, dr: DeviceRelation, ds: DeviceRelation, strategy: str, delta1: int, delta2: int,
                 want_counts: bool, *, min_count: int = 1, upper_only: bool = False, off_diagonal: bool = False,
                 row_min=None, chunk_rows: Optional[int] = None, ws: Optional[Workspace] = None,
                 host_left_deg_r=None, host_left_deg_s=None, pair_operand: bool = True):
        import torch
        self.torch = torch
        self.lib = nat.load()
        self.dr, self.ds = dr, ds
        if dr.dom_right != ds.dom_right:
            raise ValueError("relations must share the right (y) dictionary")
        self.strategy = strategy
        self.d1, self.d2 = int(delta1), int(delta2)
        self.counts = bool(want_counts)
        self.min_count = int(min_count)
        self.upper_only = bool(upper_only)
        # emission cell filter: 0 all, 1 z > x (SSJ), 2 z != x (SCJ); row_min: a
        # per-x count threshold (int32 device vector over x, e.g. |a| for SCJ)
        self.cell_filter = 1 if self.upper_only else (2 if off_diagonal else 0)
        self.row_min = row_min
        if (self.cell_filter or self.min_count > 1 or row_min is not None) and not self.counts:
            raise ValueError("min_count / row_min / cell filters act on the count path; pass want_counts=True")
        if self.cell_filter and dr.dom_left != ds.dom_left:
            raise ValueError("upper_only / off_diagonal need a self-join (x and z in one dictionary)")
        # c-prefilter only when the caller discards counts < min_count (SSJ);
        # the light_intermediate statistic then counts the pruned witnesses only
        self.prefilter = self.min_count if (self.counts and self.min_count > 1) else 0
        self.dom_x, self.dom_z, self.dom_y = dr.dom_left, ds.dom_left, dr.dom_right
        self.wpr = _rup(max(self.dom_z, 1), 1024) // 32     # rows start on 1024-cell segments
        self.ldc = _rup(max(self.dom_z, 1), 1024)
        self.ws = ws or Workspace()
        self.stats = EngineStats()
        self.hpos = None
        self.A = None
        self.B = None
        self.pairs = False
        self.allow_pairs = bool(pair_operand)   # False: B stays one z per row (heavy_matrices reads it)
        self.kpad = 0
        # heavy part of a projection: "mma" (tcgen05 product into a chunk
        # bitmap) or "or" (heavy-y bit rows OR-ed per row inside the fused
        # tail, no product and no bitmap round trip); chosen in prepare()
        self.heavy_kernel = None
        self.hbits = None
        self.lz_ptr = None
        self.lz_idx = None
        self._host_ldeg_r = host_left_deg_r
        self._host_ldeg_s = host_left_deg_s
        # uint16 count cells when no count can reach 2^16: a count is at most
        # the smaller of the two left degrees (env MMJ_COUNT16=0 forces int32)
        self.count16 = (self.counts and __import__("os").environ.get("MMJ_COUNT16", "1") != "0"
                        and min(self._max_deg(host_left_deg_r, dr), self._max_deg(host_left_deg_s, ds)) < 65536)
        self.cell_bytes = 2 if self.count16 else 4
        row_bytes = (self.ldc * self.cell_bytes) if self.counts else (self.wpr * 4)
        if chunk_rows is None:
            budget = DEFAULT_COUNT_CHUNK_BYTES if self.counts else DEFAULT_BITMAP_CHUNK_BYTES
            chunk_rows = max(BM, (budget // max(row_bytes, 1)) // BM * BM)
        self.chunk_rows = max(BM, _rup(int(chunk_rows), BM))
        self.nnz = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.wit = torch.zeros(1, dtype=torch.int64, device="cuda")
        # fused light+merge+emit kernel for the projection when a row group's
        # bitmap fits in shared memory (dom_z up to ~1.2M)
        self.group_rows = max(1, min(32, (48 * 1024) // (self.wpr * 4)))
        self.fused = (not self.counts) and self.dom_z < (1 << 31)
        # merge + scan + emission as one kernel (decoupled look-back); env
        # MMJ_FUSED_EMIT=0 selects the three-kernel path for A/B runs
        self._splits = None
        self.one_kernel_tail = self.fused and __import__("os").environ.get("MMJ_FUSED_EMIT", "1") != "0"
        self._prepared = False
        self._sizes_dev = None
        self._n_async = 0
        self.timer = None          # optional PhaseTimer (bench instrumentation)
        self._stream = None

    # ------------------------------------------------------------ prepare
    def _st(self):
        # the launching stream, looked up once per prepare() (a
        # torch.cuda.current_stream() call costs ~17 us of host time)
        if self._stream is None:
            self._stream = nat.stream_handle()
        return self._stream

    def prepare(self):
        if self._prepared:
            return
        self._stream = None
        torch = self.torch
        st = self._st()
        dr, ds = self.dr, self.ds
        self.nnz.zero_()
        self.wit.zero_()
        if self.strategy == PARTITIONED:
            dom_y = self.dom_y
            flag = self.ws.get("yflag", dom_y, torch.uint8)
            scan = self.ws.get("yscan", dom_y + 1, torch.int32)
            # engine buffers come from the workspace: an engine re-created for
            # every step (bench.py) reuses them instead of allocating
            self.hpos = self.ws.get("e_hpos", max(dom_y, 1), torch.int32)
            nat.call("mmj_heavy_y_positions", nat.ptr(dr.right_deg), nat.ptr(ds.right_deg), dom_y, self.d1,
                     nat.ptr(flag), nat.ptr(scan), nat.ptr(self.hpos), nat.ptr(self.ws.scan_ws(dom_y)), st)
            # one device -> host copy for K and the heavy-part choice's counts
            or_stats = self._heavy_or_stats()
            vals = torch.cat([scan[dom_y:dom_y + 1].long()] + ([or_stats] if or_stats is not None else [])).cpu()
            k = int(vals[0])
            self.stats.k_heavy = k
            heavy_x = self._any_heavy(self._host_ldeg_r, dr)
            heavy_z = self._any_heavy(self._host_ldeg_s, ds)
            if k > 0 and heavy_x and heavy_z and self._heavy_or(vals[1:].tolist()):
                # the heavy rows of S_h at one bit per cell (K x wpr words)
                self.heavy_kernel = "or"
                self.hbits = self.ws.get("e_hbits", k * self.wpr, torch.int32).view(k, self.wpr)
                nat.call("mmj_build_heavy_rows", nat.ptr(ds.fwd_row), nat.ptr(ds.fwd_idx), ds.n, nat.ptr(ds.left_deg),
                         self.d2, nat.ptr(self.hpos), nat.ptr(self.hbits), k, self.wpr, st)
            elif k > 0 and heavy_x and heavy_z:
                self.heavy_kernel = "mma"
                kpad = _rup(k, BK)
                self.kpad = kpad
                arows = _rup(max(self.dom_x, 1), BN)
                brows = _rup(max(self.dom_z, 1), 1024)   # product covers every word of the padded rows
                self.pairs = (self.allow_pairs and not self.counts
                              and __import__("os").environ.get("MMJ_PAIR", "1") != "0"
                              and (k <= 127 or self._max_deg(self._host_ldeg_r, dr) <= 127
                                   or self._max_deg(self._host_ldeg_s, ds) <= 127))
                self.A = self.ws.get("e_A", arows * kpad, torch.uint8).view(arows, kpad)
                nat.call("mmj_build_operand", nat.ptr(dr.fwd_row), nat.ptr(dr.fwd_idx), dr.n,
                         nat.ptr(dr.left_deg), self.d2, nat.ptr(self.hpos), nat.ptr(self.A), 0, arows, kpad, st)
                if self.pairs:
                    # z pairs share one accumulator (weights 1, 128): every
                    # count is < 128 because one side's heavy degrees are <= 127
                    self.B = self.ws.get("e_B", (brows // 2) * kpad, torch.uint8).view(brows // 2, kpad)
                    nat.call("mmj_build_operand_pairs", nat.ptr(ds.fwd_row), nat.ptr(ds.fwd_idx), ds.n,
                             nat.ptr(ds.left_deg), self.d2, nat.ptr(self.hpos), nat.ptr(self.B), 0, brows, kpad, st)
                else:
                    self.B = self.ws.get("e_B", brows * kpad, torch.uint8).view(brows, kpad)
                    nat.call("mmj_build_operand", nat.ptr(ds.fwd_row), nat.ptr(ds.fwd_idx), ds.n,
                             nat.ptr(ds.left_deg), self.d2, nat.ptr(self.hpos), nat.ptr(self.B), 0, brows, kpad, st)
            self.stats.kpad = self.kpad
            # light-z lists of S for pass 3
            n = ds.n
            lflag = self.ws.get("lzflag", n, torch.uint8)
            lpos = self.ws.get("lzpos", n + 1, torch.int32)
            self.lz_ptr = self.ws.get("e_lz_ptr", dom_y + 1, torch.int32)
            self.lz_idx = self.ws.get("e_lz_idx", max(n, 1), torch.int32)
            nat.call("mmj_light_z_csr", nat.ptr(ds.rev_ptr), nat.ptr(ds.rev_idx), n, dom_y, nat.ptr(ds.left_deg),
                     self.d2, nat.ptr(lflag), nat.ptr(lpos), nat.ptr(self.lz_ptr), nat.ptr(self.lz_idx),
                     nat.ptr(self.ws.scan_ws(n)), st)
        self._prepared = True

    def _or_candidate(self):
        """The projection's heavy part may take the in-tile OR form (fused
        tail, no counts); None when forced by env MMJ_HEAVY=mma|or."""
        if not self.fused or self.counts or not self.allow_pairs:
            return False
        env = __import__("os").environ.get("MMJ_HEAVY", "")
        return (env == "or") if env in ("mma", "or") else None

    def _heavy_or_stats(self):
        """Device int64 [#heavy x, #heavy-x tuples with heavy y] for the OR
        choice (launched, not synchronised), or None if not needed."""
        if self._or_candidate() is not None:
            return None
        torch = self.torch
        dr = self.dr
        stats = self.ws.get("e_orstats", 2, torch.int64)
        nat.call("mmj_heavy_row_stats", nat.ptr(dr.fwd_row), nat.ptr(dr.fwd_idx), dr.n, nat.ptr(dr.left_deg),
                 dr.dom_left, self.d2, nat.ptr(self.hpos), nat.ptr(stats), self._st())
        return stats

    def _heavy_or(self, stats) -> bool:
        """Projection heavy part as a sparse boolean product (OR of heavy-y
        bit rows) instead of the dense tcgen05 product.  Per output cell the
        product reads 2 B of TMEM (z-pair accumulators) whatever R_h's
        density; the OR reads 4 B x (heavy y of the row) / 32 from L2 and runs
        inside the emission tail.  Taken when R_h's heavy rows carry at most
        OR_MAX_MEAN_DEG heavy y on average (cfg2: 4.2 of K = 128) and the
        fused projection tail is in use; env MMJ_HEAVY=mma|or overrides.
        `stats` = the host values of _heavy_or_stats()."""
        forced = self._or_candidate()
        if forced is not None:
            return forced
        nh, nt = (int(v) for v in stats)
        return nt <= OR_MAX_MEAN_DEG * max(nh, 1)

    def _bitmap_mode(self) -> int:
        # every product entry counts <= K shared heavy y: with K <= 255 the
        # epilogue may pack counts as bytes
        if self.pairs:
            return nat.MODE_BITMAP_PAIR
        return nat.MODE_BITMAP_U8 if 0 < self.stats.k_heavy <= 255 else nat.MODE_BITMAP

    @staticmethod
    def _max_deg(host_deg, d: DeviceRelation) -> int:
        if host_deg is not None:
            return _host_max(host_deg)
        return int(d.left_deg.max().item()) if d.left_deg.numel() else 0

    def _any_heavy(self, host_deg, d: DeviceRelation) -> bool:
        return self._max_deg(host_deg, d) > self.d2

    # ------------------------------------------------------------ chunks
    def chunk_bounds(self, x_begin: int = 0, x_end: Optional[int] = None):
        x_end = self.dom_x if x_end is None else x_end
        x = x_begin
        while x < x_end:
            nx = min(x_end, x + self.chunk_rows)
            yield x, nx
            x = nx

    def _ph(self, name: str, start: bool):
        if self.timer is not None:
            (self.timer.start if start else self.timer.stop)(name)

    def run_chunk(self, x0: int, x1: int, sync: bool = True, codes_key: str = "codes") -> ChunkResult:
        """Evaluate output rows [x0, x1).  With ``sync=False`` no host sync
        happens: the code buffer is sized for the worst case (rows*dom_z) and
        the chunk's sizes are fetched later by :meth:`finish`."""
        torch = self.torch
        st = self._st()
        dr, ds = self.dr, self.ds
        rows = x1 - x0
        if self.counts:
            buf = self.ws.get("cnt", rows * self.ldc, torch.int16 if self.count16 else torch.int32)
            ld = self.ldc
            mode = ((nat.MODE_COUNT16 if self.count16 else nat.MODE_COUNT32)
                    | (nat.MODE_UPPER if self.cell_filter == 1 else 0))
        else:
            buf = self.ws.get("bm", rows * self.wpr, torch.int32)
            ld = self.wpr
            mode = self._bitmap_mode()
        # heavy part (writes every cell of the chunk) or zero fill; the in-tile
        # OR path (hbits) computes it inside the tail kernel instead
        if self.A is not None:
            self._ph("heavy_mma", True)
            nat.call("mmj_heavy_mma", nat.ptr(self.A), self.A.shape[0], nat.ptr(self.B), self.B.shape[0],
                     self.kpad, 0, self.kpad, x0, rows, mode, 0, nat.ptr(buf), ld, nat.ptr(self.nnz), 0, st)
            self._ph("heavy_mma", False)
        elif self.hbits is None:
            buf.zero_()
        if self.fused:
            return self._fused_tail(x0, x1, rows, buf, sync, codes_key)
        # light passes (x-driven; FULL_JOIN when hpos is None)
        t0 = int(dr.fwd_ptr_host[x0])
        t1 = int(dr.fwd_ptr_host[x1])
        ntup = t1 - t0
        lens = self.ws.get("len", ntup, torch.int32)
        offs = self.ws.get("offs", ntup + 1, torch.int64)
        hp = nat.ptr(self.hpos) if self.strategy == PARTITIONED else 0
        lzp = nat.ptr(self.lz_ptr) if self.lz_ptr is not None else 0
        lzi = nat.ptr(self.lz_idx) if self.lz_idx is not None else 0
        self._ph("light", True)
        nat.call("mmj_light_lengths", nat.ptr(dr.fwd_row), nat.ptr(dr.fwd_idx), t0, ntup, nat.ptr(dr.left_deg),
                 self.d2, hp, nat.ptr(ds.rev_ptr), nat.ptr(ds.rev_idx), lzp, lzi, self.prefilter, int(self.upper_only),
                 nat.ptr(lens), nat.ptr(offs), nat.ptr(self.ws.scan_ws(ntup)), st)
        nat.call("mmj_light_expand", nat.ptr(dr.fwd_row), nat.ptr(dr.fwd_idx), t0, ntup, nat.ptr(dr.left_deg),
                 self.d2, hp, nat.ptr(ds.rev_ptr), nat.ptr(ds.rev_idx), lzp, lzi, self.prefilter, int(self.upper_only),
                 nat.ptr(offs), -1, (2 if self.count16 else 1) if self.counts else 0, x0, nat.ptr(buf), ld, st)
        self._ph("light", False)
        # merge: segment sizes -> offsets -> codes
        self._ph("segments", True)
        if self.counts:
            ncell = rows * self.ldc
            nseg = int(self.lib.mmj_count_segment_count(ncell))
            segcnt = self.ws.get("segcnt", nseg, torch.int32)
            segoff = self.ws.get("segoff", nseg + 1, torch.int64)
            rm = nat.ptr(self.row_min) if self.row_min is not None else 0
            nat.call("mmj_count_segments", nat.ptr(buf), self.cell_bytes, rows, self.ldc, self.dom_z, x0,
                     self.min_count, rm,
                     self.cell_filter, nat.ptr(segcnt), nat.ptr(segoff), nat.ptr(self.ws.scan_ws(nseg)), st)
        else:
            nwords = rows * self.wpr
            nseg = int(self.lib.mmj_bitmap_segment_count(nwords))
            segcnt = self.ws.get("segcnt", nseg, torch.int32)
            segoff = self.ws.get("segoff", nseg + 1, torch.int64)
            nat.call("mmj_bitmap_segments", nat.ptr(buf), nwords, nat.ptr(segcnt), nat.ptr(segoff),
                     nat.ptr(self.ws.scan_ws(nseg)), st)
        self._ph("segments", False)
        if sync:
            sizes = torch.stack([segoff[nseg], offs[ntup]]).cpu()
            total, light = int(sizes[0]), int(sizes[1])
            cap = total
        else:
            slot = self._async_slot()
            slot[0:1].copy_(segoff[nseg:nseg + 1], non_blocking=True)
            slot[1:2].copy_(offs[ntup:ntup + 1], non_blocking=True)
            total = light = -1
            cap = rows * self.dom_z
        codes = self.ws.get("codes", cap, torch.int64)
        counts = None
        self._ph("emit", True)
        if self.counts:
            counts = self.ws.get("counts", cap, torch.int32)
            if cap:
                nat.call("mmj_count_emit", nat.ptr(buf), self.cell_bytes, rows, self.ldc, self.dom_z, x0, self.dom_z,
                         self.min_count, rm, self.cell_filter, nat.ptr(segoff), nat.ptr(codes), nat.ptr(counts), st)
        elif cap:
            nat.call("mmj_bitmap_emit", nat.ptr(buf), rows * self.wpr, self.wpr, nat.ptr(segoff), x0, self.dom_z,
                     nat.ptr(codes), st)
        self._ph("emit", False)
        self.stats.chunks += 1
        if not sync:
            return ChunkResult(x0, x1, -1, codes, counts, -1)
        self.stats.light_intermediate += light
        self.stats.out_size += total
        return ChunkResult(x0, x1, total, codes[:total], None if counts is None else counts[:total], light)

    def _fused_tail(self, x0, x1, rows, buf, sync, codes_key="codes"):
        """Light witnesses merged into the bitmap and the sorted codes emitted:
        one kernel (mmj_merge_emit: merge, segment scan, decoupled look-back,
        emission) or, with MMJ_FUSED_EMIT=0, the three-kernel path
        (mmj_tile_merge -> mmj_exclusive_scan_i32 -> mmj_emit_codes)."""
        # the fused kernel learns the chunk's output size only as it runs, so
        # its code buffer is sized for every cell of the chunk; synchronous
        # callers with larger chunks take the exact-size three-kernel path
        if self.one_kernel_tail and (not sync or rows * self.dom_z * 8 <= SYNC_FUSED_CAP_BYTES):
            return self._merge_emit_tail(x0, x1, rows, buf, sync, codes_key)
        torch = self.torch
        st = self._st()
        dr, ds = self.dr, self.ds
        nseg = rows * self.wpr // 32
        segcnt = self.ws.get("segcnt", nseg, torch.int32)
        segoff = self.ws.get("segoff", nseg + 1, torch.int64)
        hp = nat.ptr(self.hpos) if self.strategy == PARTITIONED else 0
        lzp = nat.ptr(self.lz_ptr) if self.lz_ptr is not None else 0
        lzi = nat.ptr(self.lz_idx) if self.lz_idx is not None else 0
        wit0 = int(self.wit.item()) if sync else 0
        self._ph("light_merge", True)
        nat.call("mmj_tile_merge", nat.ptr(buf), self._has_heavy(), x0, rows, self.wpr, self.dom_z,
                 nat.ptr(dr.fwd_ptr), nat.ptr(dr.fwd_idx), nat.ptr(dr.left_deg), self.d2, hp, nat.ptr(ds.rev_ptr),
                 nat.ptr(ds.rev_idx), lzp, lzi, nat.ptr(self.hbits) if self.hbits is not None else 0,
                 nat.ptr(self.nnz), nat.ptr(segcnt), nat.ptr(self.wit), st)
        self._ph("light_merge", False)
        self._ph("segments", True)
        nat.call("mmj_exclusive_scan_i32", nat.ptr(segcnt), nat.ptr(segoff), nseg, nat.ptr(self.ws.scan_ws(nseg)), st)
        self._ph("segments", False)
        if sync:
            total = int(segoff[nseg].item())
            cap = total
        else:
            cap = rows * self.dom_z
        codes = self.ws.get(codes_key, cap, torch.int64)
        self._ph("emit", True)
        if cap:
            nat.call("mmj_emit_codes", nat.ptr(buf), nat.ptr(segoff), rows, self.wpr, x0, self.dom_z,
                     nat.ptr(codes), st)
        self._ph("emit", False)
        self.stats.chunks += 1
        if not sync:
            slot = self._async_slot()
            slot[0:1].copy_(segoff[nseg:nseg + 1], non_blocking=True)
            return ChunkResult(x0, x1, -1, codes, None, -1, slot[0:1])
        light = int(self.wit.item()) - wit0
        self.stats.out_size += total
        return ChunkResult(x0, x1, total, codes[:total], None, light)

    def _has_heavy(self) -> int:
        """mmj_merge_emit / mmj_tile_merge heavy source: 0 none, 1 the chunk
        bitmap written by the tcgen05 product, 2 the heavy-y bit rows."""
        return 2 if self.hbits is not None else int(self.A is not None)

    def _tail_tables(self):
        """(full, light-z) column-block split tables of the S-side lists for
        the fused kernel (first list position of every column block), built
        once per engine; 0 when a row is a single tile or the table would be
        large (the kernel then bisects long lists)."""
        if self._splits is None:
            torch = self.torch
            st = self._st()
            ncb = int(self.lib.mmj_merge_emit_col_blocks(self.wpr))
            n = self.dom_y * (ncb + 1)
            keep = []
            spf = spl = 0
            if ncb > 1 and n <= (64 << 20):
                full = self.ws.get("e_split_full", max(n, 1), torch.int32)
                nat.call("mmj_list_splits", nat.ptr(self.ds.rev_ptr), nat.ptr(self.ds.rev_idx), self.dom_y, self.wpr,
                         nat.ptr(full), st)
                keep.append(full)
                spf = nat.ptr(full)
                if self.lz_ptr is not None:
                    lzt = self.ws.get("e_split_lz", max(n, 1), torch.int32)
                    nat.call("mmj_list_splits", nat.ptr(self.lz_ptr), nat.ptr(self.lz_idx), self.dom_y, self.wpr,
                             nat.ptr(lzt), st)
                    keep.append(lzt)
                    spl = nat.ptr(lzt)
            self._splits = (spf, spl, keep)
        return self._splits[:2]

    def _merge_emit_tail(self, x0, x1, rows, buf, sync, codes_key):
        torch = self.torch
        st = self._st()
        dr, ds = self.dr, self.ds
        hp = nat.ptr(self.hpos) if self.strategy == PARTITIONED else 0
        lzp = nat.ptr(self.lz_ptr) if self.lz_ptr is not None else 0
        lzi = nat.ptr(self.lz_idx) if self.lz_idx is not None else 0
        wit0 = int(self.wit.item()) if sync else 0
        wsb = int(self.lib.mmj_merge_emit_workspace_size(rows, self.wpr))
        ws = self.ws.get("fuse_ws", wsb, torch.uint8)
        # capacity: the chunk's cells (the output size is known only after the kernel)
        cap = rows * self.dom_z
        codes = self.ws.get(codes_key, cap, torch.int64)
        slot = self._async_slot()
        spf, spl = self._tail_tables()
        self._ph("merge_emit", True)
        heavy_src = self.hbits if self.hbits is not None else buf
        nat.call("mmj_merge_emit", nat.ptr(heavy_src), self._has_heavy(), x0, rows, self.wpr, self.dom_z,
                 nat.ptr(dr.fwd_ptr), nat.ptr(dr.fwd_idx), nat.ptr(dr.left_deg), self.d2, hp, nat.ptr(ds.rev_ptr),
                 nat.ptr(ds.rev_idx), lzp, lzi, spf, spl, nat.ptr(self.wit), nat.ptr(self.nnz), nat.ptr(codes),
                 nat.ptr(slot),
                 nat.ptr(ws), wsb, st)
        self._ph("merge_emit", False)
        self.stats.chunks += 1
        if not sync:
            return ChunkResult(x0, x1, -1, codes, None, -1, slot[0:1])
        self._n_async -= 1          # consumed here, not by finish()
        total = int(slot[0].item())
        light = int(self.wit.item()) - wit0
        self.stats.out_size += total
        return ChunkResult(x0, x1, total, codes[:total], None, light)

    def _async_slot(self):
        """Device slot (2 x int64) receiving one async chunk's (size, light)."""
        torch = self.torch
        if self._sizes_dev is None or self._n_async >= self._sizes_dev.shape[0]:
            grow = max(64, 2 * (0 if self._sizes_dev is None else self._sizes_dev.shape[0]))
            new = torch.zeros((grow, 2), dtype=torch.int64, device="cuda")
            if self._sizes_dev is not None:
                new[: self._sizes_dev.shape[0]].copy_(self._sizes_dev)
            self._sizes_dev = new
        slot = self._sizes_dev[self._n_async]
        self._n_async += 1
        return slot

    def finish(self):
        # one device -> host copy (synchronises the stream): heavy pairs,
        # witnesses and the asynchronous chunks' (size, light) sums
        torch = self.torch
        parts = [self.nnz, self.wit]
        if self._n_async:
            parts.append(self._sizes_dev[: self._n_async].sum(dim=0))
        vals = torch.cat(parts).cpu().tolist()
        self.stats.heavy_pairs = int(vals[0])
        if self.fused:
            self.stats.light_intermediate = int(vals[1])
        if self._n_async:
            self.stats.out_size += int(vals[2])
            if not self.fused:
                self.stats.light_intermediate += int(vals[3])
            self._n_async = 0
        return self.stats

    def reset_stats(self):
        self.stats = EngineStats(k_heavy=self.stats.k_heavy, kpad=self.stats.kpad)
        self.nnz.zero_()
        self.wit.zero_()
        self._n_async = 0

    def run(self, consumer: Callable[[ChunkResult], None], x_begin: int = 0, x_end: Optional[int] = None):
        self.prepare()
        for x0, x1 in self.chunk_bounds(x_begin, x_end):
            consumer(self.run_chunk(x0, x1))
        return self.finish()
