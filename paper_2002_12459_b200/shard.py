"""Multi-GPU sharding of the join-project path.

Each output row x depends only on R[x] and all of S, so a join shards into
contiguous dense-x ranges with S replicated and no data-path collective:
rank r owns the codes [x_lo(r)*dom_z, x_hi(r)*dom_z), and the rank-order
concatenation of the shards' outputs is the globally sorted output.  Ranges
are balanced by witness work w(x) = sum_{y in R[x]} deg_S(y) (the Zipf skew
makes per-x work uneven), not by row count.  BSI shards the query batch into
contiguous position slices.  One process per GPU (torchrun); collectives are
only used for the barrier / max-over-ranks timing and size exchange.
"""

from __future__ import annotations

import numpy as np


def x_work(r, s) -> np.ndarray:
    """Prefix sums of witness work over dense x (length dom_x + 1)."""
    per_tuple = np.asarray(s.right_deg, dtype=np.int64)[np.asarray(r.fwd_indices)]
    csum = np.concatenate([[0], np.cumsum(per_tuple)])
    return csum[np.asarray(r.fwd_indptr)]


def x_ranges(r, s, world: int) -> list:
    """Contiguous [lo, hi) dense-x ranges, one per rank, covering [0, dom_x)
    with (near-)equal witness work."""
    dom = r.rel.dom_left
    if world <= 1:
        return [(0, dom)]
    w = x_work(r, s)
    total = int(w[-1])
    cuts = [0]
    for k in range(1, world):
        c = int(np.searchsorted(w, total * k / world))
        cuts.append(min(max(c, cuts[-1]), dom))
    cuts.append(dom)
    return [(cuts[i], cuts[i + 1]) for i in range(world)]


def shard_of(r, s, rank: int, world: int) -> tuple:
    return x_ranges(r, s, world)[rank]


def batch_slice(nq: int, rank: int, world: int) -> tuple:
    """Contiguous query positions of a BSI batch owned by `rank`."""
    base, extra = divmod(nq, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def two_path_join_shard(r, s, plan=None, rank: int = 0, world: int = 1, want_counts: bool = False,
                        chunk_rows=None):
    """This rank's part of two_path_join: an OutputSet over its x range
    (codes are global codes; concatenating ranks 0..world-1 in order gives
    the full result)."""
    import numpy as _np

    from .joinproject import OutputSet, two_path_join_chunks
    lo, hi = shard_of(r, s, rank, world)
    parts = list(two_path_join_chunks(r, s, plan=plan, want_counts=want_counts, chunk_rows=chunk_rows,
                                      x_range=(lo, hi)))
    codes = _np.concatenate([p.codes for p in parts]) if parts else _np.empty(0, _np.int64)
    counts = (_np.concatenate([p.counts for p in parts]) if parts else _np.empty(0, _np.int64)) if want_counts else None
    dims = (r.rel.dom_left, s.rel.dom_left)
    return OutputSet(codes, dims, counts, {"x_range": (lo, hi), "rank": rank, "world": world})
