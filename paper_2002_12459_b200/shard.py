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


def combine_checksums(n_local: int, s_local: int, w_local: int, group=None) -> tuple:
    """Whole-output (|OUT|, sum, weighted sum) of the rank-order concatenation
    of the shards' code runs, every rank computing its own with base 0
    (mmj_code_checksum: s = sum c_i, w = sum (base + i + 1) c_i mod 2^64, so a
    run shifted by `base` codes adds base * s).  One all-gather of three
    words per rank; every rank returns the same triple."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return int(n_local), int(s_local) & _M64, int(w_local) & _M64
    dev = _group_device(group)
    mine = torch.tensor([_i64(n_local), _i64(s_local), _i64(w_local)], dtype=torch.int64, device=dev)
    parts = [torch.empty(3, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    n = s = w = 0
    for p in parts:
        pn, ps, pw = (int(v) & _M64 for v in p.cpu().tolist())
        w = (w + pw + n * ps) & _M64
        s = (s + ps) & _M64
        n += pn
    return n, s, w


def gather_batch_answers(ans_local, nq: int, group=None):
    """Answers of a position-sharded BSI batch back in batch order on every
    rank: rank r holds the int8 answers of batch_slice(nq, r, world); slices
    are padded to the longest for the all-gather (NCCL needs equal sizes) and
    cut back in rank order.  Returns a tensor of nq answers on ans_local's
    device."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return ans_local[:nq]
    rank = dist.get_rank(group)
    lo, hi = batch_slice(nq, rank, world)
    if int(ans_local.numel()) < hi - lo:
        raise ValueError(f"rank {rank}: {ans_local.numel()} answers for the {hi - lo}-query slice")
    width = max(hi_ - lo_ for lo_, hi_ in (batch_slice(nq, k, world) for k in range(world)))
    width = max(width, 1)
    dev = _group_device(group)
    pad = torch.full((width,), -2, dtype=torch.int8, device=dev)
    pad[: hi - lo] = ans_local[: hi - lo].to(dev)
    parts = [torch.empty(width, dtype=torch.int8, device=dev) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    out = torch.cat([parts[k][: b - a] for k, (a, b) in enumerate(batch_slice(nq, k, world) for k in range(world))])
    return out.to(ans_local.device)


_M64 = (1 << 64) - 1


def _i64(v: int) -> int:
    """uint64 bit pattern as a signed int64 (torch has no uint64 all-gather)."""
    v = int(v) & _M64
    return v - (1 << 64) if v >= (1 << 63) else v


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


REL_FIELDS = ("fwd_ptr", "fwd_idx", "fwd_row", "rev_ptr", "rev_idx", "left_deg", "right_deg")


def replicate_relation(dr, src: int = 0, group=None):
    """Replicate a device relation (the S side, or S_h's source) from rank
    `src` to every rank of the process group: one broadcast per CSR array
    (NCCL over NVLink on GPUs; any backend whose tensors live where `dr`'s
    do).  Non-source ranks pass an object with the same fields, or None and
    receive a fresh one; sizes travel first so they need no host copy of S.
    SURVEY.md 8(e): S is replicated, R sharded by x range."""
    import torch
    import torch.distributed as dist
    from .device import DeviceRelation
    rank = dist.get_rank(group)
    if rank == src:
        dev = dr.fwd_ptr.device
        meta = torch.tensor([dr.n, dr.dom_left, dr.dom_right], dtype=torch.int64, device=dev)
    else:
        dev = _group_device(group)
        meta = torch.zeros(3, dtype=torch.int64, device=dev)
    dist.broadcast(meta, src, group=group)
    n, dom_l, dom_r = (int(v) for v in meta.tolist())
    if rank != src:
        dr = DeviceRelation()
        dr.fwd_ptr_host = None
        dr.n, dr.dom_left, dr.dom_right = n, dom_l, dom_r
        dr.device = dev
        sizes = {"fwd_ptr": dom_l + 1, "fwd_idx": n, "fwd_row": n, "rev_ptr": dom_r + 1, "rev_idx": n,
                 "left_deg": dom_l, "right_deg": dom_r}
        for k in REL_FIELDS:
            setattr(dr, k, torch.empty(sizes[k], dtype=torch.int32, device=dev))
        dr.h2d_bytes = 0
    for k in REL_FIELDS:
        dist.broadcast(getattr(dr, k), src, group=group)
    if getattr(dr, "fwd_ptr_host", None) is None:
        dr.fwd_ptr_host = dr.fwd_ptr.cpu().numpy().astype(np.int64)
    return dr


def global_right_degrees(local_deg, group=None):
    """deg_R(y) of an x-sharded R: the sum of the shards' y-degree vectors
    (all-reduce; the heavy/light split of joinproject.py:178-180 needs the
    global degree).  In place on `local_deg`, returned for chaining."""
    import torch.distributed as dist
    dist.all_reduce(local_deg, op=dist.ReduceOp.SUM, group=group)
    return local_deg


def _group_device(group):
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")
