"""Multi-process (gloo, world_size 2, CPU) tests of the x-range sharding:
ranges cover the domain, balance the witness work, and the rank-order
concatenation of per-rank outputs equals the single-process output.  The
per-rank compute here is the CPU oracle (the GPU engine runs the same ranges
in bench.py); the max-over-ranks timing / size exchange uses torch.distributed
exactly as bench.py does."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, random_pairs, zipf_pairs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rels(seed=5):
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce
    rng = np.random.default_rng(seed)
    rp = np.array(zipf_pairs(rng, 4000, 300, 500, 1.1))
    sp = np.array(zipf_pairs(rng, 4000, 280, 500, 1.1))
    a, b = semi_join_reduce(Relation.from_raw_pairs("R", rp), Relation.from_raw_pairs("S", sp))
    return rp, sp, build_indexed(a), build_indexed(b)


def test_ranges_cover_and_balance():
    from paper_2002_12459_b200 import shard
    _, _, r, s = _rels()
    for world in (1, 2, 3, 8):
        rg = shard.x_ranges(r, s, world)
        assert rg[0][0] == 0 and rg[-1][1] == r.rel.dom_left
        assert all(a[1] == b[0] for a, b in zip(rg, rg[1:]))
        w = shard.x_work(r, s)
        loads = [w[hi] - w[lo] for lo, hi in rg]
        assert max(loads) <= w[-1] / world + w[-1] * 0.05 + max(np.diff(w))
    assert [shard.batch_slice(10, k, 3) for k in range(3)] == [(0, 4), (4, 7), (7, 10)]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import sys
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import mmjoin_oracle as o
    from paper_2002_12459_b200 import shard
    rp, sp, r, s = _rels()
    lo, hi = shard.shard_of(r, s, rank, world)
    # per-rank compute (oracle restricted to the rank's x range, in r's dense ids)
    OR, OS = o.semi_join_many([o.encode(rp), o.encode(sp)])
    full = o.two_path(OR, OS, None)
    mine = full.codes[(full.codes // full.dims[1] >= lo) & (full.codes // full.dims[1] < hi)]
    # size exchange + max-over-ranks timing, as bench.py
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([len(mine)], dtype=torch.int64))
    t = torch.tensor([0.01 * (rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    gathered = [None] * world
    dist.all_gather_object(gathered, mine.tolist())
    if rank == 0:
        cat = np.concatenate([np.asarray(g, dtype=np.int64) for g in gathered])
        out.put((cat.tolist() == full.codes.tolist(), [int(x) for x in sizes], float(t)))
    dist.destroy_process_group()


def test_gloo_two_ranks_concatenate_to_full():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, 2, port, q)) for k in range(2)]
    for p in procs:
        p.start()
    ok, sizes, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert ok
    assert sum(sizes) > 0 and all(x > 0 for x in sizes)
    assert tmax == pytest.approx(0.02)


def _replicate_worker(rank, world, port, out):
    try:
        _replicate_body(rank, world, port, out)
    except Exception as e:  # noqa: BLE001 - report to the parent
        out.put((rank, repr(e)))


def _replicate_body(rank, world, port, out):
    import torch
    import torch.distributed as dist

    from paper_2002_12459_b200.device import DeviceRelation
    from paper_2002_12459_b200.relation import Relation, build_indexed
    from paper_2002_12459_b200.shard import global_right_degrees, replicate_relation
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    rng = np.random.default_rng(5)
    sp = np.array(random_pairs(rng, 3000, 200, 90), dtype=np.int64)
    S = build_indexed(Relation.from_raw_pairs("S", sp))
    src = None
    if rank == 0:          # a CPU stand-in for the device copy (gloo broadcasts CPU tensors)
        src = DeviceRelation()
        src.n, src.dom_left, src.dom_right = S.rel.n, S.rel.dom_left, S.rel.dom_right
        host = {"fwd_ptr": S.fwd_indptr, "fwd_idx": S.fwd_indices, "rev_ptr": S.rev_indptr,
                "rev_idx": S.rev_indices, "left_deg": S.left_deg, "right_deg": S.right_deg,
                "fwd_row": np.repeat(np.arange(S.rel.dom_left), S.left_deg)}
        for k, v in host.items():
            setattr(src, k, torch.from_numpy(np.ascontiguousarray(v, dtype=np.int32)))
    got = replicate_relation(src, 0)
    ok = (got.n == S.rel.n and np.array_equal(got.rev_idx.numpy(), S.rev_indices)
          and np.array_equal(got.fwd_ptr.numpy(), S.fwd_indptr) and np.array_equal(got.fwd_ptr_host, S.fwd_indptr))
    # x-sharded R: per-shard y degrees all-reduce to the global ones
    rp = np.array(random_pairs(rng, 4000, 300, 90), dtype=np.int64)
    mine = rp[(rp[:, 0] % world) == rank]
    local = torch.from_numpy(np.bincount(mine[:, 1], minlength=90).astype(np.int64))
    glob = global_right_degrees(local)
    ok = ok and np.array_equal(glob.numpy(), np.bincount(rp[:, 1], minlength=90))
    out.put((rank, bool(ok)))
    dist.destroy_process_group()


def test_gloo_replicate_relation_and_global_degrees():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_replicate_worker, args=(k, 2, port, q)) for k in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=120) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    assert res == [(0, True), (1, True)]


# ---- bench.py's rank orchestration (shard.combine_checksums /
# shard.gather_batch_answers, the calls bench.py's verify() makes on every
# rank) with the CPU oracle standing in for the per-rank kernel call only

M64 = (1 << 64) - 1


def host_checksum(codes):
    """numpy restatement of mmj_code_checksum with base 0 (scan.cu)."""
    c = np.asarray(codes, dtype=np.int64).astype(np.uint64)
    with np.errstate(over="ignore"):
        s = int(c.sum(dtype=np.uint64))
        w = int((np.arange(1, len(c) + 1, dtype=np.uint64) * c).sum(dtype=np.uint64))
    return len(c), s & M64, w & M64


def _orch_worker(rank, world, port, out):
    try:
        out.put((rank, _orch_body(rank, world, port)))
    except Exception as e:  # noqa: BLE001 - report to the parent
        import traceback
        out.put((rank, traceback.format_exc() + repr(e)))


def _orch_body(rank, world, port):
    import torch

    from oracle import mmjoin_oracle as o
    from paper_2002_12459_b200 import shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    res = {}
    # two-path (cfg2's orchestration): witness-balanced x range -> this rank's
    # sorted codes -> whole-job (|OUT|, sum, wsum) stamp
    rp, sp, r, s = _rels(7)
    lo, hi = shard.shard_of(r, s, rank, world)
    OR, OS = o.semi_join_many([o.encode(rp), o.encode(sp)])
    full = o.two_path(OR, OS, None)
    x = full.codes // full.dims[1]
    mine = full.codes[(x >= lo) & (x < hi)]                 # stand-in for the engine's chunks
    stamp = shard.combine_checksums(*host_checksum(mine))
    res["two_path"] = stamp == host_checksum(full.codes)
    res["nonempty"] = len(mine) > 0
    # BSI (cfg5's orchestration): contiguous batch slice -> answers -> batch
    # order on every rank, uneven slice lengths included
    rng = np.random.default_rng(11)
    ra = np.array(random_pairs(rng, 3000, 400, 300), dtype=np.int64)
    sa = np.array(random_pairs(rng, 3000, 400, 300), dtype=np.int64)
    OR5, OS5 = o.encode(ra), o.encode(sa)
    nq = 1001 + world                                        # not a multiple of world
    qa = rng.integers(-5, 410, nq)
    qb = rng.integers(-5, 410, nq)
    qlo, qhi = shard.batch_slice(nq, rank, world)
    local = torch.from_numpy(o.bsi(OR5, OS5, qa[qlo:qhi], qb[qlo:qhi]))
    got = shard.gather_batch_answers(local, nq).numpy()
    exp = o.bsi(OR5, OS5, qa, qb)
    res["bsi"] = bool(np.array_equal(got, exp)) and (exp == -1).any() and (exp == 1).any()
    dist.destroy_process_group()
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_bench_orchestration_two_path_and_bsi(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_orch_worker, args=(k, world, port, q)) for k in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=240) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
    for rank, r in res:
        assert isinstance(r, dict), r
        assert r == {"two_path": True, "nonempty": True, "bsi": True}, (rank, r)
