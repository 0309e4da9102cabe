"""Device ingest (csrc/ingest.cu, ingest.py) against the oracle's restatement
of relation.py:37-69 / 119-140 / 148-186 (pinned to the reference's fixtures in
test_oracle_golden.py): identical dictionaries, dense pairs, both CSR
directions and degrees, and identical join outputs downstream."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _raw(rng, n, lo, hi, dup=0.2):
    a = rng.integers(lo, hi, size=n)
    b = rng.integers(lo, hi, size=n)
    p = np.stack([a, b], axis=1).astype(np.int64)
    k = int(dup * n)
    if k and n:
        p = np.concatenate([p, p[rng.integers(0, n, size=k)]])
        p = p[rng.permutation(len(p))]
    return p


def _check(dev, orel):
    assert dev.rel.n == orel.n
    assert np.array_equal(dev.rel.left_values, np.asarray(orel.left_values, dtype=np.int64))
    assert np.array_equal(dev.rel.right_values, np.asarray(orel.right_values, dtype=np.int64))
    assert np.array_equal(dev.rel.pairs, orel.pairs)
    fp, fi = orel.fwd()
    rp, ri = orel.rev()
    assert np.array_equal(dev.fwd_indptr, fp) and np.array_equal(dev.fwd_indices, fi)
    assert np.array_equal(dev.rev_indptr, rp) and np.array_equal(dev.rev_indices, ri)
    assert np.array_equal(dev.left_deg, orel.left_deg) and np.array_equal(dev.right_deg, orel.right_deg)
    d = dev.device
    rows = np.repeat(np.arange(orel.dom_left), orel.left_deg)
    assert np.array_equal(d.fwd_row.cpu().numpy(), rows)


@pytest.mark.parametrize("seed,n,lo,hi", [(0, 1, 0, 5), (1, 500, -50, 50), (2, 20000, 0, 3000),
                                          (3, 50000, -(1 << 62), 1 << 62), (4, 30000, 0, 40)])
def test_from_raw_pairs_device(oracle, seed, n, lo, hi):
    from paper_2002_12459_b200.ingest import from_raw_pairs_device
    raw = _raw(np.random.default_rng(seed), n, lo, hi)
    _check(from_raw_pairs_device("R", raw), oracle.encode(raw))


def _repr_heavy(rng, n):
    # right values whose repr order differs from numeric order: mixed digit
    # lengths, negatives, extremes
    pool = np.array([0, 1, 9, 10, 11, 99, 100, 101, 1000, -1, -9, -10, -100, 12, 2, 20, 200,
                     (1 << 63) - 1, -(1 << 63), 123456789012345, 98765], dtype=np.int64)
    a = rng.integers(0, 200, size=n)
    b = pool[rng.integers(0, len(pool), size=n)]
    return np.stack([a, b], axis=1).astype(np.int64)


@pytest.mark.parametrize("k", [2, 3])
def test_semi_join_reduce_device(oracle, k):
    from paper_2002_12459_b200.ingest import semi_join_reduce_device
    rng = np.random.default_rng(10 + k)
    raws = [_repr_heavy(rng, 3000) for _ in range(k)]
    raws.append(_raw(rng, 20000, 0, 150))
    raws[-1][:, 1] = np.where(raws[-1][:, 1] < 60, raws[-1][:, 1], raws[-1][:, 1] * 7)
    got = semi_join_reduce_device(raws)
    exp = oracle.semi_join_many([oracle.encode(r) for r in raws])
    assert all(g.rel.right_values is got[0].rel.right_values for g in got)
    for g, e in zip(got, exp):
        _check(g, e)


def test_ingest_edge_cases(oracle):
    from paper_2002_12459_b200.ingest import from_raw_pairs_device, semi_join_reduce_device
    empty = np.empty((0, 2), dtype=np.int64)
    d = from_raw_pairs_device("E", empty)
    assert d.rel.n == 0 and d.rel.dom_left == 0 and list(d.fwd_indptr) == [0]
    # disjoint right domains: everything filtered
    a = np.array([[1, 1], [2, 2]], dtype=np.int64)
    b = np.array([[1, 3], [2, 4]], dtype=np.int64)
    r, s = semi_join_reduce_device([a, b])
    assert r.rel.n == 0 and s.rel.n == 0 and r.rel.dom_right == 0
    # all duplicates
    c = np.array([[5, 6]] * 100, dtype=np.int64)
    _check(from_raw_pairs_device("C", c), oracle.encode(c))


def test_device_ingested_join_matches_host(oracle):
    from conftest import zipf_pairs
    from paper_2002_12459_b200.ingest import semi_join_reduce_device
    from paper_2002_12459_b200.joinproject import two_path_join
    rng = np.random.default_rng(7)
    rp = np.array(zipf_pairs(rng, 20000, 700, 900, 1.1))
    sp = np.array(zipf_pairs(rng, 20000, 650, 900, 1.1))
    r, s = semi_join_reduce_device([rp, sp])
    got = two_path_join(r, s, want_counts=True)
    OR, OS = oracle.semi_join_many([oracle.encode(rp), oracle.encode(sp)])
    exp = oracle.two_path(OR, OS, None, want_counts=True)
    assert list(got.dims) == list(exp.dims)
    assert np.array_equal(got.codes, exp.codes)
    assert np.array_equal(got.counts, exp.counts)


@pytest.mark.parametrize("shared", [False, True])
def test_bsi_on_device_ingested(oracle, shared):
    from conftest import zipf_pairs
    from paper_2002_12459_b200.apps import bsi_answer_batch_arrays
    from paper_2002_12459_b200.ingest import from_raw_pairs_device, semi_join_reduce_device
    rng = np.random.default_rng(31 + shared)
    rp = np.array(zipf_pairs(rng, 30000, 3000, 2000, 1.0)) * np.array([7, 3]) - np.array([500, 40])
    sp = np.array(zipf_pairs(rng, 30000, 2500, 2600, 1.0)) * np.array([5, 3]) - np.array([9, 40])
    q = np.stack([rng.integers(-600, 21500, 20000), rng.integers(-20, 12600, 20000)], axis=1)
    if shared:
        r, s = semi_join_reduce_device([rp, sp])
        OR, OS = oracle.semi_join_many([oracle.encode(rp), oracle.encode(sp)])
    else:
        r, s = from_raw_pairs_device("R", rp), from_raw_pairs_device("S", sp)
        OR, OS = oracle.encode(rp), oracle.encode(sp)
    exp = oracle.bsi(OR, OS, q[:, 0], q[:, 1])
    assert (exp == -1).any() and (exp == 1).any() and (exp == 0).any()
    for hb in (128, 512):
        got = bsi_answer_batch_arrays(r, s, q[:, 0], q[:, 1], heavy_bits=hb)
        assert np.array_equal(got, exp), hb


def test_ingest_from_cuda_tensor_and_errors(oracle):
    import torch
    from paper_2002_12459_b200 import _native as nat
    from paper_2002_12459_b200.ingest import from_raw_pairs_device
    raw = _raw(np.random.default_rng(99), 5000, -1000, 1000)
    _check(from_raw_pairs_device("R", torch.from_numpy(raw).cuda()), oracle.encode(raw))
    # a workspace smaller than mmj_ingest_workspace_bytes(n) is an argument error
    t = torch.from_numpy(raw).cuda()
    out = torch.empty_like(t)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        nat.call("mmj_ingest_dedup", nat.ptr(t), t.shape[0], nat.ptr(out), nat.ptr(cnt), nat.ptr(ws), 16,
                 nat.stream_handle())
    buf = torch.zeros(1024, dtype=torch.int32, device="cuda")
    seg = torch.zeros(2, dtype=torch.int32, device="cuda")
    off = torch.zeros(3, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):   # cell_bytes must be 2 or 4
        nat.call("mmj_count_segments", nat.ptr(buf), 3, 1, 1024, 1000, 0, 1, 0, 0, nat.ptr(seg), nat.ptr(off),
                 nat.ptr(ws), nat.stream_handle())
    with pytest.raises(ValueError):   # pitch not a multiple of 1024
        nat.call("mmj_count_segments", nat.ptr(buf), 4, 1, 1000, 1000, 0, 1, 0, 0, nat.ptr(seg), nat.ptr(off),
                 nat.ptr(ws), nat.stream_handle())
