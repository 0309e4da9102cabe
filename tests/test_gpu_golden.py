"""GPU parity against outputs frozen from the REFERENCE implementation
(tests/golden/*.npz, made by tests/golden/make_golden.py).  Bit-exact codes,
counts, dims and stats through the drop-in entry points."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _rels(z, i, self_join):
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce
    R = Relation.from_raw_pairs("R", z[f"i{i}_R"])
    if self_join:
        r = build_indexed(R)
        return r, r
    a, b = semi_join_reduce(R, Relation.from_raw_pairs("S", z[f"i{i}_S"]))
    return build_indexed(a), build_indexed(b)


def test_twopath_golden():
    from paper_2002_12459_b200.joinproject import two_path_join
    from paper_2002_12459_b200.optimizer import ThresholdPlan
    z = np.load(os.path.join(GOLDEN, "twopath.npz"))
    meta = json.loads(str(z["meta"]))
    cache = {}
    for m in meta:
        key = (m["inst"], m["self_join"])
        if key not in cache:
            cache[key] = _rels(z, *key)
        r, s = cache[key]
        st, d1, d2 = m["plan"]
        plan = None if st == "default" else ThresholdPlan(st, d1, d2)
        res = two_path_join(r, s, plan=plan, want_counts=m["counts"])
        k = m["key"]
        assert list(res.dims) == m["dims"], k
        assert np.array_equal(res.codes, z[k + "_codes"]), k
        if m["counts"]:
            assert np.array_equal(res.counts, z[k + "_counts"]), k
        for sk in ("light_intermediate", "heavy_pairs", "intermediate"):
            if sk in m["stats"]:
                assert res.stats[sk] == m["stats"][sk], (k, sk)
        p = res.stats["plan"]
        if "plan" in m["stats"]:
            assert [p.strategy, p.delta1, p.delta2] == m["stats"]["plan"], k


def test_worked_example_golden():
    from paper_2002_12459_b200.joinproject import heavy_matrices, partition_two_path, two_path_join
    from paper_2002_12459_b200.matmul import CountMatrix, multiply_counts
    from paper_2002_12459_b200.optimizer import ThresholdPlan
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce
    with open(os.path.join(GOLDEN, "example.json")) as f:
        ex = json.load(f)
    a, b = semi_join_reduce(Relation.from_raw_pairs("R", [tuple(p) for p in ex["R"]]),
                            Relation.from_raw_pairs("S", [tuple(p) for p in ex["S"]]))
    r, s = build_indexed(a), build_indexed(b)
    pr, ps = partition_two_path(r, s, 2, 2)
    assert sorted(pr.light.raw_pair_set()) == [tuple(p) for p in ex["light_R"]]
    assert sorted(pr.heavy.raw_pair_set()) == [tuple(p) for p in ex["heavy_R"]]
    assert sorted(ps.heavy.raw_pair_set()) == [tuple(p) for p in ex["heavy_S"]]
    m1, m2 = heavy_matrices(r, s, 2, 2)
    o1 = np.argsort([r.rel.left_values[i] for i in m1.row_keys])
    om = np.argsort([r.rel.right_values[i] for i in m1.col_keys])
    o2 = np.argsort([s.rel.left_values[i] for i in m2.col_keys])
    A = m1.data[o1][:, om]
    B = m2.data[om][:, o2]
    assert A.tolist() == ex["M1"] and B.tolist() == ex["M2"]
    assert multiply_counts(CountMatrix(A), CountMatrix(B)).data.tolist() == ex["product"]
    res = two_path_join(r, s, plan=ThresholdPlan("partitioned", 2, 2), want_counts=True)
    got = {f"{r.rel.left_values[x]},{s.rel.left_values[zz]}": int(c)
           for (x, zz), c in zip(res.tuples().tolist(), res.counts.tolist())}
    assert got == ex["counts"]
    assert res.total_count() == ex["out_join"]


def test_multiply_counts_golden():
    from paper_2002_12459_b200.matmul import CountMatrix, MatrixOverflowError, multiply_counts
    z = np.load(os.path.join(GOLDEN, "matmul.npz"))
    for i in range(12):
        got = multiply_counts(CountMatrix(z[f"m{i}_a"]), CountMatrix(z[f"m{i}_b"]), backend="cuda")
        assert np.array_equal(got.data, z[f"m{i}_p"]), i
    big = CountMatrix(np.array([[2 ** 62]], dtype=np.int64))
    with pytest.raises(MatrixOverflowError):
        multiply_counts(big, big)
    v = CountMatrix(np.array([[2 ** 31]], dtype=np.int64))
    with pytest.raises(MatrixOverflowError):
        multiply_counts(v, v, backend="blas")
    assert multiply_counts(v, v).data[0, 0] == 2 ** 62
    with pytest.raises(ValueError):
        multiply_counts(v, v, backend="fortran")


def test_chunked_api_concatenates_to_full():
    from paper_2002_12459_b200.joinproject import two_path_join, two_path_join_chunks
    from paper_2002_12459_b200.optimizer import ThresholdPlan
    z = np.load(os.path.join(GOLDEN, "twopath.npz"))
    meta = json.loads(str(z["meta"]))
    last = max(m["inst"] for m in meta)
    r, s = _rels(z, last, False)
    plan = ThresholdPlan("partitioned", 300, 1)
    full = two_path_join(r, s, plan=plan)
    parts = list(two_path_join_chunks(r, s, plan=plan, chunk_rows=128))
    assert len(parts) > 1
    assert np.array_equal(np.concatenate([p.codes for p in parts]), full.codes)
    assert all(np.all(np.diff(p.codes) > 0) for p in parts)


def test_sharded_outputs_concatenate_to_full():
    from paper_2002_12459_b200.joinproject import two_path_join
    from paper_2002_12459_b200.optimizer import ThresholdPlan
    from paper_2002_12459_b200.shard import two_path_join_shard
    z = np.load(os.path.join(GOLDEN, "twopath.npz"))
    meta = json.loads(str(z["meta"]))
    last = max(m["inst"] for m in meta)
    r, s = _rels(z, last, False)
    plan = ThresholdPlan("partitioned", 40, 3)
    full = two_path_join(r, s, plan=plan, want_counts=True)
    for world in (2, 3):
        parts = [two_path_join_shard(r, s, plan, k, world, want_counts=True, chunk_rows=128) for k in range(world)]
        assert np.array_equal(np.concatenate([p.codes for p in parts]), full.codes)
        assert np.array_equal(np.concatenate([p.counts for p in parts]), full.counts)


def test_chunked_api_pipelined_host_buffers():
    """two_path_join_chunks with a pair of pinned host buffers (compute of
    chunk i+1 overlapping chunk i's D2H) yields exactly the codes."""
    import torch
    from paper_2002_12459_b200.joinproject import two_path_join, two_path_join_chunks
    from paper_2002_12459_b200.optimizer import ThresholdPlan
    z = np.load(os.path.join(GOLDEN, "twopath.npz"))
    meta = json.loads(str(z["meta"]))
    last = max(m["inst"] for m in meta)
    r, s = _rels(z, last, False)
    plan = ThresholdPlan("partitioned", 300, 1)
    full = two_path_join(r, s, plan=plan)
    bufs = tuple(torch.empty(128 * s.rel.dom_left, dtype=torch.int64, pin_memory=True) for _ in range(2))
    got = [p.codes.copy() for p in two_path_join_chunks(r, s, plan=plan, chunk_rows=128, host_buffer=bufs,
                                                        upload="fresh")]
    assert len(got) > 1
    assert np.array_equal(np.concatenate(got), full.codes)
