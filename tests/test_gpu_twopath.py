"""GPU parity: two-path join / full join / multiply_counts vs the CPU oracle.

Bit-exact: identical code arrays (sorted distinct int64 mixed-radix codes),
identical int64 counts and identical ``stats`` counters, for every plan --
the output is plan-independent but the stats are not, so each
plan is checked as given.
"""

import numpy as np
import pytest

from conftest import random_pairs, zipf_pairs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2002_12459_b200 as p
    from paper_2002_12459_b200 import joinproject, matmul  # noqa: F401
    return p


def _mine(pkg, r_pairs, s_pairs, self_join=False):
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce
    R = Relation.from_raw_pairs("R", np.asarray(r_pairs, dtype=np.int64).reshape(-1, 2))
    if self_join:
        r = build_indexed(R)
        return r, r
    S = Relation.from_raw_pairs("S", np.asarray(s_pairs, dtype=np.int64).reshape(-1, 2))
    R, S = semi_join_reduce(R, S)
    return build_indexed(R), build_indexed(S)


def _oracle_rels(oracle, r_pairs, s_pairs, self_join=False):
    R = oracle.encode(np.asarray(r_pairs, dtype=np.int64).reshape(-1, 2))
    if self_join:
        return R, R
    S = oracle.encode(np.asarray(s_pairs, dtype=np.int64).reshape(-1, 2))
    return tuple(oracle.semi_join_many([R, S]))


def _check(pkg, oracle, r_pairs, s_pairs, plans, self_join=False, chunk_rows=None):
    from paper_2002_12459_b200.joinproject import two_path_join
    from paper_2002_12459_b200.optimizer import ThresholdPlan
    r, s = _mine(pkg, r_pairs, s_pairs, self_join)
    orr, oss = _oracle_rels(oracle, r_pairs, s_pairs, self_join)
    for strategy, d1, d2 in plans:
        for counts in (False, True):
            got = two_path_join(r, s, plan=ThresholdPlan(strategy, d1, d2), want_counts=counts,
                                chunk_rows=chunk_rows)
            exp = oracle.two_path(orr, oss, oracle.OPlan(strategy, d1, d2), want_counts=counts)
            assert got.dims == tuple(exp.dims)
            assert np.array_equal(got.codes, exp.codes), (strategy, d1, d2, counts)
            if counts:
                assert got.counts.dtype == np.int64
                assert np.array_equal(got.counts, exp.counts), (strategy, d1, d2)
            for key in ("light_intermediate", "heavy_pairs", "intermediate"):
                if key in exp.stats:
                    assert got.stats[key] == exp.stats[key], (key, strategy, d1, d2, counts)


@pytest.mark.parametrize("heavy", ["mma", "or"])
@pytest.mark.parametrize("seed", range(6))
def test_two_path_random_plans(pkg, oracle, seed, heavy, monkeypatch):
    """Both heavy kernels of the projection: the tcgen05 product into a chunk
    bitmap and the in-tile OR of heavy-y bit rows (the count path always
    uses the product)."""
    monkeypatch.setenv("MMJ_HEAVY", heavy)
    rng = np.random.default_rng(seed)
    n = int(rng.integers(20, 400))
    dom = int(rng.integers(5, 40))
    rp = random_pairs(rng, n, dom, dom)
    sp = random_pairs(rng, n, dom, dom)
    nn = max(len(rp), len(sp))
    plans = [("partitioned", 1, 1), ("partitioned", 2, 3), ("partitioned", 5, 2),
             ("partitioned", nn, nn), ("fulljoin", nn, nn)]
    _check(pkg, oracle, rp, sp, plans)


@pytest.mark.parametrize("heavy", ["", "mma", "or"])
@pytest.mark.parametrize("chunk_rows", [None, 128])
def test_two_path_zipf_medium(pkg, oracle, chunk_rows, heavy, monkeypatch):
    monkeypatch.setenv("MMJ_HEAVY", heavy)
    rng = np.random.default_rng(11)
    rp = zipf_pairs(rng, 20000, 1500, 3000, 1.2)
    sp = zipf_pairs(rng, 20000, 1300, 3000, 1.1)
    plans = [("partitioned", 10, 10), ("partitioned", 300, 1), ("partitioned", 40, 3)]
    _check(pkg, oracle, rp, sp, plans, chunk_rows=chunk_rows)


def test_two_path_self_join_default_plan(pkg, oracle):
    from paper_2002_12459_b200.joinproject import two_path_join
    rng = np.random.default_rng(3)
    rp = zipf_pairs(rng, 30000, 2000, 2000, 1.2)
    r, _ = _mine(pkg, rp, None, self_join=True)
    R, _ = _oracle_rels(oracle, rp, None, self_join=True)
    got = two_path_join(r, r, want_counts=True)
    exp = oracle.two_path(R, R, None, want_counts=True)
    assert got.stats["plan"].delta1 == exp.stats["plan"].delta1
    assert got.stats["plan"].delta2 == exp.stats["plan"].delta2
    assert np.array_equal(got.codes, exp.codes)
    assert np.array_equal(got.counts, exp.counts)
    assert got.stats["light_intermediate"] == exp.stats["light_intermediate"]
    assert got.stats["heavy_pairs"] == exp.stats["heavy_pairs"]
    assert got.total_count() == r.out_join_with(r)


def test_full_join_dedup(pkg, oracle):
    from paper_2002_12459_b200.joinproject import full_join_dedup
    rng = np.random.default_rng(5)
    rp = random_pairs(rng, 300, 25, 20)
    sp = random_pairs(rng, 300, 25, 20)
    r, s = _mine(pkg, rp, sp)
    R, S = _oracle_rels(oracle, rp, sp)
    for counts in (False, True):
        got = full_join_dedup(r, s, want_counts=counts)
        exp = oracle.full_join(R, S, counts)
        assert np.array_equal(got.codes, exp.codes)
        assert got.stats["intermediate"] == exp.stats["intermediate"] == r.out_join_with(s)
        if counts:
            assert np.array_equal(got.counts, exp.counts)


@pytest.mark.parametrize("hi", [2, 5, 300, 10 ** 6])
def test_multiply_counts_exact(pkg, hi):
    from paper_2002_12459_b200.matmul import CountMatrix, multiply_counts
    rng = np.random.default_rng(hi)
    for _ in range(6):
        u, v, w = (int(x) for x in rng.integers(1, 300, 3))
        a = rng.integers(0, hi, (u, v)).astype(np.int64)
        b = rng.integers(0, hi, (v, w)).astype(np.int64)
        got = multiply_counts(CountMatrix(a), CountMatrix(b)).data
        assert np.array_equal(got, a @ b)


def test_multiply_counts_large_k(pkg):
    from paper_2002_12459_b200.matmul import CountMatrix, multiply_counts
    rng = np.random.default_rng(1)
    a = rng.integers(0, 2, (300, 40000)).astype(np.int64)
    b = rng.integers(0, 256, (40000, 260)).astype(np.int64)
    got = multiply_counts(CountMatrix(a), CountMatrix(b)).data
    assert np.array_equal(got, a @ b)


@pytest.mark.parametrize("dom_z", [700, 30000, 300000])
def test_fused_row_emit_wide_rows(pkg, oracle, dom_z):
    """Row-group sizes from many rows per CTA (narrow z domain) to one
    60 KB row per CTA; plans with and without a heavy part."""
    rng = np.random.default_rng(dom_z)
    rp = zipf_pairs(rng, 6000, 400, 900, 1.1)
    sp = zipf_pairs(rng, 8000, dom_z, 900, 1.1)
    plans = [("partitioned", 20, 1), ("partitioned", 5, 5), ("fulljoin", 1, 1)]
    _check(pkg, oracle, rp, sp, plans)


def _pair_boundary_pairs(rng, deg_x0, n_y=300):
    """x0 holds deg_x0 heavy y; z 0..15 reach all of them (count = deg_x0 on
    both accumulator slots of several z pairs); filler tuples make every y heavy at
    delta1 = 1 and keep the other degrees small."""
    r = [(0, y) for y in range(deg_x0)]
    # z 0..15 cover both slots of the first pair rows (z = k + 8j -> row 2k + j/2)
    s = [(0, y) for y in range(n_y)] + [(z, y) for z in range(1, 16) for y in range(deg_x0)]
    for y in range(n_y):
        r += [(1 + int(rng.integers(0, 400)), y), (401 + y, y)]
        s += [(2 + int(rng.integers(0, 400)), y), (403 + y, y)]
    return sorted(set(r)), sorted(set(s))


@pytest.mark.parametrize("deg_x0", [126, 127, 128])
@pytest.mark.parametrize("heavy", ["mma", "or"])
def test_pair_operand_count_boundary(pkg, oracle, deg_x0, heavy, monkeypatch):
    """BITMAP_PAIR packs two cells as c0 + 128*c1 (engine.py: on iff one
    side's heavy degrees are <= 127): counts of exactly 127 on both slots must
    not carry, and 128 must switch the pair form off.  The tcgen05 product is
    forced (MMJ_HEAVY=mma; the default picks the in-tile OR for these sparse
    heavy rows, which has no pair operand) and the OR path checked too."""
    monkeypatch.setenv("MMJ_HEAVY", heavy)
    from paper_2002_12459_b200.joinproject import _collect, _engine
    from paper_2002_12459_b200.optimizer import ThresholdPlan
    rng = np.random.default_rng(deg_x0)
    rp, sp = _pair_boundary_pairs(rng, deg_x0)
    r, s = _mine(pkg, rp, sp)
    plan = ThresholdPlan("partitioned", 1, 1)
    eng = _engine(r, s, plan, False)
    eng.prepare()
    assert eng.heavy_kernel == heavy
    if heavy == "mma":
        assert eng.pairs == (deg_x0 <= 127 or int(np.max(s.left_deg)) <= 127)
    got = _collect(eng)
    R, S = _oracle_rels(oracle, rp, sp)
    exp = oracle.two_path(R, S, oracle.OPlan("partitioned", 1, 1))
    assert np.array_equal(got[0], exp.codes)


@pytest.mark.parametrize("case", ["disjoint_y", "single_pair", "one_hub_y", "one_x_row", "skinny_z"])
def test_two_path_edge_cases(pkg, oracle, case):
    """Empty semi-join result, a single output pair, one y shared by every
    tuple (K = 1 heavy column), a single output row, a single output column:
    every plan, with and without counts, bit-exact vs the oracle."""
    if case == "disjoint_y":
        rp = [(x, 2 * x) for x in range(50)]
        sp = [(z, 2 * z + 1) for z in range(50)]
    elif case == "single_pair":
        rp = [(7, 3), (8, 4)]
        sp = [(9, 3), (10, 5)]
    elif case == "one_hub_y":
        rp = [(x, 0) for x in range(300)] + [(x, 1 + x % 7) for x in range(300)]
        sp = [(z, 0) for z in range(260)] + [(z, 1 + z % 5) for z in range(0, 260, 3)]
    elif case == "one_x_row":
        rp = [(5, y) for y in range(200)]
        sp = [(z, y % 200) for z in range(40) for y in range(z, z + 15)]
    else:
        rp = [(x, y) for x in range(120) for y in range(x % 9, x % 9 + 4)]
        sp = [(3, y) for y in range(20)]
    nn = max(len(rp), len(sp))
    plans = [("partitioned", 1, 1), ("partitioned", 2, 1), ("partitioned", 3, 4), ("partitioned", nn, nn),
             ("fulljoin", nn, nn)]
    _check(pkg, oracle, rp, sp, plans)
