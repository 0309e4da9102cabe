"""Pin the CPU oracle (oracle/mmjoin_oracle.py) to the reference.

Every fixture under tests/golden/ was produced by the reference package itself
(tests/golden/make_golden.py); the oracle must reproduce each bit-exactly.
CPU only.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

from oracle import mmjoin_oracle as o


def _load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def _plan(p):
    st, d1, d2 = p
    return None if st == "default" else o.OPlan(st, int(d1), int(d2))


@pytest.fixture(scope="module")
def twopath():
    z = _load("twopath.npz")
    return z, json.loads(str(z["meta"]))


def test_twopath_fixtures(twopath):
    z, meta = twopath
    rels = {}
    for m in meta:
        i = m["inst"]
        if i not in rels:
            R = o.encode(z[f"i{i}_R"])
            if m["self_join"]:
                rels[i] = (R, R)
            else:
                rels[i] = tuple(o.semi_join_many([R, o.encode(z[f"i{i}_S"])]))
        r, s = rels[i]
        res = o.two_path(r, s, _plan(m["plan"]), want_counts=m["counts"])
        key = m["key"]
        assert list(res.dims) == m["dims"], key
        assert np.array_equal(res.codes, z[key + "_codes"]), key
        if m["counts"]:
            assert np.array_equal(res.counts, z[key + "_counts"]), key
        for k in ("light_intermediate", "heavy_pairs", "intermediate"):
            if k in m["stats"]:
                assert res.stats[k] == m["stats"][k], (key, k)
        if "plan" in m["stats"]:
            p = res.stats["plan"]
            assert [p.strategy, p.delta1, p.delta2] == m["stats"]["plan"], key


def test_example_fixture():
    with open(os.path.join(GOLDEN, "example.json")) as f:
        ex = json.load(f)
    R = o.encode([tuple(p) for p in ex["R"]])
    S = o.encode([tuple(p) for p in ex["S"]])
    r, s, lr, ls = o.partition(R, S, 2, 2)
    raw_r = np.array(r.raw_pairs(), dtype=object)
    raw_s = np.array(s.raw_pairs(), dtype=object)
    assert sorted(map(tuple, raw_r[lr].tolist())) == [tuple(p) for p in ex["light_R"]]
    assert sorted(map(tuple, raw_r[~lr].tolist())) == [tuple(p) for p in ex["heavy_R"]]
    assert sorted(map(tuple, raw_s[~ls].tolist())) == [tuple(p) for p in ex["heavy_S"]]
    m1, m2, hx, hy, hz = o.heavy_operands(r, s, 2, 2)
    o1 = np.argsort([r.left_values[i] for i in hx])
    om = np.argsort([r.right_values[i] for i in hy])
    o2 = np.argsort([s.left_values[i] for i in hz])
    a, b = m1[o1][:, om], m2[om][:, o2]
    assert a.tolist() == ex["M1"] and b.tolist() == ex["M2"]
    # the pinned product (reference test_joinproject.py:62; paper's (6,6)=3 is a transcription error)
    assert o.matmul_exact(a, b).tolist() == ex["product"] == [[1, 2, 1], [2, 3, 2], [2, 2, 1]]
    res = o.two_path(r, s, o.OPlan("partitioned", 2, 2), want_counts=True)
    t = res.tuples()
    got = {f"{r.left_values[x]},{s.left_values[zz]}": int(c) for (x, zz), c in zip(t.tolist(), res.counts.tolist())}
    assert got == ex["counts"]
    assert int(res.counts.sum()) == ex["out_join"] == o.out_join(r, s)
    T = o.encode([tuple(p) for p in ex["T"]])
    U = o.encode([tuple(p) for p in ex["U"]])
    st = o.star([T, U], 2, 2, want_counts=True)
    rels = o.ensure_reduced([T, U])
    got = {",".join(str(rels[i].left_values[v]) for i, v in enumerate(tt)): int(c)
           for tt, c in zip(st.tuples().tolist(), st.counts.tolist())}
    assert got == ex["star_TU_counts"]
    assert list(o.closed_form_thresholds(1000, 1000)) == ex["closed_form_1000_1000"] == [10, 10]


def test_star_fixtures():
    z = _load("star.npz")
    meta = json.loads(str(z["meta"]))
    for m in meta:
        i, k = m["inst"], m["k"]
        rels = o.semi_join_many([o.encode(z[f"s{i}_rel{j}"]) for j in range(k)])
        res = o.star(rels, m["d1"], m["d2"], want_counts=m["counts"])
        assert np.array_equal(res.codes, z[m["key"] + "_codes"]), m["key"]
        assert list(res.dims) == m["dims"]
        assert list(res.stats["heavy_dims"]) == m["heavy_dims"], m["key"]
        if m["counts"]:
            assert np.array_equal(res.counts, z[m["key"] + "_counts"]), m["key"]


def test_star_cap_error():
    rng = np.random.default_rng(11)
    rels = [o.encode(rng.integers(0, 12, (200, 2)) * np.array([1, 1]) % np.array([12, 6])) for _ in range(3)]
    rels = o.semi_join_many(rels)
    with pytest.raises(o.OracleStarCap):
        o.star(rels, 1, 1, cap=2)


def test_ssj_fixtures():
    z = _load("ssj.npz")
    meta = json.loads(str(z["meta"]))
    for m in meta:
        fam = o.encode(z[f"f{m['inst']}_pairs"])
        got = o.ssj(fam, m["c"])
        exp = {(int(a), int(b)): int(n) for a, b, n in z[m["key"]].tolist()}
        assert got == exp, m["key"]
        assert list(got) == list(exp), "insertion order = ascending code"


def test_bsi_fixtures():
    z = _load("bsi.npz")
    meta = json.loads(str(z["meta"]))
    for m in meta:
        i = m["inst"]
        R, S = o.encode(z[f"b{i}_R"]), o.encode(z[f"b{i}_S"])
        q = z[f"b{i}_batch"]
        ans = o.bsi(R, S, q[:, 0], q[:, 1])
        assert np.array_equal(ans, z[f"b{i}_ans"]), i


def test_matmul_fixtures():
    z = _load("matmul.npz")
    for i in range(12):
        a, b = z[f"m{i}_a"], z[f"m{i}_b"]
        assert np.array_equal(o.matmul_exact(a, b), z[f"m{i}_p"])
        assert np.array_equal(o.matmul_exact(a, b, "int64"), z[f"m{i}_p"])


def test_matmul_errors():
    big = np.array([[2 ** 62]], dtype=np.int64)
    with pytest.raises(o.OracleOverflow):
        o.matmul_exact(big, big)
    v = np.array([[2 ** 31]], dtype=np.int64)
    with pytest.raises(o.OracleOverflow):
        o.matmul_exact(v, v, "blas")
    assert o.matmul_exact(v, v, "int64")[0, 0] == 2 ** 62
    with pytest.raises(ValueError):
        o.matmul_exact(np.ones((2, 3), np.int64), np.ones((4, 2), np.int64))


def test_plan_constants():
    with open(os.path.join(GOLDEN, "plans.json")) as f:
        p = json.load(f)
    for row in p["closed_form"]:
        assert list(o.closed_form_thresholds(row["n"], row["est"])) == row["closed"]
    for row in p["estimate"]:
        assert o.estimate_output_size(row["dom_x"], row["out_join"], row["n"]) == row["est"]


def test_cfg1_reference_checksum_pins_oracle_stats():
    """Full-size cfg1 statistics frozen from the reference: the oracle's
    degree-only counters (plan, light intermediate) must agree exactly."""
    path = os.path.join(GOLDEN, "cfg1_reference.json")
    if not os.path.exists(path):
        pytest.skip("cfg1 reference fixture not generated")
    with open(path) as f:
        ref = json.load(f)
    from paper_2002_12459_b200 import datagen
    R = o.encode(datagen.config("cfg1").relations[0])
    plan = o.default_plan(R, R)
    assert [plan.strategy, plan.delta1, plan.delta2] == ref["plan"]
    # light intermediate = sum over R tuples of their list lengths (degree arithmetic)
    ly, lx, lz = o.light_masks(R, R, plan.delta1, plan.delta2)
    rd = R.right_deg
    x, y = R.pairs[:, 0], R.pairs[:, 1]
    p1 = int((rd[y] * ly[y]).sum())
    p2 = int((rd[y] * (lx[x] & ~ly[y])).sum())
    hx_per_y = np.bincount(y[~lx[x]], minlength=R.dom_right)
    p3 = int((hx_per_y[y] * (lz[x] & ~ly[y])).sum())
    assert p1 + p2 + p3 == ref["light_intermediate"]
