"""Cost-based planner against outputs frozen from
the REFERENCE planner (tests/golden/planner.json, made by make_golden.py
gen_planner): DegreeStats queries, modeled_costs, optimize_thresholds and
estimate_runtime on fixed inputs and synthetic calibration tables; plus the
calibration table's TSV round trip and the GPU planner's argmin."""

import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLDEN, "planner.json")) as f:
        meta = json.load(f)
    arrays = np.load(os.path.join(GOLDEN, "planner.npz"))
    return meta, arrays


def _tables():
    from paper_2002_12459_b200.calibration import CalibrationTable
    return {"t1": CalibrationTable({(100, 1): 1_000, (200, 1): 8_000, (400, 1): 64_000}),
            "t2": CalibrationTable({(16, 1): 10, (32, 1): 90, (64, 1): 700, (64, 2): 400, (128, 2): 3000})}


def _instance(arrays, i, self_join):
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce
    R = Relation.from_raw_pairs("R", arrays[f"p{i}_R"])
    if self_join:
        r = build_indexed(R)
        return r, r
    a, b = semi_join_reduce(R, Relation.from_raw_pairs("S", arrays[f"p{i}_S"]))
    return build_indexed(a), build_indexed(b)


def test_estimate_runtime_golden(golden):
    from paper_2002_12459_b200.calibration import estimate_runtime
    meta, _ = golden
    tabs = _tables()
    for row in meta["estimate_runtime"]:
        u, v, w, co = row["uvw_co"]
        assert estimate_runtime(tabs[row["table"]], u, v, w, co) == pytest.approx(row["nanos"], rel=1e-12)


def test_degree_stats_costs_and_sweep_golden(golden):
    from paper_2002_12459_b200 import optimizer as opt
    from paper_2002_12459_b200.relation import degree_stats
    meta, arrays = golden
    table = _tables()["t1"]
    for i, inst in enumerate(meta["instances"]):
        r, s = _instance(arrays, i, inst["self_join"])
        assert max(r.n, s.n) == inst["n"] and r.out_join_with(s) == inst["out_join"]
        st_r, st_s = degree_stats(r, partner=s), degree_stats(s)
        q = inst["stats"]
        for f in ("count_left", "count_right", "cdfx", "sum_y", "sum_x"):
            assert [getattr(st_r, f)(d) for d in q["deltas"]] == q["r"][f], (inst["name"], f)
            assert [getattr(st_s, f)(d) for d in q["deltas"]] == q["s"][f], (inst["name"], f)
        assert [st_r.max_left_deg, st_r.max_right_deg] == q["r_max"]
        assert [st_s.max_left_deg, st_s.max_right_deg] == q["s_max"]
        for c in inst["costs"]:
            d1, d2 = c["d"]
            got = opt.modeled_costs(st_r, st_s, r.rel.dom_left, d1, d2, opt.DEFAULT_COSTS, table)
            assert got == pytest.approx(tuple(c["cost"]), rel=1e-12)
        for p in inst["plans"]:
            kw = {"step": p["step"]} if "step" in p else {"consts": opt.CostConstants(*p["consts"])}
            pl = opt.optimize_thresholds(st_r, st_s, r.rel.dom_left, inst["out_join"], table=table, **kw)
            exp = p["plan"]
            assert [pl.strategy, pl.delta1, pl.delta2, pl.iterations] == [exp[0], exp[1], exp[2], exp[5]], inst["name"]
            assert (pl.light_cost, pl.heavy_cost) == pytest.approx((exp[3], exp[4]), rel=1e-12)


def test_optimizer_errors_and_cutoff(golden):
    from paper_2002_12459_b200 import optimizer as opt
    from paper_2002_12459_b200.calibration import CalibrationError
    from paper_2002_12459_b200.relation import degree_stats
    meta, arrays = golden
    z = meta["instances"][1]
    r, s = _instance(arrays, 1, False)
    st_r, st_s = degree_stats(r, partner=s), degree_stats(s)
    with pytest.raises(CalibrationError):
        opt.optimize_thresholds(st_r, st_s, r.rel.dom_left, z["out_join"])
    with pytest.raises(ValueError):
        opt.optimize_thresholds(st_r, st_s, r.rel.dom_left, z["out_join"], table=_tables()["t1"], step=1.5)
    pl = opt.optimize_thresholds(st_r, st_s, r.rel.dom_left, 15 * z["n"])
    assert pl.strategy == opt.FULL_JOIN and pl.iterations == 0
    with pytest.raises(ValueError):
        opt.CostConstants(T_s=0.0).validate()
    c = opt.measure_cost_constants(n=20_000)
    assert c.T_s > 0 and c.T_m > 0 and c.T_I > 0
    with pytest.raises(ValueError):
        degree_stats(r, partner=_instance(arrays, 2, True)[0])


def test_calibration_table_tsv(tmp_path):
    from paper_2002_12459_b200.calibration import CalibrationError, CalibrationTable, estimate_runtime
    t = CalibrationTable({(64, 1): 500, (32, 1): 900, (128, 1): 4000, (64, 2): 300})
    t.regularize()
    assert t.entries[(32, 1)] <= t.entries[(64, 1)] <= t.entries[(128, 1)]
    path = tmp_path / "cal.tsv"
    t.save(path)
    assert path.read_text().startswith("# mmjoin-calibration v1\n")
    assert CalibrationTable.load(path).entries == t.entries
    bad = tmp_path / "bad.tsv"
    bad.write_text("not a calibration file\n")
    with pytest.raises(CalibrationError):
        CalibrationTable.load(bad)
    with pytest.raises(CalibrationError):
        estimate_runtime(CalibrationTable(), 1, 1, 1)


def test_gpu_plan_is_model_argmin(golden):
    from paper_2002_12459_b200 import optimizer as opt
    meta, arrays = golden
    r, s = _instance(arrays, 1, False)
    costs = opt.GpuCosts(witness_s_bitmap=3e-11, witness_s_count=2e-10, cell_s=1e-13, cell_k_s=4e-16)
    pl = opt.gpu_plan(r, s, costs=costs)
    rd, sd = np.asarray(r.right_deg), np.asarray(s.right_deg)
    u, w = int((np.asarray(r.left_deg) > 1).sum()), int((np.asarray(s.left_deg) > 1).sum())

    def model(d1):
        light = (rd <= d1) & (sd <= d1)
        k = int((~light).sum())
        kp = -(-k // 128) * 128
        return int((rd * sd)[light].sum()) * costs.witness_s_bitmap + costs.heavy_seconds(u, kp, w)
    cand = sorted(set(np.maximum(rd, sd).tolist()) | {1})
    best = min(model(d) for d in cand)
    assert pl.strategy == opt.PARTITIONED and pl.delta2 == 1
    assert math.isclose(pl.total_cost, best, rel_tol=1e-9)


def test_star_threshold_is_model_argmin():
    """star.choose_threshold returns the product-degree cut whose modelled
    time (light witnesses + per-heavy-y product + K-independent read-out) is
    smallest among the 128-aligned heavy-y counts; the heavy set it induces
    has exactly that many y."""
    import math

    from paper_2002_12459_b200 import star
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce_many
    rng = np.random.default_rng(12)
    raws = []
    for _ in range(3):
        y = np.minimum(rng.zipf(1.3, 40000), 3000) - 1
        raws.append(np.unique(np.stack([rng.integers(0, 400, 40000), y], axis=1), axis=0))
    idxs = [build_indexed(r) for r in semi_join_reduce_many(
        [Relation.from_raw_pairs(f"R{j}", p) for j, p in enumerate(raws)])]
    thr = star.choose_threshold(idxs)
    prod = np.stack([np.asarray(r.right_deg, dtype=np.float64) for r in idxs]).prod(axis=0)
    order = np.sort(prod[prod > 0])[::-1]
    cells = float(math.prod(r.rel.dom_left for r in idxs))

    def model(k):
        ke = min(k, len(order))
        return (order[ke:].sum() / star.LIGHT_RATE + 2.0 * cells * (-(-ke // 128) * 128) / star.MMA_RATE
                + cells / star.CELL_RATE)
    cands = [order.sum() / star.LIGHT_RATE] + [model(k) for k in range(128, min(len(order), 8192) + 128, 128)]
    k_chosen = int((prod > thr).sum()) if math.isfinite(thr) else 0
    t_chosen = model(k_chosen) if k_chosen else order.sum() / star.LIGHT_RATE
    # y tied with the cut value stay light, so the heavy count may fall a few short of the 128-aligned optimum
    assert t_chosen <= min(cands) * 1.02


def test_ssj_host_compaction_plan_is_remembered():
    """apps._compact_host_plan: kept-set count, CSR offsets and degrees from
    the family's frozen degree vector, remembered per (family, c)."""
    from paper_2002_12459_b200.apps import SetFamily, _compact_host_plan
    from paper_2002_12459_b200.relation import Relation
    rng = np.random.default_rng(3)
    pairs = np.unique(np.stack([np.minimum(rng.zipf(1.5, 5000), 300), rng.integers(0, 200, 5000)], axis=1), axis=0)
    idx = SetFamily(Relation.from_raw_pairs("sets", pairs)).indexed
    nk, ptr, hdeg = _compact_host_plan(idx, 3)
    ldeg = np.asarray(idx.left_deg)
    assert nk == int((ldeg >= 3).sum()) and np.array_equal(hdeg, ldeg[ldeg >= 3])
    assert np.array_equal(ptr, np.concatenate([[0], np.cumsum(ldeg[ldeg >= 3])]))
    assert not ptr.flags.writeable and not hdeg.flags.writeable
    assert _compact_host_plan(idx, 3)[1] is ptr            # remembered
    nk5, ptr5, _ = _compact_host_plan(idx, 5)              # another c replaces it
    assert nk5 == int((ldeg >= 5).sum()) and ptr5 is not ptr
