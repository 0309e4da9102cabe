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
