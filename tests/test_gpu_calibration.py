"""Calibration on the tcgen05 kernel: the measured
table is monotone and round-trips; re-measured GPU costs drive gpu_plan to a
valid plan whose output is bit-identical to the oracle's."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_calibrate_on_device(tmp_path):
    from paper_2002_12459_b200.matmul import CalibrationTable, calibrate, estimate_runtime
    t = calibrate((256, 1024, 2048), cores=(1, 2), runs=3)
    assert set(t.entries) == {(p, c) for p in (256, 1024, 2048) for c in (1, 2)}
    for c in (1, 2):
        v = [t.entries[(p, c)] for p in (256, 1024, 2048)]
        assert all(x > 0 for x in v) and v == sorted(v)
    path = tmp_path / "cal.tsv"
    t.save(path)
    assert CalibrationTable.load(path).entries == t.entries
    assert estimate_runtime(t, 4096, 4096, 4096) > t.entries[(2048, 1)]


def test_measured_gpu_costs_drive_the_plan(oracle):
    from conftest import zipf_pairs
    from paper_2002_12459_b200.joinproject import two_path_join
    from paper_2002_12459_b200.optimizer import gpu_plan, measure_gpu_costs
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce
    costs = measure_gpu_costs()
    assert 0 < costs.witness_s_bitmap < 1e-6 and 0 < costs.witness_s_count < 1e-6
    assert 0 < costs.cell_s < 1e-9 and 0 < costs.cell_k_s < 1e-11
    rng = np.random.default_rng(3)
    rp = np.array(zipf_pairs(rng, 40000, 2000, 1500, 1.1))
    sp = np.array(zipf_pairs(rng, 40000, 1800, 1500, 1.1))
    a, b = semi_join_reduce(Relation.from_raw_pairs("R", rp), Relation.from_raw_pairs("S", sp))
    r, s = build_indexed(a), build_indexed(b)
    plan = gpu_plan(r, s, costs=costs)
    plan.validate()
    got = two_path_join(r, s, plan=plan)
    OR, OS = oracle.semi_join_many([oracle.encode(rp), oracle.encode(sp)])
    assert np.array_equal(got.codes, oracle.two_path(OR, OS, None).codes)
