"""GPU parity of the one-kernel projection tail (mmj_merge_emit: light merge,
segment scan, decoupled look-back and emission in one kernel) against the CPU
oracle and against the three-kernel path (tile merge -> scan -> emission).

The wide-row cases make a row span several column-block tiles (dom_z >
8192 * 32), so the precomputed list split tables and the look-back across
many tiles are exercised; bit-exact codes and identical light statistics.
"""

import numpy as np
import pytest

from conftest import zipf_pairs

pytestmark = pytest.mark.gpu


def _rels(r_pairs, s_pairs):
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce
    R, S = semi_join_reduce(Relation.from_raw_pairs("R", r_pairs), Relation.from_raw_pairs("S", s_pairs))
    return build_indexed(R), build_indexed(S)


def _wide(seed, nx, nr, nz, ns, dom_y, s_exp):
    rng = np.random.default_rng(seed)
    r_pairs = zipf_pairs(rng, nr, nx, dom_y, s_exp)            # (x, y)
    s_zy = zipf_pairs(rng, ns, nz, dom_y, s_exp)               # (z, y)
    return r_pairs, s_zy


@pytest.mark.parametrize("heavy", ["mma", "or"])
@pytest.mark.parametrize("plan", [("partitioned", 40, 1), ("partitioned", 8, 3), ("fulljoin", 0, 0)])
def test_wide_rows_match_oracle(oracle, plan, heavy, monkeypatch):
    from paper_2002_12459_b200.joinproject import two_path_join
    from paper_2002_12459_b200.optimizer import ThresholdPlan
    monkeypatch.setenv("MMJ_HEAVY", heavy)   # tcgen05 product / in-tile OR of heavy-y bit rows
    r_pairs, s_pairs = _wide(71, 32, 4_000, 3_000_000, 1_000_000, 3000, 1.1)
    r, s = _rels(r_pairs, s_pairs)
    assert s.rel.dom_left > 3 * 8192 * 32     # four column blocks per row (dom_z ~ 790k)
    strategy, d1, d2 = plan
    if strategy == "fulljoin":
        d1 = d2 = max(r.n, s.n)
    got = two_path_join(r, s, plan=ThresholdPlan(strategy, d1, d2))
    orr, oss = oracle.semi_join_many([oracle.encode(r_pairs), oracle.encode(s_pairs)])
    exp = oracle.two_path(orr, oss, oracle.OPlan(strategy, d1, d2))
    assert np.array_equal(got.codes, exp.codes)
    for key in ("light_intermediate", "heavy_pairs", "intermediate"):
        if key in exp.stats:
            assert got.stats[key] == exp.stats[key], key


def test_fused_equals_three_kernel_path_on_cfg2_chunks():
    """cfg2 (dom_z ~ 500k: two column blocks per row) chunk by chunk: the
    fused kernel's codes equal the three-kernel path's, for the first, a
    middle and the last 2048-row chunk."""
    import torch

    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.device import device_relation
    from paper_2002_12459_b200.engine import TwoPathEngine
    from paper_2002_12459_b200.optimizer import gpu_plan
    wl = datagen.config("cfg2")
    r, s = _rels(wl.relations[0], wl.relations[1])
    plan = gpu_plan(r, s)
    dr, ds = device_relation(r), device_relation(s)
    eng = TwoPathEngine(dr, ds, plan.strategy, plan.delta1, plan.delta2, False, chunk_rows=2048,
                        host_left_deg_r=r.left_deg, host_left_deg_s=s.left_deg)
    assert eng.one_kernel_tail
    eng.prepare()
    bounds = list(eng.chunk_bounds(0, r.rel.dom_left))
    for x0, x1 in (bounds[0], bounds[len(bounds) // 2], bounds[-1]):
        w0 = int(eng.wit.item())
        fused = eng.run_chunk(x0, x1, sync=False, codes_key="fa")
        n = int(fused.total_dev.item())
        fused_codes = fused.codes[:n].clone()
        w1 = int(eng.wit.item())
        eng.one_kernel_tail = False
        three = eng.run_chunk(x0, x1, sync=True, codes_key="fb")
        eng.one_kernel_tail = True
        w2 = int(eng.wit.item())
        assert three.n == n > 0
        assert torch.equal(fused_codes, three.codes)
        assert w1 - w0 == w2 - w1 == three.light
