"""GPU parity at BASELINE sizes.

* cfg1 (two-path self-join, 200k tuples) in full, against the checksum of the
  REFERENCE's own full output (tests/golden/cfg1_reference.json, 387,365,144
  codes, made by make_golden.py --cfg1) and its stats;
* cfg2 (5M + 5M two-path, 128,713,977,893 output tuples) through the exact
  engine bench.py times: |OUT|, per-chunk checksums equal to the three-kernel
  tail, and the boundary rows of every chunk vs the oracle (pi(sigma_X R join
  S) = sigma_X pi(R join S), compared in raw-value space);
* cfg3 (3 x 300k star) x1-slices vs the oracle; cfg4 (SSJ, 2M pairs, c=4)
  set-slices vs the oracle; cfg5 (BSI) at full scale and at 1/8 scale vs
  the oracle on every query.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _checksum(codes):
    u = np.asarray(codes, dtype=np.int64).view(np.uint64)
    return {"n": int(len(u)), "sum": int(u.sum(dtype=np.uint64)),
            "wsum": int((u * (np.arange(len(u), dtype=np.uint64) + np.uint64(1))).sum(dtype=np.uint64))}


@pytest.fixture(scope="module")
def cfg1():
    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.relation import Relation, build_indexed
    with open(os.path.join(GOLDEN, "cfg1_reference.json")) as f:
        ref = json.load(f)
    r = build_indexed(Relation.from_raw_pairs("R", datagen.config("cfg1").relations[0]))
    return r, ref


def test_cfg1_full_default_plan_matches_reference(cfg1):
    from paper_2002_12459_b200.joinproject import two_path_join
    r, ref = cfg1
    res = two_path_join(r, r)
    p = res.stats["plan"]
    assert [p.strategy, p.delta1, p.delta2] == ref["plan"]
    assert res.stats["light_intermediate"] == ref["light_intermediate"]
    assert res.stats["heavy_pairs"] == ref["heavy_pairs"]
    ck = _checksum(res.codes)
    assert ck == {k: ref["checksum"][k] for k in ("n", "sum", "wsum")}
    assert res.codes[ref["checksum"]["sample_idx"]].tolist() == ref["checksum"]["sample"]


def test_cfg1_full_gpu_plan_same_output(cfg1):
    from paper_2002_12459_b200.joinproject import two_path_join
    from paper_2002_12459_b200.optimizer import gpu_plan
    r, ref = cfg1
    res = two_path_join(r, r, plan=gpu_plan(r, r))
    assert _checksum(res.codes) == {k: ref["checksum"][k] for k in ("n", "sum", "wsum")}


def _raw_pairs_of(codes, dz, lv_x, lv_z):
    return np.stack([np.asarray(lv_x)[codes // dz], np.asarray(lv_z)[codes % dz]], axis=1)


def test_cfg2_bench_configuration_exact(oracle, monkeypatch):
    """The exact engine bench.py times on cfg2 (gpu_plan, 16384-row chunks,
    asynchronous chunks, the one-kernel tail k_merge_emit, all 31 chunks):
      * |OUT| = 128,713,977,893 (bench.CFG2_OUT) and every chunk strictly
        increasing, chunks in code order;
      * per-chunk sizes and order-sensitive 64-bit checksums equal to the
        three-kernel tail's (k_tile_merge -> scan -> k_emit_pf16) and to the
        fused tail fed by the tcgen05 heavy product instead of the in-tile
        OR of heavy-y bit rows;
      * the first and last 3 x of EVERY chunk (186 rows, each covering all
        column blocks / tile boundaries of its row) equal the oracle's
        sigma_X two-path, compared in raw-value space.
    Reference: joinproject.py:155-225."""
    import torch

    import bench
    from paper_2002_12459_b200 import _native as nat
    args = bench._args(["--config", "cfg2"])
    wl = bench.TwoPath(args, 0, 1)
    wl.setup()
    r, s = wl.r, wl.s
    dz = s.rel.dom_left
    st = nat.stream_handle

    def run(one_kernel, heavy=""):
        monkeypatch.setenv("MMJ_HEAVY", heavy)
        eng = wl.engine()
        eng.one_kernel_tail = one_kernel
        eng.prepare()
        assert eng.chunk_rows == 16384
        assert eng.heavy_kernel == (heavy or "or")      # the bench's default: the in-tile OR
        sizes, sums, rows = [], [], {}
        prev = -1
        for a, b in eng.chunk_bounds(wl.x_lo, wl.x_hi):
            ch = eng.run_chunk(a, b, sync=False)          # bench.TwoPath.step's call
            n = int(ch.total_dev.item())
            c = ch.codes[:n]
            if n > 1:
                assert bool((c[1:] > c[:-1]).all().item())
            if n:
                assert int(c[0].item()) > prev
                prev = int(c[-1].item())
            acc = torch.zeros(2, dtype=torch.int64, device="cuda")
            nat.call("mmj_code_checksum", nat.ptr(c), n, 0, nat.ptr(acc), st())
            sizes.append(n)
            sums.append(tuple(acc.cpu().tolist()))
            if one_kernel:
                cut = torch.tensor([(a + 3) * dz, (b - 3) * dz], dtype=torch.int64, device="cuda")
                i0, i1 = (int(v) for v in torch.searchsorted(c, cut).cpu())
                rows[(a, b)] = (c[:i0].cpu().numpy(), c[i1:].cpu().numpy())
        stats = eng.finish()
        return sizes, sums, rows, stats

    sizes, sums, rows, stats = run(True)
    assert len(sizes) == 31 and sum(sizes) == bench.CFG2_OUT == stats.out_size
    sizes3, sums3, _, stats3 = run(False)
    assert sizes3 == sizes and sums3 == sums
    assert (stats3.light_intermediate, stats3.heavy_pairs) == (stats.light_intermediate, stats.heavy_pairs)
    # the same chunks with the heavy part from the tcgen05 product (an
    # independent computation of the heavy cells): identical output and stats
    sizes_m, sums_m, _, stats_m = run(True, "mma")
    assert sizes_m == sizes and sums_m == sums
    assert (stats_m.light_intermediate, stats_m.heavy_pairs) == (stats.light_intermediate, stats.heavy_pairs)
    # oracle on the 6 boundary rows of every chunk, one sigma_X join
    lv_r, lv_s = np.asarray(r.rel.left_values), np.asarray(s.rel.left_values)
    xs = np.concatenate([np.r_[a:a + 3, b - 3:b] for a, b in rows])
    got = np.concatenate([np.concatenate(v) for v in rows.values()])
    Rraw, Sraw = wl.Rraw, wl.Sraw
    A, B = oracle.semi_join_many([oracle.encode(Rraw[np.isin(Rraw[:, 0], lv_r[xs])]), oracle.encode(Sraw)])
    exp = oracle.two_path(A, B, None)
    g = np.stack([lv_r[got // dz], lv_s[got % dz]], axis=1)
    e = np.stack([np.asarray(A.left_values)[exp.codes // exp.dims[1]],
                  np.asarray(B.left_values)[exp.codes % exp.dims[1]]], axis=1)
    gk = np.sort(g[:, 0] * (1 << 31) + g[:, 1])
    ek = np.sort(e[:, 0] * (1 << 31) + e[:, 1])
    assert len(gk) > 4e7 and np.array_equal(gk, ek)


def test_cfg3_star_x1_slices(oracle):
    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.joinproject import star_join
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce_many
    wl = datagen.config("cfg3")
    # x1-slice: restrict R1 to a few x1 values (the output restricted to those x1)
    raws = wl.relations
    xs = np.unique(raws[0][:, 0])[[0, 1, 2500, 4999]]
    r0 = raws[0][np.isin(raws[0][:, 0], xs)]
    rels = semi_join_reduce_many([Relation.from_raw_pairs("R0", r0)] +
                                 [Relation.from_raw_pairs(f"R{j}", raws[j]) for j in (1, 2)])
    idxs = [build_indexed(x) for x in rels]
    got = star_join(idxs, 100, 1, heavy_rows_cap=1 << 40)
    orels = oracle.semi_join_many([oracle.encode(r0), oracle.encode(raws[1]), oracle.encode(raws[2])])
    # the reference algorithm itself: heavy part as the Khatri-Rao x W^T float64
    # product over y heavy in >= 2 relations, light sub-joins + diamonds
    exp = oracle.star(orels, 100, 1, cap=1 << 40)
    assert np.array_equal(got.codes, exp.codes)
    assert len(exp.codes) == len(xs) * 5000 * 5000     # every x1 reaches the whole 5k x 5k square


def test_cfg4_ssj_set_slices(oracle):
    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.apps import SetFamily, ssj_mmjoin_arrays
    from paper_2002_12459_b200.relation import Relation
    pairs = datagen.config("cfg4").relations[0]
    fam = SetFamily(Relation.from_raw_pairs("sets", pairs))
    a, b, n = ssj_mmjoin_arrays(fam, 4)
    assert len(a) > 1e8 and np.all(a < b) and np.all(n >= 4)
    code = a * fam.relation.dom_left + b
    assert np.all(np.diff(code) > 0)
    # slice check: pairs whose smaller set is one of a few sets, vs the oracle
    # two-path of (sigma_{a in A'} family) x family with counts
    lv = np.asarray(fam.relation.left_values)
    for sl in ([0, 1, 2], [50000, 50001], [int(lv.size) - 3, int(lv.size) - 1]):
        raws = lv[sl]
        sub = pairs[np.isin(pairs[:, 0], raws)]
        A, B = oracle.semi_join_many([oracle.encode(sub), oracle.encode(pairs)])
        res = oracle.two_path(A, B, None, want_counts=True)
        t = res.tuples()
        ra = np.asarray(A.left_values)[t[:, 0]]
        rb = np.asarray(B.left_values)[t[:, 1]]
        keep = (ra < rb) & (res.counts >= 4)      # raw set ids are the dense ids' order (sorted input)
        exp = set(zip(ra[keep].tolist(), rb[keep].tolist(), res.counts[keep].tolist()))
        m = np.isin(lv[a], raws)
        got = set(zip(lv[a[m]].tolist(), lv[b[m]].tolist(), n[m].tolist()))
        assert got == exp


def test_cfg5_bsi_full_scale_all_queries(oracle):
    """cfg5 at BASELINE size (64M + 64M tuples, the 4M-query batch plus 4096
    queries with ids no relation holds): every answer equals the oracle's
    per-query set intersection (apps.py:314-351 restated), None markers
    included; relations ingested on the device as bench.py does."""
    import torch

    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.apps import bsi_answer_batch_arrays
    from paper_2002_12459_b200.ingest import from_raw_pairs_device
    wl = datagen.config("cfg5")
    raws = [torch.from_numpy(np.ascontiguousarray(x, dtype=np.int64)) for x in wl.relations]
    r = from_raw_pairs_device("R", raws[0])
    s = from_raw_pairs_device("S", raws[1])
    rng = np.random.default_rng(5)
    extra = rng.integers(0, 4_000_000, (4096, 2))
    extra[::2, 0] += 4_000_000          # unknown x
    extra[1::4, 1] = -7 - extra[1::4, 1]  # unknown z
    q = np.concatenate([wl.batch, extra])
    exp = oracle.bsi(oracle.encode(wl.relations[0]), oracle.encode(wl.relations[1]), q[:, 0], q[:, 1])
    for form in ("auto", "walk", "records"):      # auto = the bench's "lists" form (span tables) at cfg5
        got = bsi_answer_batch_arrays(r, s, q[:, 0], q[:, 1], form=form)
        assert np.array_equal(got, exp), form
    assert (exp[-4096:] == -1).sum() >= 2048 and 0.55 < (exp[:-4096] == 1).mean() < 0.7


def test_cfg5_bsi_eighth_scale_all_queries(oracle):
    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.apps import bsi_answer_batch_arrays
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce
    wl = datagen.config("cfg5", scale=0.125)
    R, S = semi_join_reduce(Relation.from_raw_pairs("R", wl.relations[0]), Relation.from_raw_pairs("S", wl.relations[1]))
    # "known" ids follow the UNREDUCED relations (apps.py:324-325)
    r0 = build_indexed(Relation.from_raw_pairs("R", wl.relations[0]))
    s0 = build_indexed(Relation.from_raw_pairs("S", wl.relations[1]))
    q = wl.batch
    got = bsi_answer_batch_arrays(r0, s0, q[:, 0], q[:, 1])
    exp = oracle.bsi(oracle.encode(wl.relations[0]), oracle.encode(wl.relations[1]), q[:, 0], q[:, 1])
    assert np.array_equal(got, exp)
    assert 0.5 < (exp == 1).mean() < 0.75
    del R, S
