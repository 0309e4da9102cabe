"""GPU parity for the applications: SSJ / SCJ on the exact count path and
batched boolean set intersection, against reference-frozen fixtures and the
oracle (bit-exact: same pairs, same overlap counts, same True/False/None)."""

import json
import os

import numpy as np
import torch
import pytest

from conftest import GOLDEN, random_pairs, zipf_pairs

pytestmark = pytest.mark.gpu


def test_ssj_golden():
    from paper_2002_12459_b200.apps import SetFamily, scj_join_project, ssj_mmjoin
    from paper_2002_12459_b200.relation import Relation
    z = np.load(os.path.join(GOLDEN, "ssj.npz"))
    meta = json.loads(str(z["meta"]))
    fams = {}
    for m in meta:
        i = m["inst"]
        if i not in fams:
            fams[i] = SetFamily(Relation.from_raw_pairs("sets", z[f"f{i}_pairs"]))
        got = ssj_mmjoin(fams[i], m["c"])
        exp = {(int(a), int(b)): int(n) for a, b, n in z[m["key"]].tolist()}
        assert got == exp, m["key"]
        assert list(got) == list(exp)
    for i, fam in fams.items():
        assert sorted(scj_join_project(fam)) == [tuple(p) for p in z[f"f{i}_scj"].tolist()]


def test_ssj_threshold_validation():
    from paper_2002_12459_b200.apps import SetFamily, ssj_mmjoin
    fam = SetFamily.from_dict({"a": [1]})
    with pytest.raises(ValueError):
        ssj_mmjoin(fam, 0)


@pytest.mark.parametrize("c", [1, 3, 6])
def test_ssj_zipf_family_vs_oracle(oracle, c):
    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.apps import SetFamily, ssj_mmjoin_arrays
    from paper_2002_12459_b200.optimizer import PARTITIONED, ThresholdPlan
    from paper_2002_12459_b200.relation import Relation
    pairs = datagen.set_family_pairs(9, 30000, 2000, 300, 1.5, 800, 1.1)
    fam = SetFamily(Relation.from_raw_pairs("sets", pairs))
    ofam = oracle.encode(pairs)
    ea, eb, en = oracle.ssj_arrays(ofam, c)
    for plan in (None, ThresholdPlan(PARTITIONED, 26, 26), ThresholdPlan(PARTITIONED, 200, 1)):
        a, b, n = ssj_mmjoin_arrays(fam, c, plan=plan, chunk_rows=256)
        assert np.array_equal(a, ea) and np.array_equal(b, eb) and np.array_equal(n, en)


@pytest.mark.parametrize("c", [2, 4])
def test_ssj_compaction_matches_full_matrix(oracle, c):
    """Sets smaller than c dropped and the rest renumbered before the count
    join (mmj_compact_rows), codes mapped back (mmj_decode_compact_codes):
    identical arrays to the uncompacted count matrix and to the oracle."""
    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.apps import SetFamily, _compact_family, _ssj_device, _split
    from paper_2002_12459_b200.relation import Relation
    pairs = datagen.set_family_pairs(5, 40000, 4000, 400, 1.5, 1500, 1.1)
    fam = SetFamily(Relation.from_raw_pairs("sets", pairs))
    comp = _compact_family(fam.indexed, c)
    assert comp is not None, "the Zipf(1.5) family has a large share of sets below c"
    dc, orig, hdeg = comp
    ldeg = np.asarray(fam.indexed.left_deg)
    assert dc.dom_left == int((ldeg >= c).sum()) and dc.n == int(ldeg[ldeg >= c].sum())
    assert np.array_equal(orig.cpu().numpy(), np.flatnonzero(ldeg >= c))
    assert np.array_equal(dc.left_deg.cpu().numpy(), hdeg)
    # both CSR directions of the compacted family vs a host rebuild
    idx = fam.indexed
    rows = np.repeat(np.arange(len(ldeg)), ldeg)
    kept = ldeg[rows] >= c
    new_id = np.cumsum(ldeg >= c) - 1
    r2, y2 = new_id[rows[kept]], np.asarray(idx.fwd_indices)[kept]
    assert np.array_equal(dc.fwd_row.cpu().numpy(), r2) and np.array_equal(dc.fwd_idx.cpu().numpy(), y2)
    assert np.array_equal(dc.fwd_ptr.cpu().numpy(), dc.fwd_ptr_host)
    order = np.lexsort((r2, y2))
    rdeg = np.bincount(y2, minlength=dc.dom_right)
    assert np.array_equal(dc.rev_idx.cpu().numpy(), r2[order])
    assert np.array_equal(dc.right_deg.cpu().numpy(), rdeg)
    assert np.array_equal(dc.rev_ptr.cpu().numpy(), np.concatenate([[0], np.cumsum(rdeg)]))
    got = _ssj_device(fam, c, None, 512, compact=True)
    ref = _ssj_device(fam, c, None, 512, compact=False)
    assert torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1])
    a, b = _split(got[0].cpu().numpy(), fam.relation.dom_left)
    ea, eb, en = oracle.ssj_arrays(oracle.encode(pairs), c)
    assert np.array_equal(a, ea) and np.array_equal(b, eb) and np.array_equal(got[1].cpu().numpy(), en)


def test_ssj_compaction_edges(oracle):
    """c above every set size (nothing kept), c = 1 (no compaction), a family
    where every set survives: same arrays as the oracle."""
    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.apps import SetFamily, _compact_family, ssj_mmjoin_arrays
    from paper_2002_12459_b200.relation import Relation
    pairs = datagen.set_family_pairs(7, 6000, 800, 60, 1.5, 300, 1.1)
    fam = SetFamily(Relation.from_raw_pairs("sets", pairs))
    big = int(np.asarray(fam.indexed.left_deg).max()) + 1
    assert _compact_family(fam.indexed, big) is None
    a, b, n = ssj_mmjoin_arrays(fam, big)
    assert len(a) == len(b) == len(n) == 0
    for c in (1, 2, 5):
        ea, eb, en = oracle.ssj_arrays(oracle.encode(pairs), c)
        a, b, n = ssj_mmjoin_arrays(fam, c)
        assert np.array_equal(a, ea) and np.array_equal(b, eb) and np.array_equal(n, en)


def test_compact_abi_errors():
    from paper_2002_12459_b200 import _native as nat
    nat.require_cuda()
    lib = nat.load()
    assert lib.mmj_compact_rows(*([0] * 6), 0, 0, 0, -1, *([0] * 11), 0, 0) == nat.MMJ_ERR_ARG
    assert lib.mmj_decode_compact_codes(0, 1, 0, 0, 0, 10, 0, 0) == nat.MMJ_ERR_ARG


def test_bsi_golden():
    from paper_2002_12459_b200.apps import bsi_answer_batch, bsi_answer_batch_arrays
    from paper_2002_12459_b200.relation import Relation, build_indexed
    z = np.load(os.path.join(GOLDEN, "bsi.npz"))
    meta = json.loads(str(z["meta"]))
    for m in meta:
        i = m["inst"]
        r = build_indexed(Relation.from_raw_pairs("R", z[f"b{i}_R"]))
        s = build_indexed(Relation.from_raw_pairs("S", z[f"b{i}_S"]))
        q = z[f"b{i}_batch"]
        got = bsi_answer_batch_arrays(r, s, q[:, 0], q[:, 1])
        assert np.array_equal(got, z[f"b{i}_ans"]), i
        lst = bsi_answer_batch(r, s, [tuple(p) for p in q.tolist()])
        assert lst == [None if v < 0 else bool(v) for v in z[f"b{i}_ans"].tolist()]
    assert bsi_answer_batch(r, s, []) == []


def test_bsi_string_ids_and_heavy_bits(oracle):
    from paper_2002_12459_b200.apps import bsi_answer_batch
    from paper_2002_12459_b200.relation import Relation, build_indexed
    rng = np.random.default_rng(44)
    rp = [(f"a{a}", f"y{y}") for a, y in random_pairs(rng, 400, 50, 30)]
    sp = [(f"b{b}", f"y{y}") for b, y in random_pairs(rng, 400, 50, 30)]
    r = build_indexed(Relation.from_raw_pairs("R", rp))
    s = build_indexed(Relation.from_raw_pairs("S", sp))
    batch = [(f"a{int(a)}", f"b{int(b)}") for a, b in rng.integers(0, 55, (300, 2))]
    got = bsi_answer_batch(r, s, batch)
    radj, sadj = {}, {}
    for a, y in rp:
        radj.setdefault(a, set()).add(y)
    for b, y in sp:
        sadj.setdefault(b, set()).add(y)
    for (a, b), g in zip(batch, got):
        if a not in radj or b not in sadj:
            assert g is None
        else:
            assert g == bool(radj[a] & sadj[b])


def test_bsi_float_values_and_mixed_query_ids():
    """Raw values keep Python equality (apps.py:321-350): float y-values
    never collapse onto their integer part (R y 1.5 / 2.5 vs S y 1.7 share
    nothing), an integer-valued y equal to a float one (2 == 2.0) still
    matches, and query ids 5.0 / True resolve like dict.get while 5.5 and
    '5' are unknown (None)."""
    from paper_2002_12459_b200.apps import bsi_answer_batch
    from paper_2002_12459_b200.relation import Relation, build_indexed
    rng = np.random.default_rng(45)
    rp = [(int(a), float(y) + 0.5) for a, y in random_pairs(rng, 300, 40, 25)] + [(1, 1.5), (5, 2.0)]
    sp = [(int(b), float(y) + 0.7) for b, y in random_pairs(rng, 300, 40, 25)] + [(3, 1.7), (6, 2)]
    r = build_indexed(Relation.from_raw_pairs("R", rp))
    s = build_indexed(Relation.from_raw_pairs("S", sp))
    batch = [(int(a), int(b)) for a, b in rng.integers(0, 45, (200, 2))]
    batch += [(1, 3), (5, 6), (5.0, 6), (True, 3), (5.5, 6), ("5", 6), (5, 6.0)]
    got = bsi_answer_batch(r, s, batch)
    radj, sadj = {}, {}
    for a, y in rp:
        radj.setdefault(a, set()).add(y)
    for b, y in sp:
        sadj.setdefault(b, set()).add(y)
    for (a, b), g in zip(batch, got):
        if radj.get(a) is None or sadj.get(b) is None:
            assert g is None, (a, b)
        else:
            assert g == bool(radj[a] & sadj[b]), (a, b)
    assert got[-7:-4] == [False, True, True] and got[-3:-1] == [None, None]


@pytest.mark.parametrize("heavy_bits,form", [(128, "records"), (512, "records"), (256, "lists"), (256, "auto")])
def test_bsi_zipf_vs_oracle(oracle, heavy_bits, form):
    from paper_2002_12459_b200.apps import bsi_answer_batch_arrays
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce
    rng = np.random.default_rng(heavy_bits)
    rp = np.array(zipf_pairs(rng, 60000, 4000, 8000, 1.0))
    sp = np.array(zipf_pairs(rng, 60000, 4000, 8000, 1.0))
    q = rng.integers(0, 4100, (20000, 2))
    exp = oracle.bsi(oracle.encode(rp), oracle.encode(sp), q[:, 0], q[:, 1])
    # unshared dictionaries (mapped on the host) and pre-reduced shared ones
    r = build_indexed(Relation.from_raw_pairs("R", rp))
    s = build_indexed(Relation.from_raw_pairs("S", sp))
    got = bsi_answer_batch_arrays(r, s, q[:, 0], q[:, 1], heavy_bits=heavy_bits, form=form)
    assert np.array_equal(got, exp)
    assert (exp == -1).any() and (exp == 1).any() and (exp == 0).any()


@pytest.mark.parametrize("spread", [1, 1000])
def test_bsi_direct_table_vs_search(oracle, spread, monkeypatch):
    """Query ids resolved through the direct-address tables (dense raw id
    ranges) and through the binary search (DIRECT_SPREAD = 0, and ids spread
    x1000 so no table is built): identical answers, equal to the oracle."""
    from paper_2002_12459_b200 import bsi
    from paper_2002_12459_b200.apps import bsi_answer_batch_arrays
    from paper_2002_12459_b200.relation import Relation, build_indexed
    rng = np.random.default_rng(77 + spread)
    rp = np.array(zipf_pairs(rng, 40000, 3000, 6000, 1.0))
    sp = np.array(zipf_pairs(rng, 40000, 3000, 6000, 1.0))
    rp[:, 0] *= spread
    sp[:, 0] *= spread
    q = rng.integers(0, 3100, (15000, 2)) * spread
    q[::7] += 1     # ids between the spread values (unknown unless spread == 1)
    exp = oracle.bsi(oracle.encode(rp), oracle.encode(sp), q[:, 0], q[:, 1])
    r = build_indexed(Relation.from_raw_pairs("R", rp))
    s = build_indexed(Relation.from_raw_pairs("S", sp))
    for form in ("lists", "records"):
        got = bsi_answer_batch_arrays(r, s, q[:, 0], q[:, 1], form=form)
        assert np.array_equal(got, exp)
    monkeypatch.setattr(bsi, "DIRECT_SPREAD", 0)
    r._mmj_bsi_cache = None
    for form in ("lists", "records"):
        got2 = bsi_answer_batch_arrays(r, s, q[:, 0], q[:, 1], form=form)
        assert np.array_equal(got2, exp)


@pytest.mark.parametrize("max_bits,sig_bits", [(16, 32), (4, 32), (16, 0), (4, 5)])
def test_bsi_span_tables_vs_id_walk(oracle, max_bits, sig_bits, monkeypatch):
    """The lists form through the span tables (raw id -> list offset and
    length in one 32-bit entry) and through the id table + fwd_ptr walk:
    identical answers, equal to the oracle.  With 4 length bits the lists of
    15 or more y saturate the length field and take the fwd_ptr search."""
    from paper_2002_12459_b200 import bsi
    from paper_2002_12459_b200.apps import bsi_answer_batch_arrays
    from paper_2002_12459_b200.relation import Relation, build_indexed
    monkeypatch.setattr(bsi, "SPAN_MAX_LEN_BITS", max_bits)
    monkeypatch.setattr(bsi, "SIG_BITS", sig_bits)     # heavy-y signature width (0: lists only)
    rng = np.random.default_rng(90 + max_bits)

    def side(n_ids, seed):
        g = np.random.default_rng(seed)
        # short lists (mean ~3) plus a few ids with exactly 14, 15, 16 and 60 y; id 7 left out
        lens = g.integers(1, 6, n_ids)
        lens[[3, 11, 19, 40]] = [14, 15, 16, 60]
        rows = np.repeat(np.arange(n_ids), lens)
        ys = np.concatenate([g.choice(500, k, replace=False) for k in lens])
        keep = rows != 7
        p = np.stack([rows[keep] + 100, ys[keep]], axis=1)
        return p[g.permutation(len(p))]
    rp, sp = side(3000, 1), side(2500, 2)
    q = rng.integers(95, 3200, (30000, 2))
    q[:8] = [[103, 103], [111, 111], [119, 119], [140, 140], [111, 140], [107, 103], [103, 107], [3099, 2599]]
    exp = oracle.bsi(oracle.encode(rp), oracle.encode(sp), q[:, 0], q[:, 1])
    r = build_indexed(Relation.from_raw_pairs("R", rp))
    s = build_indexed(Relation.from_raw_pairs("S", sp))
    sides = bsi.prepare(r, s)
    assert sides[0].span is not None and sides[1].span is not None and sides[0].span[3] == max_bits
    for form in ("lists", "walk"):
        got = bsi_answer_batch_arrays(r, s, q[:, 0], q[:, 1], form=form)
        assert np.array_equal(got, exp), form
    assert (exp == -1).any() and (exp == 1).any() and (exp == 0).any()
    assert exp[5] == -1 and exp[6] == -1


@pytest.mark.parametrize("form", ["lists", "walk", "records"])
def test_bsi_long_lists_chunked_merge(oracle, form):
    """Lists around and beyond the 32-entry chunk of the warp-cooperative
    intersection (1 .. 257 y per id): disjoint interleaved lists, a single
    common y at the very end / start / a chunk boundary, and equal lists --
    every (a, b) combination against the oracle."""
    from paper_2002_12459_b200.apps import bsi_answer_batch_arrays
    from paper_2002_12459_b200.relation import Relation, build_indexed
    lens = [1, 2, 31, 32, 33, 63, 64, 65, 100, 257]
    rp, sp = [], []
    for i, n in enumerate(lens):
        rp += [(i, 2 * k) for k in range(n)]                          # even y: 0, 2, ...
        sp += [(i, 2 * k + 1) for k in range(n)]                      # odd y: disjoint from every R list
        sp += [(100 + i, 2 * (n - 1))]                                # + R_i's last y only ...
        sp += [(100 + i, 2 * k + 1) for k in range(n)]                # ... after n odd ones
        sp += [(200 + i, 0)] + [(200 + i, 2 * k + 1) for k in range(n)]   # R's first y, then odd ones
        sp += [(300 + i, 2 * k) for k in range(n)]                    # equal to R_i
        sp += [(400 + i, 62)] + [(400 + i, 2 * k + 1) for k in range(max(n, 40))]   # y = 62: entry 31 of an R list
    rp, sp = np.array(rp), np.array(sp)
    ra = np.arange(len(lens))
    sb = np.concatenate([base + ra for base in (0, 100, 200, 300, 400)])
    q = np.array([(a, b) for a in ra for b in sb] + [(99, 0), (0, 99)])
    exp = oracle.bsi(oracle.encode(rp), oracle.encode(sp), q[:, 0], q[:, 1])
    r = build_indexed(Relation.from_raw_pairs("R", rp))
    s = build_indexed(Relation.from_raw_pairs("S", sp))
    got = bsi_answer_batch_arrays(r, s, q[:, 0], q[:, 1], form=form)
    assert np.array_equal(got, exp)
    by_block = exp[:-2].reshape(len(lens), 5, len(lens))      # [a, S block, b]
    assert (by_block[:, 0, :] == 0).all() and (exp == 1).sum() > 100 and (exp[-2:] == -1).all()


def test_bsi_tables_abi_errors():
    from paper_2002_12459_b200 import _native as nat
    nat.require_cuda()
    lib = nat.load()
    assert lib.mmj_bsi_direct_table(0, 0, 0, 0, 0, 0, 0) == nat.MMJ_ERR_ARG
    assert lib.mmj_bsi_answer(0, 0, 1, 0, 0, 1, 0, 0, 1, 0, 0, 1, 0, 0, 1, 0, 0, 0, 0, 6, 0, 0) == nat.MMJ_ERR_ARG
    assert lib.mmj_bsi_records(0, 0, 1, 0, 12, 0, 0, 0) == nat.MMJ_ERR_ARG
    # 6 length bits leave 26 offset bits: 2^26 - 1 tuples do not fit
    assert lib.mmj_bsi_span_table(0, 0, 0, 0, 8, 0, 0, 0, (1 << 26) - 1, 6, 0, 0) == nat.MMJ_ERR_ARG
    assert lib.mmj_bsi_span_table(0, 0, 0, 0, 8, 0, 0, 0, 10, 0, 0, 0) == nat.MMJ_ERR_ARG
    assert lib.mmj_bsi_answer_spans(0, 0, 1, 0, 0, 1, 6, 0, 1, 0, 0, 0, 1, 6, 0, 1, 0, 0, 0) == nat.MMJ_ERR_ARG


def test_star_golden():
    from paper_2002_12459_b200.joinproject import star_join
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce_many
    z = np.load(os.path.join(GOLDEN, "star.npz"))
    meta = json.loads(str(z["meta"]))
    for m in meta:
        i, k = m["inst"], m["k"]
        rels = semi_join_reduce_many([Relation.from_raw_pairs(f"R{j}", z[f"s{i}_rel{j}"]) for j in range(k)])
        idxs = [build_indexed(x) for x in rels]
        for thr in (None, 0.0, float("inf"), 3.0):     # all-heavy, all-light and mixed device splits
            res = star_join(idxs, m["d1"], m["d2"], want_counts=m["counts"], threshold=thr)
            assert list(res.dims) == m["dims"]
            assert np.array_equal(res.codes, z[m["key"] + "_codes"]), (m["key"], thr)
            assert list(res.stats["heavy_dims"]) == m["heavy_dims"], m["key"]
            if m["counts"]:
                assert np.array_equal(res.counts, z[m["key"] + "_counts"]), (m["key"], thr)


def test_star_errors_and_k2_equals_two_path():
    from paper_2002_12459_b200.errors import StarResourceError
    from paper_2002_12459_b200.joinproject import star_join, two_path_join
    from paper_2002_12459_b200.optimizer import ThresholdPlan
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce_many
    rng = np.random.default_rng(11)
    rels = semi_join_reduce_many([Relation.from_raw_pairs(f"R{i}", random_pairs(rng, 200, 12, 6)) for i in range(3)])
    idxs = [build_indexed(x) for x in rels]
    with pytest.raises(StarResourceError):
        star_join(idxs, 1, 1, heavy_rows_cap=2)
    with pytest.raises(ValueError):
        star_join(idxs[:1], 2, 2)
    with pytest.raises(ValueError):
        star_join(idxs, 0, 2)
    a = star_join(idxs[:2], 2, 2)
    b = two_path_join(idxs[0], idxs[1], plan=ThresholdPlan("partitioned", 2, 2))
    assert np.array_equal(a.codes, b.codes)


def test_star_zipf_k3_vs_oracle(oracle):
    from paper_2002_12459_b200.joinproject import star_join
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce_many
    rng = np.random.default_rng(7)
    raws = [np.array(zipf_pairs(rng, 3000, 60, 400, 1.3)) for _ in range(3)]
    rels = semi_join_reduce_many([Relation.from_raw_pairs(f"R{i}", r) for i, r in enumerate(raws)])
    idxs = [build_indexed(x) for x in rels]
    orels = oracle.semi_join_many([oracle.encode(r) for r in raws])
    exp = oracle.star(orels, 100, 1, want_counts=True, cap=1 << 30)
    got = star_join(idxs, 100, 1, want_counts=True, heavy_rows_cap=1 << 30)
    assert np.array_equal(got.codes, exp.codes) and np.array_equal(got.counts, exp.counts)
    assert list(got.stats["heavy_dims"]) == list(exp.stats["heavy_dims"])


def test_ssj_ordered_and_scj_on_device(oracle):
    """Device consumers: ssj_ordered's (-overlap, a, b) order
    from one stable device sort, and scj's containment filter fused into the
    count emission (per-row threshold |a|, diagonal excluded)."""
    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.apps import (SetFamily, scj_join_project_arrays, ssj_ordered,
                                            ssj_ordered_arrays)
    from paper_2002_12459_b200.relation import Relation
    pairs = datagen.set_family_pairs(11, 20000, 1500, 200, 1.4, 600, 1.1)
    fam = SetFamily(Relation.from_raw_pairs("sets", pairs))
    ofam = oracle.encode(pairs)
    ea, eb, en = oracle.ssj_arrays(ofam, 2)
    order = np.lexsort((eb, ea, -en))
    a, b, n = ssj_ordered_arrays(fam, 2)
    assert np.array_equal(a, ea[order]) and np.array_equal(b, eb[order]) and np.array_equal(n, en[order])
    assert ssj_ordered(fam, 2)[:50] == [((int(x), int(y)), int(k)) for x, y, k in
                                        zip(ea[order][:50], eb[order][:50], en[order][:50])]
    full = oracle.two_path(ofam, ofam, None, want_counts=True)
    dz = full.dims[1]
    x, z = full.codes // dz, full.codes % dz
    sizes = ofam.left_deg
    keep = (x != z) & (full.counts == sizes[x])
    sa, sb = scj_join_project_arrays(fam)
    assert np.array_equal(sa, x[keep]) and np.array_equal(sb, z[keep])
    assert keep.sum() > 0


@pytest.mark.parametrize("case", ["singletons", "identical_sets", "one_big_set"])
def test_ssj_edge_families(oracle, case):
    """All sets of size 1 (no pair reaches c >= 2), several identical sets
    (every pair at overlap = |set|), one large set among singletons."""
    from paper_2002_12459_b200.apps import SetFamily, ssj_mmjoin, ssj_mmjoin_arrays
    from paper_2002_12459_b200.relation import Relation
    if case == "singletons":
        pairs = np.array([(a, a % 13) for a in range(200)], dtype=np.int64)
    elif case == "identical_sets":
        pairs = np.array([(a, e) for a in range(30) for e in range(10, 22)], dtype=np.int64)
    else:
        pairs = np.array([(0, e) for e in range(500)] + [(a, a * 3) for a in range(1, 150)], dtype=np.int64)
    fam = SetFamily(Relation.from_raw_pairs("sets", pairs))
    for c in (1, 2, 12):
        ea, eb, en = oracle.ssj_arrays(oracle.encode(pairs), c)
        a, b, n = ssj_mmjoin_arrays(fam, c)
        assert np.array_equal(a, ea) and np.array_equal(b, eb) and np.array_equal(n, en), (case, c)
    if case == "identical_sets":
        got = ssj_mmjoin(fam, 12)
        assert len(got) == 30 * 29 // 2 and set(got.values()) == {12}
