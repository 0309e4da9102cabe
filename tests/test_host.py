"""CPU tests of the host side of the drop-in (no GPU): data model and
dictionary encoding vs the reference's ids (golden fixtures), planner,
error types, and the C ABI library's exported symbols."""

import ctypes
import io
import json
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, random_pairs

from oracle import mmjoin_oracle as o
from paper_2002_12459_b200 import errors, optimizer as opt, relation as rl


def _oracle_pair(r_raw, s_raw):
    return tuple(o.semi_join_many([o.encode(r_raw), o.encode(s_raw)]))


def test_first_seen_ids_match_oracle_and_reference():
    z = np.load(os.path.join(GOLDEN, "twopath.npz"))
    for i in range(5):
        R, S = z[f"i{i}_R"], z[f"i{i}_S"]
        perm = np.random.default_rng(i).permutation(len(R))
        Rp = R[perm]
        a = rl.semi_join_reduce(rl.Relation.from_raw_pairs("R", Rp), rl.Relation.from_raw_pairs("S", S))
        b = o.semi_join_many([o.encode(Rp), o.encode(S)])
        for x, y in zip(a, b):
            assert np.array_equal(x.pairs, y.pairs)
            assert list(x.left_values) == list(y.left_values)
            assert list(x.right_values) == list(y.right_values)


def test_generic_values_and_list_input():
    pairs = [("a", "x"), ("b", "y"), ("a", "x"), ("c", "x"), ("b", "z")]
    r = rl.Relation.from_raw_pairs("R", pairs)
    assert r.left_values == ["a", "b", "c"] and r.right_values == ["x", "y", "z"]
    assert r.n == 4 and r.pairs.tolist() == [[0, 0], [1, 1], [2, 0], [1, 2]]
    ints = rl.Relation.from_raw_pairs("I", [(5, 1), (3, 2), (5, 1)])
    assert list(ints.left_values) == [5, 3] and ints.left_ids.get(3) == 1 and ints.left_ids.get(4) is None
    assert 5 in ints.left_ids and ints.left_ids[5] == 0
    with pytest.raises(KeyError):
        ints.left_ids[4]


def test_semi_join_repr_order_and_shared_dict():
    r = rl.Relation.from_raw_pairs("R", [(1, 10), (2, 9), (3, 100)])
    s = rl.Relation.from_raw_pairs("S", [(7, 100), (8, 9), (9, 10), (9, 11)])
    a, b = rl.semi_join_reduce(r, s)
    assert a.right_values is b.right_values
    assert list(a.right_values) == [10, 100, 9]          # sorted by repr (relation.py:123)
    assert b.n == 3


def test_parse_edge_list_errors():
    rel = rl.parse_edge_list(io.StringIO("# c\n1 2\n\n3 4\n"))
    assert rel.n == 2
    with pytest.raises(errors.ParseError) as e:
        rl.parse_edge_list(io.StringIO("1 2\n3\n"))
    assert e.value.line_no == 2


def test_indexed_relation_csr_and_out_join():
    rng = np.random.default_rng(3)
    R = np.array(random_pairs(rng, 300, 25, 20))
    S = np.array(random_pairs(rng, 300, 25, 20))
    a, b = rl.semi_join_reduce(rl.Relation.from_raw_pairs("R", R), rl.Relation.from_raw_pairs("S", S))
    r, s = rl.build_indexed(a), rl.build_indexed(b)
    OR, OS = _oracle_pair(R, S)
    assert np.array_equal(r.fwd_indptr, OR.fwd()[0]) and np.array_equal(r.fwd_indices, OR.fwd()[1])
    assert np.array_equal(r.rev_indptr, OR.rev()[0]) and np.array_equal(r.rev_indices, OR.rev()[1])
    assert r.out_join_with(s) == o.out_join(OR, OS)
    unrelated = rl.build_indexed(rl.Relation.from_raw_pairs("X", R))
    with pytest.raises(ValueError):
        r.out_join_with(unrelated)
    vals, lens = rl.gather_ranges(r.rev_indptr, r.rev_indices, np.array([0, 1]))
    assert np.array_equal(vals, np.concatenate([r.rev(0), r.rev(1)]))


def test_default_plan_matches_oracle():
    z = np.load(os.path.join(GOLDEN, "twopath.npz"))
    meta = json.loads(str(z["meta"]))
    for m in meta:
        if m["plan"][0] != "default" or m["counts"]:
            continue
        i = m["inst"]
        R, S = z[f"i{i}_R"], z[f"i{i}_S"]
        if m["self_join"]:
            r = rl.build_indexed(rl.Relation.from_raw_pairs("R", R))
            s = r
        else:
            a, b = rl.semi_join_reduce(rl.Relation.from_raw_pairs("R", R), rl.Relation.from_raw_pairs("S", S))
            r, s = rl.build_indexed(a), rl.build_indexed(b)
        p = opt.default_plan(r, s)
        assert [p.strategy, p.delta1, p.delta2] == m["stats"]["plan"]


def test_plan_validation_and_tsv():
    with pytest.raises(errors.PlanError):
        opt.ThresholdPlan("bogus", 1, 1).validate()
    with pytest.raises(errors.PlanError):
        opt.ThresholdPlan(opt.PARTITIONED, 0, 1).validate()
    p = opt.ThresholdPlan(opt.PARTITIONED, 12, 3, 1.5, 2.5, 4)
    assert opt.ThresholdPlan.from_tsv_line(p.to_tsv_line()) == p
    assert opt.closed_form_thresholds(1000, 1000) == (10, 10)
    with pytest.raises(ValueError):
        opt.closed_form_thresholds(0, 1)


def test_gpu_plan_is_valid_partition():
    from paper_2002_12459_b200 import datagen
    raw = datagen.distinct_pairs(2, 30000, 3000, 2000, 1.0)
    r = rl.build_indexed(rl.Relation.from_raw_pairs("R", raw))
    p = opt.gpu_plan(r, r)
    p.validate()
    assert p.strategy == opt.PARTITIONED and p.delta2 == 1 and p.delta1 >= 1


def test_datagen_shapes_and_determinism():
    from paper_2002_12459_b200 import datagen
    a = datagen.distinct_pairs(2, 5000, 1000, 400, 1.0)
    b = datagen.distinct_pairs(2, 5000, 1000, 400, 1.0)
    assert np.array_equal(a, b) and len(a) == 5000
    key = a[:, 0] * 400 + a[:, 1]
    assert np.all(np.diff(key) > 0)              # distinct and sorted by (x, y)
    w = datagen.config("cfg1", scale=0.05)
    assert w.self_join and len(w.relations[0]) == 10000
    fam = datagen.set_family_pairs(4, 20000, 1000, 200, 1.5, 500, 1.1)
    assert len(fam) == 20000 and len(np.unique(fam[:, 0] * 500 + fam[:, 1])) == 20000


# ---------------------------------------------------------------- C ABI
HEADER = os.path.join(ROOT, "include", "mmjoin_b200.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(mmj_[a-z0-9_]+)\s*\(", txt)))


def test_capi_exports_every_declared_symbol():
    from paper_2002_12459_b200 import _native
    path = _native.lib_path()
    if not path.exists():
        pytest.skip("libmmjoin_b200.so not built")
    lib = ctypes.CDLL(str(path))
    names = _declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # every declared symbol also has a ctypes signature in the loader
    assert set(names) <= set(_native.exported_symbols())


def test_capi_host_only_queries():
    from paper_2002_12459_b200 import _native
    if not _native.lib_path().exists():
        pytest.skip("libmmjoin_b200.so not built")
    lib = _native.load()
    assert lib.mmj_abi_version() == 1
    assert lib.mmj_scan_workspace_bytes(10 ** 6) > 0
    assert lib.mmj_tile_count(2048, 15648 // 32 * 32) > 0
    assert lib.mmj_bitmap_segment_count(64) == 2
    # fused tail: 16-byte ticket + one status word per tile (4096 or 8192 words);
    # cfg2 rows of 15648 words split in column blocks
    ncb = lib.mmj_merge_emit_col_blocks(15648)
    assert ncb in (2, 4)
    assert lib.mmj_merge_emit_col_blocks(1024) == 1
    assert lib.mmj_merge_emit_workspace_size(16384, 15648) == 16 + 8 * 16384 * ncb
    assert lib.mmj_merge_emit_workspace_size(100, 32) == 16 + 8 * 1   # >= 128 rows per tile


def test_capi_argument_errors_without_gpu():
    """Argument checks run before any CUDA call (no GPU needed)."""
    import ctypes
    from paper_2002_12459_b200 import _native
    if not _native.lib_path().exists():
        pytest.skip("libmmjoin_b200.so not built")
    lib = _native.load()
    # a pitch that is not a multiple of 32 words
    rc = lib.mmj_merge_emit(None, 0, 0, 4, 33, 1000, None, None, None, 1, None, None, None, None, None, None, None,
                            None, None, None, None, None, 0, None)
    assert rc == 1 and b"multiple of 32" in lib.mmj_last_error()
    # a workspace smaller than mmj_merge_emit_workspace_size
    rc = lib.mmj_merge_emit(None, 0, 0, 4, 32, 1000, None, None, None, 1, None, None, None, None, None, None, None,
                            None, None, None, None, ctypes.c_void_p(16), 8, None)
    assert rc == 5 and b"workspace" in lib.mmj_last_error()
    # heavy product modes outside the enum
    rc = lib.mmj_heavy_mma(None, 256, None, 256, 128, 0, 128, 0, 128, 6, 0, None, 8, None, 0, None)
    assert rc == 1 and b"unknown mode" in lib.mmj_last_error()


def test_capi_new_entry_points_argument_errors_without_gpu():
    """SSJ compaction / code decode / BSI direct tables: argument checks run
    before any CUDA call."""
    from paper_2002_12459_b200 import _native
    if not _native.lib_path().exists():
        pytest.skip("libmmjoin_b200.so not built")
    lib = _native.load()
    assert lib.mmj_compact_rows(*([None] * 6), 0, 0, 0, -1, *([None] * 11), 0, None) == 1
    assert b"min_deg" in lib.mmj_last_error()
    assert lib.mmj_compact_rows(*([None] * 6), -5, 0, 0, 2, *([None] * 11), 0, None) == 1
    assert lib.mmj_decode_compact_codes(None, 4, 0, None, None, 10, None, None) == 1
    assert b"domains" in lib.mmj_last_error()
    assert lib.mmj_bsi_direct_table(None, None, 0, 0, 0, None, None) == 1
    assert b"range" in lib.mmj_last_error()
    assert lib.mmj_bsi_answer(None, None, 1, None, None, 1, None, 0, 1, None, None, 1, None, 0, 1, None, None, None,
                              None, 6, None, None) == 1
    assert b"words" in lib.mmj_last_error()
    assert lib.mmj_bsi_record_words(8) == 16 and lib.mmj_bsi_record_words(32) == 48
    assert lib.mmj_bsi_span_table(None, None, 0, 0, 8, None, None, None, (1 << 26) - 1, 6, None, None) == 1
    assert b"length bits" in lib.mmj_last_error()
    assert lib.mmj_bsi_answer_spans(None, None, 1, None, 0, 1, 6, None, 1, None, None, 0, 1, 6, None, 1, None, None,
                                    None) == 1
    assert b"span tables" in lib.mmj_last_error()
    assert lib.mmj_split_codes(None, 4, 0, None, None, None) == 1
    assert b"split_codes" in lib.mmj_last_error()


def test_engine_host_degree_max_memo():
    from paper_2002_12459_b200.engine import _host_max
    a = np.array([3, 9, 2], dtype=np.int64)
    b = np.array([3, 9, 2], dtype=np.int64)
    assert _host_max(a) == 9 and _host_max(a) == 9
    assert _host_max(b) == 9
    assert _host_max(np.empty(0, dtype=np.int64)) == 0
    assert _host_max([1, 40, 7]) == 40          # list input (reference objects may hold lists)
    c = np.array([1, 2, 3])
    assert _host_max(c) == 3
    c[0] = 50                                   # writeable arrays are never memoised: no stale maximum
    assert _host_max(c) == 50
    d = np.array([4, 5])
    d.flags.writeable = False                   # IndexedRelation freezes its degree vectors
    assert _host_max(d) == 5 and _host_max(d) == 5


def test_product_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2002_12459_b200.joinproject import two_path_join
    r = rl.build_indexed(rl.Relation.from_raw_pairs("R", [(1, 2), (2, 2)]))
    with pytest.raises(RuntimeError, match="CUDA"):
        two_path_join(r, r)


def test_checked_variant_exports_and_has_checks():
    """The bounds-checked build (build.py --check) exports the same C ABI and
    carries the MMJ_DCHECK trap sites (their message is in its device code)."""
    from paper_2002_12459_b200 import build
    path = build.CHECK_LIB
    if not path.exists():
        pytest.skip("libmmjoin_b200_check.so not built")
    lib = ctypes.CDLL(str(path))
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    blob = path.read_bytes()
    assert b"MMJ_DCHECK failed" in blob
    assert b"MMJ_DCHECK failed" not in build.LIB.read_bytes()
