"""GPU parity for the applications: SSJ / SCJ on the exact count path and
batched boolean set intersection, against reference-frozen fixtures and the
oracle (bit-exact: same pairs, same overlap counts, same True/False/None)."""

import json
import os

import numpy as np
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


@pytest.mark.parametrize("heavy_bits", [128, 512])
def test_bsi_zipf_vs_oracle(oracle, heavy_bits):
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
    got = bsi_answer_batch_arrays(r, s, q[:, 0], q[:, 1], heavy_bits=heavy_bits)
    assert np.array_equal(got, exp)
    assert (exp == -1).any() and (exp == 1).any() and (exp == 0).any()
