"""Small invocations of every kernel family for compute-sanitizer runs:

    compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
    compute-sanitizer --tool synccheck python tools/sanitize_cases.py

Covers the fused projection tail (k_merge_emit: heavy bits from the tcgen05
product and from the in-tile OR, decoupled look-back across several tiles
and column blocks), the three-kernel tail, the count path (heavy_mma COUNT32 /
COUNT16, light expansion, count emission), star, SSJ (compaction), BSI (both
forms) and device ingest.  Each case is checked against the CPU oracle so a
sanitizer run is also a parity run.  Exits non-zero on any mismatch.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    from conftest import zipf_pairs
    from oracle import mmjoin_oracle as o
    from paper_2002_12459_b200.apps import SetFamily, bsi_answer_batch_arrays, ssj_mmjoin_arrays
    from paper_2002_12459_b200.ingest import semi_join_reduce_device
    from paper_2002_12459_b200.joinproject import star_join, two_path_join, two_path_join_chunks
    from paper_2002_12459_b200.optimizer import PARTITIONED, ThresholdPlan
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce

    torch.cuda.set_device(0)
    from paper_2002_12459_b200 import _native
    print(f"library: {_native._LIB_PATH.name}", flush=True)
    rng = np.random.default_rng(3)
    # dom_z large enough for two column blocks of the fused tail (8192 words = 262144 cells)
    rp = np.array(zipf_pairs(rng, 30000, 600, 2000, 1.0))
    sp = np.array(zipf_pairs(rng, 30000, 300000, 2000, 1.0))
    R, S = semi_join_reduce(Relation.from_raw_pairs("R", rp), Relation.from_raw_pairs("S", sp))
    r, s = build_indexed(R), build_indexed(S)
    OR, OS = o.semi_join_many([o.encode(rp), o.encode(sp)])
    bad = []
    for d1, d2, counts, heavy in [(40, 1, False, "or"), (40, 1, False, "mma"), (40, 2, True, ""), (5, 5, False, "mma"),
                                  (10**9, 10**9, False, "")]:
        if heavy:
            os.environ["MMJ_HEAVY"] = heavy
        else:
            os.environ.pop("MMJ_HEAVY", None)
        plan = ThresholdPlan(PARTITIONED, d1, d2)
        got = two_path_join(r, s, plan=plan, want_counts=counts)
        exp = o.two_path(OR, OS, o.OPlan(PARTITIONED, d1, d2), want_counts=counts)
        ok = np.array_equal(got.codes, exp.codes) and (not counts or np.array_equal(got.counts, exp.counts))
        print(f"two_path d=({d1},{d2}) counts={counts} heavy={heavy or '-'}: {'ok' if ok else 'MISMATCH'}", flush=True)
        if not ok:
            bad.append(("two_path", d1, d2, counts, heavy))
    os.environ.pop("MMJ_HEAVY", None)
    # small synchronous chunks: the three-kernel tail
    parts = list(two_path_join_chunks(r, s, ThresholdPlan(PARTITIONED, 40, 1), chunk_rows=64))
    cat = np.concatenate([p.codes for p in parts])
    exp = o.two_path(OR, OS, o.OPlan(PARTITIONED, 40, 1))
    ok = np.array_equal(cat, exp.codes)
    print(f"two_path chunks of 64 rows: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        bad.append("chunks")
    # star k=3
    rels = [np.array(zipf_pairs(rng, 4000, 60, 300, 1.2)) for _ in range(3)]
    from paper_2002_12459_b200.relation import semi_join_reduce_many
    red = semi_join_reduce_many([Relation.from_raw_pairs(f"R{i}", x) for i, x in enumerate(rels)])
    idx = [build_indexed(x) for x in red]
    got = star_join(idx, 3, 1)
    ors = o.semi_join_many([o.encode(x) for x in rels])
    exp = o.star(ors, 3, 1, cap=1 << 40)
    ok = np.array_equal(got.codes, exp.codes)
    print(f"star k=3: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        bad.append("star")
    # SSJ with compaction
    fam_pairs = np.array(zipf_pairs(rng, 20000, 3000, 1500, 1.1))
    fam = SetFamily(Relation.from_raw_pairs("sets", fam_pairs))
    a, b, n = ssj_mmjoin_arrays(fam, 3)
    ea, eb, en = o.ssj_arrays(o.encode(fam_pairs), 3)
    ok = np.array_equal(a, ea) and np.array_equal(b, eb) and np.array_equal(n, en)
    print(f"ssj c=3: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        bad.append("ssj")
    # BSI: span tables, id-table walk, records
    q = rng.integers(-3, 620, (5000, 2))
    expb = o.bsi(o.encode(rp), o.encode(sp), q[:, 0], q[:, 1])
    r0 = build_indexed(Relation.from_raw_pairs("R", rp))
    s0 = build_indexed(Relation.from_raw_pairs("S", sp))
    for form in ("lists", "walk", "records"):
        got = bsi_answer_batch_arrays(r0, s0, q[:, 0], q[:, 1], form=form)
        ok = np.array_equal(got, expb)
        print(f"bsi {form}: {'ok' if ok else 'MISMATCH'}", flush=True)
        if not ok:
            bad.append(("bsi", form))
    # device ingest + projection
    dr, ds = semi_join_reduce_device([rp, sp])
    got = two_path_join(dr, ds, plan=ThresholdPlan(PARTITIONED, 40, 1))
    ok = np.array_equal(got.codes, o.two_path(OR, OS, o.OPlan(PARTITIONED, 40, 1)).codes)
    print(f"ingest + two_path: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        bad.append("ingest")
    torch.cuda.synchronize()
    print("ALL OK" if not bad else f"FAILED {bad}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
