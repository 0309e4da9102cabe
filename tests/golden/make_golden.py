"""Freeze outputs of the REFERENCE implementation into golden fixtures.

Run in the build container only (it imports the read-only reference package
from /root/reference/pkg/src; nothing at test time reads /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--cfg1]

Writes tests/golden/*.npz.  Inputs are seeded and regenerated here so the
fixtures are self-contained (raw input pairs are stored with the outputs).
Generators follow the reference tests' own distributions
(pkg/tests/conftest.py:15-29) and SURVEY.md section 8(d).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from mmjoin import apps, joinproject as jp, optimizer as opt  # noqa: E402
from mmjoin.matmul import CountMatrix, multiply_counts  # noqa: E402
from mmjoin.relation import Relation, build_indexed, semi_join_reduce, semi_join_reduce_many  # noqa: E402


def random_pairs(rng, n, dom_left, dom_right):
    pairs = {(int(a), int(b)) for a, b in zip(rng.integers(0, dom_left, n), rng.integers(0, dom_right, n))}
    return sorted(pairs)


def zipf_pairs(rng, n, dom_left, dom_right, s):
    w = 1.0 / np.arange(1, dom_right + 1, dtype=np.float64) ** s
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    keys = np.empty(0, dtype=np.int64)
    while len(keys) < n:
        m = int((n - len(keys)) * 1.3) + 64
        x = rng.integers(0, dom_left, m)
        y = np.minimum(np.searchsorted(cdf, rng.random(m), side="right"), dom_right - 1)
        keys = np.unique(np.concatenate([keys, x * dom_right + y]))
    keys = rng.permutation(keys)[:n]
    keys.sort()
    return [tuple(map(int, p)) for p in np.stack([keys // dom_right, keys % dom_right], axis=1)]


def reduced(r_pairs, s_pairs):
    r, s = semi_join_reduce(Relation.from_raw_pairs("R", r_pairs), Relation.from_raw_pairs("S", s_pairs))
    return build_indexed(r), build_indexed(s)


def codes_checksum(codes: np.ndarray) -> dict:
    c = np.asarray(codes, dtype=np.int64)
    u = c.view(np.uint64)
    idx = np.linspace(0, max(len(c) - 1, 0), num=min(len(c), 64)).astype(np.int64) if len(c) else np.zeros(0, np.int64)
    return {"n": int(len(c)), "sum": int(u.sum(dtype=np.uint64)),
            "wsum": int((u * (np.arange(len(u), dtype=np.uint64) + np.uint64(1))).sum(dtype=np.uint64)),
            "sample_idx": idx.tolist(), "sample": c[idx].tolist() if len(c) else []}


def gen_twopath(out):
    arrays, meta = {}, []
    inst = 0
    for seed in range(10):
        rng = np.random.default_rng(1000 + seed)
        n = int(rng.integers(20, 500))
        dom = int(rng.integers(5, 45))
        rp = random_pairs(rng, n, dom, dom)
        sp = random_pairs(rng, n, dom, int(rng.integers(5, 45)))
        cases = [(rp, sp, False)]
        if seed < 3:
            cases.append((rp, rp, True))
        for r_pairs, s_pairs, self_join in cases:
            if self_join:
                r = build_indexed(Relation.from_raw_pairs("R", r_pairs))
                s = r
            else:
                r, s = reduced(r_pairs, s_pairs)
            nn = max(r.n, s.n, 1)
            plans = [("partitioned", 1, 1), ("partitioned", 2, 3), ("partitioned", 5, 2),
                     ("partitioned", nn, nn), ("fulljoin", nn, nn), ("default", 0, 0)]
            arrays[f"i{inst}_R"] = np.asarray(r_pairs, dtype=np.int64).reshape(-1, 2)
            arrays[f"i{inst}_S"] = np.asarray(s_pairs, dtype=np.int64).reshape(-1, 2)
            for pi, (st, d1, d2) in enumerate(plans):
                plan = None if st == "default" else opt.ThresholdPlan(st, d1, d2)
                for wc in (False, True):
                    res = jp.two_path_join(r, s, plan=plan, want_counts=wc)
                    key = f"i{inst}_p{pi}_c{int(wc)}"
                    arrays[key + "_codes"] = res.codes.astype(np.int64)
                    if wc:
                        arrays[key + "_counts"] = res.counts.astype(np.int64)
                    stats = {k: (v if not isinstance(v, opt.ThresholdPlan) else [v.strategy, v.delta1, v.delta2])
                             for k, v in res.stats.items()}
                    meta.append({"key": key, "inst": inst, "plan": [st, d1, d2], "counts": wc,
                                 "self_join": self_join, "dims": list(res.dims), "stats": stats})
            inst += 1
    # a skewed medium instance (Zipf y) with several plans incl. GPU-style ones
    rng = np.random.default_rng(77)
    rp = zipf_pairs(rng, 6000, 600, 2000, 1.2)
    sp = zipf_pairs(rng, 6000, 500, 2000, 1.1)
    r, s = reduced(rp, sp)
    arrays[f"i{inst}_R"] = np.asarray(rp, dtype=np.int64)
    arrays[f"i{inst}_S"] = np.asarray(sp, dtype=np.int64)
    for pi, (st, d1, d2) in enumerate([("default", 0, 0), ("partitioned", 300, 1), ("partitioned", 40, 3)]):
        plan = None if st == "default" else opt.ThresholdPlan(st, d1, d2)
        for wc in (False, True):
            res = jp.two_path_join(r, s, plan=plan, want_counts=wc)
            key = f"i{inst}_p{pi}_c{int(wc)}"
            arrays[key + "_codes"] = res.codes.astype(np.int64)
            if wc:
                arrays[key + "_counts"] = res.counts.astype(np.int64)
            stats = {k: (v if not isinstance(v, opt.ThresholdPlan) else [v.strategy, v.delta1, v.delta2])
                     for k, v in res.stats.items()}
            meta.append({"key": key, "inst": inst, "plan": [st, d1, d2], "counts": wc, "self_join": False,
                         "dims": list(res.dims), "stats": stats})
    arrays["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(out, "twopath.npz"), **arrays)
    print("twopath:", len(meta), "cases")


def gen_example(out):
    """The reference's frozen worked examples (pkg/tests/conftest.py:119-129)
    and the pinned heavy-matrix product (test_joinproject.py:46-62)."""
    sys.path.insert(0, "/root/reference/pkg/tests")
    import conftest as rc   # reference test module: fixture data only
    r, s = reduced(rc.EXAMPLE_R, rc.EXAMPLE_S)
    pr, ps = jp.partition_two_path(r, s, 2, 2)
    m1, m2 = jp.heavy_matrices(r, s, 2, 2)
    rows = [r.rel.left_values[i] for i in m1.row_keys]
    mids = [r.rel.right_values[i] for i in m1.col_keys]
    cols = [s.rel.left_values[i] for i in m2.col_keys]
    o1, om, o2 = np.argsort(rows), np.argsort(mids), np.argsort(cols)
    a = m1.data[o1][:, om]
    b = m2.data[om][:, o2]
    prod = multiply_counts(CountMatrix(a), CountMatrix(b)).data
    res = jp.two_path_join(r, s, plan=opt.ThresholdPlan("partitioned", 2, 2), want_counts=True)
    counts = {f"{r.rel.left_values[x]},{s.rel.left_values[z]}": int(c)
              for (x, z), c in zip(res.tuples().tolist(), res.counts.tolist())}
    rels = semi_join_reduce_many([Relation.from_raw_pairs("T", rc.EXAMPLE_T), Relation.from_raw_pairs("U", rc.EXAMPLE_U)])
    idxs = [build_indexed(x) for x in rels]
    st = jp.star_join(idxs, 2, 2, want_counts=True)
    star = {",".join(str(rels[i].left_values[v]) for i, v in enumerate(t)): int(c)
            for t, c in zip(st.tuples().tolist(), st.counts.tolist())}
    meta = {"R": rc.EXAMPLE_R, "S": rc.EXAMPLE_S, "T": rc.EXAMPLE_T, "U": rc.EXAMPLE_U,
            "light_R": sorted(pr.light.raw_pair_set()), "heavy_R": sorted(pr.heavy.raw_pair_set()),
            "light_S": sorted(ps.light.raw_pair_set()), "heavy_S": sorted(ps.heavy.raw_pair_set()),
            "M1": a.tolist(), "M2": b.tolist(), "product": prod.tolist(), "counts": counts,
            "out_join": r.out_join_with(s), "star_TU_counts": star,
            "bsi_batch_size": apps.bsi_batch_size(1000, 10 ** 6),
            "closed_form_1000_1000": list(opt.closed_form_thresholds(1000, 1000))}
    with open(os.path.join(out, "example.json"), "w") as f:
        json.dump(meta, f, indent=0)
    print("example: ok")


def gen_star(out):
    arrays, meta = {}, []
    for i, (k, seed) in enumerate([(2, 0), (3, 1), (4, 2), (3, 3), (3, 4), (2, 5)]):
        rng = np.random.default_rng(3000 + seed)
        n = int(rng.integers(20, 120))
        rel_pairs = [random_pairs(rng, n, 10 if k == 4 else 14, 8) for _ in range(k)]
        rels = semi_join_reduce_many([Relation.from_raw_pairs(f"R{j}", p) for j, p in enumerate(rel_pairs)])
        idxs = [build_indexed(x) for x in rels]
        for j, p in enumerate(rel_pairs):
            arrays[f"s{i}_rel{j}"] = np.asarray(p, dtype=np.int64)
        for pi, (d1, d2) in enumerate([(1, 1), (2, 2), (3, 1), (100, 100)]):
            for wc in (False, True):
                res = jp.star_join(idxs, d1, d2, want_counts=wc)
                key = f"s{i}_p{pi}_c{int(wc)}"
                arrays[key + "_codes"] = res.codes.astype(np.int64)
                if wc:
                    arrays[key + "_counts"] = res.counts.astype(np.int64)
                meta.append({"key": key, "inst": i, "k": k, "d1": d1, "d2": d2, "counts": wc,
                             "dims": list(res.dims), "heavy_dims": list(res.stats.get("heavy_dims", []))})
    arrays["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(out, "star.npz"), **arrays)
    print("star:", len(meta), "cases")


def gen_ssj(out):
    arrays, meta = {}, []
    for i in range(8):
        rng = np.random.default_rng(4000 + i)
        n_sets = int(rng.integers(15, 60))
        fam = {}
        for a in range(n_sets):
            size = int(rng.integers(1, 12))
            fam[1000 + 7 * a] = sorted({int(e) for e in rng.integers(0, 40, size)})
        f = apps.SetFamily.from_dict(fam)
        pairs = np.array([(a, e) for a, es in fam.items() for e in es], dtype=np.int64)
        arrays[f"f{i}_pairs"] = pairs
        for c in (1, 2, 3):
            res = apps.ssj_mmjoin(f, c)
            trip = np.array([(a, b, n) for (a, b), n in res.items()], dtype=np.int64).reshape(-1, 3)
            arrays[f"f{i}_c{c}"] = trip
            meta.append({"key": f"f{i}_c{c}", "inst": i, "c": c, "n": len(trip)})
        scj = sorted(apps.scj_join_project(f))
        arrays[f"f{i}_scj"] = np.array(scj, dtype=np.int64).reshape(-1, 2)
    arrays["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(out, "ssj.npz"), **arrays)
    print("ssj:", len(meta), "cases")


def gen_bsi(out):
    arrays, meta = {}, []
    for i in range(6):
        rng = np.random.default_rng(5000 + i)
        rp = random_pairs(rng, 300, 40, 30)
        sp = random_pairs(rng, 300, 40, 30)
        r = build_indexed(Relation.from_raw_pairs("R", rp))
        s = build_indexed(Relation.from_raw_pairs("S", sp))
        batch = [(int(a), int(b)) for a, b in rng.integers(0, 44, (200, 2))]
        batch += [(999, 0), (0, 999), (-5, -5)]
        ans = apps.bsi_answer_batch(r, s, batch)
        enc = np.array([-1 if v is None else int(v) for v in ans], dtype=np.int8)
        arrays[f"b{i}_R"] = np.asarray(rp, dtype=np.int64)
        arrays[f"b{i}_S"] = np.asarray(sp, dtype=np.int64)
        arrays[f"b{i}_batch"] = np.asarray(batch, dtype=np.int64)
        arrays[f"b{i}_ans"] = enc
        meta.append({"inst": i, "none": int((enc == -1).sum()), "true": int((enc == 1).sum())})
    arrays["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(os.path.join(out, "bsi.npz"), **arrays)
    print("bsi:", meta)


def gen_matmul(out):
    arrays = {}
    rng = np.random.default_rng(6000)
    for i in range(12):
        u, v, w = (int(x) for x in rng.integers(1, 70, 3))
        hi = [2, 6, 300, 10 ** 6][i % 4]
        a = rng.integers(0, hi, (u, v)).astype(np.int64)
        b = rng.integers(0, hi, (v, w)).astype(np.int64)
        arrays[f"m{i}_a"] = a
        arrays[f"m{i}_b"] = b
        arrays[f"m{i}_p"] = multiply_counts(CountMatrix(a), CountMatrix(b)).data
    np.savez_compressed(os.path.join(out, "matmul.npz"), **arrays)
    print("matmul: 12")


def gen_plans(out):
    rows = []
    for n, est in [(1000, 1000), (100, 7), (10 ** 6, 10 ** 9), (5, 1), (200000, 87300000), (4980842, 13200000000)]:
        rows.append({"n": n, "est": est, "closed": list(opt.closed_form_thresholds(n, est))})
    ests = []
    for dom_x, oj, n in [(20000, 873000000, 200000), (50, 1000, 300), (0, 10, 10), (10, 0, 5), (499981, 163000000000, 4981499)]:
        ests.append({"dom_x": dom_x, "out_join": oj, "n": n, "est": opt.estimate_output_size(dom_x, oj, n)})
    with open(os.path.join(out, "plans.json"), "w") as f:
        json.dump({"closed_form": rows, "estimate": ests}, f, indent=0)
    print("plans: ok")


def gen_planner(out):
    """Cost-based planner of the reference (relation.py:205-277 DegreeStats /
    degree_stats, optimizer.py:57-197 CostConstants / modeled_costs /
    optimize_thresholds, matmul/calibration.py:20-104 table + estimate_runtime)
    on fixed inputs and the reference tests' synthetic calibration table
    (test_optimizer.py:16-19), so no timing enters the fixture."""
    from mmjoin.matmul import CalibrationTable, estimate_runtime
    from mmjoin.relation import degree_stats, generate_community_graph
    table = CalibrationTable({(100, 1): 1_000, (200, 1): 8_000, (400, 1): 64_000})
    table2 = CalibrationTable({(16, 1): 10, (32, 1): 90, (64, 1): 700, (64, 2): 400, (128, 2): 3000})
    est = []
    for t, name in ((table, "t1"), (table2, "t2")):
        for u, v, w, co in [(100, 100, 100, 1), (150, 230, 90, 1), (1000, 10, 10, 1), (64, 64, 64, 2),
                            (300, 300, 300, 3), (5, 7, 11, 1)]:
            est.append({"table": name, "uvw_co": [u, v, w, co], "nanos": estimate_runtime(t, u, v, w, co)})
    insts = []
    arrays = {}
    rng = np.random.default_rng(4242)
    sources = [("random", random_pairs(rng, 3000, 200, 150), random_pairs(rng, 3000, 180, 150)),
               ("zipf", zipf_pairs(rng, 8000, 700, 900, 1.1), zipf_pairs(rng, 8000, 650, 900, 1.2))]
    for nodes, k, p_, seed in [(210, 3, 0.85, 4), (300, 3, 0.5, 1), (420, 3, 0.35, 2)]:
        rel = generate_community_graph(nodes, k, p_, seed=seed)
        sources.append((f"community{nodes}", list(rel.raw_pairs()), None))
    for i, (name, rp, sp) in enumerate(sources):
        if sp is None:
            r = s = build_indexed(Relation.from_raw_pairs("R", rp))
        else:
            r, s = reduced(rp, sp)
        arrays[f"p{i}_R"] = np.asarray(rp, dtype=np.int64).reshape(-1, 2)
        if sp is not None:
            arrays[f"p{i}_S"] = np.asarray(sp, dtype=np.int64).reshape(-1, 2)
        st_r = degree_stats(r, partner=s)
        st_s = degree_stats(s)
        deltas = sorted({1, 2, 3, 5, 8, 13, 40, 100, 1000, int(st_r.max_left_deg), int(st_s.max_right_deg)})
        q = {"deltas": deltas,
             "r": {f: [int(getattr(st_r, f)(d)) for d in deltas] for f in ("count_left", "count_right", "cdfx", "sum_y", "sum_x")},
             "s": {f: [int(getattr(st_s, f)(d)) for d in deltas] for f in ("count_left", "count_right", "cdfx", "sum_y", "sum_x")},
             "r_max": [int(st_r.max_left_deg), int(st_r.max_right_deg)], "s_max": [int(st_s.max_left_deg), int(st_s.max_right_deg)]}
        n = max(r.n, s.n)
        oj = r.out_join_with(s)
        costs = []
        for d1, d2 in [(1, 1), (2, 3), (5, 2), (10, 10), (n, n), (40, 1)]:
            costs.append({"d": [d1, d2], "cost": list(opt.modeled_costs(st_r, st_s, r.rel.dom_left, d1, d2,
                                                                       opt.DEFAULT_COSTS, table))})
        plans = []
        for step in (0.05, 0.2):
            pl = opt.optimize_thresholds(st_r, st_s, r.rel.dom_left, oj, table=table, step=step)
            plans.append({"step": step, "plan": [pl.strategy, pl.delta1, pl.delta2, pl.light_cost, pl.heavy_cost,
                                                 pl.iterations]})
        cc = opt.CostConstants(1.0, 5.0, 3.0, 1)
        pl = opt.optimize_thresholds(st_r, st_s, r.rel.dom_left, oj, consts=cc, table=table)
        plans.append({"consts": [1.0, 5.0, 3.0, 1], "plan": [pl.strategy, pl.delta1, pl.delta2, pl.light_cost,
                                                             pl.heavy_cost, pl.iterations]})
        insts.append({"name": name, "self_join": sp is None, "n": n, "out_join": int(oj), "stats": q,
                      "costs": costs, "plans": plans})
    np.savez_compressed(os.path.join(out, "planner.npz"), **arrays)
    with open(os.path.join(out, "planner.json"), "w") as f:
        json.dump({"estimate_runtime": est, "instances": insts}, f)
    print("planner:", len(insts), "instances")


def gen_cfg1(out):
    """Full BASELINE cfg1 through the reference (about 3 min, ~50 GB RAM):
    checksums of the 387M output codes + stats."""
    from paper_2002_12459_b200 import datagen
    raw = datagen.config("cfg1").relations[0]
    rel = Relation.from_raw_pairs("R", [tuple(p) for p in raw.tolist()])
    idx = build_indexed(rel)
    t0 = time.time()
    res = jp.two_path_join(idx, idx)
    dt = time.time() - t0
    plan = res.stats["plan"]
    meta = {"config": "cfg1", "seconds": dt, "plan": [plan.strategy, plan.delta1, plan.delta2],
            "light_intermediate": int(res.stats["light_intermediate"]), "heavy_pairs": int(res.stats["heavy_pairs"]),
            "dims": list(res.dims), "checksum": codes_checksum(res.codes)}
    with open(os.path.join(out, "cfg1_reference.json"), "w") as f:
        json.dump(meta, f, indent=0)
    print("cfg1:", meta["checksum"]["n"], f"{dt:.1f}s")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg1", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    if a.cfg1:
        gen_cfg1(HERE)
    else:
        for name, fn in [("twopath", gen_twopath), ("example", gen_example), ("star", gen_star), ("ssj", gen_ssj),
                         ("bsi", gen_bsi), ("matmul", gen_matmul), ("plans", gen_plans), ("planner", gen_planner)]:
            if not a.only or name in a.only.split(","):
                fn(HERE)
