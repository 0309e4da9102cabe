"""Throughput of every BASELINE config on one B200 (bench.py covers the
headline cfg2 with the full bench contract; this tool reports the others).

    python tools/bench_configs.py [cfg1 cfg3 cfg4 cfg5 ...] > profiles/rN_configs.jsonl

Each line: config, workload, output size, device time per evaluation (CUDA
events, inputs resident in HBM, 1 warm-up + best of 3), throughput and the
main kernels' shares.  Parity at these sizes is covered by
tests/test_gpu_fullsize.py.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _timed(fn, reps=3):
    import torch
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / 1e3
        best = (t, out) if best is None or t < best[0] else best
    return best


def cfg1():
    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.device import device_relation
    from paper_2002_12459_b200.engine import TwoPathEngine
    from paper_2002_12459_b200.optimizer import default_plan, gpu_plan
    from paper_2002_12459_b200.relation import Relation, build_indexed
    r = build_indexed(Relation.from_raw_pairs("R", datagen.config("cfg1").relations[0]))
    dr = device_relation(r)
    res = []
    for name, plan in (("gpu_plan", gpu_plan(r, r)), ("reference_default_plan", default_plan(r, r))):
        def run():
            eng = TwoPathEngine(dr, dr, plan.strategy, plan.delta1, plan.delta2, False, chunk_rows=20480,
                                host_left_deg_r=r.left_deg, host_left_deg_s=r.left_deg)
            eng.run_pipelined(0, r.rel.dom_left)
            return eng.finish()
        t, st = _timed(run)
        res.append({"config": "cfg1", "variant": name, "plan": [plan.strategy, plan.delta1, plan.delta2],
                    "out": st.out_size, "seconds": t, "tuples_per_s": st.out_size / t,
                    "light_intermediate": st.light_intermediate, "heavy_pairs": st.heavy_pairs,
                    "reference_cpu_seconds_same_container": 147.1})
    return res


def cfg3():
    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce_many
    from paper_2002_12459_b200.star import StarEngine
    wl = datagen.config("cfg3")
    rels = semi_join_reduce_many([Relation.from_raw_pairs(f"R{j}", r) for j, r in enumerate(wl.relations)])
    idxs = [build_indexed(x) for x in rels]
    tot = {}

    def run():
        n = [0]

        def sink(a, b, codes, counts):
            n[0] += int(codes.numel())
        eng = StarEngine(idxs, False)
        eng.run(sink)
        tot["k"] = eng.kh
        tot["light"] = int(eng.wit.item())
        return n[0]
    t, n = _timed(run, reps=2)
    return [{"config": "cfg3", "workload": wl.description, "out": n, "seconds": t, "tuples_per_s": n / t,
             "k_heavy": tot["k"], "light_witnesses": tot["light"]}]


def cfg4():
    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.apps import SetFamily
    from paper_2002_12459_b200.optimizer import gpu_plan
    from paper_2002_12459_b200.relation import Relation
    fam = SetFamily(Relation.from_raw_pairs("sets", datagen.config("cfg4").relations[0]))
    from paper_2002_12459_b200.optimizer import ThresholdPlan
    idx = fam.indexed
    plans = [gpu_plan(idx, idx, counts=True, min_count=4, upper_only=True)]
    for spec in filter(None, os.environ.get("MMJ_CFG4_PLANS", "").split(";")):
        d1, d2 = (int(v) for v in spec.split(","))
        plans.append(ThresholdPlan("partitioned", d1, d2))
    from paper_2002_12459_b200.apps import _ssj_engine
    rows = []
    for plan in plans:
        for compact in (True, False):
            def run():
                # compaction (sets below c dropped), engine, count join and
                # the decode of every chunk's codes are all inside the timing
                eng, decode = _ssj_engine(idx, 4, plan, compact=compact)
                n = [0]

                def sink(ch):
                    decode(ch.codes)
                    n[0] += ch.n
                eng.run(sink)
                eng.finish()
                return n[0]
            t, n = _timed(run)
            # one more pass with CUDA-event phase brackets (separate from the timed runs)
            from bench import PhaseTimer
            eng, _ = _ssj_engine(idx, 4, plan, compact=compact)
            eng.timer = PhaseTimer()
            eng.run(lambda ch: None)
            phases = {k: round(v, 3) for k, v in eng.timer.totals().items()}
            rows.append({"config": "cfg4", "workload": "SSJ c=4, 2M (set, element) pairs, 100k sets", "plan":
                         [plan.strategy, plan.delta1, plan.delta2], "compact_sets": compact,
                         "matrix_rows": eng.dom_x, "out_pairs": n, "seconds": t, "pairs_per_s": n / t,
                         "k_heavy": int(eng.kpad), "chunks": eng.stats.chunks, "phase_ms": phases})
    return rows


def ingest():
    """Device ingest (ingest.py) of every config's raw pairs: H2D of the raw
    int64 pairs + dedup + dictionaries (+ semi-join) + both CSRs, vs the host
    numpy path (relation.py) on the same arrays."""
    import torch

    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.ingest import from_raw_pairs_device, semi_join_reduce_device
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce_many
    rows = []
    for cfg in ("cfg2", "cfg5"):
        wl = datagen.config(cfg)
        raws = [np.ascontiguousarray(r, dtype=np.int64) for r in wl.relations]
        pinned = [torch.from_numpy(r).pin_memory() for r in raws]
        semi = cfg == "cfg2"

        def dev():
            if semi:
                out = semi_join_reduce_device(pinned)
            else:
                out = [from_raw_pairs_device(f"R{j}", t) for j, t in enumerate(pinned)]
            torch.cuda.synchronize()
            return out
        dev()
        t0 = time.perf_counter()
        out = dev()
        t_dev = time.perf_counter() - t0
        t0 = time.perf_counter()
        rels = [Relation.from_raw_pairs(f"R{j}", r) for j, r in enumerate(raws)]
        if semi:
            rels = semi_join_reduce_many(rels)
        host = [build_indexed(r) for r in rels]
        t_host = time.perf_counter() - t0
        same = all(np.array_equal(d.rel.left_values, h.rel.left_values) and np.array_equal(d.fwd_indices, h.fwd_indices)
                   and np.array_equal(d.rev_indptr, h.rev_indptr) for d, h in zip(out, host))
        n = sum(len(r) for r in raws)
        rows.append({"config": cfg, "stage": "ingest (raw pairs -> dictionaries + CSR)", "raw_tuples": n,
                     "semi_join": semi, "device_seconds_incl_h2d": t_dev, "device_tuples_per_s": n / t_dev,
                     "host_numpy_seconds": t_host, "identical": bool(same)})
    return rows


def cfg5():
    import torch

    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.bsi import BsiEngine, prepare
    from paper_2002_12459_b200.ingest import from_raw_pairs_device
    wl = datagen.config("cfg5")
    raws = [torch.from_numpy(np.ascontiguousarray(r, dtype=np.int64)).pin_memory() for r in wl.relations]
    qa = torch.from_numpy(wl.batch[:, 0].copy()).cuda()
    qb = torch.from_numpy(wl.batch[:, 1].copy()).cuda()
    nq = len(wl.batch)
    holder = {}

    def ingest_prepare():
        r = from_raw_pairs_device("R", raws[0])
        s = from_raw_pairs_device("S", raws[1])
        holder["sides"] = prepare(r, s)
        return r, s
    t_ing, _ = _timed(ingest_prepare, reps=2)
    sR, sS, dom_y = holder["sides"]

    def full():
        eng = BsiEngine(sR, sS, dom_y, 256)
        eng.build()
        holder["eng"] = eng
        return eng.answer(qa, qb, nq)
    t_full, ans = _timed(full)
    eng = holder["eng"]
    t_ans, _ = _timed(lambda: eng.answer(qa, qb, nq))
    a = ans.cpu().numpy()
    in_bytes = 8 * (raws[0].shape[0] + raws[1].shape[0]) + 9 * nq
    return [{"config": "cfg5", "workload": wl.description, "queries": nq, "true": int((a == 1).sum()),
             "none": int((a == -1).sum()), "seconds_build_plus_answer": t_full, "answers_per_s": nq / t_full,
             "seconds_answer_only": t_ans, "answers_per_s_answer_only": nq / t_ans,
             "seconds_raw_pairs_to_device_index": t_ing,
             "note": "device ingest (H2D of 2 x 64M pinned raw pairs, dedup, dictionaries, CSR) + BSI y-space "
                     "union/remap, then heavy-y bitsets + light lists (build) and the batch answer",
             "lower_bound_bytes": in_bytes, "achieved_GBps_vs_lower_bound": in_bytes / t_full / 1e9}]


if __name__ == "__main__":
    import torch
    torch.cuda.set_device(0)
    names = sys.argv[1:] or ["cfg1", "cfg3", "cfg4", "cfg5", "ingest"]
    for nm in names:
        for row in globals()[nm]():
            print(json.dumps(row), flush=True)
