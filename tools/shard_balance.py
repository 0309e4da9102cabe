"""Load balance of the x-range sharding on cfg2,
measured on ONE B200: for N = 1, 2, 4, 8 every rank's shard step
(engine set-up, operand build, heavy product + fused tail over its x range)
is run in turn and timed with CUDA events.  Ranks share nothing on the data
path (S is replicated once), so the slowest shard bounds an N-GPU step;
``projected_efficiency`` = T(N=1) / (N * max shard time) is what the
sharding leaves on the table before NVLink set-up costs.  This is a
load-balance measurement, not a multi-GPU run (only one GPU is available).

    python tools/shard_balance.py [--worlds 1,2,4,8]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    import torch

    import bench
    from paper_2002_12459_b200.device import Workspace, device_relation
    from paper_2002_12459_b200.engine import TwoPathEngine
    from paper_2002_12459_b200.shard import x_ranges

    torch.cuda.set_device(0)
    wl, r, s = bench._build("cfg2")
    plan = bench._plan(argparse.Namespace(plan="gpu"), r, s)
    dr, ds = device_relation(r), device_relation(s)
    ws = Workspace()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def shard_step(x_lo, x_hi):
        eng = TwoPathEngine(dr, ds, plan.strategy, plan.delta1, plan.delta2, False, chunk_rows=16384, ws=ws,
                            host_left_deg_r=r.left_deg, host_left_deg_s=s.left_deg)
        eng.prepare()
        for a, b in eng.chunk_bounds(x_lo, x_hi):
            eng.run_chunk(a, b, sync=False)
        return eng.finish()

    shard_step(0, 16384)      # warm-up
    t1 = None
    for world in (int(v) for v in args.worlds.split(",")):
        ranges = x_ranges(r, s, world)
        per = []
        for lo, hi in ranges:
            best = None
            for _ in range(args.reps):
                flush.fill_(1)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                st = shard_step(lo, hi)
                e1.record()
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / 1e3
                best = t if best is None or t < best else best
            per.append({"x_range": [int(lo), int(hi)], "ms": round(best * 1e3, 2), "out": int(st.out_size)})
        tmax = max(p["ms"] for p in per) / 1e3
        tot = sum(p["out"] for p in per)
        if world == 1:
            t1 = tmax
        print(json.dumps({"config": "cfg2", "world": world, "shards": per, "out_total": tot,
                          "max_shard_ms": round(tmax * 1e3, 2),
                          "imbalance_max_over_mean": round(tmax / (sum(p["ms"] for p in per) / 1e3 / world), 4),
                          "projected_tuples_per_s": tot / tmax,
                          "projected_efficiency": (t1 / (world * tmax)) if t1 else None,
                          "note": "shards run one after another on one B200; not a multi-GPU measurement"}),
              flush=True)


if __name__ == "__main__":
    main()
