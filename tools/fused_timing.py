"""Per-tile phase timing of the fused projection tail (profiling aid).

Needs a -DMMJ_DEBUG_TIMING build (MMJ_NVCC_EXTRA=-DMMJ_DEBUG_TIMING python -m
paper_2002_12459_b200.build --force).  Runs the cfg2 heavy product + fused tail on
one chunk and prints, over the chunk's tiles, the distribution of the phases
(ticket -> heavy bits landed -> light merge done -> segment scan done ->
look-back done -> emission done), in microseconds.

    python tools/fused_timing.py [chunk_rows] [x0]
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2002_12459_b200 import _native as nat
    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.device import device_relation
    from paper_2002_12459_b200.engine import TwoPathEngine
    from paper_2002_12459_b200.optimizer import gpu_plan
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    x0 = int(sys.argv[2]) if len(sys.argv) > 2 else 200_000
    wl = datagen.config("cfg2")
    R, S = semi_join_reduce(Relation.from_raw_pairs("R", wl.relations[0]), Relation.from_raw_pairs("S", wl.relations[1]))
    r, s = build_indexed(R), build_indexed(S)
    plan = gpu_plan(r, s)
    dr, ds = device_relation(r), device_relation(s)
    eng = TwoPathEngine(dr, ds, plan.strategy, plan.delta1, plan.delta2, False, chunk_rows=rows,
                        host_left_deg_r=r.left_deg, host_left_deg_s=s.left_deg)
    eng.prepare()
    lib = nat.load()
    ntiles = int(lib.mmj_merge_emit_workspace_size(rows, eng.wpr) - 16) // 8
    buf = torch.zeros(ntiles * 8, dtype=torch.int64, device="cuda")
    for it in range(3):
        lib.mmj_debug_timing_buffer(nat.ptr(buf) if it == 2 else None)
        ch = eng.run_chunk(x0, x0 + rows, sync=False, codes_key="c")
        torch.cuda.synchronize()
    lib.mmj_debug_timing_buffer(None)
    t = buf.view(ntiles, 8).cpu().numpy().astype(np.float64)
    t0 = t[:, 0].min()
    ph = {"heavy_bits": t[:, 1] - t[:, 0], "light_merge": t[:, 2] - t[:, 1], "scan": t[:, 3] - t[:, 2],
          "lookback": t[:, 4] - t[:, 3], "emission": t[:, 5] - t[:, 4], "total": t[:, 5] - t[:, 0]}
    out = {"ntiles": ntiles, "kernel_us": (t[:, 5].max() - t0) / 1e3}
    for k, v in ph.items():
        v = v / 1e3
        out[k] = {"mean": float(v.mean()), "p50": float(np.median(v)), "p90": float(np.percentile(v, 90)),
                  "p99": float(np.percentile(v, 99)), "max": float(v.max())}
    # how late a tile's predecessor published its aggregate relative to this tile reaching the look-back
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
