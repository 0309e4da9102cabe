"""Host-side timing of the SSJ compaction and engine set-up on cfg4 (diagnostic)."""
import sys, time; sys.path.insert(0, '/root/repo')
import numpy as np
import torch
from paper_2002_12459_b200 import datagen, _native as nat
from paper_2002_12459_b200.apps import SetFamily, _ssj_engine, _ssj_plan
from paper_2002_12459_b200.relation import Relation
from paper_2002_12459_b200.device import DeviceRelation, device_relation
from paper_2002_12459_b200.ingest import IngestWorkspace
fam = SetFamily(Relation.from_raw_pairs("sets", datagen.config("cfg4").relations[0]))
idx = fam.indexed
device_relation(idx)
plan = _ssj_plan(idx, None, 4)
for rep in range(4):
    T = [("start", time.perf_counter())]
    def mark(n):
        torch.cuda.synchronize(); T.append((n, time.perf_counter()))
    c = 4
    ldeg = np.asarray(idx.left_deg); keep = ldeg >= c; nk = int(keep.sum()); mark("host flags")
    dr = device_relation(idx); n, dom, dom_y = dr.n, dr.dom_left, dr.dom_right; mark("device_relation")
    bufs = [torch.empty(max(k, 1), dtype=torch.int32, device="cuda") for k in (dom, dom, dom + 1, n, n, dom, dom_y + 1, n, dom_y)]
    sizes = torch.zeros(2, dtype=torch.int64, device="cuda"); mark("allocs")
    ws_buf, nb = IngestWorkspace().get(max(n, dom, dom_y)); mark("ingest ws")
    nat.call("mmj_compact_rows", nat.ptr(dr.fwd_ptr), nat.ptr(dr.fwd_idx), nat.ptr(dr.fwd_row), nat.ptr(dr.rev_ptr),
             nat.ptr(dr.rev_idx), nat.ptr(dr.left_deg), n, dom, dom_y, c, *[nat.ptr(b) for b in bufs], nat.ptr(sizes),
             nat.ptr(ws_buf), nb, nat.stream_handle()); mark("compact kernel")
    fp = np.concatenate([[0], np.cumsum(ldeg[keep], dtype=np.int64)]); mark("host ptr")
    eng, dec = _ssj_engine(idx, 4, plan); mark("_ssj_engine total")
    eng.prepare(); mark("engine prepare")
    cnt = [0]
    eng.run(lambda ch: (dec(ch.codes), cnt.__setitem__(0, cnt[0] + ch.n))); mark("run+decode")
    eng.finish(); mark("finish")
    print(" | ".join(f"{T[i][0]} {1e3 * (T[i][1] - T[i - 1][1]):.3f}" for i in range(1, len(T))))
