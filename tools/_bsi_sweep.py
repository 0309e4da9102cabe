"""cfg5 BSI: build and answer time vs heavy_bits (diagnostic)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from tools.bench_configs import _timed
from paper_2002_12459_b200 import datagen
from paper_2002_12459_b200.bsi import BsiEngine, prepare
from paper_2002_12459_b200.ingest import from_raw_pairs_device
wl = datagen.config("cfg5")
raws = [torch.from_numpy(np.ascontiguousarray(r, dtype=np.int64)).cuda() for r in wl.relations]
qa = torch.from_numpy(wl.batch[:, 0].copy()).cuda()
qb = torch.from_numpy(wl.batch[:, 1].copy()).cuda()
nq = len(wl.batch)
r = from_raw_pairs_device("R", raws[0]); s = from_raw_pairs_device("S", raws[1])
sR, sS, dom_y = prepare(r, s)
ref = None
for hb in (128, 256, 512, 1024, 2048):
    holder = {}
    def full():
        eng = BsiEngine(sR, sS, dom_y, hb); eng.build(); holder["e"] = eng
        return eng.answer(qa, qb, nq)
    tf, ans = _timed(full)
    eng = holder["e"]
    ta, _ = _timed(lambda: eng.answer(qa, qb, nq))
    a = ans.cpu().numpy()
    if ref is None: ref = a
    print(json.dumps({"heavy_bits": hb, "delta1": eng.delta1, "build_plus_answer_ms": tf * 1e3, "answer_ms": ta * 1e3,
                      "same_answers": bool(np.array_equal(a, ref))}), flush=True)
