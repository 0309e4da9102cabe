import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2002_12459_b200 import datagen
from paper_2002_12459_b200.ingest import from_raw_pairs_device
from paper_2002_12459_b200.bsi import BsiEngine, prepare
wl = datagen.config("cfg5")
r = from_raw_pairs_device("R", wl.relations[0]); s = from_raw_pairs_device("S", wl.relations[1])
qa = torch.from_numpy(wl.batch[:, 0].copy()).cuda(); qb = torch.from_numpy(wl.batch[:, 1].copy()).cuda()
nq = len(wl.batch)
def T(name, f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); out = f(); torch.cuda.synchronize(); print(f"{name:10s} {1e3*(time.perf_counter()-t0):8.2f} ms", flush=True); return out
for rep in range(2):
    r._mmj_bsi_cache = None
    sR, sS, dom_y = T("prepare", lambda: prepare(r, s))
    eng = T("init", lambda: BsiEngine(sR, sS, dom_y, 256))
    T("build", eng.build)
    T("answer", lambda: eng.answer(qa, qb, nq))
