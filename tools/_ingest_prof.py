import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2002_12459_b200 import datagen, ingest
wl = datagen.config("cfg5")
raw = torch.from_numpy(np.ascontiguousarray(wl.relations[0], dtype=np.int64)).pin_memory()
ws = ingest.IngestWorkspace()
ingest.from_raw_pairs_device("R", raw, ws)
torch.cuda.synchronize()
def T(name, f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize(); print(f"{name:12s} {1e3*(time.perf_counter()-t0):8.1f} ms"); return r
t = T("h2d", lambda: ingest._raw_tensor(raw))
d = T("dedup", lambda: ingest._dedup(t, ws))
n = d.shape[0]; flat = d.reshape(-1)
l = T("first_seen_l", lambda: ingest._first_seen(flat, 2, n, ws))
r = T("first_seen_r", lambda: ingest._first_seen(flat[1:], 2, n, ws))
rv = T("rv_d2h", lambda: r[1].cpu().numpy())
x = T("index", lambda: ingest.DeviceIndexedRelation("R", l[0], r[0], l[1], rv, None, ws, right_values_dev=r[1]))
c = T("csr_fwd", lambda: ingest._csr(l[0], r[0], n, int(l[1].numel()), len(rv), ws, True))
T("total", lambda: ingest.from_raw_pairs_device("R", raw, ws))
