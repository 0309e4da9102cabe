"""Micro-benchmarks on the B200: HBM write ceiling (torch fill_/copy_) vs the
fused emission kernel on a synthetic 49%-dense bitmap (no light work)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2002_12459_b200 import _native as nat

def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best

nat.require_cuda()
N = 1 << 30  # int64 elements = 8 GB
x = torch.empty(N, dtype=torch.int64, device="cuda")
y = torch.empty(N, dtype=torch.int64, device="cuda")
res = {}
res["fill_GBps"] = 8 * N / t(lambda: x.fill_(7)) / 1e9
res["copy_GBps(r+w)"] = 16 * N / t(lambda: y.copy_(x)) / 1e9
del y
# emission-only: rows x dom_z bitmap with ~49% density
rows, dom_z = int(sys.argv[1]) if len(sys.argv) > 1 else 2048, 499987
wpr = -(-dom_z // 256) * 8
bm = torch.randint(0, 2**31, (rows * wpr,), dtype=torch.int32, device="cuda") & torch.randint(0, 2**31, (rows * wpr,), dtype=torch.int32, device="cuda") | torch.randint(0, 2**31, (rows * wpr,), dtype=torch.int32, device="cuda")
bm = bm.view(rows, wpr)
bm[:, dom_z // 32 + 1:] = 0
bm[:, dom_z // 32] &= (1 << (dom_z % 32)) - 1
bm = bm.contiguous().view(-1)
lib = nat.load()
ntiles = lib.mmj_row_emit_tiles(rows, wpr)
status = torch.zeros(ntiles + 2, dtype=torch.int64, device="cuda")
fwd_ptr = torch.zeros(rows + 1, dtype=torch.int32, device="cuda")
zero = torch.zeros(16, dtype=torch.int32, device="cuda")
wit = torch.zeros(1, dtype=torch.int64, device="cuda")
codes = x
st = nat.stream_handle()
def emit():
    status.zero_()
    nat.call("mmj_row_light_emit", nat.ptr(bm), 0, rows, wpr, dom_z, 1, nat.ptr(fwd_ptr), nat.ptr(zero),
             nat.ptr(zero), 1, 0, nat.ptr(zero), nat.ptr(zero), 0, 0, nat.ptr(codes), nat.ptr(status), 0,
             nat.ptr(wit), nat.ptr(status[ntiles + 1:]), st)
te = t(emit)
n = int(status[ntiles + 1].item())
res.update(rows=rows, codes=n, emit_ms=te * 1e3, emit_write_GBps=8 * n / te / 1e9)
print(json.dumps(res))
