import sys, time; sys.path.insert(0, '/root/repo')
import torch
from paper_2002_12459_b200 import datagen, apps
from paper_2002_12459_b200.apps import SetFamily, _compact_family
from paper_2002_12459_b200.relation import Relation
from paper_2002_12459_b200.device import device_relation
from paper_2002_12459_b200 import _native as nat
fam = SetFamily(Relation.from_raw_pairs("sets", datagen.config("cfg4").relations[0]))
device_relation(fam.indexed)
orig_call = nat.call
tot = {}
def timed_call(name, *args):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter(); a.record(); orig_call(name, *args); b.record(); torch.cuda.synchronize()
    tot.setdefault(name, []).append((a.elapsed_time(b), (time.perf_counter() - t) * 1e3))
nat.call = timed_call
for i in range(5):
    torch.cuda.synchronize(); t = time.perf_counter()
    _compact_family(fam.indexed, 4)
    torch.cuda.synchronize(); print("compact ms", (time.perf_counter() - t) * 1e3)
print(tot)
