import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
os.environ.setdefault("CUDA_LAUNCH_BLOCKING", "1")
import numpy as np
from conftest import zipf_pairs
from paper_2002_12459_b200.joinproject import two_path_join
from paper_2002_12459_b200.optimizer import ThresholdPlan
from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce
from oracle import mmjoin_oracle as o
for (nx, nr, nz, ns, dy) in [(50, 2000, 300, 3000, 200), (32, 4000, 3_000_000, 1_000_000, 3000)]:
    rng = np.random.default_rng(3)
    rp = zipf_pairs(rng, nr, nx, dy, 1.1); sp = zipf_pairs(rng, ns, nz, dy, 1.1)
    R, S = semi_join_reduce(Relation.from_raw_pairs("R", rp), Relation.from_raw_pairs("S", sp))
    r, s = build_indexed(R), build_indexed(S)
    for plan in [("partitioned", 40, 1), ("fulljoin", 10**7, 10**7)]:
        got = two_path_join(r, s, plan=ThresholdPlan(*plan))
        a, b = o.semi_join_many([o.encode(rp), o.encode(sp)])
        exp = o.two_path(a, b, o.OPlan(*plan))
        print(nz, plan, len(got.codes), len(exp.codes), np.array_equal(got.codes, exp.codes), flush=True)
