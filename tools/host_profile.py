"""cProfile of one bench workload's step on the host (diagnostic):

    python tools/host_profile.py cfg4 [steps]

Runs the bench's setup + warm-up, then `steps` steps under cProfile with a
device sync after each, and prints the top functions by cumulative and by
own time -- where the host time of a host-bound step (cfg1, cfg4) goes."""

import cProfile
import io
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    args = bench._args(["--config", cfg])
    torch.cuda.set_device(0)
    wl = bench.WORKLOADS[cfg](args, 0, 1)
    wl.setup()
    for _ in range(3):
        wl.units(wl.step())
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(steps):
        wl.units(wl.step())
        torch.cuda.synchronize()
    pr.disable()
    for key in ("cumulative", "tottime"):
        s = io.StringIO()
        pstats.Stats(pr, stream=s).sort_stats(key).print_stats(35)
        print(s.getvalue())


if __name__ == "__main__":
    main()
