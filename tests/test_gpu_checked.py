"""Bounds-checked library run (the stand-in for compute-sanitizer, which this
GPU pool does not run): tools/sanitize_cases.py -- fused projection tail
(tcgen05 and in-tile-OR heavy parts, several column blocks, decoupled
look-back), three-kernel tail, count path, star, SSJ, BSI (both forms),
device ingest -- against libmmjoin_b200_check.so, built with every
MMJ_DCHECK compiled in (build.py --check): any out-of-range index traps the
kernel and fails the run; every case is also compared with the CPU oracle."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT


@pytest.mark.gpu
def test_sanitize_cases_with_bounds_checks():
    lib = os.path.join(ROOT, "paper_2002_12459_b200", "_lib", "libmmjoin_b200_check.so")
    assert os.path.exists(lib), "build the checked variant: python -m paper_2002_12459_b200.build --check"
    env = dict(os.environ, MMJ_LIB_VARIANT="check")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")], env=env,
                       capture_output=True, text=True, timeout=1200)
    out = p.stdout + p.stderr
    if os.path.isdir(os.path.join(ROOT, "gpurun_out")):
        with open(os.path.join(ROOT, "gpurun_out", "checked_cases.log"), "w") as f:
            f.write(out)
    assert p.returncode == 0, out[-4000:]
    assert "ALL OK" in out and "MMJ_DCHECK failed" not in out, out[-4000:]
    assert "libmmjoin_b200_check.so" in out, out[-2000:]
