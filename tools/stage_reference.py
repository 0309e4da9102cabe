"""Install the unmodified reference package into baseline/_ref and stage its
own test suite under baseline/_ref/_tests (both git-ignored; both travel to
the GPU box with the gpurun snapshot, like the built .so).

    python tools/stage_reference.py [--force]

Install: ``pip install --no-index --no-build-isolation --no-deps --target
baseline/_ref`` from a /tmp copy of /root/reference/pkg (the build writes into
its source tree; --no-deps because numpy/click are already in the image and
the offline wheelhouse does not carry them).  The Cython kernel
(matmul/_kernel_cy) is compiled by that install.  The staged tests are the
reference's pkg/tests verbatim; tests/test_gpu_reference_suite.py runs them
with tests/refsuite/mmj_dropin.py substituting the hot-path entry points.
Does nothing when /root/reference is absent (the GPU box) or when both are
already staged.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SRC = "/root/reference/pkg"
DEST = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(DEST, "_tests")


def stage(force: bool = False) -> bool:
    if not os.path.isdir(REF_SRC):
        return os.path.isdir(os.path.join(DEST, "mmjoin"))
    if force or not os.path.isdir(os.path.join(DEST, "mmjoin")):
        shutil.rmtree(DEST, ignore_errors=True)
        with tempfile.TemporaryDirectory() as tmp:
            src = os.path.join(tmp, "pkg")
            shutil.copytree(REF_SRC, src)
            subprocess.run([sys.executable, "-m", "pip", "install", "-q", "--no-index", "--no-build-isolation",
                            "--no-deps", "--find-links", "/opt/wheelhouse", "--target", DEST, src],
                           check=True, cwd=tmp)
    if force or not os.path.isdir(TESTS):
        shutil.rmtree(TESTS, ignore_errors=True)
        shutil.copytree(os.path.join(REF_SRC, "tests"), TESTS,
                        ignore=shutil.ignore_patterns("__pycache__", "*.pyc"))
    return True


if __name__ == "__main__":
    print("staged" if stage("--force" in sys.argv) else "reference absent")
