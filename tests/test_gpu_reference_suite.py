"""The reference's own test suite (pkg/tests, staged verbatim under
baseline/_ref/_tests by tools/stage_reference.py) run against the B200
drop-in: tests/refsuite/mmj_dropin.py substitutes the six hot-path entry
points of the unmodified reference package (baseline/_ref/mmjoin) with this
package's, so every join / product / SSJ / BSI call in those tests -- on
reference-built IndexedRelation, SetFamily and CountMatrix objects -- runs
the CUDA path.

Deselected: test_acceptance.py::test_criterion_09_performance_smoke, a
wall-clock ratio between two CPU strategies of the reference (the reference
fails it on this machine too); it is not a correctness
criterion.
"""

import os
import re
import subprocess
import sys

import pytest

from conftest import ROOT

SUITE = os.path.join(ROOT, "baseline", "_ref", "_tests")
PLUGIN_DIR = os.path.join(ROOT, "tests", "refsuite")
FILES = ["test_joinproject.py", "test_apps.py", "test_matmul.py", "test_acceptance.py", "test_cli.py",
         "test_optimizer.py", "test_relation.py"]
DESELECT = ["test_acceptance.py::test_criterion_09_performance_smoke"]


def run_suite(files=FILES, extra=()):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([PLUGIN_DIR, SUITE, env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-c", os.path.join(PLUGIN_DIR, "pytest.ini"),
           "--rootdir", SUITE, "-p", "mmj_dropin"] + [f"--deselect={os.path.join(SUITE, d)}" for d in DESELECT]
    cmd += [os.path.join(SUITE, f) for f in files] + list(extra)
    return subprocess.run(cmd, cwd=SUITE, env=env, capture_output=True, text=True, timeout=1500)


@pytest.mark.gpu
def test_reference_suite_on_dropin():
    if not os.path.isdir(os.path.join(SUITE)) or not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "mmjoin")):
        pytest.fail("reference suite not staged: run python tools/stage_reference.py (or __graft_entry__.build())")
    p = run_suite()
    out = p.stdout + p.stderr
    with open(os.path.join(ROOT, "gpurun_out", "reference_suite.log") if os.path.isdir(
            os.path.join(ROOT, "gpurun_out")) else os.devnull, "w") as f:
        f.write(out)
    assert p.returncode == 0, out[-6000:]
    m = re.search(r"(\d+) passed", out)
    assert m and int(m.group(1)) >= 100, out[-3000:]
    calls = dict(re.findall(r"(\w+)=(\d+)", out.split("mmj_dropin calls:")[-1].splitlines()[0]))
    for name in ("two_path_join", "star_join", "full_join_dedup", "multiply_counts", "ssj_mmjoin",
                 "bsi_answer_batch", "scj_join_project"):
        assert int(calls.get(name, 0)) > 0, (name, calls)
