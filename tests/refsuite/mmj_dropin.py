"""pytest plugin: run the reference's own test suite against the B200 drop-in.

Module substitution: the unmodified reference package
(``baseline/_ref/mmjoin``, installed by ``tools/stage_reference.py``) supplies
everything that is not on the hot path -- ``Relation``, ``IndexedRelation``,
``SetFamily``, the planner, the CLI, the BSI simulator -- and its six hot-path
entry points are replaced by this package's before any test
module binds them:

  mmjoin.joinproject.two_path_join / full_join_dedup / star_join   (joinproject.py:155, 228, 281)
  mmjoin.matmul.multiply_counts (+ core, joinproject bindings)     (matmul/core.py:95)
  mmjoin.apps.ssj_mmjoin / ssj_ordered / scj_join_project          (apps.py:65, 291, 297)
  mmjoin.apps.bsi_answer_batch                                     (apps.py:314)
  mmjoin.apps.two_path_join (the binding apps.py:13 made)
  StarResourceError / MatrixOverflowError (joinproject.py:28, core.py:33)

so the reference's tests feed reference-built ``IndexedRelation`` /
``SetFamily`` / ``CountMatrix`` objects straight into the CUDA path.  Loaded
with ``-p mmj_dropin`` (tests/refsuite on PYTHONPATH); the patched names are
listed in ``SUBSTITUTED`` and every substituted call is counted in ``CALLS``
so the wrapper test can prove the GPU path ran.
"""

from __future__ import annotations

import functools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(ROOT, "baseline", "_ref")
for p in (REF, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)

import mmjoin  # noqa: E402  (the reference package from baseline/_ref)
import mmjoin.apps as ref_apps  # noqa: E402
import mmjoin.joinproject as ref_jp  # noqa: E402
import mmjoin.matmul as ref_mm  # noqa: E402
import mmjoin.matmul.core as ref_core  # noqa: E402

from paper_2002_12459_b200 import apps as b_apps  # noqa: E402
from paper_2002_12459_b200 import errors as b_errors  # noqa: E402
from paper_2002_12459_b200 import joinproject as b_jp  # noqa: E402
from paper_2002_12459_b200 import matmul as b_mm  # noqa: E402

assert os.path.realpath(os.path.dirname(mmjoin.__file__)).startswith(os.path.realpath(REF)), mmjoin.__file__

CALLS: dict = {}
SUBSTITUTED = []


def _counted(name, fn):
    @functools.wraps(fn)
    def wrapper(*a, **k):
        CALLS[name] = CALLS.get(name, 0) + 1
        return fn(*a, **k)
    return wrapper


def _sub(module, attr, fn, name):
    setattr(module, attr, fn)
    SUBSTITUTED.append(f"{module.__name__}.{attr}")


def install():
    tp = _counted("two_path_join", b_jp.two_path_join)
    for m in (ref_jp, ref_apps):
        _sub(m, "two_path_join", tp, "two_path_join")
    _sub(ref_jp, "full_join_dedup", _counted("full_join_dedup", b_jp.full_join_dedup), "full_join_dedup")
    _sub(ref_jp, "star_join", _counted("star_join", b_jp.star_join), "star_join")
    mc = _counted("multiply_counts", b_mm.multiply_counts)
    for m in (ref_mm, ref_core, ref_jp):
        _sub(m, "multiply_counts", mc, "multiply_counts")
    for nm in ("ssj_mmjoin", "ssj_ordered", "scj_join_project", "bsi_answer_batch"):
        _sub(ref_apps, nm, _counted(nm, getattr(b_apps, nm)), nm)
    # the drop-in's exception types (same names and bases as the reference's),
    # exported where the reference module exports its own
    _sub(ref_jp, "StarResourceError", b_errors.StarResourceError, "StarResourceError")
    for m in (ref_mm, ref_core):
        _sub(m, "MatrixOverflowError", b_errors.MatrixOverflowError, "MatrixOverflowError")


install()


def pytest_terminal_summary(terminalreporter):
    terminalreporter.write_line(f"mmj_dropin substituted: {', '.join(SUBSTITUTED)}")
    terminalreporter.write_line("mmj_dropin calls: " + ", ".join(f"{k}={v}" for k, v in sorted(CALLS.items())))
