"""Result text formats (formats.py / format.cu) against the reference CLI's
own output (tests/golden/cli.json, frozen by tests/golden/make_cli_golden.py
from cli.py twopath / star / ssj / scj on mixed numeric / alphanumeric
tokens): the same inputs parsed and joined by this package, formatted on the
device, byte-identical to what the CLI printed (click.echo adds the final
newline)."""

import io
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

CASES = json.load(open(os.path.join(GOLDEN, "cli.json")))


@pytest.fixture(scope="module")
def pkg():
    import paper_2002_12459_b200 as p
    from paper_2002_12459_b200 import _native
    _native.require_cuda()
    return p


def _opt(args, name, default=None, conv=int):
    return conv(args[args.index(name) + 1]) if name in args else default


def _parse(text, name):
    from paper_2002_12459_b200.relation import parse_edge_list
    return parse_edge_list(io.StringIO(text), name)


def _run(case):
    from paper_2002_12459_b200 import formats
    from paper_2002_12459_b200.apps import SetFamily, scj_join_project_arrays, ssj_mmjoin_arrays, ssj_ordered_arrays
    from paper_2002_12459_b200.joinproject import star_join, two_path_join
    from paper_2002_12459_b200.optimizer import PARTITIONED, ThresholdPlan
    from paper_2002_12459_b200.relation import build_indexed, semi_join_reduce, semi_join_reduce_many
    args, files = case["args"], case["files"]
    cmd = args[0]
    if cmd == "twopath":
        R, S = semi_join_reduce(_parse(files[_opt(args, "--left", conv=str)], "R"),
                                _parse(files[_opt(args, "--right", conv=str)], "S"))
        d1, d2 = _opt(args, "--delta1"), _opt(args, "--delta2")
        plan = ThresholdPlan(PARTITIONED, d1, d2) if d1 is not None and d2 is not None else None
        res = two_path_join(build_indexed(R), build_indexed(S), plan=plan, want_counts="--counts" in args)
        return formats.twopath_lines(res, R, S)
    if cmd == "star":
        paths = [args[i + 1] for i, a in enumerate(args) if a == "--input"]
        rels = semi_join_reduce_many([_parse(files[p], f"R{i}") for i, p in enumerate(paths)])
        res = star_join([build_indexed(x) for x in rels], _opt(args, "--delta1", 2), _opt(args, "--delta2", 2),
                        want_counts="--counts" in args)
        return formats.star_lines(res, rels)
    fam = SetFamily(_parse(files[_opt(args, "--sets", conv=str)], "sets"))
    if cmd == "ssj":
        c = _opt(args, "--c", 1)
        if _opt(args, "--method", "mmjoin", str) == "ordered":
            a, b, n = ssj_ordered_arrays(fam, c)
            return formats.ssj_lines(fam, a, b, n, ordered=True)
        a, b, n = ssj_mmjoin_arrays(fam, c)
        return formats.ssj_lines(fam, a, b, n)
    a, b = scj_join_project_arrays(fam)
    return formats.scj_lines(fam, a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(CASES)), ids=[" ".join(c["args"][:1] + [a for a in c["args"] if a.startswith("--") and a not in ("--left", "--right", "--input", "--sets")]) for c in CASES])
def test_cli_text_matches_reference(pkg, k):
    case = CASES[k]
    got = _run(case)
    assert got + "\n" == case["output"]


@pytest.mark.gpu
def test_lines_edge_cases(pkg):
    """Empty output, one line, prefix-related values ("1" < "10" < "1a" <
    "2"), counts, and unsorted (ordered) emission."""
    from paper_2002_12459_b200 import formats
    col = formats.Column(["10", "1", "2", "1a", "b", "-3"])
    assert formats.lines(np.empty(0, np.int64), (6, 6), [col, col]) == ""
    assert formats.lines(np.array([7]), (6, 6), [col, col]) == "1 1"
    codes = np.arange(36, dtype=np.int64)
    vals = ["10", "1", "2", "1a", "b", "-3"]
    exp = sorted(f"{vals[c // 6]} {vals[c % 6]}" for c in range(36))
    assert formats.lines(codes, (6, 6), [col, col]) == "\n".join(exp)
    cnt = np.array([3, 12, 1] * 12)
    exp = sorted(f"{vals[c // 6]} {vals[c % 6]} {n}" for c, n in zip(range(36), cnt.tolist()))
    assert formats.lines(codes, (6, 6), [col, col], cnt) == "\n".join(exp)
    order = [f"{vals[c // 6]} {vals[c % 6]}" for c in codes[::-1].tolist()]
    assert formats.lines(codes[::-1].copy(), (6, 6), [col, col], sort=False) == "\n".join(order)
    with pytest.raises(ValueError):
        formats.lines(np.array([7]), (6, 6), [col])
