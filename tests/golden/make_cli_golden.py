"""Freeze the REFERENCE CLI's text output (cli.py twopath / star / ssj /
scj) on small seeded inputs into tests/golden/cli.json.

Run in the build container only (imports the read-only reference package
from /root/reference/pkg/src through click's CliRunner; nothing at test time
reads /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_cli_golden.py

Inputs mix numeric and alphanumeric tokens of different lengths ("7",
"12", "x3", "10") so the string sort of the lines differs from the
numeric / dense-id order.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from click.testing import CliRunner  # noqa: E402
from mmjoin.cli import main  # noqa: E402


def _tok(rng, v, kinds):
    k = kinds[v % len(kinds)]
    return f"{k}{v}" if k else str(v)


def _edges(rng, n, dl, dr, lk, rk, zipf=None):
    pairs = set()
    while len(pairs) < n:
        a = int(rng.integers(0, dl))
        b = int(min(rng.zipf(zipf) - 1, dr - 1)) if zipf else int(rng.integers(0, dr))
        pairs.add((a, b))
    pairs = sorted(pairs)
    rng.shuffle(pairs)
    return "\n".join(f"{_tok(rng, a, lk)} {_tok(rng, b, rk)}" for a, b in pairs) + "\n"


def main_():
    rng = np.random.default_rng(2002)
    runner = CliRunner()
    cases = []
    with tempfile.TemporaryDirectory() as d:
        def put(name, text):
            p = os.path.join(d, name)
            with open(p, "w") as f:
                f.write(text)
            return p

        def run(args, files):
            paths = {k: put(k, v) for k, v in files.items()}
            argv = [paths.get(a, a) for a in args]
            res = runner.invoke(main, argv, catch_exceptions=False)
            assert res.exit_code == 0, res.output
            cases.append({"args": args, "files": files, "output": res.output})

        r = _edges(rng, 900, 120, 60, ["", "x", ""], ["", "y"], zipf=1.6)
        s = _edges(rng, 900, 150, 60, ["z", ""], ["", "y"], zipf=1.6)
        run(["twopath", "--left", "R.txt", "--right", "S.txt"], {"R.txt": r, "S.txt": s})
        run(["twopath", "--left", "R.txt", "--right", "S.txt", "--counts"], {"R.txt": r, "S.txt": s})
        run(["twopath", "--left", "R.txt", "--right", "S.txt", "--delta1", "3", "--delta2", "2", "--counts"],
            {"R.txt": r, "S.txt": s})
        rels = {f"T{i}.txt": _edges(rng, 400, 40, 25, ["", "w"], [""], zipf=1.8) for i in range(3)}
        run(["star", "--input", "T0.txt", "--input", "T1.txt", "--input", "T2.txt", "--delta1", "4", "--delta2", "2"],
            rels)
        run(["star", "--input", "T0.txt", "--input", "T1.txt", "--counts"], rels)
        sets = _edges(rng, 1500, 200, 80, ["s", ""], ["e"], zipf=1.4)
        run(["ssj", "--sets", "F.txt", "--c", "2"], {"F.txt": sets})
        run(["ssj", "--sets", "F.txt", "--c", "3", "--method", "ordered"], {"F.txt": sets})
        run(["scj", "--sets", "F.txt"], {"F.txt": sets})
    with open(os.path.join(HERE, "cli.json"), "w") as f:
        json.dump(cases, f)
    print({c["args"][0]: len(c["output"]) for c in cases})


if __name__ == "__main__":
    main_()
