"""Shared test setup: repo root on sys.path, the `gpu` marker, seeded input
generators and decoding helpers.  The CPU oracle (oracle/mmjoin_oracle.py)
is test infrastructure and is imported only from tests."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built libmmjoin_b200.so")


def random_pairs(rng, n, dom_left, dom_right):
    """About n distinct (left, right) int pairs, sorted (same distribution as
    the reference's test generator, pkg/tests/conftest.py:15-20)."""
    pairs = {(int(a), int(b)) for a, b in zip(rng.integers(0, dom_left, n), rng.integers(0, dom_right, n))}
    return sorted(pairs)


def zipf_pairs(rng, n, dom_left, dom_right, s):
    """n distinct (x, y) with x uniform, y bounded Zipf(s), sorted by (x, y)."""
    w = 1.0 / np.arange(1, dom_right + 1, dtype=np.float64) ** s
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    keys = np.empty(0, dtype=np.int64)
    while len(keys) < n:
        m = int((n - len(keys)) * 1.3) + 64
        x = rng.integers(0, dom_left, m)
        y = np.minimum(np.searchsorted(cdf, rng.random(m), side="right"), dom_right - 1)
        keys = np.unique(np.concatenate([keys, x * dom_right + y]))
    keys = rng.permutation(keys)[:n]
    keys.sort()
    return np.stack([keys // dom_right, keys % dom_right], axis=1)


def counts_dict(res, r, s):
    """OutputSet -> {(raw a, raw c): count} via the relations' dictionaries."""
    t = res.tuples()
    lv_r, lv_s = r.rel.left_values, s.rel.left_values
    return {(lv_r[a], lv_s[c]): int(n) for (a, c), n in zip(t.tolist(), res.counts.tolist())}


def raw_set(res, r, s):
    t = res.tuples()
    lv_r, lv_s = r.rel.left_values, s.rel.left_values
    return {(lv_r[a], lv_s[c]) for a, c in t.tolist()}


@pytest.fixture(scope="session")
def oracle():
    from oracle import mmjoin_oracle
    return mmjoin_oracle
