"""Seeded synthetic workloads for the five BASELINE.json configurations
(SURVEY.md section 8(d)); shared by bench.py, the tests and the CPU baseline.

* bounded Zipf(s) on [0, n): P(k) ~ (k+1)^-s, inverse CDF by searchsorted;
* distinct tuples: draw rounds of int(deficit*1.3)+4096 (x, then y) from one
  RNG per relation, keep first occurrences in draw order, truncate to n;
* every relation is sorted by (x, y) before encoding, so dense ids are
  monotone in raw values and codes order equals raw lexicographic order.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

SEEDS = {"cfg1": (1,), "cfg2": (2, 3), "cfg3": (10, 11, 12), "cfg4": (4,), "cfg5": (20, 21, 22)}


def zipf_cdf(n: int, s: float) -> np.ndarray:
    w = np.arange(1, n + 1, dtype=np.float64) ** (-s)
    c = np.cumsum(w)
    return c / c[-1]


def zipf_draw(rng, cdf: np.ndarray, m: int) -> np.ndarray:
    return np.minimum(np.searchsorted(cdf, rng.random(m), side="right"), len(cdf) - 1).astype(np.int64)


def distinct_pairs(seed: int, n: int, xdom: int, ydom: int, s: float) -> np.ndarray:
    """n distinct (x, y): x uniform on [0, xdom), y bounded Zipf(s) on [0, ydom),
    sorted by (x, y)."""
    rng = np.random.default_rng(seed)
    cdf = zipf_cdf(ydom, s)
    kept = np.empty(0, dtype=np.int64)
    while len(kept) < n:
        m = int((n - len(kept)) * 1.3) + 4096
        x = rng.integers(0, xdom, m, dtype=np.int64)
        y = zipf_draw(rng, cdf, m)
        keys = np.concatenate([kept, x * ydom + y])
        _, first = np.unique(keys, return_index=True)
        first.sort()
        kept = keys[first]
    kept = np.sort(kept[:n])
    return np.stack([kept // ydom, kept % ydom], axis=1)


def set_family_pairs(seed: int = 4, n_pairs: int = 2_000_000, n_sets: int = 100_000, max_size: int = 2000,
                     size_s: float = 1.5, n_elems: int = 50_000, elem_s: float = 1.1) -> np.ndarray:
    """cfg4: (set, element) pairs; set sizes bounded Zipf(size_s) on [1, max_size]
    rescaled to sum n_pairs (largest remainder, floor 1), each set topped up to
    its size with distinct Zipf(elem_s) elements (lowest ids kept)."""
    rng = np.random.default_rng(seed)
    sizes = zipf_draw(rng, zipf_cdf(max_size, size_s), n_sets) + 1
    scaled = sizes * (n_pairs / sizes.sum())
    base = np.maximum(np.floor(scaled).astype(np.int64), 1)
    rem = n_pairs - int(base.sum())
    if rem > 0:
        order = np.argsort(-(scaled - np.floor(scaled)), kind="stable")
        base[order[:rem]] += 1
    elif rem < 0:
        order = np.argsort(-base, kind="stable")
        i = 0
        while rem < 0:
            j = order[i % len(order)]
            if base[j] > 1:
                base[j] -= 1
                rem += 1
            i += 1
    sizes = np.minimum(base, n_elems)
    cdf = zipf_cdf(n_elems, elem_s)
    out_sets, out_elems = [], []
    need = sizes.copy()
    have = [np.empty(0, dtype=np.int64) for _ in range(n_sets)]
    pending = np.arange(n_sets)
    while len(pending):
        draw = np.repeat(pending, 2 * need[pending])
        elems = zipf_draw(rng, cdf, len(draw))
        key = np.unique(draw * n_elems + elems)
        sids, es = key // n_elems, key % n_elems
        bounds = np.searchsorted(sids, pending)
        ends = np.searchsorted(sids, pending, side="right")
        nxt = []
        for p, b, e in zip(pending.tolist(), bounds.tolist(), ends.tolist()):
            h = np.union1d(have[p], es[b:e])
            if len(h) >= sizes[p]:
                have[p] = h[: sizes[p]]
            else:
                have[p] = h
                need[p] = sizes[p] - len(h)
                nxt.append(p)
        pending = np.asarray(nxt, dtype=np.int64)
    for p in range(n_sets):
        out_sets.append(np.full(len(have[p]), p, dtype=np.int64))
        out_elems.append(have[p])
    return np.stack([np.concatenate(out_sets), np.concatenate(out_elems)], axis=1)


@dataclass
class Workload:
    name: str
    relations: list            # raw (n, 2) int64 arrays, sorted
    batch: Optional[np.ndarray] = None
    self_join: bool = False
    description: str = ""


def config(name: str, scale: float = 1.0) -> Workload:
    """Raw inputs of a BASELINE config (``scale`` < 1 shrinks tuple counts
    and domains proportionally for quick tests)."""
    def sz(v):
        return max(16, int(round(v * scale)))
    if name == "cfg1":
        r = distinct_pairs(1, sz(200_000), sz(20_000), sz(20_000), 1.2)
        return Workload(name, [r], self_join=True,
                        description="two-path self-join, 200k tuples, x U[0,20k), y Zipf(1.2) on [0,20k)")
    if name == "cfg2":
        r = distinct_pairs(2, sz(5_000_000), sz(500_000), sz(200_000), 1.0)
        s = distinct_pairs(3, sz(5_000_000), sz(500_000), sz(200_000), 1.0)
        return Workload(name, [r, s],
                        description="two-path, 5M+5M tuples, x,z U[0,500k), y Zipf(1.0) on [0,200k)")
    if name == "cfg3":
        rels = [distinct_pairs(sd, sz(300_000), sz(5_000), sz(30_000), 1.3) for sd in (10, 11, 12)]
        return Workload(name, rels,
                        description="3-way star, 3 x 300k tuples, x U[0,5k), y Zipf(1.3) on [0,30k)")
    if name == "cfg4":
        fam = set_family_pairs(4, sz(2_000_000), sz(100_000), 2000, 1.5, sz(50_000), 1.1)
        return Workload(name, [fam], self_join=True,
                        description="SSJ, 2M (set, element) pairs, 100k sets, c=4")
    if name == "cfg5":
        r = distinct_pairs(20, sz(64_000_000), sz(4_000_000), sz(8_000_000), 1.0)
        s = distinct_pairs(21, sz(64_000_000), sz(4_000_000), sz(8_000_000), 1.0)
        rng = np.random.default_rng(22)
        q = rng.integers(0, sz(4_000_000), (sz(4_000_000), 2), dtype=np.int64)
        return Workload(name, [r, s], batch=q,
                        description="BSI, 64M+64M tuples, 4M queries, x/z U[0,4M), y Zipf(1.0) on [0,8M)")
    raise ValueError(f"unknown config {name!r}")
