"""Threshold planning for the two-path operator.

Mirrors the calibration-free part of the reference planner
(optimizer.py:14-54, 103-138, 200-208): ``ThresholdPlan``, the full-join
cutoff, the output-size estimate and the closed-form (Case 1/2) thresholds
behind ``default_plan``.  ``gpu_plan`` adds the B200 cost model: the output
is plan-independent, so the device may pick (delta1, delta2)
that move witnesses between the HBM-bound light expansion and the tensor-core
heavy product.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import PlanError

FULL_JOIN = "fulljoin"
PARTITIONED = "partitioned"
FULL_JOIN_CUTOFF = 20          # optimizer.py:18

__all__ = ["FULL_JOIN", "PARTITIONED", "FULL_JOIN_CUTOFF", "PlanError", "ThresholdPlan",
           "estimate_output_size", "closed_form_thresholds", "default_plan", "gpu_plan"]


@dataclass
class ThresholdPlan:
    """optimizer.py:25-54."""
    strategy: str
    delta1: int
    delta2: int
    light_cost: float = 0.0
    heavy_cost: float = 0.0
    iterations: int = 0

    def validate(self) -> None:
        if self.strategy not in (FULL_JOIN, PARTITIONED):
            raise PlanError(f"unknown strategy {self.strategy!r}")
        if self.strategy == PARTITIONED and (self.delta1 < 1 or self.delta2 < 1):
            raise PlanError("partitioned plans need delta1, delta2 >= 1")

    @property
    def total_cost(self) -> float:
        return self.light_cost + self.heavy_cost

    def to_tsv_line(self) -> str:
        return "\t".join(str(x) for x in (self.strategy, self.delta1, self.delta2,
                                          self.light_cost, self.heavy_cost, self.iterations))

    @classmethod
    def from_tsv_line(cls, line: str) -> "ThresholdPlan":
        s, d1, d2, cl, ch, it = line.rstrip("\n").split("\t")
        plan = cls(s, int(d1), int(d2), float(cl), float(ch), int(it))
        plan.validate()
        return plan


def estimate_output_size(dom_x: int, out_join: int, n: int) -> int:
    """optimizer.py:103-114: geometric mean of the |OUT| lower/upper bounds."""
    if out_join < 0 or n < 1:
        raise ValueError("out_join >= 0 and n >= 1 required")
    if out_join == 0 or dom_x == 0:
        return 0
    lower = max(dom_x, (out_join / n) ** 2)
    upper = min(dom_x * dom_x, out_join)
    est = math.ceil(math.sqrt(lower * upper))
    if upper >= 1:
        est = max(1, min(est, upper))
    return int(est)


def _ceil_cbrt_ratio(num: int, den: int) -> int:
    """optimizer.py:117-124: smallest k >= 1 with k^3 * den >= num (exact)."""
    k = max(1, round((num / den) ** (1.0 / 3.0)))
    while k ** 3 * den < num:
        k += 1
    while k > 1 and (k - 1) ** 3 * den >= num:
        k -= 1
    return k


def closed_form_thresholds(n: int, out_est: int) -> tuple[int, int]:
    """optimizer.py:127-138: omega=2 minimisers, clamped to [1, n]."""
    if n < 1 or out_est < 1:
        raise ValueError("n >= 1 and out_est >= 1 required")
    if out_est <= n:
        d1 = _ceil_cbrt_ratio(out_est, 1)
        d2 = _ceil_cbrt_ratio(n ** 3, out_est ** 2)
    else:
        d1 = d2 = _ceil_cbrt_ratio(2 * n * n, n + out_est)
    clamp = lambda d: max(1, min(d, n))  # noqa: E731
    return clamp(d1), clamp(d2)


def default_plan(r, s) -> ThresholdPlan:
    """optimizer.py:200-208: full-join cutoff, then the closed form."""
    n = max(r.n, s.n)
    out_join = r.out_join_with(s)
    if out_join <= FULL_JOIN_CUTOFF * n or n == 0:
        return ThresholdPlan(FULL_JOIN, max(n, 1), max(n, 1), float(out_join), 0.0, 0)
    out_est = max(1, estimate_output_size(r.rel.dom_left, out_join, n))
    d1, d2 = closed_form_thresholds(n, out_est)
    return ThresholdPlan(PARTITIONED, d1, d2, 0.0, 0.0, 0)


# ---------------------------------------------------------------------------
# B200 cost model
# ---------------------------------------------------------------------------
# Light witnesses cost one L2 atomic each; the heavy product costs 2*U*W ops
# per heavy y on the int8 tensor cores, and the bitmap it writes is the same
# for every plan.  Rates are per-B200 planning constants (measured orders of
# magnitude, refined by bench runs), not correctness parameters.
LIGHT_WITNESS_RATE = 2.0e11        # light witnesses / s (bitmap atomicOr, L2 resident)
LIGHT_COUNT_RATE = 2.0e10          # light witnesses / s (int32 count atomics over a chunk larger than L2)
MMA_OPS_RATE = 2.0e15              # int8 ops / s sustained (K is padded to 128)
K_BLOCK = 128


def gpu_plan(r, s, candidates=None, *, counts: bool = False, min_count: int = 1,
             upper_only: bool = False) -> ThresholdPlan:
    """Pick (delta1, delta2=1) minimising modelled B200 time.

    delta2 = 1 makes (almost) every x and z heavy, so the light side is pass 1
    (light y) only; delta1 then trades sum_{y light} degR*degS light
    witnesses against K = #heavy y columns of the tensor-core product.
    The count path (``counts``) pays more per light witness; with SSJ's
    pruning (``min_count`` > 1 drops sets smaller than c, ``upper_only``
    keeps z > x) only the surviving witnesses and half the product count.
    """
    n = max(r.n, s.n)
    out_join = r.out_join_with(s)
    if n == 0 or out_join <= FULL_JOIN_CUTOFF * n:
        return ThresholdPlan(FULL_JOIN, max(n, 1), max(n, 1), float(out_join), 0.0, 0)
    rdeg = np.asarray(r.right_deg, dtype=np.int64)
    sdeg = np.asarray(s.right_deg, dtype=np.int64)
    m = np.maximum(rdeg, sdeg)
    if min_count > 1:
        def kept(idx):
            ok = np.asarray(idx.left_deg) >= min_count
            rows = np.repeat(ok, np.diff(idx.fwd_indptr))
            return np.bincount(idx.fwd_indices[rows], minlength=len(idx.right_deg)).astype(np.int64)
        prod = kept(r) * kept(s)
    else:
        prod = rdeg * sdeg
    order = np.argsort(m, kind="stable")
    ms = m[order]
    cum_light = np.concatenate([[0], np.cumsum(prod[order])])
    u = int((np.asarray(r.left_deg) > 1).sum())
    w = int((np.asarray(s.left_deg) > 1).sum())
    light_rate = LIGHT_COUNT_RATE if counts else LIGHT_WITNESS_RATE
    share = 0.5 if upper_only else 1.0
    if candidates is None:
        candidates = sorted({int(v) for v in np.unique(ms)} | {1})
    best = None
    for d1 in candidates:
        n_light = int(np.searchsorted(ms, d1, side="right"))
        k = len(ms) - n_light
        light = int(cum_light[n_light])
        kpad = -(-k // K_BLOCK) * K_BLOCK
        t = share * (light / light_rate + 2.0 * u * w * kpad / MMA_OPS_RATE)
        if best is None or t < best[0]:
            best = (t, d1, light, 2.0 * u * w * kpad)
    _, d1, light, mma = best
    return ThresholdPlan(PARTITIONED, max(1, d1), 1, float(light), float(mma), 0)
