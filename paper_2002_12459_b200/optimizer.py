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
           "estimate_output_size", "closed_form_thresholds", "default_plan", "gpu_plan",
           "CostConstants", "DEFAULT_COSTS", "measure_cost_constants", "modeled_costs", "optimize_thresholds",
           "GpuCosts", "DEFAULT_GPU_COSTS", "measure_gpu_costs"]


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
# The reference's cost-based sweep (optimizer.py:57-197), same interface
# ---------------------------------------------------------------------------
@dataclass
class CostConstants:
    """optimizer.py:57-68: nanos per scan step (T_s), per allocated cell
    (T_m) and per random insert (T_I); ``co`` the core (here: GPU) budget."""
    T_s: float = 2.0
    T_m: float = 30.0
    T_I: float = 8.0
    co: int = 1

    def validate(self) -> None:
        if min(self.T_s, self.T_m, self.T_I) <= 0 or self.co < 1:
            raise ValueError("cost constants must be strictly positive")


DEFAULT_COSTS = CostConstants()


def measure_cost_constants(n: int = 200_000, seed: int = 0, co: int = 1) -> CostConstants:
    """optimizer.py:74-100: host micro-benchmarks for T_s / T_m / T_I (the
    reference's CPU cost model; the B200 planner uses :func:`measure_gpu_costs`)."""
    import random
    import time
    rng = random.Random(seed)
    vals = list(range(n))
    t0 = time.perf_counter_ns()
    acc = 0
    for v in vals:
        acc += v
    t_s = (time.perf_counter_ns() - t0) / n
    t0 = time.perf_counter_ns()
    cells = [[0] * 4 for _ in range(n // 8)]
    t_m = (time.perf_counter_ns() - t0) / max(1, n // 8)
    slots = [0] * n
    pos = [rng.randrange(n) for _ in range(n // 4)]
    t0 = time.perf_counter_ns()
    for q in pos:
        slots[q] = q
        vals.append(q)
    t_i = (time.perf_counter_ns() - t0) / max(1, 2 * (n // 4))
    del cells
    out = CostConstants(max(t_s, 0.1), max(t_m, 0.1), max(t_i, 0.1), co)
    out.validate()
    return out


def modeled_costs(stats_r, stats_s, dom_x: int, delta1: int, delta2: int, consts: CostConstants,
                  table) -> tuple:
    """optimizer.py:141-160: (t_light, t_heavy) of one threshold pair.
    ``stats_r`` is built with the join partner (its sum_x weighs by the
    partner's list lengths)."""
    from .calibration import estimate_runtime
    t_light = (consts.T_I * stats_s.sum_y(delta1) + consts.T_I * stats_r.sum_x(delta2)
               + consts.T_m * dom_x + consts.T_s * stats_s.cdfx(delta1) * dom_x)
    u = dom_x - stats_r.count_left(delta2)
    v = stats_s.dom_right - stats_s.count_right(delta1)
    w = stats_s.dom_left - stats_s.count_left(delta2)
    if min(u, v, w) <= 0:
        return t_light, 0.0
    t_heavy = estimate_runtime(table, u, v, w, consts.co) + consts.T_m * (u * v + u * w)
    return t_light, float(t_heavy)


def optimize_thresholds(stats_r, stats_s, dom_x: int, out_join: int, consts: CostConstants = DEFAULT_COSTS,
                        table=None, step: float = 0.05) -> ThresholdPlan:
    """optimizer.py:163-197: geometric delta1 sweep from n down (delta2 tied
    to delta1 through the output estimate), stopping at the first strict
    increase of the modelled cost."""
    from .calibration import CalibrationError
    if not 0 < step < 1:
        raise ValueError("step must be in (0, 1)")
    n = max(stats_r.n_tuples, stats_s.n_tuples)
    if out_join <= FULL_JOIN_CUTOFF * n:
        return ThresholdPlan(FULL_JOIN, n, n, float(out_join), 0.0, 0)
    if table is None or not table.entries:
        raise CalibrationError("optimizer needs a calibration table; run calibrate")
    out_est = max(1, estimate_output_size(dom_x, out_join, n))
    d1 = d2 = n
    cur = (math.inf, 0.0)
    it = 0
    while True:
        prev, pd1, pd2 = cur, d1, d2
        d1 = max(1, math.floor((1 - step) * d1))
        d2 = max(1, min(n, round(n * d1 / out_est)))
        cur = modeled_costs(stats_r, stats_s, dom_x, d1, d2, consts, table)
        it += 1
        if cur[0] + cur[1] > prev[0] + prev[1]:
            return ThresholdPlan(PARTITIONED, pd1, pd2, prev[0], prev[1], it)
        if d1 == 1:
            return ThresholdPlan(PARTITIONED, d1, d2, cur[0], cur[1], it)


# ---------------------------------------------------------------------------
# B200 cost model
# ---------------------------------------------------------------------------
# Light witnesses cost one L2 atomic each; the heavy product costs 2*U*W ops
# per heavy y on the int8 tensor cores, and the bitmap it writes is the same
# for every plan.  The per-B200 constants live in GpuCosts (measured by
# measure_gpu_costs); they are planning inputs, not correctness parameters.
K_BLOCK = 128


@dataclass
class GpuCosts:
    """Per-B200 planning constants (seconds): one light witness on the
    bitmap (projection) and on the count path, and the heavy product as
    ``u*w*(cell_s + k*cell_k_s)`` for u heavy x, w heavy z and k (padded)
    heavy y -- the tcgen05 kernel's epilogue cost per output cell plus its
    MMA cost per cell and K unit, divided over ``co`` x-sharded GPUs.
    Defaults: :func:`measure_gpu_costs` on a B200 (z-pair heavy product of
    8192 x 131072 cells at K = 128 / 1024; engine light passes on a seeded
    Zipf instance); call it again to re-measure on other hardware."""
    witness_s_bitmap: float = 4.8e-12       # measure_gpu_costs() on a B200, round 1
    witness_s_count: float = 7.3e-11
    cell_s: float = 1.03e-13
    cell_k_s: float = 2.27e-16
    cell_k_s_count: float = 7.0e-16          # count epilogue kernel, one cell per column (cfg4 slope)
    co: int = 1

    def heavy_seconds(self, u: int, k: int, w: int, pair: bool = True) -> float:
        """``pair``: the z-pair operand (two cells per MMA column) of the
        projection; the count path multiplies one cell per column."""
        if u <= 0 or k <= 0 or w <= 0:
            return 0.0
        return float(u) * w * (self.cell_s + k * (self.cell_k_s if pair else self.cell_k_s_count)) / self.co


DEFAULT_GPU_COSTS = GpuCosts()


def _time_heavy(rows: int, zcols: int, k: int, seed: int, counts: bool = False) -> float:
    """seconds of one heavy product of rows x zcols cells at K = k (z-pair
    bitmap, or int32 counts)"""
    import torch
    from . import _native as nat
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = (torch.rand((rows, k), generator=g, device="cuda") < 0.05).to(torch.uint8)
    b = ((torch.rand((zcols // 2, k), generator=g, device="cuda") < 0.05).to(torch.uint8)
         + 128 * (torch.rand((zcols // 2, k), generator=g, device="cuda") < 0.05).to(torch.uint8))
    nnz = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = nat.stream_handle()
    if counts:
        b = (torch.rand((zcols, k), generator=g, device="cuda") < 0.05).to(torch.uint8)
        out = torch.empty(rows * zcols, dtype=torch.int32, device="cuda")
        args = (nat.ptr(b), zcols, k, 0, k, 0, rows, nat.MODE_COUNT32, 0, nat.ptr(out), zcols)
    else:
        out = torch.empty(rows * (zcols // 32), dtype=torch.int32, device="cuda")
        args = (nat.ptr(b), zcols // 2, k, 0, k, 0, rows, nat.MODE_BITMAP_PAIR, 0, nat.ptr(out), zcols // 32)

    def run():
        nat.call("mmj_heavy_mma", nat.ptr(a), rows, *args, nat.ptr(nnz), 0, st)
    run()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return sorted(ts)[1]


def measure_gpu_costs(seed: int = 0, co: int = 1) -> GpuCosts:
    """Re-measure :class:`GpuCosts` on this GPU: the heavy product's per-cell
    epilogue and per-cell-per-K costs from the kernel at K = 128 and 1024, and
    the light-witness costs from the engine's own merge / count-expansion on a
    seeded Zipf two-path whose plan makes every y light."""
    import torch

    from .device import device_relation
    from .engine import TwoPathEngine
    from .relation import Relation, build_indexed, semi_join_reduce
    rows, zc = 8192, 131072
    t1, t2 = _time_heavy(rows, zc, 128, seed), _time_heavy(rows, zc, 1024, seed)
    cells = float(rows) * zc
    cell_k = max((t2 - t1) / (cells * (1024 - 128)), 1e-19)
    cell = max(t1 / cells - 128 * cell_k, 1e-16)
    c1, c2 = _time_heavy(rows, 16384, 128, seed, True), _time_heavy(rows, 16384, 1024, seed, True)
    cell_k_count = max((c2 - c1) / (float(rows) * 16384 * (1024 - 128)), 1e-19)
    rng = np.random.default_rng(seed)

    def zipf(n, dl, dr, a):
        w = 1.0 / np.arange(1, dr + 1, dtype=np.float64) ** a
        cdf = np.cumsum(w) / w.sum()
        x = rng.integers(0, dl, n)
        y = np.minimum(np.searchsorted(cdf, rng.random(n), side="right"), dr - 1)
        return np.stack([x, y], axis=1)
    r, s = semi_join_reduce(Relation.from_raw_pairs("R", zipf(400_000, 60_000, 40_000, 1.0)),
                            Relation.from_raw_pairs("S", zipf(400_000, 60_000, 40_000, 1.0)))
    r, s = build_indexed(r), build_indexed(s)
    dr, ds = device_relation(r), device_relation(s)
    big = max(r.n, s.n)
    per = {}
    for counts in (False, True):
        eng = TwoPathEngine(dr, ds, PARTITIONED, big, big, counts, host_left_deg_r=r.left_deg,
                            host_left_deg_s=s.left_deg)
        eng.run(lambda ch: None)          # warm-up
        eng.reset_stats()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = eng.run(lambda ch: None)
        e1.record()
        e1.synchronize()
        per[counts] = (e0.elapsed_time(e1) * 1e-3) / max(1, st.light_intermediate)
    return GpuCosts(witness_s_bitmap=per[False], witness_s_count=per[True], cell_s=cell, cell_k_s=cell_k,
                    cell_k_s_count=cell_k_count, co=co)


def gpu_plan(r, s, candidates=None, *, counts: bool = False, min_count: int = 1,
             upper_only: bool = False, costs: GpuCosts = None) -> ThresholdPlan:
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
    costs = costs or DEFAULT_GPU_COSTS
    t_wit = costs.witness_s_count if counts else costs.witness_s_bitmap
    share = 0.5 if upper_only else 1.0
    if candidates is None:
        candidates = sorted({int(v) for v in np.unique(ms)} | {1})
    best = None
    for d1 in candidates:
        n_light = int(np.searchsorted(ms, d1, side="right"))
        k = len(ms) - n_light
        light = int(cum_light[n_light])
        kpad = -(-k // K_BLOCK) * K_BLOCK
        t_light, t_heavy = light * t_wit, costs.heavy_seconds(u, kpad, w, pair=not counts)
        # upper_only: the product skips tiles below the diagonal and the
        # expansion drops z <= x (empirically both about halve)
        t = share * (t_light + t_heavy)
        if best is None or t < best[0]:
            best = (t, d1, t_light, t_heavy)
    _, d1, t_light, t_heavy = best
    return ThresholdPlan(PARTITIONED, max(1, d1), 1, float(t_light), float(t_heavy), 0)
