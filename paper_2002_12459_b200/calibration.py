"""Measured heavy-product cost table, re-measured on the tcgen05 kernel
(SURVEY.md section 8(f1)).

Same interface and TSV format as the reference's
``mmjoin.matmul.calibration`` (calibration.py:13-104): a
:class:`CalibrationTable` maps (probe dim p, cores co) to the nanoseconds of a
p x p x p product, :func:`estimate_runtime` scales the nearest probe by volume,
and tables written by either implementation load in the other.  What is
measured differs: :func:`calibrate` times the engine's own heavy product
(``mmj_heavy_mma`` in the bitmap epilogue the join uses, CUDA events on the
device) instead of a CPU BLAS call, and ``co`` counts GPUs -- a
co-GPU entry is the per-GPU share of the x-sharded product (p/co rows, the
partition ``shard.py`` uses), since the shards run in parallel.
"""

from __future__ import annotations

import statistics
from typing import Optional, Sequence

import numpy as np

from . import _native as nat

__all__ = ["FORMAT_VERSION", "DEFAULT_PROBE_DIMS", "CalibrationError", "CalibrationTable", "calibrate",
           "estimate_runtime"]

FORMAT_VERSION = "mmjoin-calibration v1"
# larger than the reference's (128..1024): below ~1000^3 a device product is
# launch-latency bound and says nothing about the heavy part of a real join
DEFAULT_PROBE_DIMS = (256, 512, 1024, 2048, 4096, 8192)


class CalibrationError(RuntimeError):
    """calibration.py:17-18."""


class CalibrationTable:
    """calibration.py:21-63: (probe dim p, cores co) -> measured nanos."""

    def __init__(self, entries: Optional[dict] = None):
        self.entries: dict = {(int(p), int(c)): int(v) for (p, c), v in dict(entries or {}).items()}

    def __len__(self):
        return len(self.entries)

    def dims_for(self, co: int) -> list:
        return sorted(p for p, c in self.entries if c == co)

    def cores_available(self) -> list:
        return sorted({c for _, c in self.entries})

    def regularize(self) -> None:
        """nanos made nondecreasing in p for every core count"""
        for co in self.cores_available():
            run = 0
            for p in self.dims_for(co):
                run = max(run, self.entries[(p, co)])
                self.entries[(p, co)] = run

    def save(self, path) -> None:
        lines = [f"# {FORMAT_VERSION}"] + [f"{p}\t{c}\t{v}" for (p, c), v in sorted(self.entries.items())]
        with open(path, "w", encoding="utf-8") as f:
            f.write("\n".join(lines) + "\n")

    @classmethod
    def load(cls, path) -> "CalibrationTable":
        with open(path, encoding="utf-8") as f:
            first = f.readline().strip()
            if FORMAT_VERSION not in first:
                raise CalibrationError(f"unrecognized calibration file {path}")
            entries = {}
            for line in f:
                line = line.strip()
                if line:
                    p, c, v = line.split("\t")
                    entries[(int(p), int(c))] = int(v)
        return cls(entries)


def estimate_runtime(table: CalibrationTable, u: int, v: int, w: int, co: int = 1) -> float:
    """calibration.py:94-104: nanos of the nearest probe (by cube root of the
    volume, then by core count) scaled by u*v*w / p^3."""
    if not table.entries:
        raise CalibrationError("calibration table is empty; run calibrate first")
    c = min(table.cores_available(), key=lambda k: (abs(k - co), k))
    target = (u * v * w) ** (1.0 / 3.0)
    p = min(table.dims_for(c), key=lambda d: (abs(d - target), d))
    return table.entries[(p, c)] * (u * v * w) / (p ** 3)


def _probe_operands(p: int, seed: int, density: float):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed + p)
    kpad = -(-p // 128) * 128
    rows = -(-p // 1024) * 1024
    a = torch.zeros((rows, kpad), dtype=torch.uint8, device="cuda")
    b = torch.zeros((rows, kpad), dtype=torch.uint8, device="cuda")
    a[:p, :p] = (torch.rand((p, p), generator=g, device="cuda") < density).to(torch.uint8)
    b[:p, :p] = (torch.rand((p, p), generator=g, device="cuda") < density).to(torch.uint8)
    return a, b, kpad, rows


def calibrate(probe_dims: Sequence[int] = DEFAULT_PROBE_DIMS, cores: Sequence[int] = (1,), seed: int = 0,
              runs: int = 3, density: float = 0.05) -> CalibrationTable:
    """calibration.py:66-91 on the B200: for each probe p, the median over
    ``runs`` >= 3 CUDA-event timings of the heavy product of two seeded 0/1
    p x p operands (row density ``density``, as sparse as a join's heavy
    rows) into a bitmap, in nanos; then regularised to be monotone in p."""
    import torch
    nat.require_cuda()
    runs = max(int(runs), 3)
    table = CalibrationTable()
    st = nat.stream_handle()
    nnz = torch.zeros(1, dtype=torch.int64, device="cuda")
    for p in probe_dims:
        p = int(p)
        a, b, kpad, rows = _probe_operands(p, seed, density)
        wpr = rows // 32
        mode = nat.MODE_BITMAP_U8 if p <= 255 else nat.MODE_BITMAP
        for co in cores:
            m = max(1, -(-p // int(co)))          # one shard of the x-sharded product
            out = torch.empty(m * wpr, dtype=torch.int32, device="cuda")

            def run():
                nat.call("mmj_heavy_mma", nat.ptr(a), rows, nat.ptr(b), rows, kpad, 0, kpad, 0, m, mode, 0,
                         nat.ptr(out), wpr, nat.ptr(nnz), 0, st)
            run()
            samples = []
            for _ in range(runs):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run()
                e1.record()
                e1.synchronize()
                samples.append(e0.elapsed_time(e1) * 1e6)
            table.entries[(p, int(co))] = int(statistics.median(samples))
        del a, b
    table.regularize()
    return table
