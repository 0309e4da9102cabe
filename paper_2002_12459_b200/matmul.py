"""Exact count-matrix product on the tcgen05 tensor cores (drop-in for
``mmjoin.matmul.core``, matmul/core.py:18-133).

``multiply_counts`` keeps the reference's contract -- exact int64 product of
non-negative count matrices, ``ValueError`` on a dimension mismatch or an
unknown backend, ``MatrixOverflowError`` when the worst-case entry
``inner * max(A) * max(B)`` exceeds int64 (core.py:98-107) or, for
``backend="blas"``, 2^53 (core.py:110-113) -- and adds the ``"cuda"``
backend, which ``"auto"`` (and every legacy backend name) resolves to; there
is no CPU path.

Exactness for arbitrary non-negative int64 entries: each operand is split
into base-256 digit planes (uint8), every digit-plane pair is contracted with
``tcgen05.mma.kind::i8`` (u8 x u8 -> s32, K windows of <= 32768 so a window
sum is < 2^31) and recombined into int64 by the ``ACC64`` epilogue
(out += partial << 8*(i+j)).  All partial sums are bounded by the final
entry, which the overflow check bounds by int64.  0/1 matrices use one plane.
"""

from __future__ import annotations

import os
from typing import Optional

import numpy as np

from .calibration import (DEFAULT_PROBE_DIMS, CalibrationError, CalibrationTable, calibrate,  # noqa: F401
                          estimate_runtime)
from .errors import MatrixOverflowError

_FLOAT_EXACT_BOUND = 2 ** 53
_INT64_MAX = np.iinfo(np.int64).max
K_WINDOW = 32768
BK = 128

INT_BACKEND = "cuda"
_env = os.environ.get("MMJOIN_BACKEND")
_KNOWN = ("auto", "cuda", "blas", "cython", "numpy")

__all__ = ["CountMatrix", "MatrixOverflowError", "INT_BACKEND", "identity", "multiply_counts",
           "theoretical_cost", "CalibrationError", "CalibrationTable", "DEFAULT_PROBE_DIMS", "calibrate",
           "estimate_runtime"]


class CountMatrix:
    """Dense non-negative int64 counts with row/col keys (core.py:37-62)."""

    def __init__(self, data: np.ndarray, row_keys=None, col_keys=None):
        data = np.ascontiguousarray(data, dtype=np.int64)
        if data.ndim != 2:
            raise ValueError("CountMatrix needs a 2-d array")
        if data.size and data.min() < 0:
            raise ValueError("counts must be nonnegative")
        self.data = data
        self.row_keys = row_keys
        self.col_keys = col_keys

    @property
    def rows(self) -> int:
        return self.data.shape[0]

    @property
    def cols(self) -> int:
        return self.data.shape[1]

    def __eq__(self, other):
        return isinstance(other, CountMatrix) and np.array_equal(self.data, other.data)

    def __repr__(self):
        return f"CountMatrix({self.rows}x{self.cols})"


def identity(n: int) -> CountMatrix:
    return CountMatrix(np.eye(n, dtype=np.int64))


def _digits(maxval: int) -> int:
    return max(1, (int(maxval).bit_length() + 7) // 8)


def _rup(a: int, b: int) -> int:
    return -(-a // b) * b


def multiply_counts(a: CountMatrix, b: CountMatrix, cores: int = 1,
                    backend: Optional[str] = None) -> CountMatrix:
    """Exact integer product A @ B on the tensor cores (core.py:95-123)."""
    if a.cols != b.rows:
        raise ValueError(f"dimension mismatch: {a.rows}x{a.cols} @ {b.rows}x{b.cols}")
    if backend is None:
        backend = "auto"
    if backend not in _KNOWN:
        raise ValueError(f"unknown backend {backend!r}")
    am = int(a.data.max()) if a.data.size else 0
    bm = int(b.data.max()) if b.data.size else 0
    bound = a.cols * am * bm
    if bound > _INT64_MAX:
        raise MatrixOverflowError(f"worst-case entry {bound} exceeds int64 capacity")
    if backend == "blas" and bound > _FLOAT_EXACT_BOUND:
        raise MatrixOverflowError(f"worst-case entry {bound} is not exact in float64")
    data = _cuda_product(a.data, b.data, am, bm)
    return CountMatrix(data, row_keys=a.row_keys, col_keys=b.col_keys)


def _cuda_product(a: np.ndarray, b: np.ndarray, am: int, bm: int) -> np.ndarray:
    import torch

    from . import _native as nat
    nat.require_cuda()
    u, v = a.shape
    w = b.shape[1]
    if u == 0 or w == 0:
        return np.zeros((u, w), dtype=np.int64)
    if v == 0 or am == 0 or bm == 0:
        return np.zeros((u, w), dtype=np.int64)
    st = nat.stream_handle()
    kpad = _rup(v, BK)
    urows, wrows = _rup(u, 256), _rup(w, 256)
    da, db = _digits(am), _digits(bm)
    ta = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    tb = torch.from_numpy(np.ascontiguousarray(b)).cuda()
    pa = [torch.empty((urows, kpad), dtype=torch.uint8, device="cuda") for _ in range(da)]
    pb = [torch.empty((wrows, kpad), dtype=torch.uint8, device="cuda") for _ in range(db)]
    for i, t in enumerate(pa):
        t.zero_()
        nat.call("mmj_digit_plane", nat.ptr(ta), u, v, 0, i, nat.ptr(t), kpad, st)
    for j, t in enumerate(pb):
        t.zero_()
        nat.call("mmj_digit_plane", nat.ptr(tb), w, v, 1, j, nat.ptr(t), kpad, st)
    out = torch.zeros((u, wrows), dtype=torch.int64, device="cuda")
    for i in range(da):
        for j in range(db):
            if i + j >= 8:
                continue        # a nonzero term here would exceed the checked int64 bound
            for k0 in range(0, kpad, K_WINDOW):
                kl = min(K_WINDOW, kpad - k0)
                nat.call("mmj_heavy_mma", nat.ptr(pa[i]), urows, nat.ptr(pb[j]), wrows, kpad, k0, kl, 0, u,
                         nat.MODE_ACC64, 8 * (i + j), nat.ptr(out), wrows, 0, 0, st)
    return out[:, :w].cpu().numpy()


def theoretical_cost(u: int, v: int, w: int, omega: float = 3.0) -> float:
    """core.py:126-133: analytic model U*V*W*beta^(omega-3)."""
    if min(u, v, w) < 1:
        raise ValueError("dimensions must be >= 1")
    if not 2 <= omega <= 3:
        raise ValueError("omega must be in [2, 3]")
    beta = min(u, v, w)
    return float(u) * v * w * beta ** (omega - 3)
