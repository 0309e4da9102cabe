"""CPU oracle for the mmjoin join-project hot path.

TEST INFRASTRUCTURE -- NOT PRODUCT CODE.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this module, and only as the checker / the
timed CPU reference.  The product package ``paper_2002_12459_b200`` never
imports it and has no CPU fallback.

What it is: a numpy restatement of the reference package ``mmjoin``
(``/root/reference/pkg/src/mmjoin``; paths below are relative to
``/root/reference/pkg/src/mmjoin/``).  Every function cites the reference
lines it follows.  The light passes are written with vectorised numpy
gathers instead of the reference's per-y Python loops; the set of emitted
(x, z) keys, their multiplicities and the ``stats`` counters are identical
because the reference immediately feeds them to ``np.unique``.

Parity pinning: ``tests/golden/make_golden.py`` imports the *reference*
package (read-only, in the build container) and freezes its outputs on seeded
inputs into ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this
oracle bit-exactly against every fixture, plus the reference's own frozen
worked examples (``pkg/tests/conftest.py:119-134``) and pinned constants.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

FULL_JOIN = "fulljoin"          # optimizer.py:14
PARTITIONED = "partitioned"     # optimizer.py:15
FULL_JOIN_CUTOFF = 20           # optimizer.py:18
FLOAT_EXACT = 2 ** 53           # matmul/core.py:23
INT64_MAX = np.iinfo(np.int64).max


class OracleOverflow(OverflowError):
    """matmul/core.py:33-34 (MatrixOverflowError)."""


class OracleStarCap(RuntimeError):
    """joinproject.py:28-29 (StarResourceError)."""


# --------------------------------------------------------------------------
# data model: dictionary encoding + CSR   (relation.py:23-190)
# --------------------------------------------------------------------------

def _first_seen_ids(values: np.ndarray):
    """Dense ids in first-appearance order (relation.py:52-59)."""
    uniq, first, inv = np.unique(values, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")          # value rank -> id
    rank_to_id = np.empty(len(uniq), dtype=np.int64)
    rank_to_id[order] = np.arange(len(uniq), dtype=np.int64)
    return rank_to_id[inv], uniq[order]


def _dedup_keep_first(left: np.ndarray, right: np.ndarray):
    """`dict.fromkeys` tuple dedup keeping first occurrences (relation.py:53)."""
    if len(left) == 0:
        return left, right
    _, lid = np.unique(left, return_inverse=True)
    _, rid = np.unique(right, return_inverse=True)
    key = lid.astype(np.int64) * (int(rid.max()) + 1) + rid
    _, first = np.unique(key, return_index=True)
    first.sort()
    return left[first], right[first]


@dataclass
class ORel:
    """Encoded relation + both CSR directions (relation.py:23-35, 157-166)."""
    pairs: np.ndarray                 # (n, 2) int64 dense ids
    left_values: Sequence
    right_values: Sequence
    right_token: object = None        # identity of the right dictionary
    _csr: dict = field(default_factory=dict, repr=False)

    @property
    def n(self):
        return len(self.pairs)

    @property
    def dom_left(self):
        return len(self.left_values)

    @property
    def dom_right(self):
        return len(self.right_values)

    def _build(self, key_col, dom):
        if key_col not in self._csr:
            keys = self.pairs[:, key_col]
            vals = self.pairs[:, 1 - key_col]
            order = np.lexsort((vals, keys))          # relation.py:149
            indptr = np.zeros(dom + 1, dtype=np.int64)
            np.add.at(indptr, keys + 1, 1)            # relation.py:151-153
            np.cumsum(indptr, out=indptr)
            self._csr[key_col] = (indptr, vals[order])
        return self._csr[key_col]

    def fwd(self):
        return self._build(0, self.dom_left)

    def rev(self):
        return self._build(1, self.dom_right)

    @property
    def left_deg(self):
        return np.diff(self.fwd()[0])                 # relation.py:165

    @property
    def right_deg(self):
        return np.diff(self.rev()[0])                 # relation.py:166

    def raw_pairs(self):
        lv, rv = self.left_values, self.right_values
        return [(lv[a], rv[b]) for a, b in self.pairs.tolist()]


def encode(raw_pairs, shared_right: Optional[tuple] = None) -> ORel:
    """relation.py:37-69 (Relation.from_raw_pairs).

    ``raw_pairs`` is an (n, 2) integer array or an iterable of 2-tuples.
    ``shared_right`` is (right_values, right_ids, token) as produced by
    :func:`semi_join_many`.
    """
    arr = None
    if isinstance(raw_pairs, np.ndarray) and raw_pairs.dtype.kind in "iu":
        arr = raw_pairs.reshape(-1, 2).astype(np.int64)
    if arr is not None:
        left, right = _dedup_keep_first(arr[:, 0], arr[:, 1])
        lid, lvals = _first_seen_ids(left)
        if shared_right is None:
            rid, rvals = _first_seen_ids(right)
            rvals = rvals.tolist()
            token = object()
        else:
            rvals, rids, token = shared_right
            keys = np.asarray(rvals, dtype=np.int64)
            order = np.argsort(keys, kind="stable")
            pos = np.searchsorted(keys, right, sorter=order)
            rid = order[pos]
        pairs = np.stack([lid, rid], axis=1).astype(np.int64).reshape(-1, 2)
        return ORel(pairs, lvals.tolist(), rvals, token)
    # generic hashable values: literal first-seen dictionary walk
    seen = dict.fromkeys(tuple(p) for p in raw_pairs)
    lids: dict = {}
    lvals: list = []
    if shared_right is None:
        rvals, rids, token = [], {}, object()
    else:
        rvals, rids, token = shared_right
    out = np.empty((len(seen), 2), dtype=np.int64)
    for i, (a, b) in enumerate(seen):
        ai = lids.setdefault(a, len(lvals))
        if ai == len(lvals):
            lvals.append(a)
        if shared_right is None:
            bi = rids.setdefault(b, len(rvals))
            if bi == len(rvals):
                rvals.append(b)
        else:
            bi = rids[b]
        out[i] = (ai, bi)
    return ORel(out, lvals, rvals, token)


def semi_join_many(rels: Sequence[ORel]) -> list:
    """relation.py:119-140: shared right dictionary = intersection of the
    right domains sorted by ``repr``; tuples with other right values drop and
    each relation is re-encoded (first-seen left ids among kept tuples)."""
    common = set(rels[0].right_values)
    for r in rels[1:]:
        common &= set(r.right_values)
    rvals = sorted(common, key=repr)
    rids = {v: i for i, v in enumerate(rvals)}
    shared = (rvals, rids, object())
    out = []
    for r in rels:
        keep_right = np.fromiter((v in rids for v in r.right_values), dtype=bool,
                                 count=r.dom_right)
        kept = r.pairs[keep_right[r.pairs[:, 1]]] if r.n else r.pairs
        if _int_valued(r):
            lv = np.asarray(r.left_values, dtype=np.int64)
            rv = np.asarray(r.right_values, dtype=np.int64)
            raw = np.stack([lv[kept[:, 0]], rv[kept[:, 1]]], axis=1)
            out.append(encode(raw, shared))
        else:
            lv, rv = r.left_values, r.right_values
            out.append(encode([(lv[a], rv[b]) for a, b in kept.tolist()], shared))
    return out


def _int_valued(r: ORel) -> bool:
    vals = list(r.left_values[:64]) + list(r.right_values[:64])
    return all(isinstance(v, (int, np.integer)) and not isinstance(v, bool) for v in vals) \
        and r.dom_left > 0 and r.dom_right > 0


def shares_right(rels: Sequence[ORel]) -> bool:
    return all(r.right_token is rels[0].right_token for r in rels[1:])


def ensure_reduced(rels: Sequence[ORel]) -> list:
    """joinproject.py:92-97."""
    if shares_right(rels):
        return list(rels)
    return semi_join_many(rels)


def gather(indptr: np.ndarray, indices: np.ndarray, keys: np.ndarray):
    """relation.py:193-204 (gather_ranges): concatenated CSR rows."""
    keys = np.asarray(keys, dtype=np.int64)
    lo = indptr[keys]
    ln = indptr[keys + 1] - lo
    tot = int(ln.sum())
    if tot == 0:
        return np.empty(0, dtype=indices.dtype), ln
    start = np.cumsum(ln) - ln
    pos = np.arange(tot, dtype=np.int64) - np.repeat(start - lo, ln)
    return indices[pos], ln


# --------------------------------------------------------------------------
# planner   (optimizer.py:103-138, 200-208)
# --------------------------------------------------------------------------

@dataclass
class OPlan:
    strategy: str
    delta1: int
    delta2: int


def estimate_output_size(dom_x: int, out_join: int, n: int) -> int:
    """optimizer.py:103-114."""
    if out_join < 0 or n < 1:
        raise ValueError("out_join >= 0 and n >= 1 required")
    if out_join == 0 or dom_x == 0:
        return 0
    lo = max(dom_x, (out_join / n) ** 2)
    hi = min(dom_x * dom_x, out_join)
    est = math.ceil(math.sqrt(lo * hi))
    if hi >= 1:
        est = max(1, min(est, hi))
    return int(est)


def ceil_cbrt_ratio(num: int, den: int) -> int:
    """optimizer.py:117-124: least k >= 1 with k^3 * den >= num."""
    k = max(1, round((num / den) ** (1.0 / 3.0)))
    while k ** 3 * den < num:
        k += 1
    while k > 1 and (k - 1) ** 3 * den >= num:
        k -= 1
    return k


def closed_form_thresholds(n: int, out_est: int):
    """optimizer.py:127-138."""
    if n < 1 or out_est < 1:
        raise ValueError("n >= 1 and out_est >= 1 required")
    if out_est <= n:
        d1 = ceil_cbrt_ratio(out_est, 1)
        d2 = ceil_cbrt_ratio(n ** 3, out_est ** 2)
    else:
        d1 = d2 = ceil_cbrt_ratio(2 * n * n, n + out_est)
    return max(1, min(d1, n)), max(1, min(d2, n))


def out_join(r: ORel, s: ORel) -> int:
    """relation.py:181-186."""
    return int(np.dot(r.right_deg, s.right_deg))


def default_plan(r: ORel, s: ORel) -> OPlan:
    """optimizer.py:200-208."""
    n = max(r.n, s.n)
    oj = out_join(r, s)
    if oj <= FULL_JOIN_CUTOFF * n or n == 0:
        return OPlan(FULL_JOIN, max(n, 1), max(n, 1))
    est = max(1, estimate_output_size(r.dom_left, oj, n))
    d1, d2 = closed_form_thresholds(n, est)
    return OPlan(PARTITIONED, d1, d2)


# --------------------------------------------------------------------------
# exact count-matrix product   (matmul/core.py:69-123)
# --------------------------------------------------------------------------

def matmul_exact(a: np.ndarray, b: np.ndarray, backend: str = "auto") -> np.ndarray:
    """matmul/core.py:95-123 (multiply_counts) on plain int64 arrays."""
    a = np.ascontiguousarray(a, dtype=np.int64)
    b = np.ascontiguousarray(b, dtype=np.int64)
    if a.shape[1] != b.shape[0]:
        raise ValueError("dimension mismatch")
    amax = int(a.max()) if a.size else 0
    bmax = int(b.max()) if b.size else 0
    bound = a.shape[1] * amax * bmax
    if bound > INT64_MAX:
        raise OracleOverflow(bound)
    if backend == "auto":
        backend = "blas" if bound <= FLOAT_EXACT else "int64"
    if backend == "blas":
        if bound > FLOAT_EXACT:
            raise OracleOverflow(bound)
        return np.rint(a.astype(np.float64) @ b.astype(np.float64)).astype(np.int64)
    if backend in ("int64", "cython", "numpy"):
        out = np.zeros((a.shape[0], b.shape[1]), dtype=np.int64)
        for k0 in range(0, a.shape[1], 256):       # core.py:69-74
            out += a[:, k0:k0 + 256] @ b[k0:k0 + 256]
        return out
    raise ValueError(f"unknown backend {backend!r}")


# --------------------------------------------------------------------------
# two-path operator   (joinproject.py:100-225)
# --------------------------------------------------------------------------

@dataclass
class OOut:
    codes: np.ndarray
    dims: tuple
    counts: Optional[np.ndarray]
    stats: dict

    def tuples(self):
        out = np.empty((len(self.codes), len(self.dims)), dtype=np.int64)
        rem = self.codes
        for i in range(len(self.dims) - 1, -1, -1):
            rem, out[:, i] = np.divmod(rem, self.dims[i])
        return out


def _code_space_ok(dims):
    """joinproject.py:87-89."""
    if math.prod(max(int(d), 1) for d in dims) >= 2 ** 62:
        raise OracleStarCap("combined domain too large to encode")


def light_masks(r: ORel, s: ORel, d1: int, d2: int):
    """joinproject.py:178-180 (identical to 103 / 123-126)."""
    light_y = (r.right_deg <= d1) & (s.right_deg <= d1)
    return light_y, r.left_deg <= d2, s.left_deg <= d2


def partition(r: ORel, s: ORel, d1: int, d2: int):
    """joinproject.py:100-116: (light_mask_R, light_mask_S) over tuples."""
    if d1 < 1 or d2 < 1:
        raise ValueError("thresholds must be >= 1")
    r, s = ensure_reduced([r, s])
    light_y = (r.right_deg <= d1) & (s.right_deg <= d1)
    masks = []
    for rel in (r, s):
        masks.append((rel.left_deg[rel.pairs[:, 0]] <= d2) | light_y[rel.pairs[:, 1]])
    return r, s, masks[0], masks[1]


def heavy_operands(r: ORel, s: ORel, d1: int, d2: int):
    """joinproject.py:119-143: dense 0/1 M1[x_h, y_h], M2[y_h, z_h] plus the
    key vectors, or None when one heavy side is empty."""
    light_y, _, _ = light_masks(r, s, d1, d2)
    hx = np.flatnonzero(r.left_deg > d2)
    hy = np.flatnonzero(~light_y)
    hz = np.flatnonzero(s.left_deg > d2)
    if len(hx) == 0 or len(hy) == 0 or len(hz) == 0:
        return None
    py = np.full(r.dom_right, -1, dtype=np.int64)
    py[hy] = np.arange(len(hy))

    def dense(rel, heavy_left):
        pl = np.full(rel.dom_left, -1, dtype=np.int64)
        pl[heavy_left] = np.arange(len(heavy_left))
        a, b = pl[rel.pairs[:, 0]], py[rel.pairs[:, 1]]
        ok = (a >= 0) & (b >= 0)
        m = np.zeros((len(heavy_left), len(hy)), dtype=np.int64)
        m[a[ok], b[ok]] = 1
        return m

    return dense(r, hx), dense(s, hz).T.copy(), hx, hy, hz


def two_path(r: ORel, s: ORel, plan: Optional[OPlan] = None,
             want_counts: bool = False) -> OOut:
    """joinproject.py:155-225 (two_path_join)."""
    r, s = ensure_reduced([r, s])
    if plan is None:
        plan = default_plan(r, s)
    if plan.strategy not in (FULL_JOIN, PARTITIONED):          # optimizer.py:34-38
        raise ValueError(f"unknown strategy {plan.strategy!r}")
    if plan.strategy == PARTITIONED and (plan.delta1 < 1 or plan.delta2 < 1):
        raise ValueError("partitioned plans need delta1, delta2 >= 1")
    if plan.strategy == FULL_JOIN:
        out = full_join(r, s, want_counts)
        out.stats["plan"] = plan
        return out
    d1, d2 = plan.delta1, plan.delta2
    dims = (r.dom_left, s.dom_left)
    _code_space_ok(dims)
    dz = dims[1]
    light_y, light_x, light_z = light_masks(r, s, d1, d2)
    s_rev_ptr, s_rev_idx = s.rev()
    rx, ry = r.pairs[:, 0], r.pairs[:, 1]
    parts = [np.empty(0, dtype=np.int64)]

    # pass 1 (joinproject.py:183-186): y light in both relations.  The
    # reference walks light y and emits rev_R(y) x rev_S(y); here every R
    # tuple with a light y picks up rev_S(y) -- the same multiset of keys.
    sel = light_y[ry] & (s.right_deg[ry] > 0)
    zs, ln = gather(s_rev_ptr, s_rev_idx, ry[sel])
    parts.append(np.repeat(rx[sel], ln) * dz + zs)

    # pass 2 (joinproject.py:188-193): light x, heavy y.
    sel = light_x[rx] & ~light_y[ry]
    zs, ln = gather(s_rev_ptr, s_rev_idx, ry[sel])
    parts.append(np.repeat(rx[sel], ln) * dz + zs)

    # pass 3 (joinproject.py:195-203): light z, heavy y, heavy x.
    sz, sy = s.pairs[:, 0], s.pairs[:, 1]
    sel = light_z[sz] & ~light_y[sy]
    if sel.any():
        hp = r.pairs[~light_x[rx]]
        order = np.lexsort((hp[:, 0], hp[:, 1]))
        hptr = np.zeros(r.dom_right + 1, dtype=np.int64)
        np.add.at(hptr, hp[:, 1] + 1, 1)
        np.cumsum(hptr, out=hptr)
        xs, ln = gather(hptr, hp[order, 0], sy[sel])
        parts.append(xs * dz + np.repeat(sz[sel], ln))

    light_codes = np.concatenate(parts)
    inter = len(light_codes)

    ops = heavy_operands(r, s, d1, d2)
    if ops is None:
        hcodes = np.empty(0, dtype=np.int64)
        hcnt = np.empty(0, dtype=np.int64)
    else:
        m1, m2, hx, _, hz = ops
        prod = matmul_exact(m1, m2)                              # joinproject.py:210
        i, j = np.nonzero(prod)
        hcodes = hx[i] * dz + hz[j]
        hcnt = prod[i, j]

    stats = {"light_intermediate": inter, "plan": plan, "heavy_pairs": len(hcodes)}
    if want_counts:                                              # joinproject.py:220-222
        lc, lcnt = np.unique(light_codes, return_counts=True)
        allc = np.concatenate([lc, hcodes])
        alln = np.concatenate([lcnt.astype(np.int64), hcnt])
        u, inv = np.unique(allc, return_inverse=True)           # _merge_counts 146-152
        cnt = np.zeros(len(u), dtype=np.int64)
        np.add.at(cnt, inv, alln)
        return OOut(u, dims, cnt, stats)
    return OOut(np.unique(np.concatenate([light_codes, hcodes])), dims, None, stats)


def full_join(r: ORel, s: ORel, want_counts: bool = False) -> OOut:
    """joinproject.py:228-248 (full_join_dedup)."""
    r, s = ensure_reduced([r, s])
    dims = (r.dom_left, s.dom_left)
    _code_space_ok(dims)
    sp, si = s.rev()
    rx, ry = r.pairs[:, 0], r.pairs[:, 1]
    zs, ln = gather(sp, si, ry)
    codes = np.repeat(rx, ln) * dims[1] + zs
    stats = {"intermediate": len(codes)}
    if want_counts:
        u, c = np.unique(codes, return_counts=True)
        return OOut(u, dims, c.astype(np.int64), stats)
    return OOut(np.unique(codes), dims, None, stats)


# --------------------------------------------------------------------------
# star operator   (joinproject.py:274-378) -- small cases only (Python y loop)
# --------------------------------------------------------------------------

def _cross(lists, dims):
    """joinproject.py:274-278."""
    c = np.asarray(lists[0], dtype=np.int64)
    for lst, d in zip(lists[1:], dims[1:]):
        c = (c[:, None] * d + np.asarray(lst, dtype=np.int64)[None, :]).ravel()
    return c


def star(rels: Sequence[ORel], d1: int, d2: int, want_counts: bool = False,
         cap: int = 1 << 22) -> OOut:
    """joinproject.py:281-378 (star_join)."""
    k = len(rels)
    if not 2 <= k <= 4:
        raise ValueError("star_join supports 2 <= k <= 4 relations")
    if d1 < 1 or d2 < 1:
        raise ValueError("thresholds must be >= 1")
    rels = ensure_reduced(rels)
    dims = [r.dom_left for r in rels]
    _code_space_ok(dims)
    deg = np.stack([r.right_deg for r in rels])
    revs = [r.rev() for r in rels]
    light_left = [r.left_deg <= d2 for r in rels]
    def rev(i, y):
        p, ix = revs[i]
        return ix[p[y]:p[y + 1]]

    parts = [np.empty(0, dtype=np.int64)]
    alive = np.flatnonzero((deg > 0).all(axis=0))
    for j in range(k):                                          # 305-313
        for y in alive:
            ls = [rev(i, y) for i in range(k)]
            lj = ls[j][light_left[j][ls[j]]]
            if len(lj):
                ls[j] = lj
                parts.append(_cross(ls, dims))
    diamond = (deg <= d1).sum(axis=0) >= k - 1                  # 315-318
    for y in np.flatnonzero(diamond & (deg > 0).all(axis=0)):
        parts.append(_cross([rev(i, y) for i in range(k)], dims))

    heavy_left = [np.flatnonzero(r.left_deg > d2) for r in rels]   # 321-322
    heavy_y = np.flatnonzero((deg > d1).sum(axis=0) >= 2)
    g1 = list(range(math.ceil(k / 2)))
    g2 = list(range(math.ceil(k / 2), k))
    hcodes = np.empty(0, dtype=np.int64)
    hdims: list = []
    if len(heavy_y) and all(len(h) for h in heavy_left):
        for grp in (g1, g2):                                    # 327-333
            rows = math.prod(len(heavy_left[i]) for i in grp)
            if rows > cap:
                raise OracleStarCap(f"{rows} heavy combinations exceed the cap")
        py = np.full(rels[0].dom_right, -1, dtype=np.int64)
        py[heavy_y] = np.arange(len(heavy_y))

        def member(i):                                          # 337-344
            pl = np.full(dims[i], -1, dtype=np.int64)
            pl[heavy_left[i]] = np.arange(len(heavy_left[i]))
            a = pl[rels[i].pairs[:, 0]]
            b = py[rels[i].pairs[:, 1]]
            ok = (a >= 0) & (b >= 0)
            m = np.zeros((len(heavy_left[i]), len(heavy_y)), dtype=np.int64)
            m[a[ok], b[ok]] = 1
            return m

        def khatri_rao(grp):                                    # 346-351
            v = member(grp[0])
            for i in grp[1:]:
                v = (v[:, None, :] * member(i)[None, :, :]).reshape(-1, len(heavy_y))
            return v

        v, w = khatri_rao(g1), khatri_rao(g2)
        m = matmul_exact(v, np.ascontiguousarray(w.T))          # 353-356
        hdims = [v.shape[0], w.shape[0], len(heavy_y)]
        ri, ci = np.nonzero(m)
        c1 = np.unravel_index(ri, tuple(len(heavy_left[i]) for i in g1))
        c2 = np.unravel_index(ci, tuple(len(heavy_left[i]) for i in g2))
        cols = [heavy_left[i][c1[p]] for p, i in enumerate(g1)]
        cols += [heavy_left[i][c2[p]] for p, i in enumerate(g2)]
        hcodes = np.zeros_like(cols[0])
        for col, d in zip(cols, dims):                          # _encode 80-84
            hcodes = hcodes * d + col

    codes = np.unique(np.concatenate(parts + [hcodes]))
    stats = {"heavy_dims": hdims}
    if not want_counts:
        return OOut(codes, tuple(dims), None, stats)
    full = [np.empty(0, dtype=np.int64)]                        # 372-378
    for y in alive:
        full.append(_cross([rev(i, y) for i in range(k)], dims))
    u, c = np.unique(np.concatenate(full), return_counts=True)
    assert np.array_equal(u, codes)
    return OOut(u, tuple(dims), c.astype(np.int64), stats)


# --------------------------------------------------------------------------
# applications   (apps.py:26-72, 314-351)
# --------------------------------------------------------------------------

def ssj(fam: ORel, c: int, plan: Optional[OPlan] = None) -> dict:
    """apps.py:57-72 (ssj_mmjoin): {(a, b): overlap} over dense set ids, a < b."""
    if c < 1:
        raise ValueError("c must be >= 1")
    res = two_path(fam, fam, plan, want_counts=True)
    t = res.tuples()
    keep = (t[:, 0] < t[:, 1]) & (res.counts >= c)
    return {(int(a), int(b)): int(n)
            for (a, b), n in zip(t[keep].tolist(), res.counts[keep].tolist())}


def ssj_arrays(fam: ORel, c: int, plan: Optional[OPlan] = None):
    """Array form of :func:`ssj`: (a, b, count) sorted by code."""
    res = two_path(fam, fam, plan, want_counts=True)
    t = res.tuples()
    keep = (t[:, 0] < t[:, 1]) & (res.counts >= c)
    return t[keep, 0], t[keep, 1], res.counts[keep]


def bsi(r: ORel, s: ORel, batch_a, batch_b) -> np.ndarray:
    """apps.py:314-351 (bsi_answer_batch) restated per query.

    Returns int8 answers: 1 = True, 0 = False, -1 = None (an id unknown to the
    *unreduced* relation, apps.py:321-329).  The reference answers through a
    filtered two-path join over raw values; (a, b) is in that join exactly
    when R[a] and S[b] share a raw y value, which is what is computed here
    (vectorised: expand every known query's two adjacency lists into
    (query, y) keys and intersect the key sets).
    """
    ba = np.asarray(batch_a, dtype=np.int64)
    bb = np.asarray(batch_b, dtype=np.int64)
    ia = _lookup(np.asarray(r.left_values, dtype=np.int64), ba)
    ib = _lookup(np.asarray(s.left_values, dtype=np.int64), bb)
    ans = np.full(len(ba), -1, dtype=np.int8)
    known = np.flatnonzero((ia >= 0) & (ib >= 0))
    ans[known] = 0
    if len(known) == 0:
        return ans
    # one shared raw-y rank space for both relations
    rrv = np.asarray(r.right_values, dtype=np.int64)
    srv = np.asarray(s.right_values, dtype=np.int64)
    yvals = np.union1d(rrv, srv)
    rrank = np.searchsorted(yvals, rrv)
    srank = np.searchsorted(yvals, srv)
    rp, ri = r.fwd()
    sp, si = s.fwd()
    ny = len(yvals)
    ry, rl = gather(rp, ri, ia[known])
    sy, sl = gather(sp, si, ib[known])
    qr = np.repeat(np.arange(len(known), dtype=np.int64), rl)
    qs = np.repeat(np.arange(len(known), dtype=np.int64), sl)
    kr = qr * ny + rrank[ry]
    ks = qs * ny + srank[sy]
    hit = np.isin(kr, ks)
    yes = np.zeros(len(known), dtype=bool)
    yes[qr[hit]] = True
    ans[known[yes]] = 1
    return ans


def _lookup(vals: np.ndarray, q: np.ndarray) -> np.ndarray:
    """Dense id of each raw value in ``q`` (dictionary probe), -1 if absent."""
    if len(vals) == 0:
        return np.full(len(q), -1, dtype=np.int64)
    order = np.argsort(vals, kind="stable")
    pos = np.minimum(np.searchsorted(vals, q, sorter=order), len(vals) - 1)
    hitv = vals[order[pos]] == q
    return np.where(hitv, order[pos], -1)
