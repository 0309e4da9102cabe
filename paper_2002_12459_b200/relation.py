"""Host data model of the path: dictionary-encoded binary relations and their
CSR indexes (the *input format* of the join-project operators).

Mirrors the reference's ``mmjoin.relation`` interface (relation.py:17-204):
same class/function names, attribute names, id-assignment rules and errors,
so an ``IndexedRelation`` built here and one built by the reference carry
identical dense ids (and the engine also accepts the reference's own objects).
Integer-valued inputs are encoded with vectorised numpy instead of the
reference's per-tuple dictionary walk; the first-seen id order is reproduced
exactly.  Nothing in this module is on the timed device path -- the
reference also builds these structures before calling the operators.
"""

from __future__ import annotations

from collections.abc import Mapping
from dataclasses import dataclass, field
from typing import Iterable, Iterator, Optional, TextIO

import numpy as np

from .errors import ParseError

__all__ = [
    "ParseError", "Relation", "IndexedRelation", "ValueIndex", "parse_edge_list",
    "parse_set_family_file", "semi_join_reduce", "semi_join_reduce_many",
    "build_indexed", "gather_ranges", "DegreeStats", "degree_stats",
]


class ValueIndex(Mapping):
    """Read-only value -> dense id map over an int64 value array (ids are
    positions in ``values``); the vectorised stand-in for the reference's
    ``left_ids``/``right_ids`` dicts (relation.py:50-66)."""

    __slots__ = ("values", "_sorted", "_order")

    def __init__(self, values: np.ndarray):
        self.values = np.asarray(values, dtype=np.int64)
        self._order = np.argsort(self.values, kind="stable")
        self._sorted = self.values[self._order]

    def lookup(self, q) -> np.ndarray:
        """Vectorised probe: dense id per query value, -1 when absent."""
        q = np.asarray(q, dtype=np.int64)
        if len(self.values) == 0:
            return np.full(q.shape, -1, dtype=np.int64)
        pos = np.minimum(np.searchsorted(self._sorted, q), len(self._sorted) - 1)
        hit = self._sorted[pos] == q
        return np.where(hit, self._order[pos], -1)

    def __getitem__(self, key):
        if isinstance(key, (bool, np.bool_)) or not isinstance(key, (int, np.integer)):
            raise KeyError(key)
        i = int(self.lookup(np.array([key]))[0])
        if i < 0:
            raise KeyError(key)
        return i

    def __contains__(self, key):
        try:
            self[key]
            return True
        except KeyError:
            return False

    def get(self, key, default=None):
        try:
            return self[key]
        except KeyError:
            return default

    def __iter__(self):
        return iter(self.values.tolist())

    def __len__(self):
        return len(self.values)


def _is_int_array(a) -> bool:
    return isinstance(a, np.ndarray) and a.dtype.kind in "iu"


def _as_int_pairs(raw_pairs) -> Optional[np.ndarray]:
    """(n, 2) int64 array if every raw value is a (non-bool) integer."""
    if _is_int_array(raw_pairs):
        return raw_pairs.reshape(-1, 2).astype(np.int64, copy=False)
    if isinstance(raw_pairs, np.ndarray):
        return None
    seq = raw_pairs if isinstance(raw_pairs, (list, tuple)) else list(raw_pairs)
    if len(seq) == 0:
        return np.empty((0, 2), dtype=np.int64)
    for a, b in seq[:256]:
        if type(a) is not int or type(b) is not int:
            return None
    try:
        arr = np.asarray(seq, dtype=object)
        if arr.ndim != 2 or arr.shape[1] != 2:
            return None
        if not all(type(v) is int for v in arr.ravel()):
            return None
        return arr.astype(np.int64)
    except (OverflowError, ValueError, TypeError):
        return None


def _first_seen(values: np.ndarray):
    """Dense ids in order of first appearance and the values in id order."""
    uniq, first, inv = np.unique(values, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")
    ids_of_rank = np.empty(len(uniq), dtype=np.int64)
    ids_of_rank[order] = np.arange(len(uniq), dtype=np.int64)
    return ids_of_rank[inv.reshape(-1)], uniq[order]


def _dedup_first(arr: np.ndarray) -> np.ndarray:
    """Drop duplicate tuples keeping first occurrences in input order
    (relation.py:53, ``dict.fromkeys``)."""
    if len(arr) < 2:
        return arr
    _, li = np.unique(arr[:, 0], return_inverse=True)
    _, ri = np.unique(arr[:, 1], return_inverse=True)
    key = li.astype(np.int64) * (int(ri.max()) + 1) + ri
    _, first = np.unique(key, return_index=True)
    if len(first) == len(arr):
        return arr
    first.sort()
    return arr[first]


class Relation:
    """A deduplicated binary relation over dense value ids (relation.py:23-97)."""

    def __init__(self, name: str, pairs: np.ndarray, left_values, left_ids, right_values, right_ids):
        self.name = name
        self.pairs = pairs
        self.left_values = left_values
        self.left_ids = left_ids
        self.right_values = right_values
        self.right_ids = right_ids

    @classmethod
    def from_raw_pairs(cls, name: str, raw_pairs: Iterable[tuple], right_values=None,
                       right_ids=None) -> "Relation":
        """relation.py:37-69: encode raw (left, right) pairs, dropping duplicates;
        left ids (and right ids unless a shared dictionary is injected) are
        assigned in first-seen order."""
        shared = right_values is not None
        if shared:
            assert right_ids is not None
        arr = _as_int_pairs(raw_pairs)
        if arr is not None and (not shared or isinstance(right_ids, ValueIndex)):
            arr = _dedup_first(arr)
            lid, lvals = _first_seen(arr[:, 0])
            if shared:
                rid = right_ids.lookup(arr[:, 1])
                if (rid < 0).any():
                    raise KeyError(int(arr[:, 1][rid < 0][0]))
            else:
                rid, rvals = _first_seen(arr[:, 1])
                right_values, right_ids = rvals, ValueIndex(rvals)
            pairs = np.stack([lid, rid], axis=1).astype(np.int64).reshape(-1, 2)
            return cls(name, pairs, lvals, ValueIndex(lvals), right_values, right_ids)
        # generic hashable values: the literal first-seen dictionary walk
        if raw_pairs is not None and not isinstance(raw_pairs, (list, tuple)):
            raw_pairs = list(map(tuple, raw_pairs)) if isinstance(raw_pairs, np.ndarray) else raw_pairs
        if not shared:
            right_values, right_ids = [], {}
        left_values: list = []
        left_ids: dict = {}
        seen = dict.fromkeys(tuple(p) for p in raw_pairs)
        enc = np.empty((len(seen), 2), dtype=np.int64)
        for i, (a, b) in enumerate(seen):
            ai = left_ids.get(a)
            if ai is None:
                ai = left_ids[a] = len(left_values)
                left_values.append(a)
            if shared:
                bi = right_ids[b]
            else:
                bi = right_ids.get(b)
                if bi is None:
                    bi = right_ids[b] = len(right_values)
                    right_values.append(b)
            enc[i, 0] = ai
            enc[i, 1] = bi
        return cls(name, enc, left_values, left_ids, right_values, right_ids)

    @classmethod
    def from_encoded(cls, name: str, pairs: np.ndarray, like: "Relation") -> "Relation":
        """relation.py:71-75: a sub-relation reusing the dictionaries of `like`."""
        return cls(name, pairs, like.left_values, like.left_ids, like.right_values, like.right_ids)

    @property
    def n(self) -> int:
        return len(self.pairs)

    @property
    def dom_left(self) -> int:
        return len(self.left_values)

    @property
    def dom_right(self) -> int:
        return len(self.right_values)

    def raw_pairs(self) -> Iterator[tuple]:
        lv, rv = self.left_values, self.right_values
        if isinstance(lv, np.ndarray) and isinstance(rv, np.ndarray):
            a = lv[self.pairs[:, 0]].tolist()
            b = rv[self.pairs[:, 1]].tolist()
            return iter(zip(a, b))
        return ((lv[a], rv[b]) for a, b in self.pairs.tolist())

    def raw_pair_set(self) -> set:
        return set(self.raw_pairs())

    def raw_array(self) -> Optional[np.ndarray]:
        """(n, 2) int64 raw values, or None for non-integer dictionaries."""
        lv, rv = self.left_values, self.right_values
        if isinstance(lv, np.ndarray) and isinstance(rv, np.ndarray):
            return np.stack([lv[self.pairs[:, 0]], rv[self.pairs[:, 1]]], axis=1)
        return None

    def __repr__(self):
        return f"Relation({self.name!r}, n={self.n}, dom={self.dom_left}x{self.dom_right})"


def parse_edge_list(source: TextIO, name: str = "R") -> Relation:
    """relation.py:100-111: `left right` lines; `#` comments and blanks skipped."""
    pairs = []
    for line_no, line in enumerate(source, start=1):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        toks = line.split()
        if len(toks) != 2:
            raise ParseError(line_no, f"expected 2 tokens, got {len(toks)}")
        pairs.append((toks[0], toks[1]))
    return Relation.from_raw_pairs(name, pairs)


def parse_set_family_file(source: TextIO, name: str = "sets") -> Relation:
    """relation.py:114-116."""
    return parse_edge_list(source, name=name)


def _repr_order(values) -> list:
    return sorted(values, key=repr)


def semi_join_reduce_many(relations: list) -> list:
    """relation.py:119-140: keep tuples whose right value occurs in every
    relation; the results share one right dictionary object, ordered by
    ``repr`` of the values (relation.py:123)."""
    int_valued = all(isinstance(r.right_values, np.ndarray) and isinstance(r.left_values, np.ndarray)
                     for r in relations)
    if int_valued:
        common = relations[0].right_values
        for r in relations[1:]:
            common = np.intersect1d(common, r.right_values)
        common = np.unique(common)
        # repr of a Python int is its decimal string: sort lexicographically
        order = np.argsort(common.astype(str), kind="stable")
        right_values = common[order]
        right_ids = ValueIndex(right_values)
        out = []
        for rel in relations:
            keep = np.isin(rel.right_values, right_values)[rel.pairs[:, 1]]
            kept = rel.pairs[keep]
            raw = np.stack([rel.left_values[kept[:, 0]], rel.right_values[kept[:, 1]]], axis=1)
            out.append(Relation.from_raw_pairs(rel.name, raw, right_values=right_values, right_ids=right_ids))
        return out
    shared = set(relations[0].right_values)
    for rel in relations[1:]:
        shared &= set(rel.right_values)
    right_values = _repr_order(shared)
    right_ids = {v: i for i, v in enumerate(right_values)}
    out = []
    for rel in relations:
        kept = [(a, b) for a, b in rel.raw_pairs() if b in right_ids]
        out.append(Relation.from_raw_pairs(rel.name, kept, right_values=right_values, right_ids=right_ids))
    return out


def semi_join_reduce(r: Relation, s: Relation) -> tuple[Relation, Relation]:
    """relation.py:143-145."""
    red = semi_join_reduce_many([r, s])
    return red[0], red[1]


def _csr(keys: np.ndarray, vals: np.ndarray, dom: int) -> tuple[np.ndarray, np.ndarray]:
    """relation.py:148-154: CSR with each row's values ascending."""
    order = np.lexsort((vals, keys))
    indptr = np.zeros(dom + 1, dtype=np.int64)
    np.cumsum(np.bincount(keys, minlength=dom), out=indptr[1:])
    return indptr, vals[order]


class IndexedRelation:
    """CSR adjacency in both directions plus degrees (relation.py:157-186)."""

    def __init__(self, rel: Relation):
        self.rel = rel
        a, b = rel.pairs[:, 0], rel.pairs[:, 1]
        self.fwd_indptr, self.fwd_indices = _csr(a, b, rel.dom_left)
        self.rev_indptr, self.rev_indices = _csr(b, a, rel.dom_right)
        self.left_deg = np.diff(self.fwd_indptr)
        self.right_deg = np.diff(self.rev_indptr)
        # immutable like the reference's index (engines remember their maxima)
        for arr in (self.fwd_indptr, self.fwd_indices, self.rev_indptr, self.rev_indices, self.left_deg,
                    self.right_deg):
            arr.flags.writeable = False

    def fwd(self, a: int) -> np.ndarray:
        return self.fwd_indices[self.fwd_indptr[a]:self.fwd_indptr[a + 1]]

    def rev(self, b: int) -> np.ndarray:
        return self.rev_indices[self.rev_indptr[b]:self.rev_indptr[b + 1]]

    @property
    def n(self) -> int:
        return self.rel.n

    def shares_right_dict(self, other) -> bool:
        return self.rel.right_values is other.rel.right_values

    def out_join_with(self, other) -> int:
        """|OUT_join| = sum_y deg_R(y) * deg_S(y) (relation.py:181-186)."""
        if not self.shares_right_dict(other):
            raise ValueError("relations do not share a right dictionary; run semi_join_reduce first")
        return int(np.dot(self.right_deg.astype(np.int64), other.right_deg.astype(np.int64)))


def build_indexed(rel: Relation) -> IndexedRelation:
    return IndexedRelation(rel)


def gather_ranges(indptr: np.ndarray, indices: np.ndarray, keys: np.ndarray):
    """relation.py:193-204: concatenated CSR rows for `keys` and their lengths."""
    keys = np.asarray(keys, dtype=np.int64)
    starts = indptr[keys]
    lens = indptr[keys + 1] - starts
    total = int(lens.sum())
    if total == 0:
        return np.empty(0, dtype=indices.dtype), lens
    idx = np.arange(total, dtype=np.int64) - np.repeat(np.cumsum(lens) - lens - starts, lens)
    return indices[idx], lens


# ------------------------------------------------------------ planner inputs
@dataclass
class DegreeStats:
    """relation.py:205-252: degree vectors sorted ascending with prefix sums,
    answering the cost model's threshold queries by binary search.

    ``sum_x`` weighs each tuple (x, y) by the partner's |S.rev(y)|; lightness
    is always judged by this relation's own degrees."""
    n_tuples: int
    dom_left: int
    dom_right: int
    left_sorted: np.ndarray
    right_sorted: np.ndarray
    _cdfx_prefix: np.ndarray = field(repr=False, default=None)
    _sumy_prefix: np.ndarray = field(repr=False, default=None)
    _sumx_prefix: np.ndarray = field(repr=False, default=None)

    @staticmethod
    def _upto(sorted_vec: np.ndarray, delta) -> int:
        """number of entries <= delta"""
        return int(np.searchsorted(sorted_vec, delta, side="right"))

    def count_left(self, delta) -> int:
        """#left values with degree <= delta"""
        return self._upto(self.left_sorted, delta)

    def count_right(self, delta) -> int:
        return self._upto(self.right_sorted, delta)

    def cdfx(self, delta) -> int:
        """tuples whose right value has degree <= delta"""
        return int(self._cdfx_prefix[self._upto(self.right_sorted, delta)])

    def sum_y(self, delta) -> int:
        """sum over right values of degree <= delta of partner degree^2"""
        return int(self._sumy_prefix[self._upto(self.right_sorted, delta)])

    def sum_x(self, delta) -> int:
        """sum over left values of degree <= delta of their partner list lengths"""
        return int(self._sumx_prefix[self._upto(self.left_sorted, delta)])

    @property
    def max_left_deg(self) -> int:
        return int(self.left_sorted[-1]) if len(self.left_sorted) else 0

    @property
    def max_right_deg(self) -> int:
        return int(self.right_sorted[-1]) if len(self.right_sorted) else 0


def degree_stats(idx, partner=None) -> DegreeStats:
    """relation.py:255-277."""
    partner = idx if partner is None else partner
    if not idx.shares_right_dict(partner):
        raise ValueError("partner must share the right dictionary")
    ldeg = np.asarray(idx.left_deg, dtype=np.int64)
    rdeg = np.asarray(idx.right_deg, dtype=np.int64)
    pdeg = np.asarray(partner.right_deg, dtype=np.int64)
    zero = np.zeros(1, dtype=np.int64)
    lo = np.argsort(ldeg, kind="stable")
    # partner list length summed over each left value's forward list
    w = np.concatenate([zero, np.cumsum(pdeg[np.asarray(idx.fwd_indices, dtype=np.int64)])])
    fptr = np.asarray(idx.fwd_indptr, dtype=np.int64)
    per_left = w[fptr[1:]] - w[fptr[:-1]]
    ro = np.argsort(rdeg, kind="stable")
    rs = rdeg[ro]
    return DegreeStats(int(idx.n), int(idx.rel.dom_left), int(idx.rel.dom_right), ldeg[lo], rs,
                       np.concatenate([zero, np.cumsum(rs)]),
                       np.concatenate([zero, np.cumsum(pdeg[ro] * pdeg[ro])]),
                       np.concatenate([zero, np.cumsum(per_left[lo])]))
