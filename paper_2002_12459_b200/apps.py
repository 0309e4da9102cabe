"""Applications on the B200 join-project engine (drop-in for ``mmjoin.apps``
on the hot path: apps.py:26-72, 291-351).

  SetFamily            apps.py:26-50
  ssj_mmjoin           apps.py:57-72   exact overlap counts on the tensor-core
                                       count path; the (a < b, count >= c)
                                       filter runs inside the emission kernel
  ssj_ordered          apps.py:291-294
  scj_join_project     apps.py:297-304
  bsi_batch_size       apps.py:307-311
  bsi_answer_batch     apps.py:314-351 per-query heavy-y bitset test plus a
                                       light-list merge intersection (bsi.cu)

``*_arrays`` variants return numpy arrays for outputs too large for Python
dicts/lists (cfg4: ~2.4e8 pairs; cfg5: 4M answers).
"""

from __future__ import annotations

import math
from typing import Optional, Sequence

import numpy as np

from .optimizer import ThresholdPlan
from .relation import IndexedRelation, Relation, ValueIndex, build_indexed

__all__ = ["SetFamily", "ssj_mmjoin", "ssj_mmjoin_arrays", "ssj_ordered", "scj_join_project",
           "bsi_batch_size", "bsi_answer_batch", "bsi_answer_batch_arrays"]


class SetFamily:
    """A family of non-empty sets stored as a (set-id, element-id) relation."""

    def __init__(self, relation: Relation):
        self.relation = relation
        self.indexed = build_indexed(relation)
        self._sizes = np.asarray(self.indexed.left_deg)

    @property
    def sets(self) -> dict:
        return {a: self.indexed.fwd(a) for a in range(self.relation.dom_left)}

    @classmethod
    def from_dict(cls, sets: dict) -> "SetFamily":
        pairs = [(a, e) for a, elems in sets.items() for e in elems]
        return cls(Relation.from_raw_pairs("sets", pairs))

    def __len__(self):
        return self.relation.dom_left

    def size(self, a: int) -> int:
        return int(self._sizes[a])

    def raw_id(self, a: int):
        return self.relation.left_values[a]

    def raw_pair(self, a: int, b: int) -> tuple:
        return (self.raw_id(a), self.raw_id(b))


def _ssj_plan(idx, plan: Optional[ThresholdPlan], c: int = 1, upper_only: bool = True) -> ThresholdPlan:
    from .optimizer import gpu_plan
    return plan if plan is not None else gpu_plan(idx, idx, counts=True, min_count=c, upper_only=upper_only)


def ssj_mmjoin_arrays(family: SetFamily, c: int, plan: Optional[ThresholdPlan] = None,
                      chunk_rows: Optional[int] = None):
    """(a, b, overlap) int64 arrays of every unordered pair a < b (dense set
    ids) with |a n b| >= c, in ascending (a, b) order."""
    if c < 1:
        raise ValueError("c must be >= 1")
    from .joinproject import _engine
    idx = family.indexed
    plan = _ssj_plan(idx, plan, int(c))
    plan.validate()
    eng = _engine(idx, idx, plan, True, min_count=int(c), upper_only=True, chunk_rows=chunk_rows)
    dz = idx.rel.dom_left
    codes, counts = [], []

    def sink(ch):
        codes.append(ch.codes.cpu().numpy())
        counts.append(ch.counts.cpu().numpy())

    eng.run(sink)
    cd = np.concatenate(codes) if codes else np.empty(0, dtype=np.int64)
    cn = (np.concatenate(counts) if counts else np.empty(0, dtype=np.int32)).astype(np.int64)
    return cd // dz, cd % dz, cn


def ssj_mmjoin(family: SetFamily, c: int, plan: Optional[ThresholdPlan] = None) -> dict:
    """apps.py:65-72: {(a, b): |a n b|} over dense set ids with a < b and
    overlap >= c; insertion order = ascending code (as the reference's)."""
    a, b, n = ssj_mmjoin_arrays(family, c, plan)
    return dict(zip(zip(a.tolist(), b.tolist()), n.tolist()))


def ssj_ordered(family: SetFamily, c: int) -> list:
    """apps.py:291-294: ssj_mmjoin sorted by overlap descending, pair ascending."""
    a, b, n = ssj_mmjoin_arrays(family, c)
    order = np.lexsort((b, a, -n))
    return [((int(a[i]), int(b[i])), int(n[i])) for i in order]


def scj_join_project(family: SetFamily) -> set:
    """apps.py:297-304: ordered containment pairs (a, b), a != b, a subset of b,
    i.e. overlap(a, b) == |a| on the exact count path."""
    from .joinproject import two_path_join
    idx = family.indexed
    res = two_path_join(idx, idx, plan=_ssj_plan(idx, None, upper_only=False), want_counts=True)
    t = res.tuples()
    sizes = np.asarray(idx.left_deg)
    keep = (t[:, 0] != t[:, 1]) & (res.counts == sizes[t[:, 0]])
    return set(map(tuple, t[keep].tolist()))


def bsi_batch_size(rate: float, n: int) -> int:
    """apps.py:307-311: latency-optimal batch size ceil((B*N)^(3/5))."""
    if rate < 1 or n < 1:
        raise ValueError("rate and n must be >= 1")
    return math.ceil((rate * n) ** 0.6)


def bsi_answer_batch_arrays(r, s, batch_a, batch_b, heavy_bits: int = 256) -> np.ndarray:
    """int8 answers per query: 1 = sets intersect, 0 = disjoint, -1 = an id
    unknown to the (unreduced) relation (apps.py:321-329)."""
    from .bsi import answer_batch
    return answer_batch(r, s, batch_a, batch_b, heavy_bits=heavy_bits)


def bsi_answer_batch(r, s, batch: Sequence[tuple]) -> list:
    """apps.py:314-351: answer[i] True iff sets a_i (in R) and b_i (in S)
    intersect; unknown set ids yield None for that query."""
    if len(batch) == 0:
        return []
    ba = [a for a, _ in batch]
    bb = [b for _, b in batch]
    ans = bsi_answer_batch_arrays(r, s, ba, bb)
    return [None if v < 0 else bool(v) for v in ans.tolist()]
