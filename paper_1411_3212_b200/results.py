"""Per-query result containers.

`ResultSet` keeps the reference's dict semantics (`tickjoin/decode.py:23-37`):
issuer id -> ascending object ids, every issued query present, canonical
text via `lines()`.  `ColumnarResult` is the CSR the native tick returns
(offsets over input-query order + ids); `to_result_set` is the only place the
columnar output is turned into Python lists.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import DuplicateResult


@dataclass
class ResultSet:
    by_query: dict = field(default_factory=dict)

    @property
    def total(self) -> int:
        return sum(len(v) for v in self.by_query.values())

    def lines(self) -> list:
        out = []
        for qid, ids in sorted(self.by_query.items()):
            out.append(f"{qid}: {','.join(str(i) for i in ids)}".rstrip())
        return out


@dataclass
class ColumnarResult:
    """CSR of one tick: queries in input order, ids ascending per query."""

    qids: np.ndarray
    offsets: np.ndarray
    ids: np.ndarray

    def of(self, k: int) -> np.ndarray:
        return self.ids[self.offsets[k]:self.offsets[k + 1]]

    def to_result_set(self) -> ResultSet:
        """Issuer-keyed dict; repeated issuers are merged like decode.py:102-123."""
        qids = np.asarray(self.qids, np.int64)
        offs = self.offsets
        if len(np.unique(qids)) == len(qids):
            ids = self.ids
            return ResultSet({int(q): ids[offs[k]:offs[k + 1]].tolist() for k, q in enumerate(qids)})
        acc: dict = {}
        for k, q in enumerate(qids):
            acc.setdefault(int(q), []).append(self.ids[offs[k]:offs[k + 1]])
        out = {}
        for q, parts in acc.items():
            v = np.sort(np.concatenate(parts))
            if len(v) > 1 and np.any(v[1:] == v[:-1]):
                raise DuplicateResult(f"query {q} received a result from two subqueries")
            out[q] = v.tolist()
        return ResultSet(out)


def merge_results(chunks, issued_query_ids) -> ResultSet:
    """Per-issuer union of (query id, object ids) chunks (reference `decode.merge_results`,
    decode.py:102-123): every issued query present (empty when nothing matched), each list
    ascending; `DuplicateResult` on a pair produced twice or on results for a query that was
    never issued.  Vectorised: one lexsort over all (query, object) pairs."""
    out: dict = {int(q): [] for q in issued_query_ids}
    qs, vs = [], []
    for qid, ids in chunks:
        ids = np.asarray(ids, np.int64).ravel()
        if len(ids):
            qs.append(np.full(len(ids), int(qid), np.int64))
            vs.append(ids)
    if not qs:
        return ResultSet(out)
    q = np.concatenate(qs)
    v = np.concatenate(vs)
    order = np.lexsort((v, q))
    q, v = q[order], v[order]
    if len(v) > 1:
        same = (q[1:] == q[:-1]) & (v[1:] == v[:-1])
        if same.any():
            raise DuplicateResult(f"query {int(q[1:][same][0])} received a result from two subqueries")
    starts = np.flatnonzero(np.concatenate([[True], q[1:] != q[:-1]]))
    ends = np.concatenate([starts[1:], [len(q)]])
    for s, e in zip(starts.tolist(), ends.tolist()):
        qid = int(q[s])
        if qid not in out:
            raise DuplicateResult(f"results for a query that was never issued: {qid}")
        out[qid] = v[s:e].tolist()
    return ResultSet(out)
