"""Equi-depth histograms and the histogram selectivity estimator — SURVEY §8(f) row f4.

The reference's contrast arm (``pkg/src/escdb/catalog.py:153-326``): ``EscConfig(enabled=False,
estimator_mode="histogram")`` orders the builds by estimated instead of exact cardinalities.  It
is an experimental baseline, not the ESC path, so it is built from the device pieces already
here plus the framework's sort:

* the non-NULL values come out of the K1 scan + compaction (``FoldedAtom(col, True)`` = NOT NULL);
* they are sorted on the device (``torch.sort`` — the one library primitive on this arm);
* bucket edges are gathered at the reference's rank positions, bucket ends located with a
  device ``searchsorted``, and per-bucket distinct counts read off a prefix sum of value
  changes — the same integers ``np.sort`` / ``np.searchsorted`` / ``np.unique`` give.

Estimates are host arithmetic identical to the reference's (same float operations in the same
order), so plans and estimates match bit for bit.
"""

from __future__ import annotations

import bisect
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import executor
from . import expr as ex
from . import sorting
from .errors import Inestimable, UnsupportedColumnKind
from .storage import ColumnTable


@dataclass
class EquiDepthHistogram:
    """k buckets over a numeric column; bucket i covers (boundaries[i], boundaries[i+1]] except
    bucket 0 which is closed on both ends.  ``counts`` are exact, ``distincts`` count distinct
    values per bucket (used for equality estimates).  Arrays are host numpy (int64), as in the
    reference."""

    table: str
    column: str
    boundaries: np.ndarray
    counts: np.ndarray
    distincts: np.ndarray
    null_count: int
    row_count: int

    @property
    def non_null(self) -> int:
        return self.row_count - self.null_count


def build_histogram(table: ColumnTable, column: str, buckets: int) -> EquiDepthHistogram:
    """Reference ``build_histogram`` (``catalog.py:178-223``) on the device."""
    col = table.column(column)
    N.require_cuda(col.values, f"column {column!r}")  # no CPU fallback: the arm runs on the device
    if col.kind.is_text:
        raise UnsupportedColumnKind(f"cannot build a histogram over TEXT column {column!r}")
    if col.kind.is_float:
        raise UnsupportedColumnKind(f"cannot build an integer histogram over float column {column!r}")
    if buckets < 1:
        raise ValueError("bucket count must be >= 1")
    if col.nulls is not None and table.row_count:
        # the non-NULL values in row order (the selection excludes NULLs: no NULL outputs)
        sel = executor.select(table, ex.FoldedAtom(ex.ColumnRef(table.name, column), True), capture=[column])
        valid = executor.launch_materialize_selection(sel, [col], sel.count, False, with_nulls=False)[0][0]
    else:
        valid = col.values
    n = int(valid.numel())
    null_count = table.row_count - n
    if n == 0:
        z = np.zeros(0, dtype=np.int64)
        return EquiDepthHistogram(table.name, column, np.zeros(1, dtype=np.int64), z, z.copy(), null_count,
                                  table.row_count)
    # the framework's own stable radix sort, then the sorted column as runs (value, start)
    keys, _, dec = sorting.ordered_keys(valid)
    skeys, _ = sorting.sort_pairs(keys)
    uk, starts, _, _, stats = sorting.runs(skeys, dec, want_counts=False)
    k = min(buckets, n)
    # equi-depth split points at value boundaries; duplicates collapse buckets
    ranks = torch.tensor([0] + [min(n - 1, (i * n) // k - 1) for i in range(1, k + 1)], dtype=torch.int64,
                         device=valid.device)
    at = sorting.rank_values(uk, starts, stats, ranks).cpu().tolist()
    edges = [int(at[0])]
    for e in at[1:]:
        if e > edges[-1]:
            edges.append(int(e))
    if len(edges) == 1:
        edges.append(edges[0])
    boundaries = np.asarray(edges, dtype=np.int64)
    nb = len(boundaries) - 1
    hi, dist = sorting.hist_buckets(uk, starts, stats, n, torch.as_tensor(boundaries, device=valid.device))
    his = hi.cpu().numpy().astype(np.int64)
    los = np.concatenate(([0], his[:-1])).astype(np.int64)
    counts = (his - los).astype(np.int64)
    distincts = dist.cpu().numpy().astype(np.int64)
    return EquiDepthHistogram(table.name, column, boundaries, counts, distincts[:nb], null_count, table.row_count)


# ---- estimates (reference catalog.py:226-326) ------------------------------------------------
# Host arithmetic with the reference's float results: bucket counts are integers, so summing the
# fully covered buckets as ints and converting once equals the reference's running float sum
# (exact below 2**53); bucket searches compare the float constant with Python ints (exact), never
# through a lossy numpy promotion.
def _his(h: EquiDepthHistogram) -> list:
    return [int(x) for x in h.boundaries[1:]]


def _estimate_le(h: EquiDepthHistogram, v: float) -> float:
    """Estimated fraction of ALL rows with value <= v: whole buckets below v, plus a linear share
    (integer values) of the bucket v falls in."""
    nb = int(h.counts.size)
    if nb == 0 or h.row_count == 0:
        return 0.0
    if v != v:  # NaN: the reference's scan stops in bucket 0 with a NaN share, clamped to 0
        width = int(h.boundaries[1]) - int(h.boundaries[0])
        return (float(h.counts[0]) if width == 0 else 0.0) / h.row_count
    full = bisect.bisect_right(_his(h), v)  # buckets with hi <= v are entirely included
    covered = int(h.counts[:full].sum()) if full else 0
    share = 0.0
    if full < nb:
        lo, hi = int(h.boundaries[full]), int(h.boundaries[full + 1])
        if not v < lo:
            width = hi - lo
            frac = (v - lo + 1) / (width + 1) if width > 0 else 1.0
            share = float(h.counts[full]) * min(1.0, max(0.0, frac))
    return (float(covered) + share) / h.row_count


def _estimate_equality(h: EquiDepthHistogram, v: float) -> float:
    """count / distinct values of the bucket holding v (bucket 0 closed below), of all rows."""
    nb = int(h.counts.size)
    if nb == 0 or h.row_count == 0 or v != int(v):
        return 0.0
    b = bisect.bisect_left(_his(h), v)  # first bucket whose upper edge reaches v
    if b >= nb or (b == 0 and v < int(h.boundaries[0])):
        return 0.0
    return float(h.counts[b]) / max(1, int(h.distincts[b])) / h.row_count


def _numeric(value) -> float:
    if isinstance(value, (int, np.integer)):
        return float(value)
    if isinstance(value, float):
        return value
    raise Inestimable(f"constant {value!r} is not numeric")


def _atom_selectivity(hist_for, atom: ex.Expr) -> float:
    if isinstance(atom, ex.FoldedAtom):
        return float(bool(atom.result))
    if isinstance(atom, ex.FnCall):
        raise Inestimable(f"no synopsis can estimate {atom.name}(...)")
    if isinstance(atom, ex.ColumnCompare):
        raise Inestimable("no synopsis for column-to-column comparison")
    ref = atom.col
    if ref.kind is not None and ref.kind.is_text:
        raise Inestimable(f"no histogram over TEXT column {ref}")
    h = hist_for(ref)
    if isinstance(atom, ex.Equality):
        return _estimate_equality(h, _numeric(atom.value))
    if isinstance(atom, ex.Range):
        return max(0.0, _estimate_le(h, _numeric(atom.hi)) - _estimate_le(h, _numeric(atom.lo) - 1))
    if isinstance(atom, ex.Comparison) and atom.op in ("<", "<=", ">", ">=", "<>"):
        v = _numeric(atom.value)
        present = h.non_null / max(1, h.row_count)  # rows a comparison can hold on
        if atom.op == "<=":
            return _estimate_le(h, v)
        if atom.op == "<":
            return _estimate_le(h, v - 1)
        rest = {">": lambda: _estimate_le(h, v), ">=": lambda: _estimate_le(h, v - 1),
                "<>": lambda: _estimate_equality(h, v)}[atom.op]()
        return max(0.0, present - rest)
    raise Inestimable(f"cannot estimate {atom!r}")


def _clamp(x: float) -> float:
    return min(1.0, max(0.0, x))


def estimate_selectivity(hist_for, pred: ex.Expr) -> float:
    """Estimated fraction of rows satisfying ``pred`` in [0, 1]: conjuncts multiply
    (independence), disjuncts by inclusion-exclusion, NOT complements; UDF calls, TEXT columns
    and column comparisons raise Inestimable (the planner then uses its configured guess)."""
    if isinstance(pred, ex.And):
        acc = 1.0
        for item in pred.items:
            acc *= estimate_selectivity(hist_for, item)
        return _clamp(acc)
    if isinstance(pred, ex.Or):
        none = 1.0
        for item in pred.items:
            none *= 1.0 - estimate_selectivity(hist_for, item)
        return _clamp(1.0 - none)
    if isinstance(pred, ex.Not):
        return _clamp(1.0 - estimate_selectivity(hist_for, pred.child))
    return _clamp(_atom_selectivity(hist_for, pred))
