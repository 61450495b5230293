"""CPU ORACLE for the ESC hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / ``--impl
reference`` legs may import this module, and only as the checker or as the timed reference CPU
implementation.  The product package never imports it (there is no CPU fallback).

This is a numpy restatement of the reference's algorithm for the selectivity sub-query
(``/root/reference/pkg/src/escdb``, Python 3.12 + numpy 2.3).  Each function cites the reference
lines it follows.  It works on plain numpy columns and on predicates in the JSON form below, so
it shares no code with the product.  It is PINNED against golden vectors produced by running the
reference itself (``tests/golden/make_golden.py``; checked by ``tests/test_oracle_golden.py``).

Predicate JSON (one list per node)::

    ["eq", ref, v]            Equality            ["cmp", ref, op, v]     Comparison
    ["range", ref, lo, hi]    Range (inclusive)   ["colcmp", ref, op, ref] ColumnCompare
    ["fn", name, [ref...], op, v]  FnCall         ["folded", ref, bool]    FoldedAtom
    ["and", [...]]  ["or", [...]]  ["not", x]
    ref = [column_name, decimal_scale_or_null]

Values are ints, floats (``{"float": "nan"|"inf"|"-inf"}`` for non-finite) or strings.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


class OracleExecutionError(Exception):
    """Stands for the reference's ExecutionError (same message text)."""


@dataclass
class OColumn:
    values: np.ndarray
    nulls: np.ndarray            # bool, True = NULL (reference Column.null_mask)
    kind: str = "INT64"
    scale: int = 0
    words: list | None = None    # dictionary strings (TEXT)


@dataclass
class OTable:
    name: str
    columns: dict = field(default_factory=dict)  # name -> OColumn (insertion = base order)

    @property
    def row_count(self) -> int:
        return len(next(iter(self.columns.values())).values)


def decode_value(v):
    if isinstance(v, dict) and "float" in v:
        return float(v["float"])
    return v


_OPS = {
    "=": np.equal, "<>": np.not_equal, "<": np.less, "<=": np.less_equal,
    ">": np.greater, ">=": np.greater_equal,
}


def _compare(values, op, const):
    """executor.py:97-110 — numpy comparison (NEP 50 promotion applies)."""
    if op not in _OPS:
        raise OracleExecutionError(f"unknown comparison operator {op!r}")
    return _OPS[op](values, const)


def _text_lut(col: OColumn, op: str, value: str) -> np.ndarray:
    """executor.py:73-87 — bool LUT over the dictionary's decoded strings."""
    strings = np.asarray(col.words or [], dtype=object)
    if strings.size == 0:
        return np.zeros(0, dtype=bool)
    if op in ("<", "<=", ">", ">="):
        return np.asarray(_OPS[op](strings, value), dtype=bool)
    raise OracleExecutionError(f"unsupported TEXT comparison operator {op!r}")


def _apply_lut(lut, codes, nulls):
    """executor.py:90-94."""
    if lut.size == 0:
        return np.zeros(codes.shape, dtype=bool)
    safe = np.where(nulls, 0, codes)
    return lut[safe] & ~nulls


class _Slices:
    """executor.py:47-70 — lazily gathered (values, nulls) per column."""

    def __init__(self, table: OTable, rows):
        self.table, self.rows, self.cache = table, rows, {}

    def get(self, name):
        if name not in self.cache:
            c = self.table.columns[name]
            if self.rows is None:
                self.cache[name] = (c.values, c.nulls)
            else:
                self.cache[name] = (c.values[self.rows], c.nulls[self.rows])
        return self.cache[name]

    @property
    def size(self):
        return self.table.row_count if self.rows is None else int(self.rows.size)


def _udf(node, slices: _Slices, udfs: dict):
    """executor.py:113-146 — float64 args (DECIMAL / 10**s), np.frompyfunc, error -> first row."""
    _, name, refs, op, value = node
    fn = udfs.get(name)
    if fn is None:
        raise OracleExecutionError(f"function {name!r} has no bound implementation")
    arrays = []
    any_null = np.zeros(slices.size, dtype=bool)
    for cname, scale in refs:
        vals, nulls = slices.get(cname)
        out = vals.astype(np.float64)
        if scale:
            out = out / float(10**scale)
        arrays.append(out)
        any_null |= nulls
    try:
        raw = np.frompyfunc(fn, len(arrays), 1)(*arrays)
    except Exception as exc:  # noqa: BLE001 - mirror of the reference's catch-all
        for i in range(slices.size):
            try:
                fn(*(float(a[i]) for a in arrays))
            except Exception:  # noqa: BLE001
                raise OracleExecutionError(f"UDF {name!r} failed at row {i}: {exc}") from exc
        raise OracleExecutionError(f"UDF {name!r} failed: {exc}") from exc
    results = raw.astype(np.float64) if raw.size else np.zeros(0, dtype=np.float64)
    return _compare(results, op, decode_value(value)) & ~any_null


def _atom(node, slices: _Slices, udfs: dict):
    """executor.py:149-177."""
    tag = node[0]
    if tag == "eq":
        vals, nulls = slices.get(node[1][0])
        return (vals == decode_value(node[2])) & ~nulls
    if tag == "cmp":
        vals, nulls = slices.get(node[1][0])
        v = decode_value(node[3])
        if isinstance(v, str):
            return _apply_lut(_text_lut(slices.table.columns[node[1][0]], node[2], v), vals, nulls)
        return _compare(vals, node[2], v) & ~nulls
    if tag == "range":
        vals, nulls = slices.get(node[1][0])
        lo, hi = decode_value(node[2]), decode_value(node[3])
        if isinstance(lo, str):
            col = slices.table.columns[node[1][0]]
            return _apply_lut(_text_lut(col, ">=", lo) & _text_lut(col, "<=", hi), vals, nulls)
        return (vals >= lo) & (vals <= hi) & ~nulls
    if tag == "colcmp":
        lv, ln = slices.get(node[1][0])
        rv, rn = slices.get(node[3][0])
        return _compare(lv, node[2], rv) & ~ln & ~rn
    if tag == "fn":
        return _udf(node, slices, udfs)
    if tag == "folded":
        _, nulls = slices.get(node[1][0])
        return ~nulls if node[2] else np.zeros(slices.size, dtype=bool)
    raise OracleExecutionError(f"unknown atom {node!r}")


def eval_mask(node, slices: _Slices, udfs: dict):
    """executor.py:180-199 — whole-slice short circuit; two-valued NOT."""
    tag = node[0]
    if tag == "and":
        items = node[1]
        mask = eval_mask(items[0], slices, udfs)
        for item in items[1:]:
            if not mask.any():
                break
            mask = mask & eval_mask(item, slices, udfs)
        return mask
    if tag == "or":
        items = node[1]
        mask = eval_mask(items[0], slices, udfs)
        for item in items[1:]:
            if mask.all():
                break
            mask = mask | eval_mask(item, slices, udfs)
        return mask
    if tag == "not":
        return ~eval_mask(node[1], slices, udfs)
    return _atom(node, slices, udfs)


def count_star(table: OTable, pred, udfs=None) -> int:
    """executor.py:218-224."""
    if pred is None:
        return table.row_count
    return int(np.count_nonzero(eval_mask(pred, _Slices(table, None), udfs or {})))


def eval_predicate(table: OTable, pred, rows=None, udfs=None) -> np.ndarray:
    """executor.py:202-215 — ascending int64 row ids (``rows``: a prior selection)."""
    if pred is None:
        return np.arange(table.row_count, dtype=np.int64) if rows is None else rows
    mask = eval_mask(pred, _Slices(table, rows), udfs or {})
    if rows is None:
        return np.flatnonzero(mask).astype(np.int64)
    return rows[mask]


def take(col: OColumn, idx) -> OColumn:
    """storage.py:176-184."""
    return OColumn(col.values[idx], col.nulls[idx], col.kind, col.scale, col.words)


def materialize(table: OTable, pred, needed, udfs=None) -> dict:
    """optimizer.py:189-193 — re-evaluate, gather the needed columns in the given order."""
    rows = eval_predicate(table, pred, None, udfs)
    return {name: take(table.columns[name], rows) for name in needed}


# -------------------------------------------------------------------------------------------
# planner policy and ordering (exact, host logic)
# -------------------------------------------------------------------------------------------
def decide_pushdown(row_count: int, count: int, min_table_size=1000, max_selectivity=0.2) -> bool:
    """optimizer.py:171-177 — inclusive thresholds, exact rational comparison."""
    from fractions import Fraction

    if row_count < min_table_size or row_count <= 0:
        return False
    return Fraction(count, row_count) <= max_selectivity


def order_builds(aliases, edges, probe, effective) -> list:
    """optimizer.py:208-228 — greedy smallest adjacent effective cardinality, ties by alias.
    ``edges`` = [(alias_a, alias_b), ...]."""
    connected, remaining, order = {probe}, [a for a in aliases if a != probe], []
    while remaining:
        cands = [a for a in remaining
                 if any((a == x and y in connected) or (a == y and x in connected) for x, y in edges)]
        if not cands:
            raise OracleExecutionError("cartesian product required")
        pick = min(cands, key=lambda a: (effective[a], a))
        order.append(pick)
        connected.add(pick)
        remaining.remove(pick)
    return order


def py_mod(x: float, y: float) -> float:
    """CPython float ``%`` (what the reference's UDFs compute); used by tests."""
    return x % y


def is_finite(x) -> bool:
    return isinstance(x, (int, float)) and math.isfinite(x)


# ---------------------------------------------------------------------------------------------
# hash joins: reference executor.py:253-531, numpy restatement
# ---------------------------------------------------------------------------------------------
@dataclass
class OIndex:
    """HashTableIndex (executor.py:275-303): groups of equal keys over the non-NULL rows.  The
    group id of a key is its index among the ascending unique keys (np.unique); a group's rows
    are ascending (stable argsort of the inverse)."""

    table: OTable
    key: str
    n_entries: int
    unique_keys: np.ndarray
    group_rows: np.ndarray
    group_start: np.ndarray
    group_counts: np.ndarray

    @property
    def distinct_keys(self) -> int:
        return int(self.unique_keys.size)

    def probe_groups(self, keys: np.ndarray, valid: np.ndarray) -> np.ndarray:
        """executor.py:327-346: group id per key, -1 when absent or invalid (the open-addressed
        probe returns exactly the np.unique index of the key, restated by a sorted search)."""
        out = np.full(keys.shape, -1, dtype=np.int64)
        if self.unique_keys.size == 0:
            return out
        k = keys.astype(np.int64)
        pos = np.searchsorted(self.unique_keys, k)
        ok = valid & (pos < self.unique_keys.size)
        ok[ok] = self.unique_keys[pos[ok]] == k[ok]
        out[ok] = pos[ok]
        return out

    def lookup(self, key: int) -> np.ndarray:
        g = self.probe_groups(np.asarray([key], dtype=np.int64), np.ones(1, dtype=bool))[0]
        if g < 0:
            return np.empty(0, dtype=np.int64)
        return self.group_rows[self.group_start[g]: self.group_start[g + 1]]


def build_index(table: OTable, key: str, rows: np.ndarray) -> OIndex:
    """HashTableIndex.__init__ (executor.py:281-298)."""
    col = table.columns[key]
    key_vals = col.values[rows]
    non_null = ~col.nulls[rows]
    rows = rows[non_null]
    key_vals = key_vals[non_null].astype(np.int64)
    uk, inverse = np.unique(key_vals, return_inverse=True)
    order = np.argsort(inverse, kind="stable")
    counts = np.bincount(inverse, minlength=uk.size).astype(np.int64)
    start = np.concatenate((np.zeros(1, dtype=np.int64), np.cumsum(counts)))
    return OIndex(table, key, int(rows.size), uk, rows[order].astype(np.int64), start, counts)


def build_hash(table: OTable, key: str, residual=None, udfs=None) -> OIndex:
    """executor.py:353-358."""
    return build_index(table, key, eval_predicate(table, residual, None, udfs))


def expand_matches(index: OIndex, groups: np.ndarray):
    """_expand_matches (executor.py:373-386)."""
    counts = index.group_counts[groups]
    starts = index.group_start[groups]
    total = int(counts.sum())
    if total == 0:
        return counts, np.empty(0, dtype=np.int64)
    offsets = np.zeros(groups.size, dtype=np.int64)
    np.cumsum(counts[:-1], out=offsets[1:])
    flat = np.arange(total, dtype=np.int64)
    flat -= np.repeat(offsets, counts)
    flat += np.repeat(starts, counts)
    return counts, index.group_rows[flat]


def probe_joins(probe: OTable, probe_alias: str, probe_pred, steps, projection=None, udfs=None):
    """_probe_chunk + probe_joins (executor.py:403-531) with one chunk.  ``steps`` is a list of
    (alias, OIndex, (probe_table_alias, probe_column)); ``projection`` a list of (alias, column)
    or None.  Returns (stage counts, result columns as {name: OColumn} or None)."""
    prow = eval_predicate(probe, probe_pred, None, udfs)
    stage_out = [int(prow.size)]
    brows: dict = {}
    tables = {probe_alias: probe}
    for alias, index, (src, cname) in steps:
        rows_src = prow if src == probe_alias else brows[src]
        col = tables[src].columns[cname]
        keys = col.values[rows_src]
        valid = ~col.nulls[rows_src]
        groups = index.probe_groups(keys, valid)
        hit = groups >= 0
        prow = prow[hit]
        for a in brows:
            brows[a] = brows[a][hit]
        counts, matched = expand_matches(index, groups[hit])
        prow = np.repeat(prow, counts)
        for a in brows:
            brows[a] = np.repeat(brows[a], counts)
        brows[alias] = matched
        tables[alias] = index.table
        stage_out.append(int(prow.size))
    if projection is None:
        return stage_out, None
    rows_of = {probe_alias: prow, **brows}
    out, used = {}, set()
    for alias, cname in projection:
        c = take(tables[alias].columns[cname], rows_of[alias])
        name = cname if cname not in used else f"{alias}.{cname}"
        used.add(name)
        out[name] = c
    return stage_out, out


# ---------------------------------------------------------------------------------------------
# equi-depth histograms + estimator: reference catalog.py:178-326
# ---------------------------------------------------------------------------------------------
def build_histogram(values: np.ndarray, nulls: np.ndarray, buckets: int) -> dict:
    """catalog.py:178-223: sort the non-NULL values, edges at ranks (i*n)//k - 1 (duplicates
    collapse buckets), counts by right-searchsorted, distincts by np.unique per bucket."""
    valid = np.sort(values[~nulls].astype(np.int64))
    n = valid.size
    out = {"null_count": int(values.size - n), "row_count": int(values.size)}
    if n == 0:
        out.update(boundaries=[0], counts=[], distincts=[])
        return out
    k = min(buckets, n)
    edges = [int(valid[0])]
    for i in range(1, k + 1):
        e = int(valid[min(n - 1, (i * n) // k - 1)])
        if e > edges[-1]:
            edges.append(e)
    if len(edges) == 1:
        edges.append(edges[0])
    counts, distincts, lo = [], [], 0
    for b in range(len(edges) - 1):
        hi = n if b == len(edges) - 2 else int(np.searchsorted(valid, edges[b + 1], side="right"))
        counts.append(hi - lo)
        distincts.append(int(np.unique(valid[lo:hi]).size))
        lo = hi
    out.update(boundaries=edges, counts=counts, distincts=distincts)
    return out


def _h_le(h: dict, v: float) -> float:
    """_estimate_le (catalog.py:226-244)."""
    if not h["counts"] or h["row_count"] == 0:
        return 0.0
    total = 0.0
    for b in range(len(h["counts"])):
        lo, hi = h["boundaries"][b], h["boundaries"][b + 1]
        if v >= hi:
            total += float(h["counts"][b])
        elif v < lo:
            break
        else:
            span = hi - lo
            frac = (v - lo + 1) / (span + 1) if span > 0 else 1.0
            total += float(h["counts"][b]) * min(1.0, max(0.0, frac))
            break
    return total / h["row_count"]


def _h_eq(h: dict, v: float) -> float:
    """_estimate_equality (catalog.py:247-257)."""
    if not h["counts"] or h["row_count"] == 0:
        return 0.0
    if v != int(v):
        return 0.0
    for b in range(len(h["counts"])):
        lo, hi = h["boundaries"][b], h["boundaries"][b + 1]
        if (lo <= v <= hi) if b == 0 else (lo < v <= hi):
            return float(h["counts"][b]) / max(1, h["distincts"][b]) / h["row_count"]
    return 0.0


class OracleInestimable(Exception):
    pass


def estimate(h: dict, pred) -> float:
    """estimate_selectivity + _atom_selectivity (catalog.py:268-326) over one column's histogram;
    ``pred`` in the JSON form."""
    def num(x):
        x = decode_value(x)
        if isinstance(x, bool) or not isinstance(x, (int, float)):
            raise OracleInestimable(repr(x))
        return float(x)

    def clamp(x):
        return min(1.0, max(0.0, x))

    t = pred[0]
    if t == "and":
        s = 1.0
        for it in pred[1]:
            s *= estimate(h, it)
        return clamp(s)
    if t == "or":
        miss = 1.0
        for it in pred[1]:
            miss *= 1.0 - estimate(h, it)
        return clamp(1.0 - miss)
    if t == "not":
        return clamp(1.0 - estimate(h, pred[1]))
    if t == "folded":
        return 1.0 if pred[2] else 0.0
    if t in ("fn", "colcmp"):
        raise OracleInestimable(t)
    present = (h["row_count"] - h["null_count"]) / max(1, h["row_count"])
    if t == "eq":
        return clamp(_h_eq(h, num(pred[2])))
    if t == "range":
        return clamp(max(0.0, _h_le(h, num(pred[3])) - _h_le(h, num(pred[2]) - 1)))
    op, v = pred[2], num(pred[3])
    r = {"<=": lambda: _h_le(h, v), "<": lambda: _h_le(h, v - 1),
         ">": lambda: max(0.0, present - _h_le(h, v)), ">=": lambda: max(0.0, present - _h_le(h, v - 1)),
         "<>": lambda: max(0.0, present - _h_eq(h, v))}[op]()
    return clamp(r)
