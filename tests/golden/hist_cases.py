"""Deterministic histogram scenarios: columns (values, nulls), bucket counts and
predicates over column ``v`` (JSON form).  Shared by make_golden.py (reference outputs) and the
tests.  Includes the reference's own TestHistogram inputs (test_catalog.py:106-141)."""

from __future__ import annotations

import numpy as np


def _col(vals):
    nulls = np.array([v is None for v in vals], dtype=bool)
    return np.array([0 if v is None else v for v in vals], dtype=np.int64), nulls


def columns() -> dict:
    g = np.random.default_rng(5)
    out = {
        "ref_partition": _col(g.integers(0, 1000, size=5000).tolist() + [None] * 40),
        "ref_balance": _col(list(range(6400))),
        "ref_single": _col([3, 1, 2]),
        "ref_constant": _col([7] * 10),
        "ref_empty": _col([]),
        "uniform": _col(np.random.default_rng(17).integers(0, 1000, size=10_000).tolist()),
    }
    g = np.random.default_rng(99)
    z = (g.zipf(1.3, 20_000) % 5000).astype(np.int64)
    nulls = g.random(20_000) < 0.07
    out["zipf_nulls"] = (np.where(nulls, 0, z), nulls)
    w = g.integers(-(1 << 40), 1 << 40, 3000).astype(np.int64)
    out["wide"] = (w, np.zeros(w.size, bool))
    out["all_null"] = _col([None] * 5)
    return out


BUCKETS = (64, 8, 1, 3)

PREDICATES = (
    [["cmp", ["v", None], op, c] for op in ("<", "<=", ">", ">=", "<>") for c in
     (0, 137, 400, 499, 999, 2000, -5, 10**9, 4.5, 2500.25, 7, 1 << 39, -(1 << 39))]
    + [["eq", ["v", None], c] for c in (500, 4.5, 7, 0, 10**9, 3, -(1 << 39))]
    + [["range", ["v", None], lo, hi] for lo, hi in ((100, 299), (0, 0), (5, 4), (-10, 10**6), (2.5, 7.5))]
    + [["and", [["cmp", ["v", None], "<", 500], ["cmp", ["v", None], ">=", 100]]],
       ["or", [["cmp", ["v", None], "<", 200], ["cmp", ["v", None], ">=", 800]]],
       ["not", ["cmp", ["v", None], "<", 300]],
       ["folded", ["v", None], True], ["folded", ["v", None], False],
       ["and", [["eq", ["v", None], 5], ["or", [["cmp", ["v", None], ">", 900], ["not", ["eq", ["v", None], 3]]]]]]]
)
