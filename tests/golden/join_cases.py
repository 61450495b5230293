"""Deterministic join scenarios (hash build + probe pipeline).

Shared by ``make_golden.py`` (which runs the REFERENCE ``build_hash`` / ``probe_joins`` on them and
freezes the results in ``known.json["joins"]``) and the tests (which rebuild the same inputs and
check the oracle and the device path against those results).  All columns are INT64 with
optional NULLs, aliases are table names, predicates use the JSON form of ``oracle/esc_oracle.py``.

* ``ref_*``   — the reference's own ``test_executor.join_data`` fixture (``random.Random(13)``)
               and its TestProbeJoins scenarios (residual build, probe filter, projection,
               chained probe key, empty build side, swapped build order, NULL probe keys);
* ``fuzz_*``  — random star / snowflake pipelines with duplicate build keys, NULL keys on both
               sides, residuals and probe filters.
"""

from __future__ import annotations

import random

import numpy as np


def _table(**cols):
    out = {}
    for name, vals in cols.items():
        nulls = np.array([v is None for v in vals], dtype=bool)
        out[name] = (np.array([0 if v is None else v for v in vals], dtype=np.int64), nulls)
    return out


def _ref_join_data():
    """test_executor.py join_data (rng 13): orders 15, parts 8 + a duplicate p_id 3, lines 40."""
    rng = random.Random(13)
    n_orders, n_parts, n_lines = 15, 8, 40
    orders = []
    for i in range(1, n_orders + 1):
        orders.append(dict(o_id=i, o_ch=rng.randrange(10), o_pid=rng.randrange(1, n_parts + 1)))
    parts = [dict(p_id=i, p_cls=rng.randrange(5)) for i in range(1, n_parts + 1)]
    parts.append(dict(p_id=3, p_cls=1))
    lines = []
    for _ in range(n_lines):
        lines.append(dict(l_oid=rng.randrange(1, n_orders + 1) if rng.random() > 0.1 else None,
                          l_pid=rng.randrange(1, n_parts + 1), l_qty=rng.randrange(1, 50)))
    col = lambda recs, k: [r[k] for r in recs]  # noqa: E731
    return {
        "orders": _table(o_id=col(orders, "o_id"), o_ch=col(orders, "o_ch"), o_pid=col(orders, "o_pid")),
        "parts": _table(p_id=col(parts, "p_id"), p_cls=col(parts, "p_cls")),
        "lines": _table(l_oid=col(lines, "l_oid"), l_pid=col(lines, "l_pid"), l_qty=col(lines, "l_qty")),
    }


def _fuzz(seed: int):
    g = np.random.default_rng(np.random.SeedSequence([2026, seed]))
    n_probe = int(g.integers(2000, 8000))
    n_steps = int(g.integers(1, 5))
    tables = {}
    steps = []
    probe_cols = {}
    for s in range(n_steps):
        alias = f"b{s}"
        nb = int(g.integers(1, 400))
        key_range = int(g.integers(max(2, nb // 3), nb * 2 + 3))
        keys = g.integers(0, key_range, nb)
        knull = g.random(nb) < 0.05
        attr = g.integers(0, 20, nb)
        tables[alias] = {"k": (np.where(knull, 0, keys).astype(np.int64), knull),
                         "a": (attr.astype(np.int64), np.zeros(nb, bool)),
                         "fk": (g.integers(0, 50, nb).astype(np.int64), g.random(nb) < 0.05)}
        placed = ["probe"] + [st["alias"] for st in steps]
        src = "probe" if (s == 0 or g.random() < 0.6) else placed[int(g.integers(1, len(placed)))]
        if src == "probe":
            cname = f"f{s}"
            pk = g.integers(-2, key_range + 2, n_probe)
            pn = g.random(n_probe) < 0.05
            probe_cols[cname] = (np.where(pn, 0, pk).astype(np.int64), pn)
            probe_key = ["probe", cname]
        else:
            probe_key = [src, "fk"]
        residual = None
        if g.random() < 0.5:
            hi = int(g.integers(0, 20))
            residual = ["cmp", ["a", None], "<=", hi]
        steps.append({"alias": alias, "key": "k", "residual": residual, "probe_key": probe_key})
    probe_cols["q"] = (g.integers(0, 100, n_probe).astype(np.int64), np.zeros(n_probe, bool))
    tables["probe"] = probe_cols
    probe_pred = ["cmp", ["q", None], "<", int(g.integers(20, 101))] if g.random() < 0.6 else None
    projection = None
    if g.random() < 0.5:
        projection = [["probe", "q"]] + [[st["alias"], "a"] for st in steps] + [["probe", "q"]]
    return {"name": f"fuzz_{seed}", "tables": tables, "probe": "probe", "probe_pred": probe_pred,
            "steps": steps, "projection": projection}


def cases() -> list:
    d = _ref_join_data()
    oc = ["cmp", ["o_ch", None], "<", 6]
    qty = ["cmp", ["l_qty", None], ">", 5]
    orders = {"alias": "orders", "key": "o_id", "residual": oc, "probe_key": ["lines", "l_oid"]}
    parts = {"alias": "parts", "key": "p_id", "residual": None, "probe_key": ["lines", "l_pid"]}
    proj = [["lines", "l_qty"], ["orders", "o_ch"], ["parts", "p_cls"]]
    out = [
        {"name": "ref_count", "tables": d, "probe": "lines", "probe_pred": qty, "steps": [orders, parts],
         "projection": None},
        {"name": "ref_count_swapped", "tables": d, "probe": "lines", "probe_pred": qty, "steps": [parts, orders],
         "projection": None},
        {"name": "ref_projection", "tables": d, "probe": "lines", "probe_pred": qty, "steps": [orders, parts],
         "projection": proj},
        {"name": "ref_chained", "tables": d, "probe": "lines", "probe_pred": None,
         "steps": [{"alias": "orders", "key": "o_id", "residual": None, "probe_key": ["lines", "l_oid"]},
                   {"alias": "parts", "key": "p_id", "residual": None, "probe_key": ["orders", "o_pid"]}],
         "projection": None},
        {"name": "ref_chained_projection", "tables": d, "probe": "lines", "probe_pred": None,
         "steps": [{"alias": "orders", "key": "o_id", "residual": None, "probe_key": ["lines", "l_oid"]},
                   {"alias": "parts", "key": "p_id", "residual": None, "probe_key": ["orders", "o_pid"]}],
         "projection": [["lines", "l_qty"], ["parts", "p_cls"], ["orders", "o_pid"]]},
        {"name": "ref_empty_build", "tables": d, "probe": "lines", "probe_pred": None,
         "steps": [{"alias": "orders", "key": "o_id", "residual": ["cmp", ["o_ch", None], "<", -1],
                    "probe_key": ["lines", "l_oid"]}],
         "projection": [["lines", "l_qty"]]},
        {"name": "ref_duplicate_names", "tables": d, "probe": "lines", "probe_pred": None, "steps": [orders, parts],
         "projection": [["lines", "l_qty"], ["lines", "l_qty"]]},
        {"name": "ref_null_probe_keys", "tables": {"lines": _table(l_oid=[1, None, 1], l_qty=[1, 2, 3]),
                                                   "orders": _table(o_id=[1])},
         "probe": "lines", "probe_pred": None,
         "steps": [{"alias": "orders", "key": "o_id", "residual": None, "probe_key": ["lines", "l_oid"]}],
         "projection": None},
    ]
    out += [_fuzz(s) for s in range(24)]
    return out
