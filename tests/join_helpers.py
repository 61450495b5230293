"""Join scenario plumbing shared by the oracle and device join tests."""

from __future__ import annotations

import os
import sys

import numpy as np

from oracle import esc_oracle as O

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
import join_cases  # noqa: E402


def cases() -> list:
    return join_cases.cases()


def oracle_run(case):
    tabs = {a: O.OTable(a, {c: O.OColumn(v, n) for c, (v, n) in cols.items()}) for a, cols in case["tables"].items()}
    steps = []
    for st in case["steps"]:
        idx = O.build_hash(tabs[st["alias"]], st["key"], st["residual"])
        steps.append((st["alias"], idx, tuple(st["probe_key"])))
    proj = [tuple(p) for p in case["projection"]] if case["projection"] is not None else None
    stage_out, cols = O.probe_joins(tabs[case["probe"]], case["probe"], case["probe_pred"], steps, proj)
    rec = {"probe_out": stage_out, "result_rows": stage_out[-1],
           "build_cards": [s[1].n_entries for s in steps], "build_distinct": [s[1].distinct_keys for s in steps]}
    if cols is not None:
        rec["columns"] = [[name, c.values.tolist(), c.nulls.tolist()] for name, c in cols.items()]
    return rec


def device_tables(case, device):
    from paper_1901_01488_b200.storage import KIND_INT64, Column, ColumnTable

    return {a: ColumnTable(a, [Column(c, KIND_INT64, v, n, device=device) for c, (v, n) in cols.items()])
            for a, cols in case["tables"].items()}


def device_run(case, device):
    from paper_1901_01488_b200 import expr as ex, join, serde

    tabs = device_tables(case, device)
    steps = []
    for st in case["steps"]:
        res = serde.from_json(st["residual"], st["alias"]) if st["residual"] is not None else None
        idx = join.build_hash(tabs[st["alias"]], st["key"], res)
        steps.append(join.BuildStep(st["alias"], idx, ex.ColumnRef(*st["probe_key"])))
    pp = serde.from_json(case["probe_pred"], case["probe"]) if case["probe_pred"] is not None else None
    proj = tuple(ex.ColumnRef(a, c) for a, c in case["projection"]) if case["projection"] is not None else None
    result, stats = join.probe_joins(tabs[case["probe"]], case["probe"], pp, steps, proj)
    rec = {"probe_out": stats.probe_out, "result_rows": stats.result_rows, "build_cards": stats.build_cards,
           "build_distinct": stats.build_distinct}
    if result is not None:
        cols = []
        for c in result.columns:
            v, m = c.to_numpy()
            cols.append([c.name, np.asarray(v).tolist(), np.asarray(m).tolist()])
        rec["columns"] = cols
    return rec
