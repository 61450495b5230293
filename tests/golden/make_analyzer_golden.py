"""Freeze the REFERENCE analyzer's constant normalisation (run HERE only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_analyzer_golden.py

Writes ``analyzer_cases.json``: for literals against INT64 / DECIMAL(15,2) / DATE / TEXT columns
(comparisons with every operator, BETWEEN, UDF comparisons) the resolved atom the reference's
``frontend.analyze`` produces — or its error class and message — so
``tests/test_analyzer.py`` pins ``paper_1901_01488_b200.analyzer`` to it.
"""

from __future__ import annotations

import json
import os

import numpy as np
from escdb import expr as rex
from escdb import frontend as rfe
from escdb.catalog import Catalog as RCatalog
from escdb.errors import EscdbError
from escdb.storage import Column as RColumn, ColumnTable as RTable, Dictionary as RDict, parse_kind

HERE = os.path.dirname(os.path.abspath(__file__))

LITERALS = ["0", "7", "-3", "10.5", "10.50", "0.125", "1e3", "2.5e-1", "1050", "99999999999999999999",
            "-0.0", "123456789012345678901234567890.5", "'abc'", "'w1'", "DATE '2024-01-31'", "DATE '1970-01-01'",
            "DATE '2024-13-01'", "'2020-02-29'"]
OPS = ["=", "<>", "<", "<=", ">", ">="]


def atom_json(e):
    name = type(e).__name__
    if name == "FoldedAtom":
        return ["folded", e.col.name, bool(e.result)]
    if name == "Equality":
        return ["eq", e.col.name, _v(e.value)]
    if name == "Comparison":
        return ["cmp", e.col.name, e.op, _v(e.value)]
    if name == "Range":
        return ["range", e.col.name, _v(e.lo), _v(e.hi)]
    if name == "FnCall":
        return ["fn", e.name, [a.name for a in e.args], e.op, _v(e.value)]
    raise TypeError(name)


def _v(v):
    if isinstance(v, bool):
        return v
    if isinstance(v, int):
        return {"int": str(v)}
    if isinstance(v, float):
        return {"float": repr(v)}
    return v


def main():
    cat = RCatalog()
    d = RDict()
    for w in ("w0", "w1", "abc"):
        d.encode(w)
    cols = [RColumn("i", parse_kind("int64"), np.zeros(3, np.int64), np.zeros(3, bool)),
            RColumn("p", parse_kind("decimal(15,2)"), np.zeros(3, np.int64), np.zeros(3, bool)),
            RColumn("d", parse_kind("date"), np.zeros(3, np.int64), np.zeros(3, bool)),
            RColumn("s", parse_kind("text"), np.zeros(3, np.int64), np.zeros(3, bool), d)]
    cat.register(RTable("t", cols))
    cat.register_udf("f", 1, lambda x: x)
    cases = []

    def run(where):
        sql = f"SELECT COUNT(*) FROM t WHERE {where}"
        try:
            ra = rfe.analyze(rfe.parse(sql), cat)
            node = ra.child
            while not hasattr(node, "predicate"):
                node = node.child
            return {"ok": atom_json(node.predicate)}
        except EscdbError as exc:
            return {"error": type(exc).__name__, "message": str(exc)}

    for col in ("i", "p", "d", "s"):
        for lit in LITERALS:
            for op in OPS:
                cases.append({"where": [col, op, lit], "result": run(f"{col} {op} {lit}")})
        for lo, hi in (("1", "5"), ("5", "1"), ("1.5", "2.25"), ("'a'", "'b'"), ("'b'", "'a'"),
                       ("DATE '2020-01-01'", "DATE '2020-12-31'"), ("DATE '2021-01-01'", "DATE '2020-12-31'")):
            cases.append({"between": [col, lo, hi], "result": run(f"{col} BETWEEN {lo} AND {hi}")})
    for lit in ("3", "0.5", "1e2", "'x'"):
        cases.append({"fn": ["f", ["i"], ">", lit], "result": run(f"f(i) > {lit}")})
    with open(os.path.join(HERE, "analyzer_cases.json"), "w") as fh:
        json.dump(cases, fh, indent=0)
    print(len(cases), "cases")


if __name__ == "__main__":
    rex  # noqa: B018 (imported for the reference's node classes)
    main()
