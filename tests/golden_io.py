"""Load the golden fixtures (tests/golden/, produced by running the reference) into the forms the
oracle and the device path consume."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from oracle import esc_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# the UDFs the fixtures name (mirrors tests/golden/make_golden.py UDFS)
UDFS = {"mixy": lambda x, y: (x * 7.0 + y) % 13.0,
        "inv": lambda x: 100.0 / x,
        "fmod": lambda x, y: x % (y - 500.0),
        "fdiv": lambda x, y: (x - y) // 3.0}


def corpus() -> dict:
    with open(os.path.join(GOLDEN, "corpus.json")) as fh:
        return json.load(fh)


def known() -> dict:
    with open(os.path.join(GOLDEN, "known.json")) as fh:
        return json.load(fh)


def _kind_scale(kind: str) -> int:
    return int(kind[8:-1].split(",")[1]) if kind.startswith("DECIMAL") else 0


def raw_tables() -> dict:
    """name -> list of (col, kind, values, nulls, words) in base column order."""
    arr = np.load(os.path.join(GOLDEN, "tables.npz"))
    meta = corpus()["meta"]
    out = {}
    for tname, cols in meta.items():
        out[tname] = [(c["name"], c["kind"], arr[f"{tname}.{c['name']}.values"],
                       arr[f"{tname}.{c['name']}.nulls"], c["words"]) for c in cols]
    return out


def oracle_table(name: str, cols) -> O.OTable:
    t = O.OTable(name)
    for cname, kind, vals, nulls, words in cols:
        t.columns[cname] = O.OColumn(vals, nulls, kind, _kind_scale(kind), words)
    return t


def device_table(name: str, cols, device=None):
    from paper_1901_01488_b200.storage import Column, ColumnTable, Dictionary, parse_kind

    return ColumnTable(name, [Column(cname, parse_kind(kind), vals, nulls,
                                     Dictionary(words) if words is not None else None, device=device)
                              for cname, kind, vals, nulls, words in cols])


def digest(idx) -> str:
    return hashlib.sha256(np.asarray(idx, dtype=np.int64).tobytes()).hexdigest()


def outcome(fn, exc_types):
    try:
        return {"ok": fn()}
    except exc_types as exc:  # noqa: B030
        return {"error": "ExecutionError", "message": str(exc)}
