"""Predicate trees <-> JSON (the interchange format of the golden fixtures and the oracle).

``["eq", ref, v]``, ``["cmp", ref, op, v]``, ``["range", ref, lo, hi]``, ``["colcmp", ref, op, ref]``,
``["fn", name, [ref...], op, v]``, ``["folded", ref, bool]``, ``["and", [...]]``, ``["or", [...]]``,
``["not", x]`` with ``ref = [column, decimal_scale_or_null]``; non-finite floats are
``{"float": "nan"}`` etc.  UDF callables travel by name (``udfs`` maps name -> callable).
"""

from __future__ import annotations

import math

from . import expr as ex
from .storage import decimal


def _v_out(v):
    if isinstance(v, float) and not math.isfinite(v):
        return {"float": repr(v)}
    if hasattr(v, "item") and not isinstance(v, (int, float, str)):
        v = v.item()
    return v


def _v_in(v):
    if isinstance(v, dict) and "float" in v:
        return float(v["float"])
    return v


def _ref_out(r: ex.ColumnRef):
    k = r.kind
    scale = k.scale if k is not None and getattr(k, "is_decimal", False) else None
    return [r.name, scale]


def _ref_in(j, table):
    name, scale = j
    return ex.ColumnRef(table, name, kind=decimal(18, scale) if scale is not None else None)


def to_json(e: ex.Expr):
    if isinstance(e, ex.Equality):
        return ["eq", _ref_out(e.col), _v_out(e.value)]
    if isinstance(e, ex.Comparison):
        return ["cmp", _ref_out(e.col), e.op, _v_out(e.value)]
    if isinstance(e, ex.Range):
        return ["range", _ref_out(e.col), _v_out(e.lo), _v_out(e.hi)]
    if isinstance(e, ex.ColumnCompare):
        return ["colcmp", _ref_out(e.left), e.op, _ref_out(e.right)]
    if isinstance(e, ex.FnCall):
        return ["fn", e.name, [_ref_out(a) for a in e.args], e.op, _v_out(e.value)]
    if isinstance(e, ex.FoldedAtom):
        return ["folded", _ref_out(e.col), bool(e.result)]
    if isinstance(e, ex.And):
        return ["and", [to_json(i) for i in e.items]]
    if isinstance(e, ex.Or):
        return ["or", [to_json(i) for i in e.items]]
    if isinstance(e, ex.Not):
        return ["not", to_json(e.child)]
    raise TypeError(f"not a predicate node: {e!r}")


def from_json(j, table: str | None = None, udfs: dict | None = None) -> ex.Expr:
    udfs = udfs or {}
    tag = j[0]
    if tag == "eq":
        return ex.Equality(_ref_in(j[1], table), _v_in(j[2]))
    if tag == "cmp":
        return ex.Comparison(_ref_in(j[1], table), j[2], _v_in(j[3]))
    if tag == "range":
        return ex.Range(_ref_in(j[1], table), _v_in(j[2]), _v_in(j[3]))
    if tag == "colcmp":
        return ex.ColumnCompare(_ref_in(j[1], table), j[2], _ref_in(j[3], table))
    if tag == "fn":
        return ex.FnCall(j[1], tuple(_ref_in(a, table) for a in j[2]), j[3], _v_in(j[4]), udfs.get(j[1]))
    if tag == "folded":
        return ex.FoldedAtom(_ref_in(j[1], table), bool(j[2]))
    if tag == "and":
        return ex.And(tuple(from_json(i, table, udfs) for i in j[1]))
    if tag == "or":
        return ex.Or(tuple(from_json(i, table, udfs) for i in j[1]))
    if tag == "not":
        return ex.Not(from_json(j[1], table, udfs))
    raise ValueError(f"unknown predicate tag {tag!r}")
