"""Analyzer constant rules: literals -> storage-unit constants -> resolved atoms.

The reference analyzer (``pkg/src/escdb/frontend.py:597-715``) normalises every comparison
constant to the column's storage units before the executor sees it.  Its rules, restated here for
its own kinds and pinned to its outputs (``tests/golden/analyzer_cases.json``):

* numeric literals are exact ``Fraction``s, scaled by ``10**s`` for DECIMAL(p,s); an integral
  result stays a Python ``int`` (any size), anything else becomes a ``float`` (``_scaled_constant``,
  ``frontend.py:603-610``);
* ``=`` / ``<>`` against a fractional literal on an integer-stored column fold to
  ``FoldedAtom(False)`` / ``FoldedAtom(True)`` (``frontend.py:676-678``);
* DATE literals become epoch days, a number against a DATE is a type mismatch;
* TEXT ``=`` / ``<>`` compare dictionary codes and fold when the literal is absent from the
  dictionary; TEXT ordering keeps the string payload (``frontend.py:659-675``);
* ``BETWEEN lo AND hi`` with ``lo > hi`` folds to ``FoldedAtom(False)`` (``frontend.py:718-724``);
* a UDF is compared with ``float(literal)`` (``frontend.py:702-715``).

The reference only knows INT64 / DATE / DECIMAL / TEXT.  This build stores native widths, so it
adds rules for the new kinds (the FLOAT32 rule SURVEY Appendix A.3 asked to define):

* INT32 / INT16 / INT8: the INT64 rules unchanged — an out-of-range integral literal stays an
  exact Python int and compares mathematically (the device compiler folds it to all-true /
  all-false per operator, as numpy's NEP 50 comparison of an int32 array with a large Python int
  does);
* FLOAT32 / FLOAT64: a numeric literal becomes ``float(Fraction(literal))`` — the correctly
  rounded double a Python user writing ``col == 0.1`` passes — and is never folded: a float
  column holds fractional values, so ``=`` / ``<>`` / ordering are real comparisons.  The
  executor then compares in the column's NEP 50 domain: FLOAT64 in float64, FLOAT32 against that
  double rounded to float32 (``np.float32 array == 0.1`` semantics).  A DATE or string literal
  against a float column is a type mismatch.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

from . import expr as ex
from .errors import AnalysisError, ArityMismatch, TypeMismatch, UnknownFunction, UnsupportedPredicate
from .storage import DATE, FLOAT32, FLOAT64, ColumnKind, date_to_days

_ORDER_OPS = ("<", "<=", ">", ">=")


@dataclass(frozen=True)
class Literal:
    """A parsed literal: ``kind`` is ``"number"``, ``"string"`` or ``"date"`` and ``text`` the
    unquoted lexeme (the reference's ``AstConst``)."""

    kind: str
    text: str


def number(text) -> Literal:
    return Literal("number", str(text))


def string(text: str) -> Literal:
    return Literal("string", text)


def date(text: str) -> Literal:
    return Literal("date", text)


def _number_value(lit: Literal) -> Fraction:
    try:
        return Fraction(lit.text)
    except (ValueError, ZeroDivisionError):
        raise AnalysisError(f"bad numeric literal {lit.text!r}") from None


def _is_float(kind: ColumnKind) -> bool:
    return kind.name in (FLOAT32, FLOAT64)


def scaled_constant(value: Fraction, kind: ColumnKind):
    """Literal value in the column's storage units: exact int when integral, float otherwise
    (reference ``_scaled_constant``); float kinds always take the correctly rounded double."""
    if _is_float(kind):
        return float(value)
    scaled = value * (10 ** kind.scale if kind.is_decimal else 1)
    if scaled.denominator == 1:
        return int(scaled)
    return float(scaled)


def constant_for_column(col: ex.ColumnRef, lit: Literal):
    """(storage-unit constant, exact) — exact False when a fractional literal meets an
    integer-stored column (reference ``_const_for_column``, ``frontend.py:613-640``)."""
    kind: ColumnKind = col.kind
    if kind is None:
        raise AnalysisError(f"column {col} has no kind; resolve it against a table first")
    if kind.is_text:
        if lit.kind != "string":
            raise AnalysisError(f"type mismatch: TEXT column {col} compared to {_show(lit)}")
        return lit.text, True
    if kind.name == DATE:
        if lit.kind == "number":
            raise AnalysisError(f"type mismatch: DATE column {col} compared to a number")
        try:
            return date_to_days(lit.text), True
        except TypeMismatch:
            raise AnalysisError(f"bad date literal {lit.text!r} (expected YYYY-MM-DD)") from None
    if lit.kind != "number":
        raise AnalysisError(f"type mismatch: column {col} compared to {_show(lit)}")
    value = scaled_constant(_number_value(lit), kind)
    return value, _is_float(kind) or isinstance(value, int)


def _show(lit: Literal) -> str:
    if lit.kind == "number":
        return lit.text
    body = "'" + lit.text.replace("'", "''") + "'"
    return "DATE " + body if lit.kind == "date" else body


def compare(col: ex.ColumnRef, op: str, lit: Literal, dictionary=None) -> ex.Expr:
    """``col op literal`` as a resolved atom (reference ``_analyze_compare``, ``frontend.py:643-680``).
    ``dictionary``: the TEXT column's Dictionary (equality compares codes)."""
    if op not in ("=",) + ex.COMPARISON_OPS:
        raise AnalysisError(f"unknown comparison operator {op!r}")
    value, exact = constant_for_column(col, lit)
    if col.kind.is_text:
        if op in ("=", "<>"):
            code = dictionary.lookup(value) if dictionary is not None else None
            if code is None:  # absent from the dictionary: = never holds, <> holds off NULL
                return ex.FoldedAtom(col, op == "<>")
            return ex.Equality(col, code) if op == "=" else ex.Comparison(col, "<>", code)
        return ex.Comparison(col, op, value)  # string payload, decoded compare
    if not exact and op in ("=", "<>"):
        return ex.FoldedAtom(col, op == "<>")  # a fractional literal never equals an integer
    if op == "=":
        return ex.Equality(col, value)
    return ex.Comparison(col, op, value)


def column_compare(left: ex.ColumnRef, op: str, right: ex.ColumnRef) -> ex.Expr:
    """``col op col`` (same kind required; not over TEXT), reference ``frontend.py:647-658``."""
    if left.kind != right.kind:
        raise AnalysisError(f"type mismatch: cannot compare {left} ({left.kind}) to {right} ({right.kind})")
    if left.kind.is_text:
        raise UnsupportedPredicate(f"column-to-column comparison over TEXT: {left} {op} {right}")
    return ex.ColumnCompare(left, op, right)


def between(col: ex.ColumnRef, lo: Literal, hi: Literal) -> ex.Expr:
    """Inclusive range; folds to FALSE when lo > hi (reference ``_analyze_between``)."""
    lo_v, _ = constant_for_column(col, lo)
    hi_v, _ = constant_for_column(col, hi)
    if lo_v > hi_v:
        return ex.FoldedAtom(col, False)
    return ex.Range(col, lo_v, hi_v)


def fn_compare(catalog, name: str, args, op: str, lit: Literal) -> ex.FnCall:
    """``name(args) op number`` against a registered UDF (reference ``_analyze_fncall``)."""
    udf = catalog.udf(name)
    if udf is None:
        raise UnknownFunction(f"unknown function {name!r}")
    if udf.arity != len(args):
        raise ArityMismatch(f"function {name!r} takes {udf.arity} arguments, got {len(args)}")
    for ref in args:
        if ref.kind is not None and ref.kind.is_text:
            raise AnalysisError(f"type mismatch: TEXT column {ref} passed to {name}()")
    if lit.kind != "number":
        raise AnalysisError(f"function comparison {name}(...) {op} requires a numeric constant")
    return ex.FnCall(name, tuple(args), op, float(_number_value(lit)), fn=udf.fn)


def resolve(table, alias: str | None, column: str) -> ex.ColumnRef:
    """A ColumnRef carrying the table column's kind (what the reference's scope resolution gives)."""
    col = table.column(column)
    return ex.ColumnRef(alias or table.name, column, kind=col.kind)
