"""Analyzer constant rules against the reference analyzer's frozen outputs
(tests/golden/analyzer_cases.json, made by make_analyzer_golden.py from escdb.frontend), plus the
rules this build adds for its native-width kinds (INT32 / INT16 / INT8 like INT64; FLOAT32 /
FLOAT64 never folded, the literal as the correctly rounded double)."""

import json
import os

import pytest

from paper_1901_01488_b200 import analyzer as A
from paper_1901_01488_b200 import expr as ex
from paper_1901_01488_b200.catalog import Catalog
from paper_1901_01488_b200.errors import EscdbError
from paper_1901_01488_b200.storage import Dictionary, parse_kind

HERE = os.path.dirname(os.path.abspath(__file__))
KINDS = {"i": "int64", "p": "decimal(15,2)", "d": "date", "s": "text"}


def _lit(text: str) -> A.Literal:
    if text.startswith("DATE '"):
        return A.date(text[6:-1])
    if text.startswith("'"):
        return A.string(text[1:-1])
    return A.number(text)


def _v(v):
    if isinstance(v, bool):
        return v
    if isinstance(v, int):
        return {"int": str(v)}
    if isinstance(v, float):
        return {"float": repr(v)}
    return v


def _json(e):
    if isinstance(e, ex.FoldedAtom):
        return ["folded", e.col.name, bool(e.result)]
    if isinstance(e, ex.Equality):
        return ["eq", e.col.name, _v(e.value)]
    if isinstance(e, ex.Comparison):
        return ["cmp", e.col.name, e.op, _v(e.value)]
    if isinstance(e, ex.Range):
        return ["range", e.col.name, _v(e.lo), _v(e.hi)]
    if isinstance(e, ex.FnCall):
        return ["fn", e.name, [a.name for a in e.args], e.op, _v(e.value)]
    raise TypeError(type(e))


def _outcome(fn):
    try:
        return {"ok": _json(fn())}
    except EscdbError as exc:
        return {"error": type(exc).__name__, "message": str(exc)}


def test_reference_analyzer_cases():
    cases = json.load(open(os.path.join(HERE, "golden", "analyzer_cases.json")))
    d = Dictionary(["w0", "w1", "abc"])
    cat = Catalog()
    cat.register_udf("f", 1, lambda x: x)
    checked = 0
    for c in cases:
        want = c["result"]
        if want.get("error") == "ParseError":
            continue  # SQL lexing, not constant rules (no SQL frontend here)
        if "where" in c:
            col, op, lit = c["where"]
            ref = ex.ColumnRef("t", col, kind=parse_kind(KINDS[col]))
            got = _outcome(lambda: A.compare(ref, op, _lit(lit), d if col == "s" else None))
        elif "between" in c:
            col, lo, hi = c["between"]
            ref = ex.ColumnRef("t", col, kind=parse_kind(KINDS[col]))
            got = _outcome(lambda: A.between(ref, _lit(lo), _lit(hi)))
        else:
            name, args, op, lit = c["fn"]
            refs = [ex.ColumnRef("t", a, kind=parse_kind(KINDS[a])) for a in args]
            got = _outcome(lambda: A.fn_compare(cat, name, refs, op, _lit(lit)))
        assert got == want, c
        checked += 1
    assert checked > 300


@pytest.mark.parametrize("kind", ["int32", "int16", "int8"])
def test_narrow_integer_kinds_follow_int64_rules(kind):
    a = ex.ColumnRef("t", "a", kind=parse_kind(kind))
    b = ex.ColumnRef("t", "a", kind=parse_kind("int64"))
    for lit in ("7", "10.5", "-3", "99999999999999999999", "0.125"):
        for op in ("=", "<>", "<", ">="):
            assert _json(A.compare(a, op, A.number(lit))) == _json(A.compare(b, op, A.number(lit)))
    assert isinstance(A.between(a, A.number("5"), A.number("1")), ex.FoldedAtom)


@pytest.mark.parametrize("kind", ["float32", "float64"])
def test_float_kinds_never_fold_and_take_the_rounded_double(kind):
    f = ex.ColumnRef("t", "f", kind=parse_kind(kind))
    e = A.compare(f, "=", A.number("0.5"))
    assert isinstance(e, ex.Equality) and e.value == 0.5 and isinstance(e.value, float)
    e = A.compare(f, "<>", A.number("0.1"))
    assert isinstance(e, ex.Comparison) and e.value == 0.1
    e = A.compare(f, "<", A.number("3"))
    assert e.value == 3.0 and isinstance(e.value, float)
    assert A.between(f, A.number("-0.5"), A.number("1.0")) == ex.Range(f, -0.5, 1.0)
    with pytest.raises(EscdbError):
        A.compare(f, "=", A.string("x"))
    with pytest.raises(EscdbError):
        A.compare(f, "=", A.date("2020-01-01"))


@pytest.mark.gpu
def test_float32_rule_on_the_device_is_numpy_nep50(cuda):
    """The FLOAT32 rule end to end: analyzer constant -> device compare == numpy's
    ``float32_array <op> python_float`` (NEP 50: the double rounded to float32)."""
    import numpy as np

    from paper_1901_01488_b200 import ColumnTable, count_star
    from paper_1901_01488_b200.storage import Column

    g = np.random.default_rng(3)
    x = np.concatenate([g.standard_normal(100_000).astype(np.float32),
                        np.float32([0.1, 0.5, -0.5, 1.0, 0.30000001, 1 / 3])])
    t = ColumnTable("t", [Column("f", parse_kind("float32"), x, device=cuda)])
    f = ex.ColumnRef("t", "f", kind=parse_kind("float32"))
    ops = {"=": np.equal, "<>": np.not_equal, "<": np.less, "<=": np.less_equal, ">": np.greater,
           ">=": np.greater_equal}
    for lit in ("0.1", "0.5", "-0.5", "0.30000001", "0.3333333333333333", "1"):
        for op, npop in ops.items():
            want = int(npop(x, float(lit)).sum())
            assert count_star(t, A.compare(f, op, A.number(lit))) == want, (op, lit)
    assert count_star(t, A.between(f, A.number("-0.5"), A.number("1.0"))) == int(((x >= -0.5) & (x <= 1.0)).sum())
