"""UDF tracing: the recorded program reproduces CPython float semantics (checked with the host
reference evaluator), and untraceable UDFs are refused loudly."""

import math
import random

import pytest

from paper_1901_01488_b200 import _native as N
from paper_1901_01488_b200.errors import UnsupportedUdf
from paper_1901_01488_b200.udf import FAIL_MESSAGES, trace

CASES = [
    lambda b, d: (b * 3.0 + d) % 7.0,
    lambda x, y: (x * 7.0 + y) % 13.0,
    lambda x, y: (x - y) // 3.0,
    lambda x, y: -abs(x) + y / 2.5,
    lambda x, y: x ** 2 - 10 * y,
    lambda x, y: (x + 1) % -3.0,
    lambda x, y: +x - (-y) * 0.1,
    lambda x, y: 7 - x // -2,
    lambda x, y: 2.0,
]


@pytest.mark.parametrize("fn", CASES)
def test_traced_program_equals_python(fn):
    prog = trace(fn, 2)
    rng = random.Random(7)
    vals = [0.0, -0.0, 1.0, -1.0, 7.0, -9.0, 13.5, -2.25, 1e15, -3e-7, 2.0**53]
    for _ in range(300):
        x, y = rng.choice(vals + [rng.uniform(-1e4, 1e4)]), rng.choice(vals + [rng.uniform(-1e4, 1e4)])
        want = fn(x, y)
        got = prog.evaluate([x, y])
        assert (math.isnan(want) and math.isnan(got)) or (want == got and math.copysign(1, want) == math.copysign(1, got)), (x, y)


def test_cpython_floored_semantics():
    assert trace(lambda x, y: x % y, 2).evaluate([-9.0, 7.0]) == 5.0
    assert math.copysign(1, trace(lambda x, y: x % y, 2).evaluate([7.0, -7.0])) == -1.0


def test_may_fail_flags():
    assert not trace(lambda x: x % 7.0, 1).may_fail
    assert trace(lambda x, y: x % y, 2).may_fail
    assert trace(lambda x: x / 0.0, 1).may_fail
    assert trace(lambda x: x ** 2, 1).may_fail


@pytest.mark.parametrize("fn,msg", [
    (lambda x: math.exp(x), "float()"),
    (lambda x: x ** 3, "\\*\\* 3"),
    (lambda x: "s", "returns str"),
    (lambda x: round(x, 2), "ndigits"),
])
def test_untraceable_udfs_are_refused(fn, msg):
    with pytest.raises(UnsupportedUdf, match=msg):
        trace(fn, 1, "f")


def test_failure_messages_are_cpythons():
    assert FAIL_MESSAGES[N.FAIL_DIV] == "float division by zero"
    assert FAIL_MESSAGES[N.FAIL_FLOORDIV] == "float floor division by zero"
    try:
        1.0 % 0.0
    except ZeroDivisionError as e:
        assert FAIL_MESSAGES[N.FAIL_MOD] == str(e)


BRANCHY = [
    (lambda x, y: x if x > y else y * 0.5, 2),
    (lambda x, y: min(x, y, 0.25) - max(x, -y), 2),
    (lambda x, y: -1.0 if x < -1 else (1.0 if x > 1 else x), 2),
    (lambda x, y: x / y if y != 0 else 0.0, 2),
    (lambda x, y: math.floor(x / 10.0) % 7 + y, 2),
    (lambda x, y: math.ceil(x) // 3, 2),
    (lambda x, y: math.trunc(x) * 0.5 - math.fabs(y), 2),
    (lambda x, y: math.sqrt(abs(x)) if x == x else y, 2),
    (lambda x, y: 1.0 if (x > 0 and y > 0) or x < -5 else 2.0, 2),
    (lambda x, y: 0.0 if math.isnan(x) or math.isinf(y) else x, 2),
    (lambda x, y: x > y, 2),
    (lambda x, y: (x > 0) * 3.0 + y, 2),
]


@pytest.mark.parametrize("fn,n", BRANCHY)
def test_branchy_trace_equals_python(fn, n):
    """Path-enumerated programs (jumps, comparisons, floor/ceil/trunc/sqrt/fabs/isnan/isinf)
    reproduce CPython on every path, errors included."""
    prog = trace(fn, n)
    rng = random.Random(11)
    special = [0.0, -0.0, 1.0, -1.0, 7.0, -9.0, 13.5, -2.25, 1e15, math.nan, math.inf, -math.inf]
    for _ in range(1500):
        args = [rng.choice(special + [rng.uniform(-50, 50)]) for _ in range(n)]
        try:
            want = ("ok", float(fn(*args)))
        except (ArithmeticError, ValueError) as exc:
            want = ("err", str(exc))
        try:
            got = ("ok", prog.evaluate(args))
        except (ArithmeticError, ValueError) as exc:
            got = ("err", str(exc))
        if want[0] == got[0] == "ok" and math.isnan(want[1]):
            assert math.isnan(got[1]), args
        else:
            assert want == got, args


@pytest.mark.parametrize("fn", [lambda x: math.floor(x) + math.floor(x), lambda x: x.__float__(), lambda x: math.exp(x),
                                lambda x: math.floor(x) * 2, lambda x: x ** 3, lambda x: round(x, 1),
                                lambda x: int(x) * 2])
def test_untraceable_branchy_refused(fn):
    with pytest.raises(UnsupportedUdf):
        trace(fn, 1)


def _builtin_calls():
    return {
        "float": (lambda a, b: float(a) / 3 + b),
        "int": (lambda a, b: int(a / 7) + b),
        "round": (lambda a, b: round(a / 4) - b),
        "round_cmp": (lambda a, b: 1.0 if round(a * 0.5) == round(b * 0.5) else 0.0),
        "int_mod": (lambda a, b: int(a) % 3 if a > 0 else int(b) // 2),
        "round_fails": (lambda a, b: round(a / b)),
    }


@pytest.mark.parametrize("name", sorted(_builtin_calls()))
def test_builtin_float_int_round_trace(name):
    """float() / int() / round() called by name trace (identity, truncation, ties-to-even) and the
    program equals the Python call, errors included (NaN / inf / division by zero)."""
    fn = _builtin_calls()[name]
    prog = trace(fn, 2, name)
    g = random.Random(9)
    for _ in range(3000):
        a = g.choice([g.uniform(-50, 50), g.randint(-20, 20) + 0.5, float(g.randint(-9, 9)), 0.0, math.inf, math.nan])
        b = g.choice([g.uniform(-50, 50), float(g.randint(-20, 20)), 0.0, -2.5])
        try:
            want = ("ok", fn(a, b))
        except (ArithmeticError, ValueError) as exc:
            want = ("err", str(exc))
        try:
            got = ("ok", prog.evaluate([a, b]))
        except (ArithmeticError, ValueError) as exc:
            got = ("err", str(exc))
        if want[0] == got[0] == "ok" and isinstance(want[1], float) and math.isnan(want[1]):
            assert math.isnan(got[1]), (a, b)
        else:
            assert want == got, (a, b)
