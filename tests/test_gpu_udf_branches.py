"""UDFs with branches and math on the device vs the oracle (the reference's per-row Python call):
conditional expressions, if/else, min/max, and/or, math.floor/ceil/trunc/sqrt/fabs/isnan,
float()/int()/round(), in the
interpreter and the JIT tier, over the mixed-kind table (NULLs, DECIMAL, DATE, float32), with the
reference's error semantics (a failing op on a branch Python does not take never fails)."""

import math

import numpy as np
import pytest

from helpers import UDFS, device_table, mixed_arrays, oracle_table
from oracle import esc_oracle as O

pytestmark = pytest.mark.gpu


def _relu(x):
    return x if x > 0 else 0.0


def _piecewise(x, y):
    if x < -100:
        return y * 2.0
    elif x > 500 and y != 0:
        return x / y
    return math.floor(x / 7.0) % 5


BRANCHY = {
    "relu": _relu,
    "clip": lambda x: -50.0 if x < -50 else (50.0 if x > 50 else x),
    "mn": lambda x, y: min(x, y) * 2.0,
    "mx3": lambda x, y: max(x, y, 300.0),
    "safe": lambda x, y: x / y if y != 0 else -1.0,        # the division never fails
    "unsafe": lambda x, y: x / y if x > 900 else 0.0,      # fails only where x > 900 and y == 0
    "fl": lambda x: math.floor(x / 10.0) % 7,
    "cl": lambda x: math.ceil(x * 0.25) // 3,
    "tr": lambda x: math.trunc(x / 3.0) * 0.5,
    "sq": lambda x: math.sqrt(x) if x >= 0 else -math.sqrt(-x),
    "sqfail": lambda x: math.sqrt(x - 500.0),              # math domain error below 500
    "band": lambda x, y: 1.0 if (x > 0 and y > 0) or x < -5 else 2.0,
    "isn": lambda x: 0.0 if math.isnan(x) else math.fabs(x),
    "pw": _piecewise,
    "cmpres": lambda x, y: x > y,                          # a bool result: 1.0 / 0.0
    # builtins called by name: float() is the value, int() truncates, round() ties to even
    "flt": lambda x: float(x) / 3.0 + 1.0,
    "it": lambda x: int(x / 7.0) % 4,
    "rnd": lambda x: round(x / 4.0) * 2.0,
    "rndf": lambda x, y: round(x / y),                     # ZeroDivisionError, NaN / inf errors
}
ALL = {**UDFS, **BRANCHY}


@pytest.fixture(scope="module")
def mixed(cuda):
    arrays = mixed_arrays(50_003, seed=11)
    return arrays, device_table("data", arrays, device=cuda), oracle_table("data", arrays)


def _pred(j):
    from paper_1901_01488_b200 import serde

    return serde.from_json(j, "data", ALL)


def _outcome(fn, *args, errors=()):
    try:
        return ("ok", fn(*args))
    except errors as exc:
        return ("err", str(exc))


def _cases():
    a, b, f, val, when = ["a", None], ["b", None], ["f", None], ["val", 2], ["when", None]
    out = []
    for name, args in (("relu", [b]), ("clip", [b]), ("mn", [a, b]), ("mx3", [a, b]), ("safe", [a, b]),
                       ("unsafe", [a, b]), ("fl", [b]), ("cl", [a]), ("tr", [val]), ("sq", [b]),
                       ("sqfail", [a]), ("band", [b, f]), ("isn", [f]), ("pw", [b, a]), ("cmpres", [a, b]),
                       ("fl", [f]), ("cl", [when]), ("flt", [a]), ("it", [b]), ("rnd", [val]), ("rndf", [a, b]),
                       ("rnd", [f]), ("it", [f])):
        for op, k in ((">", 0.0), ("<=", 2.0), ("=", 1.0)):
            out.append(["fn", name, args, op, k])
    # short circuits around failing branchy UDFs (reference whole-slice semantics)
    out.append(["and", [["cmp", a, "<", 0], ["fn", "sqfail", [a], ">", 1.0]]])
    out.append(["or", [["cmp", a, ">=", 0], ["fn", "unsafe", [a, b], ">", 0.0]]])
    out.append(["not", ["fn", "pw", [b, a], ">", 1.0]])
    return out


@pytest.mark.parametrize("tier", [0, 2])
def test_branchy_udfs_match_reference(mixed, tier):
    from paper_1901_01488_b200 import _native as N, count_star, eval_predicate, materialize
    from paper_1901_01488_b200.errors import ExecutionError

    arrays, t, ot = mixed
    N.set_jit(tier, 0)
    try:
        for j in _cases():
            want = _outcome(O.count_star, ot, j, ALL, errors=(O.OracleExecutionError,))
            got = _outcome(count_star, t, _pred(j), errors=(ExecutionError,))
            assert got == want, j
            if want[0] == "ok":
                rows = eval_predicate(t, _pred(j)).to_indices().cpu().numpy()
                assert np.array_equal(rows, O.eval_predicate(ot, j, None, ALL)), j
                (c,) = materialize(t, _pred(j), ["id"])
                assert np.array_equal(c.to_numpy()[0], O.materialize(ot, j, ["id"], ALL)["id"].values), j
    finally:
        N.set_jit(1, 1 << 22)


def test_udf_error_messages_are_cpythons(mixed):
    """The new failure kinds carry CPython's exact text."""
    from paper_1901_01488_b200.udf import FAIL_MESSAGES
    from paper_1901_01488_b200 import _native as N

    assert FAIL_MESSAGES[N.FAIL_DOMAIN] == "math domain error"
    assert FAIL_MESSAGES[N.FAIL_NAN_INT] == "cannot convert float NaN to integer"
    assert FAIL_MESSAGES[N.FAIL_INF_INT] == "cannot convert float infinity to integer"
