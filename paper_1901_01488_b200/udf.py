"""Symbolic tracing of registered UDFs into float64 device programs.

The reference applies a UDF row by row as a Python callable on float arguments through
``np.frompyfunc`` (``executor.py:128-146``; registry ``catalog.py:138-150``).  A device cannot run
Python, so the callable is executed ONCE with proxy operands that record every arithmetic
operation; the recording becomes a postfix program the kernel evaluates with CPython float
semantics (``+ - *`` round-to-nearest without FMA contraction, IEEE ``/``, floored ``%`` and
``//`` exactly as CPython's ``float_rem`` / ``_float_div_mod``, unary ``-``/``+``/``abs``,
``** 2``).  Python numeric constants are converted with ``float()`` at trace time — the same
conversion CPython performs when it mixes an int with a float.

Anything a trace cannot capture — comparisons / truth tests (value-dependent control flow),
``math.*`` (needs ``float(proxy)``), non-numeric results — raises
:class:`~paper_1901_01488_b200.errors.UnsupportedUdf`, loudly, instead of silently running on
the CPU.
"""

from __future__ import annotations

import math
import numbers
from dataclasses import dataclass

from . import _native as N
from .errors import UnsupportedUdf

_BINARY = {"add": N.UDF_ADD, "sub": N.UDF_SUB, "mul": N.UDF_MUL, "truediv": N.UDF_DIV,
           "mod": N.UDF_MOD, "floordiv": N.UDF_FLOORDIV}
_MAY_FAIL_DIVISOR = {N.UDF_DIV, N.UDF_MOD, N.UDF_FLOORDIV}


def _const_float(x) -> float:
    if isinstance(x, bool):
        return float(x)
    if isinstance(x, numbers.Real):
        try:
            return float(x)
        except OverflowError as exc:  # int too large to convert to float (what CPython raises)
            raise UnsupportedUdf(f"constant {x!r}: {exc}") from None
    raise TypeError(f"unsupported operand {x!r}")


class Sym:
    """Proxy operand; every arithmetic dunder returns a new Sym recording the op."""

    __slots__ = ("node",)

    def __init__(self, node):
        self.node = node

    @staticmethod
    def _wrap(x):
        if isinstance(x, Sym):
            return x.node
        return ("const", _const_float(x))

    def _bin(self, name, other, swap=False):
        try:
            o = Sym._wrap(other)
        except TypeError:
            return NotImplemented
        a, b = (o, self.node) if swap else (self.node, o)
        return Sym((name, a, b))

    def __add__(self, o): return self._bin("add", o)
    def __radd__(self, o): return self._bin("add", o, True)
    def __sub__(self, o): return self._bin("sub", o)
    def __rsub__(self, o): return self._bin("sub", o, True)
    def __mul__(self, o): return self._bin("mul", o)
    def __rmul__(self, o): return self._bin("mul", o, True)
    def __truediv__(self, o): return self._bin("truediv", o)
    def __rtruediv__(self, o): return self._bin("truediv", o, True)
    def __mod__(self, o): return self._bin("mod", o)
    def __rmod__(self, o): return self._bin("mod", o, True)
    def __floordiv__(self, o): return self._bin("floordiv", o)
    def __rfloordiv__(self, o): return self._bin("floordiv", o, True)
    def __neg__(self): return Sym(("neg", self.node))
    def __pos__(self): return self
    def __abs__(self): return Sym(("abs", self.node))

    def __pow__(self, e, mod=None):
        if mod is None and not isinstance(e, Sym) and isinstance(e, numbers.Real):
            if e == 2:
                return Sym(("square", self.node))
            if e == 1:
                return self
            if e == 0:
                return Sym(("const", 1.0))  # CPython float_pow: x ** 0 == 1.0 for every x
        raise UnsupportedUdf(f"'** {e!r}' is not supported in a device UDF (only ** 0, 1, 2)")

    def __rpow__(self, o):
        raise UnsupportedUdf("a traced value cannot be used as an exponent")

    def _refuse(self, *_):
        raise UnsupportedUdf("value-dependent control flow / comparison inside a UDF cannot be traced")

    __bool__ = __lt__ = __le__ = __gt__ = __ge__ = __eq__ = __ne__ = _refuse
    __hash__ = None

    def __float__(self):
        raise UnsupportedUdf("float()/math.* on a UDF argument cannot be traced")

    __int__ = __index__ = __round__ = __trunc__ = __floor__ = __ceil__ = __float__


@dataclass
class UdfProgram:
    """Postfix float64 program of one UDF."""

    ops: list            # [(opcode, arg_index, const)]
    n_args: int
    may_fail: bool       # contains a division/modulo by a non-constant (or zero) divisor, or ** 2
    depth: int

    def evaluate(self, args: list[float]) -> float:
        """Host reference of the device interpreter (tests only)."""
        stack: list[float] = []
        for op, a, k in self.ops:
            if op == N.UDF_ARG:
                stack.append(args[a])
            elif op == N.UDF_CONST:
                stack.append(k)
            elif op == N.UDF_NEG:
                stack[-1] = -stack[-1]
            elif op == N.UDF_ABS:
                stack[-1] = abs(stack[-1])
            elif op == N.UDF_SQUARE:
                stack[-1] = stack[-1] ** 2
            else:
                y = stack.pop()
                x = stack[-1]
                stack[-1] = {N.UDF_ADD: x.__add__, N.UDF_SUB: x.__sub__, N.UDF_MUL: x.__mul__,
                             N.UDF_DIV: x.__truediv__, N.UDF_MOD: x.__mod__,
                             N.UDF_FLOORDIV: x.__floordiv__}[op](y)
        return stack[0]


def trace(fn, n_args: int, name: str = "udf") -> UdfProgram:
    """Record ``fn(*args)`` as a device program."""
    proxies = [Sym(("arg", i)) for i in range(n_args)]
    try:
        out = fn(*proxies)
    except UnsupportedUdf as exc:
        raise UnsupportedUdf(f"UDF {name!r} cannot run on the GPU: {exc}") from None
    except Exception as exc:  # noqa: BLE001 - anything else the callable did with a proxy
        raise UnsupportedUdf(f"UDF {name!r} cannot run on the GPU: tracing raised "
                             f"{type(exc).__name__}: {exc}") from None
    if isinstance(out, Sym):
        root = out.node
    else:
        try:
            root = ("const", _const_float(out))
        except (TypeError, UnsupportedUdf):
            raise UnsupportedUdf(f"UDF {name!r} returns {type(out).__name__}, not a number") from None

    ops: list = []
    may_fail = False

    def emit(node):
        nonlocal may_fail
        kind = node[0]
        if kind == "arg":
            ops.append((N.UDF_ARG, node[1], 0.0))
        elif kind == "const":
            ops.append((N.UDF_CONST, 0, node[1]))
        elif kind in ("neg", "abs", "square"):
            emit(node[1])
            op = {"neg": N.UDF_NEG, "abs": N.UDF_ABS, "square": N.UDF_SQUARE}[kind]
            if op == N.UDF_SQUARE:
                may_fail = True
            ops.append((op, 0, 0.0))
        else:
            op = _BINARY[kind]
            emit(node[1])
            emit(node[2])
            if op in _MAY_FAIL_DIVISOR:
                divisor = node[2]
                if divisor[0] != "const" or divisor[1] == 0.0 or math.isnan(divisor[1]):
                    may_fail = True
            ops.append((op, 0, 0.0))

    emit(root)
    depth = max_depth = 0
    for op, _, _ in ops:
        depth += 1 if op in (N.UDF_ARG, N.UDF_CONST) else (0 if op in (N.UDF_NEG, N.UDF_ABS, N.UDF_SQUARE) else -1)
        max_depth = max(max_depth, depth)
    if max_depth > 16:
        raise UnsupportedUdf(f"UDF {name!r} needs an evaluation stack deeper than 16")
    if len(ops) > 255:
        raise UnsupportedUdf(f"UDF {name!r} is longer than 255 operations")
    return UdfProgram(ops, n_args, may_fail, max_depth)


def _python_message(kind: int) -> str:
    """The exception text CPython produces for a failing float op (what the reference's
    ``ExecutionError(f"UDF {name!r} failed at row {i}: {exc}")`` embeds)."""
    try:
        if kind == N.FAIL_DIV:
            1.0 / 0.0
        elif kind == N.FAIL_MOD:
            1.0 % 0.0
        elif kind == N.FAIL_FLOORDIV:
            1.0 // 0.0
        else:
            1e308 ** 2
    except Exception as exc:  # noqa: BLE001
        return str(exc)
    return "float operation failed"


FAIL_MESSAGES = {k: _python_message(k) for k in (N.FAIL_DIV, N.FAIL_MOD, N.FAIL_FLOORDIV, N.FAIL_POW)}
