"""Symbolic tracing of registered UDFs into float64 device programs.

The reference applies a UDF row by row as a Python callable on float arguments through
``np.frompyfunc`` (``executor.py:128-146``; registry ``catalog.py:138-150``).  A device cannot run
Python, so the callable is executed with proxy operands that record every operation; the
recording becomes a postfix program the kernel evaluates with CPython float semantics (``+ - *``
round-to-nearest without FMA contraction, IEEE ``/``, floored ``%`` and ``//`` exactly as
CPython's ``float_rem`` / ``_float_div_mod``, unary ``-``/``+``/``abs``, ``** 2``).  Python
numeric constants are converted with ``float()`` at trace time — the same conversion CPython
performs when it mixes an int with a float.

**Branches.**  A comparison of a traced value (``<``, ``==``, ... also inside ``min`` / ``max``,
``if`` / ``else``, conditional expressions, ``and`` / ``or`` / ``not``, the truth value of a
number) is a symbolic condition; whenever Python asks for its truth value the tracer answers
from a decision script and re-runs the callable until every combination of answers has been
seen (path enumeration, at most 64 paths).  The paths form a decision tree that becomes forward
jumps in the program (``ESC_UDF_JMPF`` / ``ESC_UDF_JMP``), so a row evaluates only its own path's
operations — an operation that would fail on a branch Python does not take never fails on the
device either.

**math.**  ``math.floor`` / ``math.ceil`` / ``math.trunc`` (their integral results), ``math.sqrt``,
``math.fabs``, ``math.isnan`` / ``isinf`` / ``isfinite`` and the ``min`` / ``max`` / ``abs``
builtins trace; the callable runs against a copy of its globals in which the ``math`` module (or
functions imported from it) is replaced by tracing versions.  The integral results of
floor / ceil / trunc are exact doubles on the device; they may be compared, returned, combined
with floats, or reduced with ``%`` / ``//`` by an integer literal (CPython's exact integer
operations agree with the float ones there), but integer-by-integer ``+ - *`` — exact big-int
arithmetic in CPython — is refused.  Failures keep CPython's messages: ``cannot convert float
NaN to integer``, ``cannot convert float infinity to integer``, ``math domain error``.

Anything a trace cannot capture — ``float()`` / ``int()`` of a traced value, other ``math``
functions, ``**`` beyond 0/1/2, non-numeric results, more than 64 paths — raises
:class:`~paper_1901_01488_b200.errors.UnsupportedUdf`, loudly, instead of silently running on
the CPU.
"""

from __future__ import annotations

import math
import numbers
import threading
import types
from dataclasses import dataclass

from . import _native as N
from .errors import UnsupportedUdf

_BINARY = {"add": N.UDF_ADD, "sub": N.UDF_SUB, "mul": N.UDF_MUL, "truediv": N.UDF_DIV,
           "mod": N.UDF_MOD, "floordiv": N.UDF_FLOORDIV}
_CMP = {"lt": N.UDF_LT, "le": N.UDF_LE, "gt": N.UDF_GT, "ge": N.UDF_GE, "eq": N.UDF_EQ, "ne": N.UDF_NE}
_SWAPPED = {"lt": "gt", "le": "ge", "gt": "lt", "ge": "le", "eq": "eq", "ne": "ne"}
_UNARY = {"neg": N.UDF_NEG, "abs": N.UDF_ABS, "square": N.UDF_SQUARE, "floor": N.UDF_FLOOR,
          "ceil": N.UDF_CEIL, "trunc": N.UDF_TRUNC, "sqrt": N.UDF_SQRT, "rint": N.UDF_RINT}
_MAY_FAIL_UNARY = {"square", "floor", "ceil", "trunc", "sqrt", "rint"}
_MAY_FAIL_DIVISOR = {N.UDF_DIV, N.UDF_MOD, N.UDF_FLOORDIV}
_EXACT = 2 ** 53
MAX_PATHS = 64


def _const_float(x) -> float:
    if isinstance(x, bool):
        return float(x)
    if isinstance(x, numbers.Real):
        try:
            return float(x)
        except OverflowError as exc:  # int too large to convert to float (what CPython raises)
            raise UnsupportedUdf(f"constant {x!r}: {exc}") from None
    raise TypeError(f"unsupported operand {x!r}")


# ------------------------------------------------------------------------------------------------
# path enumeration: the truth values Python asks for, answered from a script
# ------------------------------------------------------------------------------------------------
class _Run:
    def __init__(self, script: list, expect: list):
        self.script = script
        self.expect = expect    # the conditions the previous run met at the scripted positions
        self.taken: list = []   # [(condition node, answer)]

    def decide(self, cond) -> bool:
        i = len(self.taken)
        if i < len(self.script):
            if self.expect[i] != cond:
                raise UnsupportedUdf("the UDF asks different questions on re-execution (not deterministic)")
            answer = self.script[i]
        else:
            answer = True
        self.taken.append((cond, answer))
        if len(self.taken) > 12:
            raise UnsupportedUdf("more than 12 nested decisions in one evaluation")
        return answer


_state = threading.local()


def _decide(cond) -> bool:
    run = getattr(_state, "run", None)
    if run is None:
        raise UnsupportedUdf("a traced comparison was used outside the traced call")
    return run.decide(cond)


class SymBool:
    """A symbolic comparison result; its truth value is a decision of the current path."""

    __slots__ = ("node",)

    def __init__(self, node):
        self.node = node

    def __bool__(self):
        return _decide(self.node)

    # a bool used as a number (True * x): decided, then the plain int takes part
    def _num(self):
        return 1 if bool(self) else 0

    def __add__(self, o): return self._num() + o
    def __radd__(self, o): return o + self._num()
    def __sub__(self, o): return self._num() - o
    def __rsub__(self, o): return o - self._num()
    def __mul__(self, o): return self._num() * o
    def __rmul__(self, o): return o * self._num()
    def __truediv__(self, o): return self._num() / o
    def __rtruediv__(self, o): return o / self._num()
    def __neg__(self): return -self._num()
    def __invert__(self): return ~self._num()
    __hash__ = None


class Sym:
    """Proxy operand; every arithmetic dunder returns a new Sym recording the op.  ``is_int``
    marks the integral results of floor / ceil / trunc (Python ints in the reference)."""

    __slots__ = ("node", "is_int")

    def __init__(self, node, is_int: bool = False):
        self.node = node
        self.is_int = is_int

    @staticmethod
    def _wrap(x):
        """(node, is_int, is_literal) of an operand."""
        if isinstance(x, Sym):
            return x.node, x.is_int, False
        if isinstance(x, SymBool):
            raise TypeError("decide first")
        is_int = isinstance(x, numbers.Integral)
        return ("const", _const_float(x)), is_int, True

    def _bin(self, name, other, swap=False):
        if isinstance(other, SymBool):
            other = other._num()
        try:
            o, o_int, o_lit = Sym._wrap(other)
        except TypeError:
            return NotImplemented
        if self.is_int and o_int:
            if name in ("add", "sub", "mul"):
                raise UnsupportedUdf("integer arithmetic on math.floor/ceil/trunc results is exact big-int "
                                     "arithmetic in Python and is not traced (multiply by a float instead)")
            if name in ("mod", "floordiv"):
                if swap or not o_lit:
                    raise UnsupportedUdf("integer % and // of floor/ceil/trunc results need an integer literal divisor")
                k = o[1]
                if k == 0.0:
                    raise UnsupportedUdf("integer division by the literal 0 always fails")
                if abs(k) > _EXACT:
                    raise UnsupportedUdf(f"integer divisor {k!r} beyond 2**53")
                return Sym((name, self.node, o), is_int=True)
        a, b = (o, self.node) if swap else (self.node, o)
        return Sym((name, a, b))

    def _cmp(self, name, other):
        if isinstance(other, SymBool):
            other = other._num()
        try:
            o, _, o_lit = Sym._wrap(other)
        except TypeError:
            return NotImplemented
        if o_lit and isinstance(other, numbers.Integral) and abs(int(other)) > _EXACT:
            raise UnsupportedUdf(f"comparison with the integer {other!r} beyond 2**53 (exact in Python)")
        return SymBool(("cmp", name, self.node, o))

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
    def __neg__(self): return Sym(("neg", self.node), self.is_int)
    def __pos__(self): return self
    def __abs__(self): return Sym(("abs", self.node), self.is_int)

    def __lt__(self, o): return self._cmp("lt", o)
    def __le__(self, o): return self._cmp("le", o)
    def __gt__(self, o): return self._cmp("gt", o)
    def __ge__(self, o): return self._cmp("ge", o)
    def __eq__(self, o): return self._cmp("eq", o)
    def __ne__(self, o): return self._cmp("ne", o)
    __hash__ = None

    def __bool__(self):  # truth value of a number: x != 0 (NaN is true, as in Python)
        return _decide(("cmp", "ne", self.node, ("const", 0.0)))

    def __pow__(self, e, mod=None):
        if mod is None and not isinstance(e, (Sym, SymBool)) and isinstance(e, numbers.Real):
            if e == 2:
                if self.is_int:
                    raise UnsupportedUdf("integer ** 2 of a floor/ceil/trunc result is exact big-int arithmetic")
                return Sym(("square", self.node))
            if e == 1:
                return self
            if e == 0:
                return Sym(("const", 1.0), self.is_int)  # CPython: x ** 0 == 1 (1.0 for a float)
        raise UnsupportedUdf(f"'** {e!r}' is not supported in a device UDF (only ** 0, 1, 2)")

    def __rpow__(self, o):
        raise UnsupportedUdf("a traced value cannot be used as an exponent")

    def _integral(self, kind):
        return self if self.is_int else Sym((kind, self.node), is_int=True)

    def __floor__(self): return self._integral("floor")
    def __ceil__(self): return self._integral("ceil")
    def __trunc__(self): return self._integral("trunc")

    def __round__(self, ndigits=None):
        if ndigits is not None:
            raise UnsupportedUdf("round(x, ndigits) of a UDF argument cannot be traced (round(x) can)")
        return self._integral("rint")

    def __float__(self):
        raise UnsupportedUdf("float()/int() of a UDF argument can only be traced when the UDF calls them by "
                             "name (math.floor/ceil/trunc, math.sqrt/fabs, round() and arithmetic trace too)")

    __int__ = __index__ = __float__


# ---- the tracing math module --------------------------------------------------------------------
def _sym_sqrt(x):
    if isinstance(x, Sym):
        return Sym(("sqrt", x.node))
    return math.sqrt(x)


def _sym_fabs(x):
    if isinstance(x, Sym):
        return Sym(("abs", x.node))  # float result (exact for the integral doubles too)
    return math.fabs(x)


def _sym_isnan(x):
    if isinstance(x, Sym):
        return SymBool(("cmp", "ne", x.node, x.node))
    return math.isnan(x)


def _sym_isinf(x):
    if isinstance(x, Sym):
        return SymBool(("cmp", "eq", ("abs", x.node), ("const", math.inf)))
    return math.isinf(x)


def _sym_isfinite(x):
    if isinstance(x, Sym):
        return SymBool(("cmp", "lt", ("abs", x.node), ("const", math.inf)))
    return math.isfinite(x)


_MATH_OVERRIDES = {"sqrt": _sym_sqrt, "fabs": _sym_fabs, "isnan": _sym_isnan, "isinf": _sym_isinf,
                   "isfinite": _sym_isfinite}


# builtins a UDF calls by name: float() of a traced value is the value itself (arguments are
# float64 already; floor/ceil/trunc/round results are integral doubles, exactly representable),
# int() truncates toward zero like math.trunc; anything else goes to the real builtin
def _sym_float(x=0.0):
    if isinstance(x, Sym):
        return Sym(x.node)
    if isinstance(x, SymBool):
        return float(x._num())
    return float(x)


def _sym_int(x=0, *base):
    if isinstance(x, Sym) and not base:
        return x._integral("trunc")
    if isinstance(x, SymBool) and not base:
        return x._num()
    return int(x, *base)


_BUILTIN_OVERRIDES = {"float": _sym_float, "int": _sym_int}


class _TracingMath(types.ModuleType):
    """``math`` with tracing sqrt / fabs / isnan / isinf / isfinite (floor / ceil / trunc trace
    through the dunder methods already); every other attribute is the real one."""

    def __init__(self):
        super().__init__("math")

    def __getattr__(self, name):
        if name in _MATH_OVERRIDES:
            return _MATH_OVERRIDES[name]
        return getattr(math, name)


_TMATH = _TracingMath()
_REAL_TO_SYM = {getattr(math, k): v for k, v in _MATH_OVERRIDES.items()}


def _traceable(fn):
    """``fn`` with ``math`` (and functions imported from it) swapped for tracing versions in a
    copy of its globals; other callables are returned unchanged."""
    if not isinstance(fn, types.FunctionType):
        return fn
    g = fn.__globals__
    patch = {}
    for name in fn.__code__.co_names:
        v = g.get(name)
        if v is math:
            patch[name] = _TMATH
        elif v in _REAL_TO_SYM if _hashable(v) else False:
            patch[name] = _REAL_TO_SYM[v]
        elif v is None and name in _BUILTIN_OVERRIDES:  # the builtin itself, not a global of that name
            patch[name] = _BUILTIN_OVERRIDES[name]
    if not patch:
        return fn
    ng = dict(g)
    ng.update(patch)
    f = types.FunctionType(fn.__code__, ng, fn.__name__, fn.__defaults__, fn.__closure__)
    f.__kwdefaults__ = fn.__kwdefaults__
    return f


def _hashable(v) -> bool:
    try:
        hash(v)
        return True
    except TypeError:
        return False


# ------------------------------------------------------------------------------------------------
@dataclass
class UdfProgram:
    """Postfix float64 program of one UDF (with forward jumps for traced branches)."""

    ops: list            # [(opcode, arg_index / jump offset, const)]
    n_args: int
    may_fail: bool       # a division/modulo by a non-constant (or zero) divisor, ** 2, floor/ceil/trunc, sqrt
    depth: int
    n_paths: int = 1

    def evaluate(self, args: list[float]) -> float:
        """Host reference of the device interpreter (tests only)."""
        stack: list[float] = []
        i = 0
        while i < len(self.ops):
            op, a, k = self.ops[i]
            i += 1
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
            elif op == N.UDF_FLOOR:
                stack[-1] = float(math.floor(stack[-1]))
            elif op == N.UDF_CEIL:
                stack[-1] = float(math.ceil(stack[-1]))
            elif op == N.UDF_TRUNC:
                stack[-1] = float(math.trunc(stack[-1]))
            elif op == N.UDF_SQRT:
                stack[-1] = math.sqrt(stack[-1])
            elif op == N.UDF_RINT:
                stack[-1] = float(round(stack[-1]))
            elif op == N.UDF_JMPF:
                if stack.pop() == 0.0:
                    i += a
            elif op == N.UDF_JMP:
                i += a
            else:
                y = stack.pop()
                x = stack[-1]
                if op in _CMP.values():
                    cmp = {N.UDF_LT: x < y, N.UDF_LE: x <= y, N.UDF_GT: x > y, N.UDF_GE: x >= y,
                           N.UDF_EQ: x == y, N.UDF_NE: x != y}[op]
                    stack[-1] = 1.0 if cmp else 0.0
                else:
                    stack[-1] = {N.UDF_ADD: x.__add__, N.UDF_SUB: x.__sub__, N.UDF_MUL: x.__mul__,
                                 N.UDF_DIV: x.__truediv__, N.UDF_MOD: x.__mod__,
                                 N.UDF_FLOORDIV: x.__floordiv__}[op](y)
        return stack[0]


def _result_node(out, name: str):
    if isinstance(out, Sym):
        return out.node
    if isinstance(out, SymBool):
        return out.node  # a comparison: 1.0 / 0.0, as astype(float64) of a Python bool
    try:
        return ("const", _const_float(out))
    except (TypeError, UnsupportedUdf):
        raise UnsupportedUdf(f"UDF {name!r} returns {type(out).__name__}, not a number") from None


def _paths(fn, n_args: int, name: str) -> list:
    """Every (decisions, result node) path of ``fn`` over symbolic arguments (DFS over answers)."""
    target = _traceable(fn)
    paths, script, expect = [], [], []
    while True:
        run = _Run(script, expect)
        proxies = [Sym(("arg", i)) for i in range(n_args)]
        prev = getattr(_state, "run", None)
        _state.run = run
        try:
            out = target(*proxies)
        except UnsupportedUdf as exc:
            raise UnsupportedUdf(f"UDF {name!r} cannot run on the GPU: {exc}") from None
        except Exception as exc:  # noqa: BLE001 - anything else the callable did with a proxy
            raise UnsupportedUdf(f"UDF {name!r} cannot run on the GPU: tracing raised "
                                 f"{type(exc).__name__}: {exc}") from None
        finally:
            _state.run = prev
        taken = run.taken
        paths.append((list(taken), _result_node(out, name)))
        if len(paths) > MAX_PATHS:
            raise UnsupportedUdf(f"UDF {name!r} has more than {MAX_PATHS} branch paths")
        while taken and taken[-1][1] is False:
            taken.pop()
        if not taken:
            return paths
        expect = [c for c, _ in taken]
        script = [v for _, v in taken[:-1]] + [False]


def _tree(paths: list, depth: int = 0):
    if len(paths) == 1 and len(paths[0][0]) == depth:
        return ("leaf", paths[0][1])
    cond = paths[0][0][depth][0]
    yes = [p for p in paths if p[0][depth][1]]
    no = [p for p in paths if not p[0][depth][1]]
    return ("if", cond, _tree(yes, depth + 1), _tree(no, depth + 1))


def trace(fn, n_args: int, name: str = "udf") -> UdfProgram:
    """Record ``fn(*args)`` as a device program."""
    paths = _paths(fn, n_args, name)
    tree = _tree(paths)
    ops: list = []
    may_fail = False

    def emit(node):
        nonlocal may_fail
        kind = node[0]
        if kind == "arg":
            ops.append([N.UDF_ARG, node[1], 0.0])
        elif kind == "const":
            ops.append([N.UDF_CONST, 0, node[1]])
        elif kind in _UNARY:
            emit(node[1])
            if kind in _MAY_FAIL_UNARY:
                may_fail = True
            ops.append([_UNARY[kind], 0, 0.0])
        elif kind == "cmp":
            emit(node[2])
            emit(node[3])
            ops.append([_CMP[node[1]], 0, 0.0])
        else:
            op = _BINARY[kind]
            emit(node[1])
            emit(node[2])
            if op in _MAY_FAIL_DIVISOR:
                divisor = node[2]
                if divisor[0] != "const" or divisor[1] == 0.0 or math.isnan(divisor[1]):
                    may_fail = True
            ops.append([op, 0, 0.0])

    def emit_tree(t):
        if t[0] == "leaf":
            emit(t[1])
            return
        _, cond, yes, no = t
        emit(cond)
        jf = len(ops)
        ops.append([N.UDF_JMPF, 0, 0.0])
        emit_tree(yes)
        j = len(ops)
        ops.append([N.UDF_JMP, 0, 0.0])
        ops[jf][1] = len(ops) - (jf + 1)
        emit_tree(no)
        ops[j][1] = len(ops) - (j + 1)

    emit_tree(tree)
    if len(ops) > 255:
        raise UnsupportedUdf(f"UDF {name!r} is longer than 255 operations")
    # stack heights along every path (forward jumps: one pass in op order)
    height = [-1] * (len(ops) + 1)
    height[0] = 0
    max_depth = 0
    for k, (op, a, _) in enumerate(ops):
        h = height[k]
        if h < 0:
            continue
        succ = [k + 1]
        if op in (N.UDF_ARG, N.UDF_CONST):
            h += 1
        elif op == N.UDF_JMPF:
            h -= 1
            succ.append(k + 1 + a)
        elif op == N.UDF_JMP:
            succ = [k + 1 + a]
        elif op in _BINARY.values() or op in _CMP.values():
            h -= 1
        max_depth = max(max_depth, h)
        for t in succ:
            height[t] = h
    if max_depth > 16:
        raise UnsupportedUdf(f"UDF {name!r} needs an evaluation stack deeper than 16")
    return UdfProgram([tuple(o) for o in ops], n_args, may_fail, max_depth, len(paths))


def _python_message(kind: int) -> str:
    """The exception text CPython produces for a failing op (what the reference's
    ``ExecutionError(f"UDF {name!r} failed at row {i}: {exc}")`` embeds)."""
    try:
        if kind == N.FAIL_DIV:
            1.0 / 0.0
        elif kind == N.FAIL_MOD:
            1.0 % 0.0
        elif kind == N.FAIL_FLOORDIV:
            1.0 // 0.0
        elif kind == N.FAIL_NAN_INT:
            math.floor(math.nan)
        elif kind == N.FAIL_INF_INT:
            math.floor(math.inf)
        elif kind == N.FAIL_DOMAIN:
            math.sqrt(-1.0)
        else:
            1e308 ** 2
    except Exception as exc:  # noqa: BLE001
        return str(exc)
    return "float operation failed"


FAIL_MESSAGES = {k: _python_message(k) for k in (N.FAIL_DIV, N.FAIL_MOD, N.FAIL_FLOORDIV, N.FAIL_POW,
                                                 N.FAIL_NAN_INT, N.FAIL_INF_INT, N.FAIL_DOMAIN)}
