"""P0: resolved predicate tree -> flat device program (``esc_program_t``).

Replaces the tree-walking numpy interpreter of the reference (``_eval_mask`` / ``_eval_atom`` /
``_eval_fncall``, ``executor.py:73-199``) with a compile step.  The program is a short list of
32-byte instructions the kernel dispatches once per lane per tile:

* every atom becomes one instruction that evaluates the atom on 4*C rows and merges the result
  into a running bit-mask accumulator with ``combine`` = SET / AND / OR (optionally negated);
* nested connectives that cannot be flattened become PUSH ... POP groups; ``NOT`` of a group
  becomes a NOT instruction (two-valued, so NOT re-admits NULL rows: ``executor.py:197-198``);
* the kernel tracks a "care" mask (rows whose value can still change the result) so a UDF that
  cannot fail is only evaluated on rows the short-circuit leaves open.

Comparison semantics are fixed here, on the host, exactly as numpy evaluates the reference's
``values <op> const`` (NEP 50): the comparison domain is ``np.result_type`` of the column dtype
and the constant — int64 (exact, also for out-of-dtype-range Python ints, which numpy compares
mathematically; constants outside int64 fold), float32 (constant rounded via float64, as numpy
does) or float64 (ints rounded to nearest).  TEXT ordering predicates become a bitmap LUT over
dictionary codes built with Python string comparisons (``executor.py:73-94``).
"""

from __future__ import annotations

import os

import ctypes as C
import threading
import warnings
import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import expr as ex
from .errors import ExecutionError
from .udf import UdfProgram, trace

# count / selection scans stage nullable columns' NULLs as packed bits (ESC_PACKED_NULLS=0: bytes)
_PACKED_NULLS = os.environ.get("ESC_PACKED_NULLS", "1") == "1"


def set_packed_nulls(on: bool) -> bool:
    """Stage packed NULL bitmaps in scans (True) or the byte masks; returns the previous setting
    (tests, measurement).  Affects predicates compiled afterwards."""
    global _PACKED_NULLS
    prev, _PACKED_NULLS = _PACKED_NULLS, bool(on)
    return prev

_I64_MIN, _I64_MAX = -(2**63), 2**63 - 1
_NP_OF_TORCH = {
    torch.int8: np.int8, torch.int16: np.int16, torch.int32: np.int32, torch.int64: np.int64,
    torch.uint8: np.uint8, torch.uint16: np.uint16, torch.uint32: np.uint32,
    torch.float32: np.float32, torch.float64: np.float64,
}
_LUT_OPS = {"<": str.__lt__, "<=": str.__le__, ">": str.__gt__, ">=": str.__ge__}


@dataclass
class CompiledPredicate:
    """Device program for one predicate over one table (cached per table)."""

    pred: ex.Expr
    program: N.EscProgram
    columns: list                 # Column per slot
    slot_of: dict                 # column name -> slot
    lut: torch.Tensor | None
    udf_index: dict               # id(FnCall node) -> udf slot
    unbound: list                 # FnCall nodes without an implementation
    n_udfs: int
    may_fail: bool                # some UDF is evaluated densely (can raise)
    col_array: object = field(default=None, repr=False)
    c_plans: dict = field(default_factory=dict, repr=False)  # prepared one-pass launches (executor)
    shapes: dict = field(default_factory=dict, repr=False)   # one-pass output templates (executor)

    @property
    def ncols(self) -> int:
        return len(self.columns)

    def column_array(self, extra=()):
        """ctypes esc_column_t[] of the slots (+ projection-only columns appended); cached (the
        columns are immutable, so their device pointers are too) — callers must not mutate it."""
        key = tuple(id(c) for c in extra)
        cache = self.col_array if isinstance(self.col_array, dict) else {}
        arr = cache.get(key)
        if arr is None:
            arr = cache[key] = self._build_column_array(extra)
            self.col_array = cache
        return arr

    def tile_rows(self) -> int:
        """Tile geometry the scan kernels use for this program (cached)."""
        tr = getattr(self, "_tile_rows", None)
        if tr is None:
            tr = self._tile_rows = int(N.load_library().esc_tile_rows(C.byref(self.program), self.column_array(),
                                                                      self.ncols))
        return tr

    def _build_column_array(self, extra=()):
        cols = list(self.columns) + list(extra)
        arr = (N.EscColumn * max(len(cols), 1))()
        for i, col in enumerate(cols):
            N.require_cuda(col.values, f"column {col.name!r}")
            arr[i].data = col.values.data_ptr() if len(col) else None
            arr[i].nulls = col.nulls.data_ptr() if col.nulls is not None and len(col) else None
            nb = col.null_bits if _PACKED_NULLS and col.nulls is not None and len(col) else None
            arr[i].null_bits = nb.data_ptr() if nb is not None else None
            arr[i].dtype = N.dtype_code(col.values)
            arr[i].flags = 0
        return arr


def _np_dtype(col) -> np.dtype:
    return np.dtype(_NP_OF_TORCH[col.values.dtype])


def _fold_int(op: str, v: int) -> bool:
    """Truth of ``x <op> v`` for every int64 ``x`` when ``v`` lies outside int64."""
    above = v > _I64_MAX
    return {"=": False, "<>": True, "<": above, "<=": above, ">": not above, ">=": not above}[op]


def _as_f32(v: float) -> float:
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        return float(np.float32(v))


def domain_const(dt: np.dtype, v, op: str):
    """(domain, constant) numpy would compare ``array[dt] <op> v`` in, or ("fold", bool)."""
    if isinstance(v, (bool, np.bool_)):
        v = int(v)
    if isinstance(v, (np.integer, np.floating)):  # strong numpy scalar (np.float64 is a float!)
        rt = np.result_type(dt, v)
        if rt.kind in "iu":
            return N.DOM_I64, int(v)
        if rt == np.float32:
            return N.DOM_F32, _as_f32(float(v))
        if rt == np.float64:
            return N.DOM_F64, float(v)
    elif isinstance(v, int):  # weak Python int
        if dt.kind in "iu":
            if _I64_MIN <= v <= _I64_MAX:
                return N.DOM_I64, int(v)
            return "fold", _fold_int(op, v)
        if dt == np.float32:
            return N.DOM_F32, _as_f32(float(v))
        return N.DOM_F64, float(v)
    elif isinstance(v, float):  # weak Python float
        if dt == np.float32:
            return N.DOM_F32, _as_f32(v)
        return N.DOM_F64, float(v)
    raise ExecutionError(f"cannot compare a {dt} column with {v!r}")


def _set_const(slot: N.EscConst, domain: int, value):
    if domain == N.DOM_I64:
        slot.i = int(value)
    else:
        slot.f = float(value)


class _Builder:
    def __init__(self, table, pred):
        self.table = table
        self.pred = pred
        self.instrs: list = []
        self.columns: list = []
        self.slot_of: dict = {}
        self.lut_words: list = []
        self.udfs: list = []
        self.udf_ops: list = []
        self.udf_index: dict = {}
        self.unbound: list = []
        self.depth = self.max_depth = 0
        self.may_fail = False

    # -- helpers -----------------------------------------------------------------------------
    def slot(self, ref: ex.ColumnRef) -> int:
        name = ref.name
        if name not in self.slot_of:
            if not self.table.has_column(name):
                raise ExecutionError(f"table {self.table.name!r} has no column {name!r}")
            if len(self.columns) >= N.MAX_COLS:
                raise ExecutionError(f"predicate references more than {N.MAX_COLS} columns")
            self.slot_of[name] = len(self.columns)
            self.columns.append(self.table.column(name))
        return self.slot_of[name]

    def instr(self, op, combine=N.COMB_SET, neg=False, **kw):
        if len(self.instrs) >= N.MAX_INSTRS:
            raise ExecutionError(f"predicate needs more than {N.MAX_INSTRS} device instructions")
        d = dict(op=op, combine=combine, neg=int(neg))
        d.update(kw)
        self.instrs.append(d)

    # -- tree ----------------------------------------------------------------------------------
    def emit(self, node, mode):
        while isinstance(node, ex.Not) and isinstance(node.child, ex.Not):
            node = node.child.child
        if isinstance(node, ex.Not) and isinstance(node.child, ex.ATOM_TYPES):
            return self.atom(node.child, mode, True)
        if isinstance(node, ex.ATOM_TYPES):
            return self.atom(node, mode, False)
        negate = isinstance(node, ex.Not)
        inner = node.child if negate else node
        if not isinstance(inner, (ex.And, ex.Or)):
            raise ExecutionError(f"unknown atom {inner!r}")
        if not inner.items:
            raise ExecutionError(f"empty {type(inner).__name__}")
        op = N.COMB_AND if isinstance(inner, ex.And) else N.COMB_OR
        if len(inner.items) == 1 and not negate:
            return self.emit(inner.items[0], mode)
        if mode == N.COMB_SET:
            self.body(inner.items, op)
            if negate:
                self.instr(N.OP_NOT)
        elif mode == op and not negate:
            for item in inner.items:
                self.emit(item, op)
        else:
            self.instr(N.OP_PUSH, mode)
            self.depth += 1
            self.max_depth = max(self.max_depth, self.depth)
            self.body(inner.items, op)
            if negate:
                self.instr(N.OP_NOT)
            self.instr(N.OP_POP, mode)
            self.depth -= 1

    def body(self, items, op):
        self.emit(items[0], N.COMB_SET)
        for item in items[1:]:
            self.emit(item, op)

    # -- atoms --------------------------------------------------------------------------------
    def atom(self, a, mode, neg):
        if isinstance(a, ex.Equality):
            return self.compare(a.col, "=", a.value, mode, neg)
        if isinstance(a, ex.Comparison):
            if isinstance(a.value, str):
                return self.lut(a.col, [(a.op, a.value)], mode, neg)
            return self.compare(a.col, a.op, a.value, mode, neg)
        if isinstance(a, ex.Range):
            if isinstance(a.lo, str):
                return self.lut(a.col, [(">=", a.lo), ("<=", a.hi)], mode, neg)
            return self.range(a, mode, neg)
        if isinstance(a, ex.ColumnCompare):
            return self.colcmp(a, mode, neg)
        if isinstance(a, ex.FnCall):
            return self.fncall(a, mode, neg)
        if isinstance(a, ex.FoldedAtom):
            if a.result:
                return self.instr(N.OP_NOTNULL, mode, neg, col_a=self.slot(a.col))
            self.slot(a.col)
            return self.instr(N.OP_FALSE, mode, neg)
        raise ExecutionError(f"unknown atom {a!r}")

    def compare(self, ref, op, value, mode, neg):
        if op not in N.CMP_CODE:
            raise ExecutionError(f"unknown comparison operator {op!r}")
        s = self.slot(ref)
        col = self.columns[s]
        if isinstance(value, str):
            raise ExecutionError(f"cannot compare column {ref} with string {value!r} by '{op}'")
        dom, k = domain_const(_np_dtype(col), value, op)
        if dom == "fold":
            if k:
                return self.instr(N.OP_NOTNULL, mode, neg, col_a=s)
            return self.instr(N.OP_FALSE, mode, neg)
        self.instr(N.OP_CMP, mode, neg, cmp=N.CMP_CODE[op], domain=dom, col_a=s, k0=k)

    def range(self, a: ex.Range, mode, neg):
        s = self.slot(a.col)
        dt = _np_dtype(self.columns[s])
        lo = domain_const(dt, a.lo, ">=")
        hi = domain_const(dt, a.hi, "<=")
        if lo[0] != "fold" and lo[0] == hi[0]:
            return self.instr(N.OP_RANGE, mode, neg, domain=lo[0], col_a=s, k0=lo[1], k1=hi[1])
        # mixed domains: (v >= lo) & (v <= hi), each compared in its own domain
        pair = ex.And((ex.Comparison(a.col, ">=", a.lo), ex.Comparison(a.col, "<=", a.hi)))
        self.emit(ex.Not(pair) if neg else pair, mode)

    def colcmp(self, a: ex.ColumnCompare, mode, neg):
        if a.op not in N.CMP_CODE:
            raise ExecutionError(f"unknown comparison operator {a.op!r}")
        sa, sb = self.slot(a.left), self.slot(a.right)
        rt = np.result_type(_np_dtype(self.columns[sa]), _np_dtype(self.columns[sb]))
        dom = N.DOM_I64 if rt.kind in "iu" else N.DOM_F32 if rt == np.float32 else N.DOM_F64
        self.instr(N.OP_COLCMP, mode, neg, cmp=N.CMP_CODE[a.op], domain=dom, col_a=sa, col_b=sb)

    def lut(self, ref, conds, mode, neg):
        s = self.slot(ref)
        col = self.columns[s]
        if col.dictionary is None:
            raise ExecutionError(f"column {ref} has no dictionary for a string comparison")
        for op, _ in conds:
            if op not in _LUT_OPS:
                raise ExecutionError(f"unsupported TEXT comparison operator {op!r}")
        words = col.dictionary.strings()
        if not words:
            return self.instr(N.OP_FALSE, mode, neg)
        hit = np.ones(len(words), dtype=bool)
        for op, value in conds:
            f = _LUT_OPS[op]
            hit &= np.fromiter((f(w, value) for w in words), dtype=bool, count=len(words))
        nwords = (len(words) + 31) // 32
        bits = np.zeros(nwords * 32, dtype=bool)
        bits[: len(words)] = hit
        packed32 = np.packbits(bits, bitorder="little").view("<u4")  # bit b of word w = code 32w+b
        offset = len(self.lut_words)
        self.lut_words.extend(int(w) for w in packed32)
        self.instr(N.OP_LUT, mode, neg, col_a=s, aux=offset, aux2=len(words))

    def fncall(self, a: ex.FnCall, mode, neg):
        arg_slots = [self.slot(r) for r in a.args]
        if a.fn is None:
            self.unbound.append(a)
            return self.instr(N.OP_FALSE, mode, neg)
        if a.op not in N.CMP_CODE:
            raise ExecutionError(f"unknown comparison operator {a.op!r}")
        if len(self.udfs) >= N.MAX_UDFS:
            raise ExecutionError(f"predicate has more than {N.MAX_UDFS} UDF calls")
        if len(a.args) > N.MAX_UDF_ARGS:
            raise ExecutionError(f"UDF {a.name!r} has more than {N.MAX_UDF_ARGS} arguments")
        prog: UdfProgram = _trace_cached(a.fn, len(a.args), a.name)
        if len(self.udf_ops) + len(prog.ops) > N.MAX_UDF_OPS:
            raise ExecutionError(f"UDF programs exceed {N.MAX_UDF_OPS} operations")
        divs = []
        for r in a.args:
            kind = r.kind
            divs.append(float(10 ** kind.scale) if kind is not None and getattr(kind, "is_decimal", False)
                        and kind.scale else 0.0)
        index = len(self.udfs)
        self.udfs.append(dict(first_op=len(self.udf_ops), n_ops=len(prog.ops), n_args=len(a.args),
                              dense=int(prog.may_fail), arg_col=arg_slots, arg_div=divs))
        self.udf_ops.extend(prog.ops)
        self.udf_index[id(a)] = index
        self.may_fail |= prog.may_fail
        try:
            k = float(a.value)
        except (TypeError, ValueError, OverflowError):
            raise ExecutionError(f"UDF comparison constant {a.value!r} is not numeric") from None
        self.instr(N.OP_UDF, mode, neg, cmp=N.CMP_CODE[a.op], domain=N.DOM_F64, aux=index, k0=k)

    # -- output -------------------------------------------------------------------------------
    def build(self) -> CompiledPredicate:
        self.emit(self.pred, N.COMB_SET)
        prog = N.EscProgram()
        prog.abi_version = N.ABI_VERSION
        prog.n_instrs = len(self.instrs)
        prog.n_udfs = len(self.udfs)
        prog.n_udf_ops = len(self.udf_ops)
        prog.max_depth = self.max_depth
        if self.max_depth > N.MAX_STACK:
            raise ExecutionError(f"predicate nests deeper than {N.MAX_STACK} groups")
        for i, d in enumerate(self.instrs):
            I = prog.instrs[i]
            I.op, I.combine, I.neg = d["op"], d["combine"], d["neg"]
            I.cmp = d.get("cmp", 0)
            dom = d.get("domain", N.DOM_I64)
            I.domain = dom
            I.col_a, I.col_b = d.get("col_a", 0), d.get("col_b", 0)
            I.aux, I.aux2 = d.get("aux", 0), d.get("aux2", 0)
            _set_const(I.k0, dom, d.get("k0", 0))
            _set_const(I.k1, dom, d.get("k1", 0))
        for i, u in enumerate(self.udfs):
            U = prog.udfs[i]
            U.first_op, U.n_ops, U.n_args, U.dense = u["first_op"], u["n_ops"], u["n_args"], u["dense"]
            for j, (s, dv) in enumerate(zip(u["arg_col"], u["arg_div"])):
                U.arg_col[j] = s
                U.arg_div[j] = dv
        for i, (op, arg, k) in enumerate(self.udf_ops):
            prog.udf_ops[i].op, prog.udf_ops[i].arg, prog.udf_ops[i].k = op, arg, k
        lut = None
        if self.lut_words:
            lut = torch.tensor(np.asarray(self.lut_words, dtype=np.uint32).view(np.int32),
                               dtype=torch.int32, device=self.table.device)
            prog.lut = lut.data_ptr()
            prog.lut_words = len(self.lut_words)
        return CompiledPredicate(self.pred, prog, self.columns, self.slot_of, lut, self.udf_index,
                                 self.unbound, len(self.udfs), self.may_fail)


_trace_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_trace_lock = threading.Lock()


def _trace_cached(fn, n_args: int, name: str) -> UdfProgram:
    try:
        with _trace_lock:
            per_fn = _trace_cache.setdefault(fn, {})
    except TypeError:  # not weak-referenceable (e.g. a builtin): trace every time
        return trace(fn, n_args, name)
    key = (n_args, name)
    if key not in per_fn:
        per_fn[key] = trace(fn, n_args, name)
    return per_fn[key]


# compiled programs, per table (weak), per predicate (+ identity of the bound UDFs)
_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_cache_lock = threading.Lock()


def _key(pred: ex.Expr):
    fns = tuple(id(a.fn) for a in ex.atoms(pred) if isinstance(a, ex.FnCall))
    try:
        hash(pred)
        return (pred, fns)
    except TypeError:
        return (id(pred), fns)


def compile_predicate(table, pred: ex.Expr) -> CompiledPredicate:
    """Compile (or fetch from the per-table cache) the device program of ``pred``."""
    with _cache_lock:
        per_table = _cache.setdefault(table, {})
        seen = per_table.get(("id", id(pred)))  # the same tree object again: no re-keying
    if seen is not None and seen[0] is pred:
        return seen[1]
    orig = pred
    pred = ex.adopt(pred)  # trees from the reference analyzer drive the engine unchanged
    key = _key(pred)
    with _cache_lock:
        hit = per_table.get(key)
    if hit is not None:
        with _cache_lock:
            per_table[("id", id(orig))] = (orig, hit)  # holds ``orig``: its id stays unique
        return hit
    cp = _Builder(table, pred).build()
    with _cache_lock:
        if len(per_table) > 512:
            per_table.clear()
        per_table[key] = cp
        per_table[("id", id(orig))] = (orig, cp)
    return cp


def program_summary(cp: CompiledPredicate) -> list[str]:
    """Human-readable listing of a compiled program (debugging / tests)."""
    names = {v: k for k, v in vars(N).items() if k.startswith("OP_") and isinstance(v, int)}
    comb = {0: "SET", 1: "AND", 2: "OR"}
    out = []
    for i in range(cp.program.n_instrs):
        I = cp.program.instrs[i]
        out.append(f"{names.get(I.op, I.op)} {comb[I.combine]}{' NEG' if I.neg else ''} "
                   f"cmp={I.cmp} dom={I.domain} a={I.col_a} b={I.col_b}")
    return out


def sizeof_program() -> int:
    return C.sizeof(N.EscProgram)
