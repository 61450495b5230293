"""Host-side predicate compiler (no GPU): program shape, NEP 50 domains, constant folding, TEXT LUT
bitmaps, nesting, limits."""

import ctypes as C

import numpy as np
import pytest

from paper_1901_01488_b200 import _native as N
from paper_1901_01488_b200 import expr as ex
from paper_1901_01488_b200.compiler import compile_predicate, domain_const
from paper_1901_01488_b200.errors import ExecutionError
from paper_1901_01488_b200.storage import (KIND_FLOAT32, KIND_INT32, KIND_INT64, KIND_INT8, KIND_TEXT, Column,
                                           ColumnTable, Dictionary, decimal)

WORDS = ["pear", "apple", "fig", "kiwi", "banana"]


@pytest.fixture(scope="module")
def t():
    n = 64
    return ColumnTable("t", [
        Column("a", KIND_INT32, np.arange(n, dtype=np.int32), device="cpu"),
        Column("b", KIND_INT64, np.arange(n, dtype=np.int64), np.arange(n) % 7 == 0, device="cpu"),
        Column("g", KIND_INT8, np.zeros(n, np.int8), device="cpu"),
        Column("f", KIND_FLOAT32, np.zeros(n, np.float32), device="cpu"),
        Column("s", KIND_TEXT, (np.arange(n) % 5).astype(np.int8), None, Dictionary(WORDS), device="cpu"),
        Column("v", decimal(15, 2), np.arange(n, dtype=np.int64), device="cpu"),
    ])


def r(c):
    return ex.ColumnRef("t", c)


def ops(cp):
    return [(cp.program.instrs[i].op, cp.program.instrs[i].combine, cp.program.instrs[i].neg)
            for i in range(cp.program.n_instrs)]


def test_flat_and_chain(t):
    cp = compile_predicate(t, ex.And((ex.Range(r("a"), 1, 5), ex.Equality(r("b"), 3), ex.Comparison(r("a"), "<", 9))))
    assert ops(cp) == [(N.OP_RANGE, N.COMB_SET, 0), (N.OP_CMP, N.COMB_AND, 0), (N.OP_CMP, N.COMB_AND, 0)]
    assert cp.program.max_depth == 0 and cp.ncols == 2


def test_nested_groups_and_not(t):
    p = ex.And((ex.Range(r("a"), 1, 5), ex.Not(ex.Or((ex.Equality(r("b"), 3), ex.Equality(r("a"), 2))))))
    cp = compile_predicate(t, p)
    assert [o[0] for o in ops(cp)] == [N.OP_RANGE, N.OP_PUSH, N.OP_CMP, N.OP_CMP, N.OP_NOT, N.OP_POP]
    assert cp.program.max_depth == 1
    # NOT of an atom is a flag, double NOT cancels, same-op nesting flattens
    cp = compile_predicate(t, ex.Or((ex.Not(ex.Equality(r("a"), 1)), ex.Not(ex.Not(ex.Or((ex.Equality(r("a"), 2),
                                                                                           ex.Equality(r("a"), 3))))))))
    assert ops(cp) == [(N.OP_CMP, N.COMB_SET, 1), (N.OP_CMP, N.COMB_OR, 0), (N.OP_CMP, N.COMB_OR, 0)]


def test_nep50_domains():
    i32, f32, i64 = np.dtype(np.int32), np.dtype(np.float32), np.dtype(np.int64)
    assert domain_const(i32, 5, "<") == (N.DOM_I64, 5)
    assert domain_const(i32, 2**40, "<") == (N.DOM_I64, 2**40)        # mathematically (numpy 2)
    assert domain_const(i32, 2**70, "<") == ("fold", True)
    assert domain_const(i32, 2**70, "=") == ("fold", False)
    assert domain_const(i64, -(2**70), ">=") == ("fold", True)
    assert domain_const(i32, 1050.5, "<") == (N.DOM_F64, 1050.5)
    dom, k = domain_const(f32, 0.1, "=")
    assert dom == N.DOM_F32 and k == float(np.float32(0.1))
    n = 2**54 + 2**30 + 1   # numpy rounds int -> float64 -> float32 (double rounding) for weak ints
    assert domain_const(f32, n, "<") == (N.DOM_F32, float(np.float32(float(n))))
    assert domain_const(f32, np.float64(0.1), "<") == (N.DOM_F64, 0.1)  # strong f64 scalar promotes
    assert domain_const(np.dtype(np.int8), np.float32(1.5), "<")[0] == N.DOM_F32


def test_folded_and_out_of_range(t):
    cp = compile_predicate(t, ex.And((ex.Comparison(r("a"), "<", 2**80), ex.FoldedAtom(r("b"), False))))
    assert [o[0] for o in ops(cp)] == [N.OP_NOTNULL, N.OP_FALSE]


def test_text_lut_bitmap(t):
    cp = compile_predicate(t, ex.Range(r("s"), "banana", "kiwi"))
    I = cp.program.instrs[0]
    assert I.op == N.OP_LUT and I.aux2 == len(WORDS)
    bits = int(cp.lut.numpy().view(np.uint32)[0])
    want = sum(1 << i for i, w in enumerate(WORDS) if "banana" <= w <= "kiwi")
    assert bits == want
    with pytest.raises(ExecutionError, match="unsupported TEXT comparison"):
        compile_predicate(t, ex.Comparison(r("s"), "=", "fig"))


def test_udf_program(t):
    fn = lambda b, d: (b * 3.0 + d) % 7.0  # noqa: E731
    # like the reference (executor.py:121) the descale follows the ColumnRef's kind
    cp = compile_predicate(t, ex.FnCall("u", (r("a"), ex.ColumnRef("t", "v", decimal(15, 2))), ">", 3, fn))
    u = cp.program.udfs[0]
    assert cp.program.n_udfs == 1 and u.n_args == 2 and not u.dense
    assert u.arg_div[0] == 0.0 and u.arg_div[1] == 100.0   # DECIMAL(15,2) argument descaled by 10**2
    assert [cp.program.udf_ops[i].op for i in range(u.n_ops)] == [
        N.UDF_ARG, N.UDF_CONST, N.UDF_MUL, N.UDF_ARG, N.UDF_ADD, N.UDF_CONST, N.UDF_MOD]
    cp = compile_predicate(t, ex.FnCall("w", (r("a"),), ">", 0, lambda x: 1.0 / x))
    assert cp.program.udfs[0].dense and cp.may_fail


def test_limits(t):
    big = ex.Or(tuple(ex.Equality(r("a"), i) for i in range(N.MAX_INSTRS + 1)))
    with pytest.raises(ExecutionError, match="instructions"):
        compile_predicate(t, big)
    with pytest.raises(ExecutionError, match="no column"):
        compile_predicate(t, ex.Equality(r("zz"), 1))


def test_cache_hits(t):
    p = ex.Comparison(r("a"), "<", 4)
    assert compile_predicate(t, p) is compile_predicate(t, ex.Comparison(r("a"), "<", 4))


def test_program_struct_is_the_abi_layout():
    assert C.sizeof(N.EscProgram) == 16 + 8 + 32 * N.MAX_INSTRS + 80 * N.MAX_UDFS + 16 * N.MAX_UDF_OPS
