"""Device path vs the oracle on seeded inputs: counts, row sets (order), compacted columns,
chained selections, UDF error semantics, tile-boundary sizes.  Bit-exact throughout."""

import random

import numpy as np
import pytest
import torch

from helpers import UDFS, Corpus, device_table, mixed_arrays, oracle_table
from oracle import esc_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mixed(cuda):
    arrays = mixed_arrays(50_003, seed=7)
    return arrays, device_table("data", arrays, device=cuda), oracle_table("data", arrays)


def _pred(j):
    from paper_1901_01488_b200 import serde

    return serde.from_json(j, "data", UDFS)


def _oracle(fn, *args):
    try:
        return ("ok", fn(*args))
    except O.OracleExecutionError as exc:
        return ("err", str(exc))


def _device(fn, *args):
    from paper_1901_01488_b200.errors import ExecutionError

    try:
        return ("ok", fn(*args))
    except ExecutionError as exc:
        return ("err", str(exc))


def test_random_counts(mixed):
    from paper_1901_01488_b200 import count_star

    arrays, t, ot = mixed
    corpus = Corpus(arrays, random.Random(2024))
    for _ in range(300):
        j = corpus.pred()
        want = _oracle(O.count_star, ot, j, UDFS)
        got = _device(count_star, t, _pred(j))
        assert got == want, j


def test_random_selections_in_order(mixed):
    from paper_1901_01488_b200 import eval_predicate

    arrays, t, ot = mixed
    corpus = Corpus(arrays, random.Random(101))
    for _ in range(120):
        j = corpus.pred()
        want = O.eval_predicate(ot, j, None, UDFS)
        got = eval_predicate(t, _pred(j)).to_indices().cpu().numpy()
        assert np.array_equal(got, want), j


def test_chained_selection(mixed):
    from paper_1901_01488_b200 import eval_predicate

    arrays, t, ot = mixed
    corpus = Corpus(arrays, random.Random(77), udfs=("mixy", "lin"))
    for _ in range(40):
        ja, jb = corpus.pred(), corpus.pred()
        first = eval_predicate(t, _pred(ja))
        got = eval_predicate(t, _pred(jb), first).to_indices().cpu().numpy()
        rows = O.eval_predicate(ot, ja, None, UDFS)
        want = O.eval_predicate(ot, jb, rows, UDFS)
        assert np.array_equal(got, want), (ja, jb)


def test_materialize_columns(mixed):
    from paper_1901_01488_b200 import materialize

    arrays, t, ot = mixed
    corpus = Corpus(arrays, random.Random(5), udfs=("mixy", "lin"))
    names = ["id", "a", "tag", "f", "val", "g8"]
    for i in range(40):
        j = corpus.pred()
        want = O.materialize(ot, j, names, UDFS)
        cols = materialize(t, _pred(j), names, stage_proj=bool(i % 2))
        for c in cols:
            v, m = c.to_numpy()
            assert np.array_equal(v, want[c.name].values), (j, c.name)
            assert np.array_equal(m, want[c.name].nulls), (j, c.name)
            assert c.dictionary is t.column(c.name).dictionary


def test_not_readmits_nulls(mixed):
    from paper_1901_01488_b200 import count_star

    arrays, t, ot = mixed
    j = ["not", ["cmp", ["a", None], "<", 10**9]]
    assert count_star(t, _pred(j)) == int(arrays["a"][2].sum()) == O.count_star(ot, j)


@pytest.mark.parametrize("n", [0, 1, 3, 127, 128, 129, 2047, 2048, 4096, 8191, 8192, 8193, 65536 + 77])
def test_tile_boundaries(cuda, n):
    from paper_1901_01488_b200 import count_star, eval_predicate, materialize

    arrays = mixed_arrays(n, seed=n + 1)
    t, ot = device_table("data", arrays, device=cuda), oracle_table("data", arrays)
    corpus = Corpus(arrays, random.Random(n), udfs=("mixy",)) if n else None
    preds = [["cmp", ["a", None], "<", 500], ["or", [["eq", ["tag", None], 3], ["range", ["b", None], 0, 100]]]]
    if corpus:
        preds += [corpus.pred() for _ in range(10)]
    for j in preds:
        assert count_star(t, _pred(j)) == O.count_star(ot, j, UDFS), j
        got = eval_predicate(t, _pred(j)).to_indices().cpu().numpy()
        assert np.array_equal(got, O.eval_predicate(ot, j, None, UDFS)), j
        (c,) = materialize(t, _pred(j), ["id"])
        assert np.array_equal(c.to_numpy()[0], O.materialize(ot, j, ["id"], UDFS)["id"].values)


def test_udf_errors_match_reference_semantics(mixed):
    """A failing UDF raises only when the whole-slice short circuit reaches it, and reports the
    first failing row with CPython's message (executor.py:128-146, 183-196)."""
    from paper_1901_01488_b200 import count_star

    arrays, t, ot = mixed
    cases = [
        ["fn", "inv", [["b", None]], ">", 0.0],                       # b has zeros (and NULL rows)
        ["and", [["cmp", ["a", None], "<", 0], ["fn", "inv", [["b", None]], ">", 0.0]]],   # prefix empty
        ["and", [["cmp", ["a", None], "<", 5], ["fn", "inv", [["b", None]], ">", 0.0]]],   # reached
        ["or", [["folded", ["id", None], True], ["fn", "inv", [["b", None]], ">", 0.0]]],  # prefix all
        ["or", [["cmp", ["a", None], ">=", 0], ["fn", "inv", [["b", None]], ">", 0.0]]],  # a has NULLs
        ["not", ["fn", "rmod", [["a", None], ["b", None]], ">", 1.0]],
        ["fn", "fdiv", [["a", None], ["a", None]], "<", 2.0],                                  # cannot fail
        ["fn", "sq", [["val", 2]], ">", 0.0],
    ]
    for j in cases:
        assert _device(count_star, t, _pred(j)) == _oracle(O.count_star, ot, j, UDFS), j


def test_unbound_function(mixed):
    from paper_1901_01488_b200 import count_star, expr as ex
    from paper_1901_01488_b200.errors import ExecutionError

    arrays, t, ot = mixed
    fc = ex.FnCall("ghost", (ex.ColumnRef("data", "a"),), ">", 1.0, None)
    with pytest.raises(ExecutionError, match="no bound implementation"):
        count_star(t, fc)
    short = ex.And((ex.Comparison(ex.ColumnRef("data", "a"), "<", -1), fc))
    assert count_star(t, short) == 0


def test_take(mixed):
    arrays, t, ot = mixed
    idx = np.array([5, 0, 49_999, 17, 17, 123], dtype=np.int64)
    for name in ("a", "tag", "f", "big"):
        c = t.column(name).take(torch.from_numpy(idx))
        v, m = c.to_numpy()
        assert np.array_equal(v, arrays[name][1][idx])
        want_m = arrays[name][2][idx] if arrays[name][2] is not None else np.zeros(len(idx), bool)
        assert np.array_equal(m, want_m)


def test_large_multi_tile_lookback(cuda):
    """~2.4M rows: hundreds of tiles through the decoupled look-back; row ids must be exactly
    the ascending hit positions."""
    from paper_1901_01488_b200 import ColumnTable, count_star, eval_predicate, expr as ex, materialize
    from paper_1901_01488_b200.storage import KIND_INT32, KIND_INT64, Column

    n = 2_400_017
    g = np.random.default_rng(3)
    x = g.integers(0, 1000, n).astype(np.int32)
    y = g.integers(0, 1 << 40, n).astype(np.int64)
    t = ColumnTable("t", [Column("x", KIND_INT32, x, device=cuda), Column("y", KIND_INT64, y, device=cuda)])
    for lo, hi in [(0, 0), (0, 9), (100, 599), (0, 999), (5, 4)]:
        p = ex.Range(ex.ColumnRef("t", "x"), lo, hi)
        want = np.flatnonzero((x >= lo) & (x <= hi))
        assert count_star(t, p) == want.size
        got = eval_predicate(t, p).to_indices().cpu().numpy()
        assert np.array_equal(got, want)
        cx, cy = materialize(t, p, ["x", "y"])
        assert np.array_equal(cy.values.cpu().numpy(), y[want])
        assert np.array_equal(cx.values.cpu().numpy(), x[want])


# ---- JIT tier: generated straight-line evaluators must agree with the oracle too ------------
@pytest.fixture()
def jit_always(cuda):
    from paper_1901_01488_b200 import _native as N

    N.set_jit(2, 0)
    yield N
    N.set_jit(1, 1 << 22)


def test_jit_random_counts_and_rows(mixed, jit_always):
    from paper_1901_01488_b200 import count_star, eval_predicate, materialize

    arrays, t, ot = mixed
    corpus = Corpus(arrays, random.Random(909))
    for i in range(60):
        j = corpus.pred()
        want = _oracle(O.count_star, ot, j, UDFS)
        assert _device(count_star, t, _pred(j)) == want, j
        if want[0] == "ok" and i % 3 == 0:
            got = eval_predicate(t, _pred(j)).to_indices().cpu().numpy()
            assert np.array_equal(got, O.eval_predicate(ot, j, None, UDFS)), j
            cols = materialize(t, _pred(j), ["id", "tag", "f"])
            want_m = O.materialize(ot, j, ["id", "tag", "f"], UDFS)
            for c in cols:
                v, m = c.to_numpy()
                assert np.array_equal(v, want_m[c.name].values) and np.array_equal(m, want_m[c.name].nulls)
    st = jit_always.jit_stats()
    assert st["nvrtc"] and st["compiled"] > 0 and st["failures"] == 0, st


def test_jit_udf_integer_lowering_and_errors(mixed, jit_always):
    """Exact int64 lowering of integral UDFs must reproduce CPython float results, including
    floored % / // on negative operands; failing UDFs keep the reference error semantics."""
    from paper_1901_01488_b200 import count_star

    arrays, t, ot = mixed
    cases = [["fn", "mixy", [["b", None], ["g8", None]], ">", 6.0],
             ["fn", "fdiv", [["b", None], ["u8", None]], "<", -40.0],
             ["fn", "sq", [["g8", None]], ">=", 100.0],
             ["fn", "nabs", [["b", None]], "<", -100.0],
             ["fn", "inv", [["b", None]], ">", 0.0],
             ["and", [["cmp", ["a", None], "<", 0], ["fn", "inv", [["b", None]], ">", 0.0]]],
             ["fn", "rmod", [["a", None], ["b", None]], ">", 1.0]]
    for j in cases:
        assert _device(count_star, t, _pred(j)) == _oracle(O.count_star, ot, j, UDFS), j


def test_onepass_lookback_kernel_matches(mixed):
    """The single-pass decoupled look-back kernel (esc_compact_onepass) is bit-identical."""
    from paper_1901_01488_b200 import executor

    arrays, t, ot = mixed
    corpus = Corpus(arrays, random.Random(31), udfs=("mixy", "lin"))
    names = ["id", "a", "tag", "f", "val"]
    for _ in range(25):
        j = corpus.pred()
        want = O.materialize(ot, j, names, UDFS)
        count, cols = executor.materialize_onepass(t, _pred(j), names)
        assert count == len(want["id"].values), j
        for c in cols:
            v, m = c.to_numpy()
            assert np.array_equal(v, want[c.name].values) and np.array_equal(m, want[c.name].nulls), (j, c.name)


def test_selection_reuse(mixed):
    """select() records the selection once; materialising from it equals re-evaluating."""
    from paper_1901_01488_b200 import executor

    arrays, t, ot = mixed
    j = ["or", [["cmp", ["a", None], "<", 100], ["eq", ["tag", None], 2]]]
    sel = executor.select(t, _pred(j))
    assert sel.count == O.count_star(ot, j)
    (a1,) = executor.materialize_selection(sel, ["a"])
    (a2,) = executor.materialize_selection(sel, ["a"], capacity=7)
    want = O.materialize(ot, j, ["a"])["a"].values
    assert np.array_equal(a1.to_numpy()[0], want)
    assert np.array_equal(a2.to_numpy()[0], want[:7])


# ---- scan-time capture and streamed compaction of dense tiles ---------------------------------
@pytest.fixture(params=["off", "default", "always", "mid", "hitlist"])
def stream_mode(request, cuda):
    """The compaction route: the scan + gathered chain with streaming of dense tiles off /
    default / always, the gathered chain with warp hit lists forced on, or the one-launch
    mid-size kernel."""
    from paper_1901_01488_b200 import _native as N

    div = {"off": 0, "default": 32, "always": 1 << 30, "mid": 32, "hitlist": 32}[request.param]
    prev = N.set_stream_div(div)
    prev_mid = N.set_mid_max_rows(1 << 40 if request.param == "mid" else 0)
    prev_hl = N.set_hit_lists(2 if request.param == "hitlist" else 1)
    yield request.param
    N.set_stream_div(prev)
    N.set_mid_max_rows(prev_mid)
    N.set_hit_lists(prev_hl)


@pytest.mark.parametrize("capture", [False, True])
@pytest.mark.parametrize("jit", [0, 2])
def test_capture_and_stream_paths(mixed, stream_mode, capture, jit):
    """Every compaction route — captured sparse segments, lane gathers, warp gathers, TMA-streamed
    dense tiles — yields the oracle's columns, null masks and row ids, in order."""
    from paper_1901_01488_b200 import _native as N, eval_predicate, executor, materialize

    arrays, t, ot = mixed
    prev_cap = executor.set_capture(capture)
    N.set_jit(jit, 0)
    try:
        corpus = Corpus(arrays, random.Random(4242 + jit), udfs=("mixy", "lin"))
        names = ["id", "a", "tag", "f", "val", "big"]
        for i in range(12):
            j = corpus.pred()
            want = _oracle(O.materialize, ot, j, names, UDFS)
            if want[0] != "ok":
                continue
            cols = materialize(t, _pred(j), names)
            for c in cols:
                v, m = c.to_numpy()
                assert np.array_equal(v, want[1][c.name].values), (j, c.name)
                assert np.array_equal(m, want[1][c.name].nulls), (j, c.name)
            if i % 4 == 0:
                got = eval_predicate(t, _pred(j)).to_indices().cpu().numpy()
                assert np.array_equal(got, O.eval_predicate(ot, j, None, UDFS)), j
    finally:
        executor.set_capture(prev_cap)
        N.set_jit(1, 1 << 22)


def test_stream_selectivity_sweep(cuda, stream_mode):
    """2.4M rows over every selectivity regime (sparse -> fully dense) and mixed widths: the
    streamed dense tiles and the gathered sparse ones stitch together in row order."""
    from paper_1901_01488_b200 import ColumnTable, count_star, eval_predicate, expr as ex, materialize
    from paper_1901_01488_b200.storage import KIND_INT32, KIND_INT64, Column, parse_kind

    n = 2_400_017
    g = np.random.default_rng(11)
    x = g.integers(0, 1_000_000, n).astype(np.int32)
    y = g.integers(0, 1 << 40, n).astype(np.int64)
    z = g.integers(-100, 100, n).astype(np.int8)
    h = g.integers(-30000, 30000, n).astype(np.int16)
    hn = g.random(n) < 0.1
    t = ColumnTable("t", [Column("x", KIND_INT32, x, device=cuda), Column("y", KIND_INT64, y, device=cuda),
                          Column("z", parse_kind("INT8"), z, device=cuda),
                          Column("h", parse_kind("INT16"), np.where(hn, 0, h).astype(np.int16), hn, device=cuda)])
    for hi in (99, 9_999, 29_999, 99_999, 499_999, 899_999, 999_999):
        p = ex.Range(ex.ColumnRef("t", "x"), 0, hi)
        want = np.flatnonzero(x <= hi)
        assert count_star(t, p) == want.size
        cx, cy, cz, ch = materialize(t, p, ["x", "y", "z", "h"])
        assert np.array_equal(cx.values.cpu().numpy(), x[want])
        assert np.array_equal(cy.values.cpu().numpy(), y[want])
        assert np.array_equal(cz.values.cpu().numpy(), z[want])
        hv, hm = ch.to_numpy()
        assert np.array_equal(hm, hn[want])
        assert np.array_equal(hv, np.where(hn, 0, h)[want])
        got = eval_predicate(t, p).to_indices().cpu().numpy()
        assert np.array_equal(got, want)
        # only predicate columns projected: sparse segments' values all come from the capture
        # slots (the mid kernel then reads no bitmap for them)
        p2 = ex.And((p, ex.Range(ex.ColumnRef("t", "z"), -90, 99)))
        want2 = np.flatnonzero((x <= hi) & (z >= -90))
        cz2, cx2 = materialize(t, p2, ["z", "x"])
        assert np.array_equal(cx2.values.cpu().numpy(), x[want2])
        assert np.array_equal(cz2.values.cpu().numpy(), z[want2])


def test_lean_bitmap_step_mixed_density(cuda, stream_mode):
    """A queued step whose projections are all predicate columns (the plan's K1 writes no bitmap
    words for captured or empty segments): clustered hits give tiles that mix dense, captured and
    empty segments, and every route (streamed dense tiles, captured copies, sparse gathers) must
    still yield the rows in order — with streaming always on, the lean rule keeps tiles holding a
    captured or empty segment off the streamed path."""
    from paper_1901_01488_b200 import ColumnTable, executor, expr as ex
    from paper_1901_01488_b200.storage import KIND_INT32, KIND_INT64, Column

    n = 3_000_029
    g = np.random.default_rng(31)
    x = g.integers(0, 1_000_000, n).astype(np.int32)
    # clusters: runs of rows that all pass, runs that pass sparsely, and runs with no hit at all
    block = np.arange(n) // 3000
    kind = block % 5
    x = np.where(kind == 0, g.integers(0, 1000, n), x).astype(np.int32)          # dense runs
    x = np.where(kind == 1, np.where(g.random(n) < 0.004, 5, 999_999), x).astype(np.int32)  # sparse
    x = np.where(kind == 2, 999_999, x).astype(np.int32)                           # empty
    y = g.integers(-(1 << 40), 1 << 40, n).astype(np.int64)
    t = ColumnTable("t", [Column("x", KIND_INT32, x, device=cuda), Column("y", KIND_INT64, y, device=cuda)])
    for hi in (999, 49_999, 199_999):
        p = ex.And((ex.Range(ex.ColumnRef("t", "x"), 0, hi), ex.Comparison(ex.ColumnRef("t", "y"), ">", -(1 << 40) + 5)))
        want = np.flatnonzero((x <= hi) & (y > -(1 << 40) + 5))
        count, cols = executor.count_and_materialize(t, p, ["y", "x"], n)
        assert count == want.size
        cy, cx = cols
        assert np.array_equal(cx.values.cpu().numpy(), x[want]), hi
        assert np.array_equal(cy.values.cpu().numpy(), y[want]), hi


def test_queued_compaction_checks_count_on_device(cuda):
    """count_and_materialize queues the compaction behind the scan with a device-side capacity
    check: a qualifying table is materialised exactly, an overflowing one yields no temp and its
    (skipped) compaction leaves nothing behind; both match the oracle's counts."""
    from paper_1901_01488_b200 import ColumnTable, executor, expr as ex
    from paper_1901_01488_b200.storage import KIND_INT32, KIND_INT64, Column

    n = 3_000_001
    g = np.random.default_rng(17)
    x = g.integers(0, 100_000, n).astype(np.int32)
    y = g.integers(-(1 << 40), 1 << 40, n).astype(np.int64)
    t = ColumnTable("t", [Column("x", KIND_INT32, x, device=cuda), Column("y", KIND_INT64, y, device=cuda)])
    for hi in (9, 999, 19_999, 60_000):
        p = ex.Range(ex.ColumnRef("t", "x"), 0, hi)
        want = np.flatnonzero(x <= hi)
        for cap in (want.size - 1, want.size, n // 5):
            count, cols = executor.count_and_materialize(t, p, ["y", "x"], cap)
            assert count == want.size
            if want.size > cap:
                assert cols is None
                continue
            cy, cx = cols
            assert np.array_equal(cy.values.cpu().numpy(), y[want])
            assert np.array_equal(cx.values.cpu().numpy(), x[want])


def test_onepass_plan_rebinds_new_outputs(cuda):
    """A small table's ESC step reuses its prepared one-pass launch (esc_step_plan_rebind): every
    run writes fresh output buffers, so the columns an earlier run handed over stay intact."""
    from paper_1901_01488_b200 import ColumnTable, executor, expr as ex
    from paper_1901_01488_b200.compiler import compile_predicate
    from paper_1901_01488_b200.storage import KIND_INT32, KIND_INT64, Column

    n = 40_000
    g = np.random.default_rng(23)
    k = np.arange(n, dtype=np.int64) * 3
    r = g.integers(0, 25, n).astype(np.int32)
    t = ColumnTable("t", [Column("k", KIND_INT64, k, device=cuda), Column("r", KIND_INT32, r, device=cuda)])
    p = ex.Range(ex.ColumnRef("t", "r"), 3, 4)
    want = np.flatnonzero((r >= 3) & (r <= 4))
    first = executor.count_and_materialize(t, p, ["k", "r"], n)
    keep = [c.values.cpu().numpy().copy() for c in first[1]]
    for _ in range(3):
        count, cols = executor.count_and_materialize(t, p, ["k", "r"], n)
        assert count == want.size
        assert np.array_equal(cols[0].values.cpu().numpy(), k[want])
        assert np.array_equal(cols[1].values.cpu().numpy(), r[want])
    assert np.array_equal(first[1][0].values.cpu().numpy(), keep[0])  # not overwritten by later runs
    assert np.array_equal(first[1][1].values.cpu().numpy(), keep[1])
    assert len(compile_predicate(t, p).c_plans) == 1  # one prepared launch, rebound each time


def test_queued_step_lends_outputs_until_released(cuda):
    """A queued step's temp columns are views of its plan's output buffers: while an earlier
    step's columns (or a view derived from them) are alive, later steps write to another plan's
    buffers; once they are dropped, the plan is reused (no new buffers)."""
    from paper_1901_01488_b200 import ColumnTable, executor, expr as ex
    from paper_1901_01488_b200.storage import KIND_INT32, KIND_INT64, Column

    n = 3_000_017
    g = np.random.default_rng(29)
    x = g.integers(0, 100_000, n).astype(np.int32)
    y = g.integers(-(1 << 40), 1 << 40, n).astype(np.int64)
    t = ColumnTable("t", [Column("x", KIND_INT32, x, device=cuda), Column("y", KIND_INT64, y, device=cuda)])
    p = ex.Range(ex.ColumnRef("t", "x"), 0, 999)
    want = np.flatnonzero(x <= 999)
    cap = n // 5
    _, first = executor.count_and_materialize(t, p, ["y", "x"], cap)
    derived = first[0].values[:10]  # a view of a view keeps the buffer lent too
    ptr0 = first[0].values.data_ptr()
    del first
    for _ in range(4):  # the same predicate again (same plan key): must not reuse the lent buffer
        count, cols = executor.count_and_materialize(t, p, ["y", "x"], cap)
        assert count == want.size and cols[0].values.data_ptr() != ptr0
        assert np.array_equal(cols[0].values.cpu().numpy(), y[want])
        del cols
    assert np.array_equal(derived.cpu().numpy(), y[want[:10]])
    del derived
    ptrs = set()
    for _ in range(3):  # everything released: steady state reuses the same buffers
        count, cols = executor.count_and_materialize(t, p, ["y", "x"], cap)
        ptrs.add(cols[0].values.data_ptr())
        assert np.array_equal(cols[1].values.cpu().numpy(), x[want])
        del cols
    assert len(ptrs) == 1


@pytest.mark.parametrize("n", [600 * 8192 + 77, 2 * 148 * 4096 * 2 + 4096 * 3 + 5])
def test_ticketed_scan_tails(cuda, n):
    """K1 hands out multi-tile tickets on large scans; counts and selections stay exact when the
    tile count is not a multiple of the ticket size (and the last tile is partial)."""
    from paper_1901_01488_b200 import ColumnTable, count_star, executor, expr as ex
    from paper_1901_01488_b200.storage import KIND_INT32, Column

    g = np.random.default_rng(n % 1000)
    cols = {c: g.integers(0, 1000, n).astype(np.int32) for c in ("a", "b", "c", "d")}
    t = ColumnTable("t", [Column(c, KIND_INT32, v, device=cuda) for c, v in cols.items()])
    r = lambda c: ex.ColumnRef("t", c)  # noqa: E731
    p1 = ex.Range(r("a"), 0, 9)
    assert count_star(t, p1) == int(np.count_nonzero(cols["a"] <= 9))
    p4 = ex.And((ex.Range(r("a"), 0, 499), ex.Range(r("b"), 100, 999), ex.Comparison(r("c"), "<", 300),
                 ex.Comparison(r("d"), ">=", 10)))
    m = (cols["a"] <= 499) & (cols["b"] >= 100) & (cols["c"] < 300) & (cols["d"] >= 10)
    want = np.flatnonzero(m)
    count, out = executor.count_and_materialize(t, p4, ["d", "a"], n)
    assert count == want.size
    assert np.array_equal(out[0].values.cpu().numpy(), cols["d"][want])
    assert np.array_equal(out[1].values.cpu().numpy(), cols["a"][want])


@pytest.mark.parametrize("packed", [True, False])
@pytest.mark.parametrize("jit", [0, 2])
def test_packed_and_byte_null_staging(mixed, packed, jit):
    """Count / selection scans stage nullable columns' NULLs as a packed 1-bit bitmap (default)
    or as the byte mask: both equal the oracle (NULL floor, two-valued NOT, UDF NULL rows)."""
    from paper_1901_01488_b200 import _native as N, compiler, count_star, eval_predicate

    arrays, t, ot = mixed
    prev = compiler.set_packed_nulls(packed)
    N.set_jit(jit, 0)
    try:
        corpus = Corpus(arrays, random.Random(99 + jit + 2 * packed))
        for _ in range(25):
            j = corpus.pred()
            want = _oracle(O.count_star, ot, j, UDFS)
            assert _device(count_star, t, _pred(j)) == want, j
            if want[0] == "ok":
                got = eval_predicate(t, _pred(j)).to_indices().cpu().numpy()
                assert np.array_equal(got, O.eval_predicate(ot, j, None, UDFS)), j
    finally:
        compiler.set_packed_nulls(prev)
        N.set_jit(1, 1 << 22)


def test_packed_null_bitmap_layout(cuda):
    """esc_pack_nulls: bit r % 32 of word r / 32, zero padding past the last row."""
    from paper_1901_01488_b200.storage import KIND_INT32, Column

    for n in (1, 31, 32, 33, 1000, 65_537):
        m = np.random.default_rng(n).random(n) < 0.3
        m[0] = True
        c = Column("x", KIND_INT32, np.zeros(n, np.int32), m, device=cuda)
        words = c.null_bits.cpu().numpy().view(np.uint32)
        bits = np.unpackbits(words.view(np.uint8), bitorder="little")
        assert np.array_equal(bits[:n].astype(bool), m) and not bits[n:].any()


def test_sparse_selection_hit_lists_at_scale(cuda):
    """A sparse selection over a table large enough that the gathered compaction picks warp hit
    lists on its own (80M rows, 3 predicate columns: 512-row segments with scan-time captures, so
    list entries of captured segments skip the captured column): rows in order, equal to numpy;
    and the same selection with the lists off."""
    from paper_1901_01488_b200 import _native as N, ColumnTable, executor, expr as ex
    from paper_1901_01488_b200.storage import KIND_INT32, KIND_INT64, Column

    n = 80_000_003
    g = np.random.default_rng(77)
    x = g.integers(0, 1_000_000, n, dtype=np.int32)
    a = g.integers(0, 1000, n, dtype=np.int32)
    b = g.integers(0, 1000, n, dtype=np.int32)
    y = g.integers(-(1 << 50), 1 << 50, n, dtype=np.int64)
    t = ColumnTable("t", [Column("x", KIND_INT32, x, device=cuda), Column("a", KIND_INT32, a, device=cuda),
                          Column("b", KIND_INT32, b, device=cuda), Column("y", KIND_INT64, y, device=cuda)])
    for hi, amin in ((999, 0), (99, 500), (1999, 990)):
        p = ex.And((ex.Range(ex.ColumnRef("t", "x"), 0, hi), ex.Comparison(ex.ColumnRef("t", "a"), ">=", amin),
                    ex.Comparison(ex.ColumnRef("t", "b"), ">=", 0)))
        want = np.flatnonzero((x <= hi) & (a >= amin))
        assert want.size * 500 <= n  # the automatic route takes the hit lists
        for mode in (1, 0):
            prev = N.set_hit_lists(mode)
            try:
                cy, cx = executor.materialize(t, p, ["y", "x"])
            finally:
                N.set_hit_lists(prev)
            assert np.array_equal(cx.values.cpu().numpy(), x[want]), (hi, mode)
            assert np.array_equal(cy.values.cpu().numpy(), y[want]), (hi, mode)
