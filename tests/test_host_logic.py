"""Host-side logic that needs no GPU: push-down policy, probe choice, greedy order, needed columns,
the COUNT sub-query tree, EXPLAIN formats, the temp store, storage and serde."""

import json
import re
from fractions import Fraction

import numpy as np
import pytest

from paper_1901_01488_b200 import expr as ex
from paper_1901_01488_b200 import ra, serde
from paper_1901_01488_b200.catalog import Catalog
from paper_1901_01488_b200.errors import (CartesianProductRequired, DeadHandle, DuplicateFunction, DuplicateTable,
                                          LengthMismatch, NoPredicate, PlanError, UnknownTable,
                                          UnsupportedPredicate)
from paper_1901_01488_b200.optimizer import (EscConfig, EscDecision, PhysicalPlan, PlanBuild, build_count_subquery,
                                             choose_probe, decide_pushdown, explain_json, explain_text,
                                             _needed_columns, order_builds)
from paper_1901_01488_b200.storage import (KIND_INT64, KIND_TEXT, Column, ColumnTable, Dictionary, TempTableStore,
                                           decimal, format_decimal, parse_kind)


def table(name, **cols):
    return ColumnTable(name, [Column(c, KIND_INT64, np.asarray(v, dtype=np.int64), device="cpu")
                              for c, v in cols.items()])


@pytest.fixture()
def star():
    cat = Catalog()
    cat.register(table("fact", f_a=range(10), f_b=range(10), f_x=range(10)))
    cat.register(table("a", a_id=range(5), a_v=range(5)))
    cat.register(table("b", b_id=range(7), b_w=range(7), b_extra=range(7)))
    return cat


def r(t, c):
    return ex.ColumnRef(t, c)


def test_policy_boundaries_inclusive():
    cfg = EscConfig()
    assert decide_pushdown(1000, 200, cfg) and not decide_pushdown(1000, 201, cfg)   # exactly 0.2
    assert decide_pushdown(1000, 50, cfg) and not decide_pushdown(999, 1, cfg)        # size gate
    assert not decide_pushdown(0, 0, EscConfig(min_table_size=0))
    assert decide_pushdown(1000, 0, cfg)
    # exact rational: 0.2 as a double is slightly above 1/5
    assert decide_pushdown(5, 1, EscConfig(min_table_size=1)) == (Fraction(1, 5) <= 0.2)


def test_config_validation():
    with pytest.raises(ValueError):
        EscConfig(max_selectivity=1.5)
    with pytest.raises(ValueError):
        EscConfig(min_table_size=-1)
    with pytest.raises(ValueError):
        EscConfig(estimator_mode="magic")


def test_join_graph_probe_and_order(star):
    where = ex.And((ex.ColumnCompare(r("fact", "f_a"), "=", r("a", "a_id")),
                    ex.ColumnCompare(r("fact", "f_b"), "=", r("b", "b_id")),
                    ex.Comparison(r("a", "a_v"), "<", 3), ex.Comparison(r("fact", "f_x"), ">", 1)))
    q = ra.query(star, ["fact", "a", "b"], where, select=[r("b", "b_w")])
    g = ra.build_join_graph(q)
    assert g.tables == ("fact", "a", "b") and len(g.edges) == 2
    assert str(g.residual("a")) == "a.a_v < 3" and g.residual("b") is None
    rows = {"fact": 10, "a": 5, "b": 7}
    assert choose_probe(g, rows) == "fact"
    assert order_builds(g, "fact", rows) == ["a", "b"]
    assert order_builds(g, "fact", {"fact": 10, "a": 9, "b": 7}) == ["b", "a"]
    assert order_builds(g, "fact", {"fact": 10, "a": 7, "b": 7}) == ["a", "b"]   # tie -> alias
    assert _needed_columns(g, q.columns, "b", star.table("b")) == ["b_id", "b_w"]
    assert _needed_columns(g, None, "a", star.table("a")) == ["a_id"]


def test_probe_ties_break_by_alias():
    g = ra.JoinGraph(("bb", "aa"), {"bb": "bb", "aa": "aa"}, (), {})
    assert choose_probe(g, {"aa": 10, "bb": 10}) == "aa"


def test_cartesian_and_cross_table_predicates(star):
    g = ra.JoinGraph(("fact", "a", "b"), {}, (ra.JoinEdge(r("fact", "f_a"), r("a", "a_id")),), {})
    with pytest.raises(CartesianProductRequired):
        order_builds(g, "fact", {"fact": 1, "a": 1, "b": 1})
    bad = ra.query(star, ["fact", "a"], ex.ColumnCompare(r("fact", "f_a"), "<", r("a", "a_id")))
    with pytest.raises(UnsupportedPredicate):
        ra.build_join_graph(bad)


def test_count_subquery_shape(star):
    pred = ex.Comparison(r("b", "b_w"), "<", 5)
    tree = build_count_subquery(star, "b", pred, ("b_id",))
    assert isinstance(tree, ra.RaAggregate)
    sel = tree.child
    assert isinstance(sel, ra.RaSelect) and sel.predicate is pred
    assert isinstance(sel.child, ra.RaProject) and isinstance(sel.child.child, ra.RaScan)
    assert [c.name for c in sel.child.columns] == ["b_id", "b_w"]   # base column order
    with pytest.raises(NoPredicate):
        build_count_subquery(star, "b", None)
    with pytest.raises(NoPredicate):
        build_count_subquery(star, "b", ex.FoldedAtom(r("b", "b_w"), True))


def _plan():
    g = ra.JoinGraph(("fact", "cust", "prod"), {"fact": "fact", "cust": "cust", "prod": "prod"},
                     (ra.JoinEdge(r("fact", "f_cid"), r("cust", "c_id")),
                      ra.JoinEdge(r("fact", "f_pid"), r("prod", "p_id"))), {})
    from paper_1901_01488_b200.storage import TempTableHandle

    h = TempTableHandle(1, (("c_id", KIND_INT64),), 200)
    d1 = EscDecision("cust", ex.Equality(r("cust", "c_band"), 3), 200, 2000, Fraction(1, 10), True, True, h, 1.25, 0.5)
    d2 = EscDecision("prod", ex.Equality(r("prod", "p_cls"), 0), 400, 1200, Fraction(1, 3), False, False, None, 0.75)
    builds = [PlanBuild("cust", h, r("cust", "c_id"), r("fact", "f_cid"), None, 200),
              PlanBuild("prod", "prod", r("prod", "p_id"), r("fact", "f_pid"), d2.predicate, 1200)]
    return PhysicalPlan("fact", "fact", 5000, ex.Comparison(r("fact", "f_qty"), "<", 50), builds, None, [d1, d2], g)


def test_explain_text_format():
    """Same line formats as the reference's EXPLAIN (optimizer.py:440-471)."""
    text = explain_text(_plan())
    lines = text.splitlines()
    assert lines[0] == "ESC table=cust count=200 sel=0.100000 pushdown=true time_ms=1.750"
    assert lines[1] == "ESC table=prod count=400 sel=0.333333 pushdown=false time_ms=0.750"
    assert lines[2] == "Aggregate COUNT(*)"
    assert lines[3] == "  HashJoin (prod.p_id = fact.f_pid)"
    assert lines[4] == "    HashJoin (cust.c_id = fact.f_cid)"
    assert lines[5] == "      Probe fact=fact rows=5000 filter=(fact.f_qty < 50)"
    assert lines[6] == "      Build cust=temp(rows=200) rows=200"
    assert lines[7] == "    Build prod=prod rows=1200 filter=(prod.p_cls = 0)"
    for ln in lines[:2]:
        assert re.fullmatch(r"ESC table=\w+ count=\d+ sel=\d\.\d{6} pushdown=(true|false) time_ms=\d+\.\d{3}", ln)


def test_explain_json_schema():
    j = explain_json(_plan())
    assert j["build_card_sum"] == 1400 and j["projection"] is None
    assert j["builds"][0] == {"alias": "cust", "source": "temp(rows=200)", "rows": 200, "key": "cust.c_id",
                              "probe_key": "fact.f_cid", "filter": None}
    d = j["decisions"][0]
    assert set(d) == {"table", "predicate", "count", "row_count", "selectivity", "qualified", "pushdown",
                      "temp_rows", "subquery_ms", "materialize_ms"}
    json.dumps(j)


def test_temp_store_semantics():
    store = TempTableStore()
    c = Column("x", KIND_INT64, np.arange(3, dtype=np.int64), device="cpu")
    h1 = store.materialize([c])
    h2 = store.materialize([c])
    assert str(h1) == "temp#1" and h2.id == 2 and h1.row_count == 3
    assert store.resolve(h1).is_temporary and store.resolve(h1).name == "$temp1"
    store.drop(h1)
    with pytest.raises(DeadHandle):
        store.drop(h1)
    with pytest.raises(DeadHandle):
        store.resolve(h1)
    assert store.live_handles() == [2] and store.sweep() == 1 and store.live_handles() == []


def test_catalog_registry():
    cat = Catalog()
    cat.register(table("t", x=[1]))
    with pytest.raises(DuplicateTable):
        cat.register(table("t", x=[1]))
    with pytest.raises(UnknownTable):
        cat.table("nope")
    cat.register_udf("F", 1, abs)
    assert cat.udf("f").fn is abs
    with pytest.raises(DuplicateFunction):
        cat.register_udf("f", 1, abs)


def test_storage_columns():
    c = Column("t", KIND_TEXT, np.array([0, 1, 0], np.int8), np.array([False, True, False]), Dictionary(["x", "y"]),
               device="cpu")
    assert c.has_nulls and c.decode_value(0) == "x" and c.decode_value(1) is None
    c2 = Column("n", KIND_INT64, np.arange(4), np.zeros(4, bool), device="cpu")
    assert c2.nulls is None and not bool(c2.null_mask.any())      # all-False masks are dropped
    with pytest.raises(LengthMismatch):
        ColumnTable("bad", [Column("a", KIND_INT64, [1, 2], device="cpu"), Column("b", KIND_INT64, [1], device="cpu")])
    assert parse_kind("decimal(15,2)") == decimal(15, 2) and parse_kind("float32").name == "FLOAT32"
    assert format_decimal(-1050, 2) == "-10.50"


def test_serde_round_trip():
    p = ex.And((ex.Range(ex.ColumnRef("t", "a"), 1, 2.5), ex.Not(ex.Or((ex.Equality(ex.ColumnRef("t", "b"), 3),
                                                                        ex.FoldedAtom(ex.ColumnRef("t", "c"), False)))),
                ex.Comparison(ex.ColumnRef("t", "s"), "<", "m"),
                ex.ColumnCompare(ex.ColumnRef("t", "a"), "<>", ex.ColumnRef("t", "b")),
                ex.FnCall("f", (ex.ColumnRef("t", "v", decimal(15, 2)),), ">", float("nan"), abs)))
    j = serde.to_json(p)
    q = serde.from_json(json.loads(json.dumps(j)), "t", {"f": abs})
    assert str(q) == str(p) and serde.to_json(q) == j


def test_histogram_arm_needs_the_device():
    """The histogram arm builds its synopses on the device: CPU-resident tables fail loudly
    (no CPU fallback); the baseline arm (no estimates) needs no device."""
    from paper_1901_01488_b200.errors import NativeUnavailable
    from paper_1901_01488_b200.optimizer import plan

    cat = Catalog()
    cat.register(table("f", k=range(4)))
    cat.register(table("d", k2=range(3), v=range(3)))
    q = ra.query(cat, ["f", "d"], ex.And((ex.ColumnCompare(r("f", "k"), "=", r("d", "k2")),
                                          ex.Comparison(r("d", "v"), "<", 1))))
    with pytest.raises(NativeUnavailable):
        plan(q, cat, EscConfig(enabled=False, estimator_mode="histogram"))
    p = plan(q, cat, EscConfig(enabled=False))   # baseline arm: no sub-queries, base cardinalities
    assert p.decisions == [] and p.build_order == ["d"] and p.build_card_sum == 3


def test_lent_step_plan_bookkeeping():
    """A queued step's plan lends its output buffers to the temp columns (views): it is reused only
    once nothing refers to them, and free lent plans return to the byte-bounded plan cache (CPU
    tensors stand in for the device buffers: the bookkeeping reads storage use counts only)."""
    import torch

    from paper_1901_01488_b200 import executor

    class _Ws:
        def __init__(self):
            self.scratch = {}

    class _Plan:
        def __init__(self, key, n):
            self.key = key
            self.out_values = [torch.empty(n, dtype=torch.int32)]
            self.out_nulls = [None]
            self.nbytes = 4 * n

    ws = _Ws()
    p1 = _Plan(("k", 1), 1000)
    view = p1.out_values[0][:10]  # a temp column's view
    executor._plan_lend(ws, p1)
    assert not executor._outputs_free(p1)
    executor._reclaim_lent(ws)
    assert ws.scratch["lent"] == [p1] and "plans" not in ws.scratch  # still lent
    derived = view[2:5]  # a view of the view keeps it lent too
    del view
    executor._reclaim_lent(ws)
    assert ws.scratch["lent"] == [p1]
    del derived
    assert executor._outputs_free(p1)
    p2 = _Plan(("k", 2), 10)
    executor._plan_lend(ws, p2)  # lending reclaims the free ones first
    assert ws.scratch["plans"] == {("k", 1): p1} and ws.scratch["lent"] == [p2]
    # the cache's byte budget drops the least recently used plans
    old = executor.STEP_PLAN_BYTES
    executor.STEP_PLAN_BYTES = 4000
    try:
        executor._plan_checkin(ws, _Plan(("k", 3), 500))
        assert list(ws.scratch["plans"]) == [("k", 3)]
    finally:
        executor.STEP_PLAN_BYTES = old
