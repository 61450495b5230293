"""Device path vs the reference's frozen outputs (tests/golden/): the reference's own PredGen
corpora (criterion 1 and the eval/count suites), semantic edge cases, NEP 50 float32, the SURVEY
Appendix B known answers, and the planner's decisions / join order / temp contents on the
test_optimizer ``shop`` fixture and the config-3 star (60M-row fact).  Bit-exact."""

import numpy as np
import pytest
import torch

import golden_io as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tables(cuda):
    raw = G.raw_tables()
    return {name: G.device_table(name, cols, device=cuda) for name, cols in raw.items()}


def _pred(j, table):
    from paper_1901_01488_b200 import serde

    return serde.from_json(j, table, G.UDFS)


def _dev(fn):
    from paper_1901_01488_b200.errors import ExecutionError

    return G.outcome(fn, (ExecutionError,))


@pytest.fixture(params=["interp", "jit"])
def tier(request, cuda):
    from paper_1901_01488_b200 import _native as N

    N.set_jit(2 if request.param == "jit" else 0, 0)
    yield request.param
    N.set_jit(1, 1 << 22)


@pytest.mark.parametrize("section,tname,cat_name", [("criterion1_custom", "custom_nulls", "data"),
                                                    ("criterion1_orders", "orders", "orders"),
                                                    ("count_custom_55", "custom_nulls", "data")])
def test_reference_corpus_counts(tables, tier, section, tname, cat_name):
    """compute_exact_selectivity == the reference's, error messages included (criterion 1)."""
    from paper_1901_01488_b200 import Catalog, compute_exact_selectivity

    t = tables[tname]
    cat = Catalog()
    cat.register(t)
    entries = G.corpus()[section]
    if tier == "jit":
        entries = entries[:25]  # every new program shape is an NVRTC compile
    for entry in entries:
        got = _dev(lambda: compute_exact_selectivity(cat, tname, _pred(entry["pred"], tname), alias=cat_name)[0])
        want = entry["result"]
        if "ok" in want:
            assert got == {"ok": want["ok"]}, entry["pred"]
        else:
            assert got.get("message") == want["message"], entry["pred"]


def test_reference_corpus_rows(tables):
    from paper_1901_01488_b200 import eval_predicate

    t = tables["custom_nulls"]
    for entry in G.corpus()["eval_custom_101"]:
        want = entry["result"]
        got = _dev(lambda: eval_predicate(t, _pred(entry["pred"], "data")).to_indices().cpu().numpy())
        if "ok" in want:
            idx = got["ok"]
            assert idx.size == want["ok"]["count"] and idx[:8].tolist() == want["ok"]["head"], entry["pred"]
            assert G.digest(idx) == want["ok"]["sha256"], entry["pred"]
        else:
            assert got.get("message") == want["message"], entry["pred"]


def test_edge_cases(tables, tier):
    from paper_1901_01488_b200 import count_star, eval_predicate

    t = tables["custom_nulls"]
    for entry in G.corpus()["edge_cases"]:
        got = _dev(lambda: count_star(t, _pred(entry["pred"], "data")))
        want = entry["count"]
        if "ok" in want:
            assert got == {"ok": want["ok"]}, entry["pred"]
            rows = eval_predicate(t, _pred(entry["pred"], "data")).to_indices().cpu().numpy()
            assert G.digest(rows) == entry["rows_sha256"]["ok"], entry["pred"]
        else:
            assert got.get("message") == want["message"], entry["pred"]


def test_float32_nep50(cuda):
    from paper_1901_01488_b200 import ColumnTable, count_star
    from paper_1901_01488_b200.storage import KIND_FLOAT32, Column

    f32 = G.corpus()["float32"]
    vals = np.asarray(f32["values"], dtype=np.float32)
    t = ColumnTable("f32", [Column("f", KIND_FLOAT32, vals, device=cuda)])
    for case in f32["cases"]:
        assert count_star(t, _pred(case["pred"], "f32")) == case["count"], case["pred"]


def _device_workload(w, cuda, name):
    from paper_1901_01488_b200.storage import Column, ColumnTable, Dictionary, parse_kind

    return ColumnTable(name, [Column(c, parse_kind(spec[0]), spec[1], None,
                                     Dictionary(spec[2]) if len(spec) > 2 else None, device=cuda)
                              for c, spec in w.columns.items()])


@pytest.mark.parametrize("name", ["config1", "config2", "config4_6M"])
def test_appendix_b_known_answers(cuda, tier, name):
    from paper_1901_01488_b200 import Catalog, eval_predicate, serde
    from paper_1901_01488_b200 import datagen
    from paper_1901_01488_b200.optimizer import EscConfig, esc_subquery

    want = G.known()["configs"][name]
    w = {"config1": datagen.config1, "config2": datagen.config2,
         "config4_6M": lambda: datagen.config4(6_000_000)}[name]()
    t = _device_workload(w, cuda, name)
    pred = serde.from_json(w.pred, name, w.udfs)
    rows = eval_predicate(t, pred).to_indices().cpu().numpy()
    assert rows.size == want["count"] and rows[:5].tolist() == want["head"]
    assert G.digest(rows) == want["rows_sha256"]
    cat = Catalog()
    cat.register(t)
    d = esc_subquery(cat, name, pred, w.project, EscConfig(max_selectivity=1.0))
    assert d.exact_count == want["count"] and d.pushed_down
    temp = cat.resolve_temp(d.temp)
    for c in temp.columns:
        v = c.values.cpu().numpy()
        got = float(v.astype(np.float64).sum()) if v.dtype.kind == "f" else int(v.astype(np.int64).sum())
        assert got == want["sums"][c.name], c.name


def test_config5_counts(cuda):
    from paper_1901_01488_b200 import count_star, datagen, serde

    want = G.known()["configs"]
    t = _device_workload(datagen.config5(6_000_000, 0.01), cuda, "c5")
    for s in datagen.CONFIG5_SELECTIVITIES:
        for conj in (False, True):
            w = datagen.config5(8, s, conj)
            assert count_star(t, serde.from_json(w.pred, "c5")) == \
                want[f"config5_s{s}_{'conj4' if conj else 'single'}"]["count"]


def _shop(cuda):
    from paper_1901_01488_b200 import Catalog
    from paper_1901_01488_b200.storage import KIND_INT64, Column, ColumnTable

    def t(name, n, **cols):
        i = np.arange(1, n + 1, dtype=np.int64)
        return ColumnTable(name, [Column(c, KIND_INT64, fn(i).astype(np.int64), device=cuda) for c, fn in cols.items()])

    cat = Catalog()
    cat.register(t("fact", 5000, f_id=lambda i: i, f_cid=lambda i: (i * 7) % 2000 + 1,
                   f_pid=lambda i: (i * 13) % 1200 + 1, f_tid=lambda i: (i * 3) % 80 + 1, f_qty=lambda i: i % 100))
    cat.register(t("cust", 2000, c_id=lambda i: i, c_band=lambda i: i % 10))
    cat.register(t("prod", 1200, p_id=lambda i: i, p_cls=lambda i: i % 3))
    cat.register(t("tiny", 80, t_id=lambda i: i, t_x=lambda i: i))
    return cat


def _shop_query(cat):
    from paper_1901_01488_b200 import expr as ex, ra

    r = ex.ColumnRef
    where = ex.And((ex.ColumnCompare(r("fact", "f_cid"), "=", r("cust", "c_id")),
                    ex.ColumnCompare(r("fact", "f_pid"), "=", r("prod", "p_id")),
                    ex.ColumnCompare(r("fact", "f_tid"), "=", r("tiny", "t_id")),
                    ex.Equality(r("cust", "c_band"), 3), ex.Equality(r("prod", "p_cls"), 0),
                    ex.Comparison(r("tiny", "t_x"), "<", 40), ex.Comparison(r("fact", "f_qty"), "<", 50)))
    return ra.query(cat, ["fact", "cust", "prod", "tiny"], where)


def test_shop_plans_match_reference(cuda):
    """Decisions, verdicts, temp sizes, join order and build_card_sum of test_optimizer's shop
    fixture under six EscConfigs, against the reference planner."""
    from paper_1901_01488_b200.optimizer import EscConfig, plan

    cat = _shop(cuda)
    q = _shop_query(cat)
    configs = {"default": EscConfig(), "min1": EscConfig(min_table_size=1),
               "min5000": EscConfig(min_table_size=5000), "nomat": EscConfig(materialize=False),
               "sel0.05": EscConfig(max_selectivity=0.05), "off": EscConfig(enabled=False),
               "histogram": EscConfig(enabled=False, estimator_mode="histogram")}
    for label, want in G.known()["shop"].items():
        p = plan(q, cat, configs[label])
        assert [[d.table, d.exact_count, d.row_count, d.qualified, d.pushed_down] for d in p.decisions] == \
            want["decisions"], label
        assert p.build_order == want["order"] and p.build_card_sum == want["build_card_sum"], label
        assert [d.temp.row_count if d.temp else None for d in p.decisions] == want["temp_rows"], label
        if label == "default":  # temp contents: c_id % 10 == 3, ascending (test_optimizer.py:171-181)
            temp = cat.resolve_temp(p.decisions[0].temp)
            ids = temp.column("c_id").values.cpu().numpy()
            assert ids.tolist() == [i for i in range(1, 2001) if i % 10 == 3]
        cat.temps.sweep()


def test_star_plan_matches_reference(cuda):
    """Config 3: exact dimension counts (incl. the 0.1995-vs-0.2 boundary), push-down verdicts,
    temp contents (the pushed dimension's join key, in row order) and the join order."""
    from paper_1901_01488_b200 import Catalog, datagen, expr as ex, ra, serde
    from paper_1901_01488_b200.optimizer import EscConfig, plan
    from paper_1901_01488_b200.storage import Column, ColumnTable, Dictionary, parse_kind

    g = datagen.config3(fact_rows=1)
    cat = Catalog()
    names = {"date": "dates"}
    for tname, cols in g.items():
        if tname == "fact":
            continue
        cat.register(ColumnTable(names.get(tname, tname), [
            Column(c, parse_kind(s[0]), s[1], None, Dictionary(s[2]) if len(s) > 2 else None, device=cuda)
            for c, s in cols.items()]))
    fact = torch.ones(60_000_000, dtype=torch.int32, device=cuda)  # never scanned by ESC: only its size matters
    cat.register(ColumnTable("fact", [Column(c, parse_kind("INT32"), fact) for c in
                                      ("f_datekey", "f_custkey", "f_suppkey", "f_partkey")]))
    r = ex.ColumnRef
    conj = [ex.ColumnCompare(r("fact", a), "=", r(names.get(d, d), b)) for _, a, d, b in datagen.CONFIG3_EDGES]
    conj += [serde.from_json(j, names.get(d, d)) for d, j in datagen.CONFIG3_WHERE.items()]
    q = ra.query(cat, ["fact", "dates", "customer", "supplier", "part"], ex.And(tuple(conj)))
    want = G.known()["star"]
    p = plan(q, cat, EscConfig())
    got = {d[0]: d for d in ([dd.table, dd.exact_count, dd.row_count, dd.qualified, dd.pushed_down]
                             for dd in p.decisions)}
    assert got == {d[0]: d for d in want["decisions"]}
    assert p.build_order == want["order"] and p.build_card_sum == want["build_card_sum"]
    for d in p.decisions:
        if d.temp is not None:
            col = cat.resolve_temp(d.temp).columns[0].values.cpu().numpy()
            assert col.size == want["temps"][d.table]["rows"]
            assert G.digest(col) == want["temps"][d.table]["sha256"], d.table
    cat.temps.sweep()
