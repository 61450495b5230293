"""Generate the golden fixtures by running the REFERENCE implementation (run HERE only).

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests python tests/golden/make_golden.py

The reference (``/root/reference/pkg``, escdb 0.1.0, numpy 2.3) does not exist on the GPU box, so
its outputs are frozen here:

* ``tables.npz``       — the reference's own test tables: ``custom_nulls``
                          (``GenSpec("custom", 0.02, 3, null_fraction=0.08)``, conftest.py) and the
                          ``orders`` table of ``GenSpec("tpch_subset", 0.001, 7)``.
* ``corpus.json``      — predicates from the reference's ``test_executor.PredGen`` (criterion-1
                          seeds 2024 / 7, eval seeds 101 / 55) with the reference's counts / row ids,
                          plus hand-picked semantic edge cases (NULL floor, two-valued NOT, folded
                          atoms, TEXT LUT ranges, NEP 50 promotions, UDF errors).
* ``known.json``       — reference results on the SURVEY Appendix B recipes (configs 1, 2, 4, 5 at
                          the pinned sizes) and the planner's decisions / join order on the
                          test_optimizer ``shop`` fixture and the config-3 star.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from escdb import expr as rex  # noqa: E402  (the reference)
from escdb import frontend as rfe  # noqa: E402
from escdb.bench import GenSpec, generate  # noqa: E402
from escdb.catalog import Catalog as RCatalog  # noqa: E402
from escdb.errors import EscdbError  # noqa: E402
from escdb.executor import count_star as rcount, eval_predicate as reval  # noqa: E402
from escdb.optimizer import (EscConfig as REscConfig, compute_exact_selectivity as rces,  # noqa: E402
                             materialize_pushdown as rmat, plan as rplan)
from escdb.storage import Column as RColumn, ColumnKind, ColumnTable as RTable, Dictionary as RDict  # noqa: E402
from escdb.storage import KIND_INT64, KIND_TEXT, append_rows  # noqa: E402
from test_executor import PredGen  # noqa: E402  (the reference's own random predicate generator)

from paper_1901_01488_b200 import datagen  # noqa: E402  (our recipes; fed to the reference below)

MIXY = "mixy"  # PredGen's UDF: lambda x, y: (x * 7.0 + y) % 13.0


def ref_json(e):
    """Reference expr -> the JSON form of paper_1901_01488_b200.serde / oracle."""
    def ref(c):
        k = c.kind
        return [c.name, k.scale if (k is not None and k.is_decimal) else None]

    def val(v):
        if isinstance(v, float) and not np.isfinite(v):
            return {"float": repr(v)}
        return v

    if isinstance(e, rex.Equality):
        return ["eq", ref(e.col), val(e.value)]
    if isinstance(e, rex.Comparison):
        return ["cmp", ref(e.col), e.op, val(e.value)]
    if isinstance(e, rex.Range):
        return ["range", ref(e.col), val(e.lo), val(e.hi)]
    if isinstance(e, rex.ColumnCompare):
        return ["colcmp", ref(e.left), e.op, ref(e.right)]
    if isinstance(e, rex.FnCall):
        return ["fn", e.name if e.name != "mixy" else MIXY, [ref(a) for a in e.args], e.op, val(e.value)]
    if isinstance(e, rex.FoldedAtom):
        return ["folded", ref(e.col), bool(e.result)]
    if isinstance(e, rex.And):
        return ["and", [ref_json(i) for i in e.items]]
    if isinstance(e, rex.Or):
        return ["or", [ref_json(i) for i in e.items]]
    if isinstance(e, rex.Not):
        return ["not", ref_json(e.child)]
    raise TypeError(e)


UDFS = {MIXY: lambda x, y: (x * 7.0 + y) % 13.0,
        "inv": lambda x: 100.0 / x,
        "fmod": lambda x, y: x % (y - 500.0),
        "fdiv": lambda x, y: (x - y) // 3.0,
        "b3d": datagen.udf_b3d}


def json_to_ref(j, table):
    """JSON predicate -> reference expr over ``table`` (kinds from the table)."""
    def ref(r):
        return rex.ColumnRef(table.name, r[0], table.column(r[0]).kind)

    def v(x):
        return float(x["float"]) if isinstance(x, dict) else x

    t = j[0]
    if t == "eq":
        return rex.Equality(ref(j[1]), v(j[2]))
    if t == "cmp":
        return rex.Comparison(ref(j[1]), j[2], v(j[3]))
    if t == "range":
        return rex.Range(ref(j[1]), v(j[2]), v(j[3]))
    if t == "colcmp":
        return rex.ColumnCompare(ref(j[1]), j[2], ref(j[3]))
    if t == "fn":
        return rex.FnCall(j[1], tuple(ref(a) for a in j[2]), j[3], v(j[4]), UDFS.get(j[1]))
    if t == "folded":
        return rex.FoldedAtom(ref(j[1]), j[2])
    if t == "and":
        return rex.And(tuple(json_to_ref(i, table) for i in j[1]))
    if t == "or":
        return rex.Or(tuple(json_to_ref(i, table) for i in j[1]))
    if t == "not":
        return rex.Not(json_to_ref(j[1], table))
    raise ValueError(t)


def digest(idx) -> str:
    return hashlib.sha256(np.asarray(idx, dtype=np.int64).tobytes()).hexdigest()


def outcome(fn):
    try:
        return {"ok": fn()}
    except EscdbError as exc:
        return {"error": type(exc).__name__, "message": str(exc)}


def table_arrays(prefix, table, out):
    meta = []
    for c in table.columns:
        out[f"{prefix}.{c.name}.values"] = np.asarray(c.values)
        out[f"{prefix}.{c.name}.nulls"] = np.asarray(c.null_mask)
        meta.append({"name": c.name, "kind": str(c.kind),
                     "words": c.dictionary.strings() if c.kind.is_text else None})
    return meta


def corpus_entries(table, name, seed, n, mode):
    gen = PredGen(table, random.Random(seed))
    cat = RCatalog()
    cat.register(table)
    out = []
    while len(out) < n:
        p = gen.pred()
        if mode == "count":
            if isinstance(p, rex.FoldedAtom) and p.result:
                continue
            res = outcome(lambda: rces(cat, name, p)[0])
        else:
            res = outcome(lambda: reval(table, p).to_indices())
            if "ok" in res:
                idx = res["ok"]
                res = {"ok": {"count": int(idx.size), "sha256": digest(idx), "head": idx[:8].tolist()}}
        out.append({"pred": ref_json(p), "result": res})
    return out


def edge_cases(table):
    """Semantic corner cases evaluated by the reference executor on ``custom_nulls``."""
    preds = [
        ["not", ["cmp", ["a", None], "<", 10**9]],             # NOT re-admits NULL rows
        ["folded", ["a", None], True], ["folded", ["a", None], False],
        ["not", ["folded", ["b", None], True]],
        ["cmp", ["tag", None], "<", "fir"], ["range", ["tag", None], "birch", "maple"],
        ["cmp", ["tag", None], ">=", "zzz"], ["range", ["tag", None], "pine", "alder"],
        ["cmp", ["a", None], "<", 2**70], ["cmp", ["a", None], ">", -(2**70)], ["eq", ["a", None], 2**70],
        ["cmp", ["a", None], "<", 500.5], ["range", ["val", 2], 1000, 2000.5], ["cmp", ["val", 2], "<>", 0.5],
        ["colcmp", ["a", None], "<=", ["b", None]],
        ["fn", "inv", [["a", None]], ">", 0.0],                 # a has zeros and NULL rows -> error
        ["and", [["cmp", ["a", None], "<", 0], ["fn", "inv", [["a", None]], ">", 0.0]]],  # short-circuited
        ["or", [["folded", ["id", None], True], ["fn", "inv", [["a", None]], ">", 0.0]]],
        ["fn", "fmod", [["a", None], ["b", None]], ">", 1.0],
        ["fn", "fdiv", [["val", 2], ["when", None]], "<", -2000.0],
        ["fn", MIXY, [["a", None], ["b", None]], ">=", 6.0],
    ]
    out = []
    for j in preds:
        p = json_to_ref(j, table)
        res = outcome(lambda: rcount(table, p))
        sel = outcome(lambda: digest(reval(table, p).to_indices()))
        out.append({"pred": j, "count": res, "rows_sha256": sel})
    return out


def float32_cases():
    """NEP 50: float32 column vs Python floats / ints (the reference executor on a native-width
    float32 Column — SURVEY §0 hazard 3)."""
    g = np.random.default_rng(np.random.SeedSequence([42, 77]))
    f = g.standard_normal(5000).astype(np.float32)
    f[:4] = np.float32([0.1, 16777216.0, -0.0, 0.5])
    t = RTable("f32", [RColumn("f", ColumnKind("FLOAT32"), f, np.zeros(f.size, bool))])
    preds = [["eq", ["f", None], 0.1], ["cmp", ["f", None], "<", 0.1], ["cmp", ["f", None], "<", 16777217],
             ["eq", ["f", None], 16777217], ["range", ["f", None], -0.5, 1.0], ["cmp", ["f", None], ">", -0.0],
             ["cmp", ["f", None], "<>", 0.5], ["cmp", ["f", None], ">=", 1e-8]]
    return {"values": f.tolist(),
            "cases": [{"pred": j, "count": rcount(t, json_to_ref(j, t))} for j in preds]}


def native(w: datagen.Workload, name: str) -> RTable:
    cols = []
    for cname, spec in w.columns.items():
        kind_name, vals = spec[0], spec[1]
        kind = {"INT32": KIND_INT64, "INT64": KIND_INT64, "FLOAT32": ColumnKind("FLOAT32"),
                "TEXT": KIND_TEXT}.get(kind_name)
        if kind_name == "DATE":
            kind = ColumnKind("DATE")
        if kind_name.startswith("DECIMAL"):
            from escdb.storage import decimal
            kind = decimal(15, 2)
        d = None
        if kind_name == "TEXT":
            d = RDict()
            for s in spec[2]:
                d.encode(s)
        cols.append(RColumn(cname, kind, vals, np.zeros(len(vals), bool), d))
    return RTable(name, cols)


def config_known():
    out = {}
    for name, w in (("config1", datagen.config1()), ("config2", datagen.config2()),
                    ("config4_6M", datagen.config4(6_000_000))):
        t = native(w, name)
        cat = RCatalog()
        cat.register(t)
        p = json_to_ref(w.pred, t)
        k = rcount(t, p)
        handle, _ = rmat(cat, name, p, w.project)
        temp = cat.resolve_temp(handle)
        idx = reval(t, p).to_indices()
        sums = {}
        for c in temp.columns:
            v = np.asarray(c.values)
            sums[c.name] = float(v.astype(np.float64).sum()) if v.dtype.kind == "f" else int(v.astype(np.int64).sum())
        out[name] = {"count": int(k), "head": idx[:5].tolist(), "rows_sha256": digest(idx), "sums": sums}
    for s in datagen.CONFIG5_SELECTIVITIES:
        for conj in (False, True):
            w = datagen.config5(6_000_000, s, conj)
            t = native(w, "c5")
            out[f"config5_s{s}_{'conj4' if conj else 'single'}"] = {"count": int(rcount(t, json_to_ref(w.pred, t)))}
    return out


def shop_known():
    """test_optimizer.py's `shop` fixture and SHOP_SQL, planned by the reference."""
    def int_table(name, n, **cols):
        schema = [(c, KIND_INT64) for c in cols]
        rows = [[str(fn(i)) for fn in cols.values()] for i in range(1, n + 1)]
        return append_rows(RTable.empty(name, schema), rows)

    cat = RCatalog()
    cat.register(int_table("fact", 5000, f_id=lambda i: i, f_cid=lambda i: (i * 7) % 2000 + 1,
                           f_pid=lambda i: (i * 13) % 1200 + 1, f_tid=lambda i: (i * 3) % 80 + 1,
                           f_qty=lambda i: i % 100))
    cat.register(int_table("cust", 2000, c_id=lambda i: i, c_band=lambda i: i % 10))
    cat.register(int_table("prod", 1200, p_id=lambda i: i, p_cls=lambda i: i % 3))
    cat.register(int_table("tiny", 80, t_id=lambda i: i, t_x=lambda i: i))
    sql = ("SELECT COUNT(*) FROM fact, cust, prod, tiny WHERE f_cid = c_id AND f_pid = p_id AND f_tid = t_id "
           "AND c_band = 3 AND p_cls = 0 AND t_x < 40 AND f_qty < 50")
    out = {}
    for label, cfg in (("histogram", REscConfig(enabled=False, estimator_mode="histogram")),
                       ("default", REscConfig()), ("min1", REscConfig(min_table_size=1)),
                       ("min5000", REscConfig(min_table_size=5000)), ("nomat", REscConfig(materialize=False)),
                       ("sel0.05", REscConfig(max_selectivity=0.05)), ("off", REscConfig(enabled=False))):
        p = rplan(rfe.analyze(rfe.parse(sql), cat), cat, cfg)
        out[label] = {"decisions": [[d.table, d.exact_count, d.row_count, d.qualified, d.pushed_down]
                                    for d in p.decisions],
                      "order": p.build_order, "build_card_sum": p.build_card_sum,
                      "temp_rows": [d.temp.row_count if d.temp else None for d in p.decisions]}
        cat.temps.sweep()
    return out


def star_known():
    g = datagen.config3(fact_rows=60_000_000)
    cat = RCatalog()
    names = {"date": "dates"}
    for tname, cols in g.items():
        rc = []
        for cname, spec in cols.items():
            if spec[0] == "TEXT":
                d = RDict()
                for s in spec[2]:
                    d.encode(s)
                rc.append(RColumn(cname, KIND_TEXT, spec[1], np.zeros(len(spec[1]), bool), d))
            else:
                rc.append(RColumn(cname, KIND_INT64, spec[1], np.zeros(len(spec[1]), bool)))
        cat.register(RTable(names.get(tname, tname), rc))
    sql = ("SELECT COUNT(*) FROM fact, dates, customer, supplier, part WHERE f_datekey = d_datekey "
           "AND f_custkey = c_custkey AND f_suppkey = s_suppkey AND f_partkey = p_partkey "
           "AND c_region = 'R1' AND (p_category = 'C03' OR p_category = 'C07') "
           "AND d_year BETWEEN 1993 AND 1994 AND (s_nation = 'N02' OR s_nation = 'N05')")
    p = rplan(rfe.analyze(rfe.parse(sql), cat), cat, REscConfig())
    res = {"decisions": [[d.table, d.exact_count, d.row_count, d.qualified, d.pushed_down] for d in p.decisions],
           "order": p.build_order, "build_card_sum": p.build_card_sum,
           "temps": {d.table: {"rows": d.temp.row_count,
                               "sha256": digest(cat.resolve_temp(d.temp).columns[0].values)} for d in p.decisions
                     if d.temp}}
    cat.temps.sweep()
    return res


def join_known():
    """Reference build_hash / probe_joins on tests/golden/join_cases.py: stage counts, result rows,
    projected columns in order (full lists: the cases are small)."""
    sys.path.insert(0, HERE)
    import join_cases
    from escdb.executor import BuildStep as RBuildStep, build_hash as rbuild, probe_joins as rprobe

    out = {}
    for case in join_cases.cases():
        tabs = {}
        for alias, cols in case["tables"].items():
            tabs[alias] = RTable(alias, [RColumn(c, KIND_INT64, v, n) for c, (v, n) in cols.items()])
        steps = []
        for st in case["steps"]:
            t = tabs[st["alias"]]
            res = json_to_ref(st["residual"], t) if st["residual"] is not None else None
            idx = rbuild(t, st["key"], res)
            src, cname = st["probe_key"]
            steps.append(RBuildStep(st["alias"], idx, rex.ColumnRef(src, cname, KIND_INT64)))
        probe = tabs[case["probe"]]
        pp = json_to_ref(case["probe_pred"], probe) if case["probe_pred"] is not None else None
        proj = None
        if case["projection"] is not None:
            proj = tuple(rex.ColumnRef(a, c, KIND_INT64) for a, c in case["projection"])
        result, stats = rprobe(probe, case["probe"], pp, steps, proj)
        rec = {"probe_out": [int(x) for x in stats.probe_out], "result_rows": int(stats.result_rows),
               "build_cards": [int(x) for x in stats.build_cards],
               "build_distinct": [int(x) for x in stats.build_distinct]}
        if result is not None:
            rec["columns"] = [[c.name, np.asarray(c.values).tolist(), np.asarray(c.null_mask).tolist()]
                              for c in result.columns]
        out[case["name"]] = rec
    return out


def histogram_known():
    """Reference build_histogram + estimate_selectivity on tests/golden/hist_cases.py, and the
    histogram arm's plans on the shop fixture."""
    sys.path.insert(0, HERE)
    import hist_cases
    from escdb.catalog import build_histogram as rbuild, estimate_selectivity as rest
    from escdb.errors import Inestimable

    out = {"histograms": {}, "estimates": {}}
    for name, (vals, nulls) in hist_cases.columns().items():
        t = RTable("t", [RColumn("v", KIND_INT64, vals, nulls)])
        for b in hist_cases.BUCKETS:
            h = rbuild(t, "v", b)
            out["histograms"][f"{name}/{b}"] = {"boundaries": h.boundaries.tolist(), "counts": h.counts.tolist(),
                                                "distincts": h.distincts.tolist(), "null_count": int(h.null_count),
                                                "row_count": int(h.row_count)}
            if b != 64:
                continue
            est = []
            for j in hist_cases.PREDICATES:
                try:
                    est.append(repr(rest(lambda ref: h, json_to_ref(j, t))))
                except (Inestimable, ValueError, OverflowError) as exc:
                    est.append(f"error:{type(exc).__name__}")
            out["estimates"][name] = est
    return out


def csv_known():
    """Reference load_csv on tests/golden/csv_cases.py: column values / NULL masks / dictionary
    words, or the exception type and message."""
    sys.path.insert(0, HERE)
    import csv_cases
    from escdb.engine import parse_schema_spec as rspec
    from escdb.storage import load_csv as rload

    out = {}
    for name, text, spec, header in csv_cases.CASES:
        try:
            t = rload(text, "t", rspec(spec), has_header=header)
            out[name] = {"columns": [[c.name, np.asarray(c.values).tolist(), np.asarray(c.null_mask).tolist(),
                                      c.dictionary.strings() if c.kind.is_text else None] for c in t.columns]}
        except Exception as exc:  # noqa: BLE001 — the reference's own exception is the fixture
            out[name] = {"error": type(exc).__name__, "message": str(exc)}
    return out


def star_execute_known():
    """The config-3 star query executed by the reference: plan with ESC, execute_plan COUNT."""
    from escdb.optimizer import execute_plan as rexec

    g = datagen.config3(fact_rows=60_000_000)
    cat = RCatalog()
    names = {"date": "dates"}
    for tname, cols in g.items():
        rc = []
        for cname, spec in cols.items():
            if spec[0] == "TEXT":
                d = RDict()
                for w in spec[2]:
                    d.encode(w)
                rc.append(RColumn(cname, KIND_TEXT, spec[1], np.zeros(len(spec[1]), bool), d))
            else:
                rc.append(RColumn(cname, KIND_INT64, spec[1], np.zeros(len(spec[1]), bool)))
        cat.register(RTable(names.get(tname, tname), rc))
    sql = ("SELECT COUNT(*) FROM fact, dates, customer, supplier, part WHERE f_datekey = d_datekey "
           "AND f_custkey = c_custkey AND f_suppkey = s_suppkey AND f_partkey = p_partkey "
           "AND c_region = 'R1' AND (p_category = 'C03' OR p_category = 'C07') "
           "AND d_year BETWEEN 1993 AND 1994 AND (s_nation = 'N02' OR s_nation = 'N05')")
    import time as _t

    p = rplan(rfe.analyze(rfe.parse(sql), cat), cat, REscConfig())
    t0 = _t.perf_counter()
    _, count, stats = rexec(p, cat)
    ms = (_t.perf_counter() - t0) * 1e3
    cat.temps.sweep()
    return {"count": int(count), "probe_out": [int(x) for x in stats.probe_out], "execute_ms_reference": ms,
            "order": p.build_order}


def main():
    if "--only-joins" in sys.argv:  # refresh just the join sections of known.json
        path = os.path.join(HERE, "known.json")
        with open(path) as fh:
            known = json.load(fh)
        known["joins"] = join_known()
        known["histogram"] = histogram_known()
        known["shop"] = shop_known()
        known["csv"] = csv_known()
        if "--skip-star" not in sys.argv:
            known["star_execute"] = star_execute_known()
        with open(path, "w") as fh:
            json.dump(known, fh, indent=1)
        print("join fixtures written")
        return
    custom = generate(GenSpec("custom", 0.02, 3, null_fraction=0.08))["data"]
    orders = generate(GenSpec("tpch_subset", 0.001, 7))["orders"]
    arrays = {}
    meta = {"custom_nulls": table_arrays("custom_nulls", custom, arrays),
            "orders": table_arrays("orders", orders, arrays)}
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **arrays)
    corpus = {
        "meta": meta,
        "criterion1_custom": corpus_entries(custom, "data", 2024, 200, "count"),
        "criterion1_orders": corpus_entries(orders, "orders", 7, 40, "count"),
        "eval_custom_101": corpus_entries(custom, "data", 101, 60, "rows"),
        "count_custom_55": corpus_entries(custom, "data", 55, 20, "count"),
        "edge_cases": edge_cases(custom),
        "float32": float32_cases(),
    }
    with open(os.path.join(HERE, "corpus.json"), "w") as fh:
        json.dump(corpus, fh, separators=(",", ":"))
    known = {"configs": config_known(), "shop": shop_known(), "star": star_known(), "joins": join_known(),
             "histogram": histogram_known(), "csv": csv_known(),
             "star_execute": star_execute_known(),
             "generator": "reference escdb 0.1.0 (pkg/src/escdb), numpy " + np.__version__}
    with open(os.path.join(HERE, "known.json"), "w") as fh:
        json.dump(known, fh, indent=1)
    print("golden fixtures written")


if __name__ == "__main__":
    main()
