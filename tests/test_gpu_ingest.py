"""Device CSV ingestion (row f3) against the reference loader's outputs: values, NULL masks and
dictionaries bit-exact, and the reference's error type and message for malformed input."""

import csv
import os
import sys

import numpy as np
import pytest

from golden_io import known

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
import csv_cases  # noqa: E402

pytestmark = pytest.mark.gpu

GOLD = known()["csv"]


@pytest.mark.parametrize("case", csv_cases.CASES, ids=lambda c: c[0])
def test_load_csv_matches_reference(cuda, case):
    from paper_1901_01488_b200.engine import parse_schema_spec
    from paper_1901_01488_b200.errors import CsvError
    from paper_1901_01488_b200.ingest import load_csv

    name, text, spec, header = case
    want = GOLD[name]
    if "error" in want:
        with pytest.raises((CsvError, OverflowError, csv.Error)) as err:
            load_csv(text, "t", parse_schema_spec(spec), has_header=header, device=cuda)
        assert str(err.value) == want["message"]
        assert {"Error": "Error", "CsvError": "CsvError", "OverflowError": "OverflowError"}[want["error"]] == \
            type(err.value).__name__
        return
    t = load_csv(text, "t", parse_schema_spec(spec), has_header=header, device=cuda)
    assert [c.name for c in t.columns] == [c[0] for c in want["columns"]]
    for col, (cname, vals, nulls, words) in zip(t.columns, want["columns"]):
        v, m = col.to_numpy()
        assert m.tolist() == nulls, cname
        assert np.where(m, 0, v).tolist() == np.where(np.asarray(nulls, bool), 0, np.asarray(vals, np.int64)).tolist(), cname
        if col.kind.is_text and words is not None:
            assert col.dictionary.strings() == words, cname


def test_engine_load_csv_file_and_roundtrip(cuda, tmp_path):
    """Engine.load_csv_file (reference engine.py:41-49) registers a device table; dump_csv writes
    the loader's format back byte-stably, and reloading it gives the same table."""
    from paper_1901_01488_b200 import Engine, count_star, expr as ex
    from paper_1901_01488_b200.engine import parse_schema_spec
    from paper_1901_01488_b200.ingest import dump_csv, load_csv

    name, text, spec, _ = next(c for c in csv_cases.CASES if c[0] == "big_lf")
    path = tmp_path / "t.csv"
    path.write_bytes(text.encode("utf-8"))
    eng = Engine()
    t = eng.load_csv_file(str(path), "t", spec)
    assert eng.catalog.table("t") is t and t.columns[0].values.is_cuda
    out = dump_csv(t)
    t2 = load_csv(out, "t", parse_schema_spec(spec), device=cuda)
    for a, b in zip(t.columns, t2.columns):
        va, ma = a.to_numpy()
        vb, mb = b.to_numpy()
        assert (ma == mb).all() and (np.where(ma, 0, va) == np.where(mb, 0, vb)).all()
    assert dump_csv(t2) == out
    assert count_star(t, ex.Comparison(ex.ColumnRef("t", "i"), ">", 0)) == int(
        ((t.columns[0].to_numpy()[0] > 0) & ~t.columns[0].to_numpy()[1]).sum())


def test_null_masks_only_where_nulls_occur(cuda):
    """The parse kernel flags the columns that hold a NULL (d_null_seen): those get a bool mask
    with exactly the NULL rows, the others none — for INT64, DECIMAL and TEXT columns, with the
    NULLs early, late and absent."""
    from paper_1901_01488_b200.ingest import NULL_TOKEN, load_csv
    from paper_1901_01488_b200.storage import parse_kind

    n = 20_011
    g = np.random.default_rng(5)
    null_i = g.random(n) < 0.01
    null_i[-1] = True                       # a NULL in the very last row
    null_t = np.zeros(n, bool)
    null_t[0] = True                        # a single NULL in the first row
    lines = []
    for r in range(n):
        i = NULL_TOKEN if null_i[r] else str(r * 7 - 5)
        t = NULL_TOKEN if null_t[r] else f"w{r % 13}"
        lines.append(f"{i},{r % 97},{t},{r}.25\n")
    schema = [("i", parse_kind("int64")), ("k", parse_kind("int64")), ("t", parse_kind("text")),
              ("d", parse_kind("decimal(15,2)"))]
    tab = load_csv("".join(lines), "n", schema, device=cuda)
    ci, ck, ct, cd = tab.columns
    assert ci.nulls is not None and np.array_equal(ci.nulls.cpu().numpy(), null_i)
    assert ct.nulls is not None and np.array_equal(ct.nulls.cpu().numpy(), null_t)
    assert ck.nulls is None and cd.nulls is None
    vi = ci.values.cpu().numpy()
    assert np.array_equal(vi[~null_i], (np.arange(n) * 7 - 5)[~null_i])
    assert np.array_equal(ck.values.cpu().numpy(), np.arange(n) % 97)
