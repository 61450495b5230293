"""Device equi-depth histograms (row f4) and the estimator against the reference's outputs:
boundaries / counts / distincts bit-exact, estimates equal as floats; plus the reference's
TestHistogram / TestEstimates properties (test_catalog.py:104-290)."""

import os
import sys

import numpy as np
import pytest

from golden_io import known

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
import hist_cases  # noqa: E402

pytestmark = pytest.mark.gpu

GOLD = known()["histogram"]
COLS = hist_cases.columns()


def _table(vals, nulls, cuda):
    from paper_1901_01488_b200.storage import KIND_INT64, Column, ColumnTable

    return ColumnTable("t", [Column("v", KIND_INT64, vals, nulls, device=cuda)])


@pytest.mark.parametrize("name", sorted(COLS))
def test_device_histograms_and_estimates(cuda, name):
    from paper_1901_01488_b200 import serde
    from paper_1901_01488_b200.histogram import build_histogram, estimate_selectivity

    vals, nulls = COLS[name]
    t = _table(vals, nulls, cuda)
    for b in hist_cases.BUCKETS:
        h = build_histogram(t, "v", b)
        got = {"boundaries": h.boundaries.tolist(), "counts": h.counts.tolist(), "distincts": h.distincts.tolist(),
               "null_count": h.null_count, "row_count": h.row_count}
        assert got == GOLD["histograms"][f"{name}/{b}"], b
        if b != 64:
            continue
        for j, want in zip(hist_cases.PREDICATES, GOLD["estimates"][name]):
            try:
                est = repr(estimate_selectivity(lambda ref: h, serde.from_json(j, "t")))
            except (ValueError, OverflowError) as exc:
                est = f"error:{type(exc).__name__}"
            assert est == want, j


def test_histogram_properties(cuda):
    from paper_1901_01488_b200.errors import Inestimable, UnsupportedColumnKind
    from paper_1901_01488_b200 import expr as ex
    from paper_1901_01488_b200.histogram import build_histogram, estimate_selectivity
    from paper_1901_01488_b200.storage import KIND_INT64, KIND_TEXT, Column, ColumnTable, Dictionary

    vals, nulls = COLS["ref_partition"]
    h = build_histogram(_table(vals, nulls, cuda), "v", 64)
    assert int(h.counts.sum()) == 5000 and h.null_count == 40 and h.non_null == 5000
    assert np.all(np.diff(h.boundaries) > 0)
    t = ColumnTable("t", [Column("v", KIND_INT64, np.arange(3), device=cuda),
                          Column("s", KIND_TEXT, np.zeros(3, np.int8), None, Dictionary(["a"]), device=cuda)])
    with pytest.raises(UnsupportedColumnKind):
        build_histogram(t, "s", 8)
    with pytest.raises(ValueError):
        build_histogram(t, "v", 0)
    hf = lambda ref: h  # noqa: E731
    with pytest.raises(Inestimable):
        estimate_selectivity(hf, ex.FnCall("f", (ex.ColumnRef("t", "v"),), "<", 3.0, lambda a: a))
    with pytest.raises(Inestimable):
        estimate_selectivity(hf, ex.ColumnCompare(ex.ColumnRef("t", "v"), "=", ex.ColumnRef("t", "w")))


def test_correlated_conjunction_underestimates(cuda):
    """Independence multiplies per-atom fractions: a copied column pair is estimated near
    (1/n)^2 when the truth is 1/n — the failure mode exact counts avoid (test_catalog.py:259)."""
    from paper_1901_01488_b200 import count_star, expr as ex
    from paper_1901_01488_b200.histogram import build_histogram, estimate_selectivity
    from paper_1901_01488_b200.storage import KIND_INT64, Column, ColumnTable

    a = np.random.default_rng(23).integers(0, 1000, size=20_000)
    t = ColumnTable("t", [Column("a", KIND_INT64, a, device=cuda), Column("b", KIND_INT64, a.copy(), device=cuda)])
    hists = {"a": build_histogram(t, "a", 64), "b": build_histogram(t, "b", 64)}
    pred = ex.And((ex.Equality(ex.ColumnRef("t", "a"), 5), ex.Equality(ex.ColumnRef("t", "b"), 5)))
    est = estimate_selectivity(lambda ref: hists[ref.name], pred)
    true = count_star(t, pred) / t.row_count
    assert true > 0 and est < true / 10
