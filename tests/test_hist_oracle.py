"""The oracle's restatement of the reference histogram arm (build_histogram, estimate_selectivity)
against the reference's own outputs (tests/golden/hist_cases.py; CPU only)."""

import os
import sys

import pytest

from golden_io import known
from oracle import esc_oracle as O

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
import hist_cases  # noqa: E402

GOLD = known()["histogram"]
COLS = hist_cases.columns()


@pytest.mark.parametrize("name", sorted(COLS))
def test_histograms_match_reference(name):
    vals, nulls = COLS[name]
    for b in hist_cases.BUCKETS:
        assert O.build_histogram(vals, nulls, b) == GOLD["histograms"][f"{name}/{b}"], b


@pytest.mark.parametrize("name", sorted(COLS))
def test_estimates_match_reference(name):
    vals, nulls = COLS[name]
    h = O.build_histogram(vals, nulls, 64)
    for j, want in zip(hist_cases.PREDICATES, GOLD["estimates"][name]):
        try:
            got = repr(O.estimate(h, j))
        except (ValueError, OverflowError) as exc:
            got = f"error:{type(exc).__name__}"
        assert got == want, j
