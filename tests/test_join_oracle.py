"""The oracle's restatement of the reference hash join (build_hash / probe_joins) against the
reference's own outputs on every join scenario (tests/golden/join_cases.py; CPU only)."""

import numpy as np
import pytest

from golden_io import known
from join_helpers import cases, oracle_run
from oracle import esc_oracle as O

GOLD = known().get("joins", {})


@pytest.mark.parametrize("case", cases(), ids=lambda c: c["name"])
def test_oracle_matches_reference(case):
    want = GOLD[case["name"]]
    got = oracle_run(case)
    for k in ("probe_out", "result_rows", "build_cards", "build_distinct"):
        assert got[k] == want[k], k
    assert got.get("columns") == want.get("columns")


def test_index_groups_follow_unique_key_order():
    """Group ids are indices into the ascending unique keys; rows of a group ascend."""
    t = O.OTable("t", {"k": O.OColumn(np.array([5, 5, 7, 0, 9], np.int64), np.array([0, 0, 0, 1, 0], bool))})
    idx = O.build_hash(t, "k")
    assert idx.n_entries == 4 and idx.distinct_keys == 3
    assert idx.probe_groups(np.array([5, 6, 7, 9, 5]), np.ones(5, bool)).tolist() == [0, -1, 1, 2, 0]
    assert idx.lookup(5).tolist() == [0, 1] and idx.lookup(0).size == 0
