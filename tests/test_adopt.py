"""Trees built by the reference's own analyzer (same IR class names and fields) are adopted by
this package unchanged: predicates, column kinds and RA trees convert node for node (CPU; skipped
where the reference source tree is not mounted)."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources not mounted")


def test_reference_sql_trees_adopt():
    sys.path.insert(0, REF)
    try:
        from escdb import frontend as rfe
        from escdb.catalog import Catalog as RCatalog
        from escdb.storage import KIND_INT64, KIND_TEXT, decimal, load_csv
    finally:
        sys.path.remove(REF)
    from paper_1901_01488_b200 import expr as ex, ra

    cat = RCatalog()
    cat.register(load_csv("1,2.50,a\n", "t", [("a", KIND_INT64), ("p", decimal(9, 2)), ("s", KIND_TEXT)]))
    cat.register(load_csv("1,3\n", "u", [("k", KIND_INT64), ("v", KIND_INT64)]))
    cat.register_udf("h", 1, lambda x: x * 2.0)
    sql = ("SELECT COUNT(*) FROM t, u WHERE a = k AND (p BETWEEN 1.00 AND 3.50 OR s = 'a') "
           "AND NOT (v < 2) AND h(a) > 1")
    tree = rfe.analyze(rfe.parse(sql), cat)
    ours = ra.adopt(tree)
    assert repr(ours) == repr(tree)  # same fields, node for node
    assert type(ours) is ra.RaAggregate and type(ours.child.predicate) is ex.And
    assert ra.adopt(ours) is ours and ex.adopt(ours.child.predicate) is ours.child.predicate
    g = ra.build_join_graph(ours)
    assert [(str(e.left), str(e.right)) for e in g.edges] == [("t.a", "u.k")]
    assert str(g.residual("t")) == "(t.p BETWEEN 100 AND 350 OR t.s = 0) AND h(t.a) > 1.0"
    assert str(g.residual("u")) == "NOT u.v < 2"
    fn = [a for a in ex.atoms(ours.child.predicate) if isinstance(a, ex.FnCall)][0]
    assert fn.fn(3.0) == 6.0 and isinstance(fn.args[0], ex.ColumnRef)
    dec = [r for a in ex.atoms(g.residual("t")) for r in ex.atom_columns(a) if r.name == "p"][0]
    from paper_1901_01488_b200.storage import ColumnKind

    assert isinstance(dec.kind, ColumnKind) and dec.kind.scale == 2
