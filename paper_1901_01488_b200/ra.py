"""Relational-algebra nodes and the join graph the ESC planner consumes.

Same node types and fields as the reference lowering (``pkg/src/escdb/frontend.py:511-557``) and
join-graph classification (``frontend.py:780-871``), so trees produced by the reference's
analyzer — or by :func:`query` below, the programmatic builder used where no SQL text is
involved — plan identically.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import expr as ex
from .errors import AnalysisError, UnsupportedPredicate
from .storage import KIND_INT64, TempTableHandle


@dataclass(frozen=True)
class RaScan:
    table: str
    alias: str
    schema: tuple


@dataclass(frozen=True)
class RaTempScan:
    handle: TempTableHandle
    alias: str
    schema: tuple


@dataclass(frozen=True)
class RaSelect:
    child: object
    predicate: ex.Expr
    schema: tuple


@dataclass(frozen=True)
class RaProject:
    child: object
    columns: tuple
    schema: tuple


@dataclass(frozen=True)
class RaJoin:
    left: object
    right: object
    pairs: tuple
    schema: tuple


@dataclass(frozen=True)
class RaAggregate:
    child: object
    agg: str
    schema: tuple


COUNT_COLUMN = ex.ColumnRef(None, "count", kind=KIND_INT64)


@dataclass(frozen=True)
class JoinEdge:
    left: ex.ColumnRef
    right: ex.ColumnRef

    def touches(self, alias: str) -> bool:
        return alias in (self.left.table, self.right.table)

    def key_for(self, alias: str) -> ex.ColumnRef:
        for side in (self.left, self.right):
            if side.table == alias:
                return side
        raise KeyError(alias)

    def other(self, alias: str) -> str:
        if self.left.table == alias:
            return self.right.table
        if self.right.table == alias:
            return self.left.table
        raise KeyError(alias)

    def __str__(self):
        return f"{self.left} = {self.right}"


@dataclass
class JoinGraph:
    tables: tuple        # aliases, FROM order
    source: dict         # alias -> base table name
    edges: tuple
    residuals: dict      # alias -> per-table predicate (absent = unfiltered)

    def residual(self, alias: str):
        return self.residuals.get(alias)


def _scans_and_predicate(ra):
    node = ra.child if isinstance(ra, (RaProject, RaAggregate)) else ra
    pred = None
    if isinstance(node, RaSelect):
        pred, node = node.predicate, node.child
    scans: list = []
    stack = [node]
    while stack:  # left-deep, keep FROM order: visit left before right
        n = stack.pop()
        if isinstance(n, RaJoin):
            stack.append(n.right)
            stack.append(n.left)
        elif isinstance(n, RaScan):
            scans.append(n)
        else:
            raise AnalysisError(f"unexpected node below Select: {type(n).__name__}")
    return scans, pred


def build_join_graph(ra) -> JoinGraph:
    """Each WHERE conjunct is a join edge (cross-table ``=`` ColumnCompare) or a residual of the
    one table it touches; anything else spanning tables is rejected."""
    scans, pred = _scans_and_predicate(ra)
    edges: list = []
    per_alias: dict = {}
    for conj in (ex.conjuncts(pred) if pred is not None else []):
        touched = ex.tables(conj)
        if isinstance(conj, ex.ColumnCompare) and conj.op == "=" and conj.left.table != conj.right.table:
            edges.append(JoinEdge(conj.left, conj.right))
        elif len(touched) == 1:
            per_alias.setdefault(next(iter(touched)), []).append(conj)
        else:
            raise UnsupportedPredicate(
                f"predicate spans tables {sorted(touched)} and is not an equi-join: {conj}")
    return JoinGraph(tuple(s.alias for s in scans), {s.alias: s.table for s in scans}, tuple(edges),
                     {a: ex.conjoin(items) for a, items in per_alias.items()})


def _schema(alias, table) -> tuple:
    return tuple(ex.ColumnRef(alias, c.name, kind=c.kind) for c in table.columns)


def query(catalog, tables, where: ex.Expr | None = None, select=None):
    """Build the canonical RA tree the reference analyzer produces (``frontend.py:738-772``):
    scans joined left-deep in FROM order, one Select on top, then Project (``select`` = list of
    column refs, or ``"*"``) or Aggregate(COUNT(*)) when ``select`` is None.

    ``tables`` is a list of table names or ``(name, alias)`` pairs."""
    node = None
    for item in tables:
        name, alias = (item, item) if isinstance(item, str) else item
        scan = RaScan(name, alias, _schema(alias, catalog.table(name)))
        node = scan if node is None else RaJoin(node, scan, (), node.schema + scan.schema)
    if where is not None:
        node = RaSelect(node, where, node.schema)
    if select is None:
        return RaAggregate(node, "count_star", (COUNT_COLUMN,))
    cols = node.schema if select == "*" else tuple(select)
    return RaProject(node, cols, cols)


def adopt(node):
    """This package's RA tree for one built by the reference analyzer (``frontend.py:511-557``:
    same class names and fields); predicates and column refs are adopted too."""
    if node is None:
        return None
    name = type(node).__name__
    if isinstance(node, (RaScan, RaTempScan, RaSelect, RaProject, RaJoin, RaAggregate)):
        return node
    schema = tuple(ex.adopt_ref(c) for c in getattr(node, "schema", ()))
    if name == "RaScan":
        return RaScan(node.table, node.alias, schema)
    if name == "RaTempScan":
        return RaTempScan(node.handle, node.alias, schema)
    if name == "RaSelect":
        return RaSelect(adopt(node.child), ex.adopt(node.predicate), schema)
    if name == "RaProject":
        return RaProject(adopt(node.child), tuple(ex.adopt_ref(c) for c in node.columns), schema)
    if name == "RaJoin":
        return RaJoin(adopt(node.left), adopt(node.right),
                      tuple((ex.adopt_ref(a), ex.adopt_ref(b)) for a, b in node.pairs), schema)
    if name == "RaAggregate":
        return RaAggregate(adopt(node.child), node.agg, schema)
    raise TypeError(f"not an RA node: {node!r}")
