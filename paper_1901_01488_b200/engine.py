"""Engine facade: one query at a time, temps never outlive the query.

Multi-GPU: each rank runs its own Engine over its shards of the same tables (one process per GPU)
and the same queries in the same order; :meth:`Engine.run` then plans on global counts and
executes with :func:`.multigpu.execute_plan_sharded`.

The reference ``Engine.run`` (``pkg/src/escdb/engine.py:56-77``) plans, executes, and sweeps every
planner temp table in a ``finally``; its ESC overhead is ``sum(subquery_ms + materialize_ms)``.
:meth:`Engine.run` does the same on the device (ESC sub-queries, then the hash-join pipeline of
``join.execute_plan`` over the temps); :meth:`Engine.optimize` stops after planning
(``keep_temps=True`` hands the temps to the caller, who must ``catalog.temps.sweep()``).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

from . import join, optimizer
from .catalog import Catalog
from .optimizer import EscConfig, PhysicalPlan
from .storage import ColumnTable


@dataclass
class QueryResult:
    """Reference ``engine.QueryResult`` (``engine.py:19-32``)."""

    count: int
    rows: ColumnTable | None  # None for COUNT(*) queries
    plan: PhysicalPlan
    stats: object
    time_ms: float  # plan + execute, sub-queries included
    overhead_ms: float  # planning-time sub-query + materialization cost

    @property
    def is_count(self) -> bool:
        return self.rows is None


@dataclass
class OptimizeResult:
    plan: PhysicalPlan
    plan_ms: float       # wall time of optimizer.plan (sub-queries included)
    overhead_ms: float   # reference definition: sum of subquery_ms + materialize_ms


class Engine:
    def __init__(self, config: EscConfig | None = None, workers: int = 1):
        self.catalog = Catalog()
        self.config = config or EscConfig()
        self.workers = workers

    def register_udf(self, name: str, arity: int, fn):
        self.catalog.register_udf(name, arity, fn)

    def load_csv_file(self, path: str, table: str, schema_spec: str, has_header: bool = False) -> ColumnTable:
        """Load a CSV file with a ``name:kind,name:kind`` schema spec into a device table and
        register it (reference ``engine.py:41-49``); parsing runs on the device."""
        from .ingest import load_csv

        with open(path, "rb") as fh:
            loaded = load_csv(fh.read(), table, parse_schema_spec(schema_spec), has_header=has_header)
        self.catalog.register(loaded)
        return loaded

    def run(self, ra) -> QueryResult:
        """Plan with ESC and execute on the device — reference ``Engine.run`` (``engine.py:56-77``)
        minus the SQL text frontend: ``ra`` is an analyzed tree (``ra.query`` builds one).  The
        pushed-down builds read their ESC temps in place; every temp is swept in ``finally``."""
        t0 = time.perf_counter()
        try:
            p = optimizer.plan(ra, self.catalog, self.config)
            if self._sharded(p):
                from .multigpu import execute_plan_sharded

                rows, count, stats = execute_plan_sharded(p, self.catalog, workers=self.workers)
            else:
                rows, count, stats = join.execute_plan(p, self.catalog, workers=self.workers)
            elapsed = (time.perf_counter() - t0) * 1000.0
        finally:
            self.catalog.temps.sweep()
        return QueryResult(count=count, rows=rows, plan=p, stats=stats, time_ms=elapsed,
                           overhead_ms=optimizer.esc_overhead_ms(p))

    def _sharded(self, p) -> bool:
        """Does the plan touch a row-partitioned table (multi-GPU: one Engine per rank, every
        rank running the same query)?"""
        return any(self.catalog.table(src).shard is not None for src in p.graph.source.values())

    def optimize(self, ra, keep_temps: bool = False) -> OptimizeResult:
        t0 = time.perf_counter()
        try:
            p = optimizer.plan(ra, self.catalog, self.config)
            elapsed = (time.perf_counter() - t0) * 1000.0
        finally:
            if not keep_temps:
                self.catalog.temps.sweep()
        return OptimizeResult(p, elapsed, optimizer.esc_overhead_ms(p))


def parse_schema_spec(spec: str) -> list:
    """``"o_orderkey:int64,o_totalprice:decimal(15,2)"`` -> [(name, ColumnKind)]; commas inside
    ``decimal(p,s)`` do not split (reference ``engine.py:80-99``)."""
    from .storage import parse_kind

    items, pending = [], []
    for part in spec.split(","):
        pending.append(part)
        chunk = ",".join(pending)
        if chunk.count("(") != chunk.count(")"):
            continue
        name, sep, kind = chunk.partition(":")
        if not sep or not name.strip():
            raise ValueError(f"bad schema item {chunk!r} (expected name:kind)")
        items.append((name.strip(), parse_kind(kind)))
        pending = []
    if pending:
        raise ValueError(f"bad schema item {','.join(pending)!r} (unbalanced parentheses)")
    return items
