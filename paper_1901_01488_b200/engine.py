"""Engine facade: one query at a time, temps never outlive the query.

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

    def run(self, ra) -> QueryResult:
        """Plan with ESC and execute on the device — reference ``Engine.run`` (``engine.py:56-77``)
        minus the SQL text frontend: ``ra`` is an analyzed tree (``ra.query`` builds one).  The
        pushed-down builds read their ESC temps in place; every temp is swept in ``finally``."""
        t0 = time.perf_counter()
        try:
            p = optimizer.plan(ra, self.catalog, self.config)
            rows, count, stats = join.execute_plan(p, self.catalog, workers=self.workers)
            elapsed = (time.perf_counter() - t0) * 1000.0
        finally:
            self.catalog.temps.sweep()
        return QueryResult(count=count, rows=rows, plan=p, stats=stats, time_ms=elapsed,
                           overhead_ms=optimizer.esc_overhead_ms(p))

    def optimize(self, ra, keep_temps: bool = False) -> OptimizeResult:
        t0 = time.perf_counter()
        try:
            p = optimizer.plan(ra, self.catalog, self.config)
            elapsed = (time.perf_counter() - t0) * 1000.0
        finally:
            if not keep_temps:
                self.catalog.temps.sweep()
        return OptimizeResult(p, elapsed, optimizer.esc_overhead_ms(p))
