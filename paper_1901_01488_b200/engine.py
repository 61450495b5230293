"""Engine facade: one query at a time, temps never outlive the query.

The reference ``Engine.run`` (``pkg/src/escdb/engine.py:56-77``) plans, executes, and sweeps every
planner temp table in a ``finally``; its ESC overhead is ``sum(subquery_ms + materialize_ms)``.
This build accelerates the planning half, so :meth:`Engine.optimize` returns the plan with the
same overhead definition and the same sweep guarantee (``keep_temps=True`` hands the temps to the
caller, who must ``catalog.temps.sweep()``).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

from . import optimizer
from .catalog import Catalog
from .optimizer import EscConfig, PhysicalPlan


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

    def optimize(self, ra, keep_temps: bool = False) -> OptimizeResult:
        t0 = time.perf_counter()
        try:
            p = optimizer.plan(ra, self.catalog, self.config)
            elapsed = (time.perf_counter() - t0) * 1000.0
        finally:
            if not keep_temps:
                self.catalog.temps.sweep()
        return OptimizeResult(p, elapsed, optimizer.esc_overhead_ms(p))
