"""B200-native exact selectivity computation (ESC, arXiv 1901.01488).

Drop-in for the hot path of the reference ``escdb`` package: the planning-time COUNT sub-query,
its push-down policy, the order-preserving materialization of qualifying rows into temp tables,
join ordering from the exact counts, and the hash-join pipeline that reuses those temps in place
— with every scan, count, compaction, hash build and probe running in hand-written sm_100a
kernels behind the C ABI in ``include/esc.h``.
"""

from . import expr
from .catalog import Catalog
from .engine import Engine, OptimizeResult, QueryResult
from .errors import EscdbError
from .executor import RowSelection, count_star, eval_predicate, execute_count, materialize
from .histogram import EquiDepthHistogram, build_histogram, estimate_selectivity
from .ingest import append_rows, dump_csv, load_csv
from .join import BuildStep, ExecStats, HashTableIndex, build_hash, execute_plan, probe_joins
from .optimizer import (
    EscConfig,
    compute_exact_selectivity,
    decide_pushdown,
    explain_json,
    explain_text,
    materialize_pushdown,
    order_builds,
    plan,
)
from .ra import build_join_graph, query
from .storage import Column, ColumnKind, ColumnTable, Dictionary

__version__ = "0.1.0"

__all__ = [
    "BuildStep", "Catalog", "EquiDepthHistogram", "append_rows", "dump_csv", "load_csv", "build_histogram", "estimate_selectivity", "Column", "ColumnKind", "ColumnTable", "Dictionary", "Engine", "EscConfig",
    "EscdbError", "ExecStats", "HashTableIndex", "OptimizeResult", "QueryResult", "RowSelection",
    "__version__", "build_hash", "build_join_graph", "execute_plan", "probe_joins",
    "compute_exact_selectivity", "count_star", "decide_pushdown", "eval_predicate",
    "execute_count", "explain_json", "explain_text", "expr", "materialize",
    "materialize_pushdown", "order_builds", "plan", "query",
]
