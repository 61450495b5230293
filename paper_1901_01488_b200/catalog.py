"""Catalog: base tables, the temp-table facade and the UDF registry.

Mirrors ``escdb.catalog.Catalog`` (reference ``pkg/src/escdb/catalog.py:63-150``) for everything
the ESC path touches.  Tables are device-resident :class:`~.storage.ColumnTable` objects; temp
tables are the compaction kernel's outputs.  Histograms of the estimator contrast arm
(``catalog.py:128-134``, built by :mod:`.histogram`) are cached per (table, column).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

from .errors import DuplicateFunction, DuplicateTable, EmptySchema, UnknownTable
from .storage import Column, ColumnTable, TempTableHandle, TempTableStore


@dataclass
class Udf:
    name: str
    arity: int
    fn: Callable


class Catalog:
    def __init__(self):
        self._tables: dict[str, ColumnTable] = {}
        self._udfs: dict[str, Udf] = {}
        self._histograms: dict = {}
        self.temps = TempTableStore()

    # -- base tables ------------------------------------------------------------------------
    def create_table(self, name: str, schema) -> ColumnTable:
        if name in self._tables:
            raise DuplicateTable(f"table {name!r} already exists")
        if not schema:
            raise EmptySchema(f"table {name!r} must have at least one column")
        table = ColumnTable.empty(name, schema)
        self._tables[name] = table
        return table

    def register(self, table: ColumnTable):
        if table.name in self._tables:
            raise DuplicateTable(f"table {table.name!r} already exists")
        self._tables[table.name] = table

    def replace(self, table: ColumnTable):
        """Swap in a rebuilt version of an existing (or new) table (drops its histograms)."""
        self._tables[table.name] = table
        self._histograms = {k: v for k, v in self._histograms.items() if k[0] != table.name}

    # -- statistics -------------------------------------------------------------------------------
    def histogram(self, table: str, column: str, buckets: int = 64):
        """Cached equi-depth histogram (reference ``catalog.py:128-134``), built on the device."""
        from .histogram import build_histogram

        key = (table, column)
        if key not in self._histograms:
            self._histograms[key] = build_histogram(self.table(table), column, buckets)
        return self._histograms[key]

    def table(self, name: str) -> ColumnTable:
        table = self._tables.get(name)
        if table is None:
            raise UnknownTable(f"unknown table {name!r}")
        return table

    def has_table(self, name: str) -> bool:
        return name in self._tables

    def table_names(self) -> list[str]:
        return sorted(self._tables)

    # -- temp tables ----------------------------------------------------------------------------
    def materialize_temp(self, columns: list[Column], shard=None) -> TempTableHandle:
        return self.temps.materialize(columns, shard)

    def resolve_temp(self, handle: TempTableHandle) -> ColumnTable:
        return self.temps.resolve(handle)

    def drop_temp(self, handle: TempTableHandle):
        self.temps.drop(handle)

    # -- UDFs -------------------------------------------------------------------------------------
    def register_udf(self, name: str, arity: int, fn: Callable):
        """Register a scalar function usable in predicates.  It receives float arguments
        (DECIMAL descaled, DATE as epoch days) and is traced into a device program on first
        use (see :mod:`.udf`)."""
        key = name.lower()
        if key in self._udfs:
            raise DuplicateFunction(f"function {name!r} already registered")
        self._udfs[key] = Udf(key, arity, fn)

    def udf(self, name: str) -> Udf | None:
        return self._udfs.get(name.lower())
