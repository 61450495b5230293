"""Device-resident columnar tables and the per-query temp-table store.

Replaces the numpy storage of the reference (``pkg/src/escdb/storage.py``):

* :class:`Column` (reference ``storage.py:156-197``) keeps ``values`` as a torch tensor in HBM at
  its NATIVE width (int8/int16/int32/int64/float32/float64) instead of widening every kind to
  int64 (``storage.py:1-7``, ``:293``); the NULL mask is a bool tensor (1 byte per row, True =
  NULL, the reference's representation) and is dropped entirely when the column has no NULLs,
  so a NULL-free column costs no mask traffic in the scan.
* :class:`ColumnKind` keeps INT64 / DATE / TEXT / DECIMAL(p,s) and adds INT32, INT16, INT8,
  FLOAT32 and FLOAT64 for the BASELINE configurations' physical widths.
* :class:`TempTableStore` / :class:`TempTableHandle` (``storage.py:325-375``) hold the compacted
  temp tables produced by the materialization kernel; dropping a handle releases its device
  buffers back to torch's caching allocator (no ``cudaFree`` on the planning path).

Tables are immutable once built (reference ``storage.py:1-7``).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from datetime import date as _date
from typing import Sequence

import numpy as np
import torch

from .errors import (
    DeadHandle,
    EmptySchema,
    LengthMismatch,
    StorageError,
    TypeMismatch,
)

EPOCH = _date(1970, 1, 1)

INT64, DATE, TEXT, DECIMAL = "INT64", "DATE", "TEXT", "DECIMAL"
INT32, INT16, INT8, FLOAT32, FLOAT64 = "INT32", "INT16", "INT8", "FLOAT32", "FLOAT64"
_INTEGER_KINDS = (INT64, INT32, INT16, INT8, DATE)
_FLOAT_KINDS = (FLOAT32, FLOAT64)


@dataclass(frozen=True)
class ColumnKind:
    """Logical column type; ``precision``/``scale`` only for DECIMAL."""

    name: str
    precision: int = 0
    scale: int = 0

    def __str__(self):
        return f"DECIMAL({self.precision},{self.scale})" if self.is_decimal else self.name

    @property
    def is_text(self) -> bool:
        return self.name == TEXT

    @property
    def is_decimal(self) -> bool:
        return self.name == DECIMAL

    @property
    def is_float(self) -> bool:
        return self.name in _FLOAT_KINDS


def decimal(precision: int, scale: int) -> ColumnKind:
    return ColumnKind(DECIMAL, precision, scale)


KIND_INT64 = ColumnKind(INT64)
KIND_DATE = ColumnKind(DATE)
KIND_TEXT = ColumnKind(TEXT)
KIND_INT32 = ColumnKind(INT32)
KIND_INT16 = ColumnKind(INT16)
KIND_INT8 = ColumnKind(INT8)
KIND_FLOAT32 = ColumnKind(FLOAT32)
KIND_FLOAT64 = ColumnKind(FLOAT64)

_SIMPLE_KINDS = {k.name: k for k in (KIND_INT64, KIND_DATE, KIND_TEXT, KIND_INT32, KIND_INT16,
                                     KIND_INT8, KIND_FLOAT32, KIND_FLOAT64)}

# default physical dtype per kind when values arrive as Python lists
_DEFAULT_DTYPE = {
    INT64: np.int64, DATE: np.int32, TEXT: np.int32, DECIMAL: np.int64, INT32: np.int32,
    INT16: np.int16, INT8: np.int8, FLOAT32: np.float32, FLOAT64: np.float64,
}

_SUPPORTED_DTYPES = (np.int8, np.int16, np.int32, np.int64, np.uint8, np.uint16, np.uint32,
                     np.float32, np.float64)


def parse_kind(text: str) -> ColumnKind:
    """``int64`` / ``date`` / ``text`` / ``decimal(15,2)`` / ``int32`` / ``float32`` ..."""
    t = text.strip().upper()
    if t in _SIMPLE_KINDS:
        return _SIMPLE_KINDS[t]
    if t.startswith("DECIMAL(") and t.endswith(")"):
        parts = t[8:-1].split(",")
        if len(parts) == 2 and all(p.strip().isdigit() for p in parts):
            return decimal(int(parts[0]), int(parts[1]))
    raise TypeMismatch(f"unknown column kind {text!r}")


def date_to_days(text: str) -> int:
    try:
        return (_date.fromisoformat(text) - EPOCH).days
    except ValueError as exc:
        raise TypeMismatch(f"bad DATE literal {text!r}: {exc}") from None


def days_to_date(days: int) -> str:
    return _date.fromordinal(EPOCH.toordinal() + int(days)).isoformat()


def format_decimal(scaled: int, scale: int) -> str:
    if scale == 0:
        return str(int(scaled))
    mag = abs(int(scaled))
    sign = "-" if scaled < 0 else ""
    q, r = divmod(mag, 10**scale)
    return f"{sign}{q}.{r:0{scale}d}"


class Dictionary:
    """Insertion-ordered bijection string <-> code (reference ``storage.py:127-153``)."""

    def __init__(self, words: Sequence[str] = ()):
        self._codes: dict[str, int] = {}
        self._words: list[str] = []
        for w in words:
            self.encode(w)

    def __len__(self):
        return len(self._words)

    def encode(self, s: str) -> int:
        code = self._codes.get(s)
        if code is None:
            code = self._codes[s] = len(self._words)
            self._words.append(s)
        return code

    def lookup(self, s: str) -> int | None:
        return self._codes.get(s)

    def decode(self, code: int) -> str:
        return self._words[code]

    def strings(self) -> list[str]:
        return list(self._words)


def default_device() -> torch.device:
    """Where new columns live: the current CUDA device, or CPU on a GPU-less host (host-side
    logic only — every kernel entry point refuses CPU columns)."""
    if torch.cuda.is_available():
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _as_tensor(x, dtype_hint, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x
    else:
        arr = np.asarray(x)
        if arr.dtype == object or arr.dtype.kind not in "iufb":
            arr = np.asarray(x, dtype=dtype_hint)
        if arr.dtype.type not in _SUPPORTED_DTYPES and arr.dtype != np.bool_:
            raise TypeMismatch(f"unsupported column dtype {arr.dtype}")
        t = torch.from_numpy(np.ascontiguousarray(arr))
    if t.dim() != 1:
        raise TypeMismatch("column data must be one-dimensional")
    return t.to(device).contiguous()


class Column:
    """One typed column: ``values`` (device tensor, native width) + optional NULL mask.

    ``values`` at NULL positions are not interpreted by atoms (they are by UDF argument
    conversion, exactly as in the reference ``executor.py:113-125``).
    """

    __slots__ = ("name", "kind", "values", "nulls", "dictionary", "_zero_mask", "_null_bits")

    def __init__(self, name: str, kind: ColumnKind, values, null_mask=None,
                 dictionary: Dictionary | None = None, device=None):
        dev = torch.device(device) if device is not None else (
            values.device if isinstance(values, torch.Tensor) else default_device())
        self.name = name
        self.kind = kind
        self.values = _as_tensor(values, _DEFAULT_DTYPE.get(kind.name, np.int64), dev)
        if self.values.dtype == torch.bool:
            self.values = self.values.to(torch.int8)
        nulls = None
        if null_mask is not None:
            if isinstance(null_mask, torch.Tensor):
                m = null_mask.to(dev).to(torch.bool).contiguous()
                if m.numel() and bool(m.any()):
                    nulls = m
            else:
                arr = np.asarray(null_mask, dtype=bool)
                if arr.any():
                    nulls = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
        if nulls is not None and nulls.numel() != self.values.numel():
            raise LengthMismatch(f"column {name!r}: null mask length differs from values")
        self.nulls = nulls
        if kind.is_text and dictionary is None:
            dictionary = Dictionary()
        self.dictionary = dictionary
        self._zero_mask = None
        self._null_bits = None

    @property
    def null_bits(self) -> "torch.Tensor | None":
        """The NULL mask packed 1 bit per row (row-linear int32 words), built once on the device
        (``esc_pack_nulls``) and staged by count / selection scans instead of the byte mask:
        N/8 bytes of NULL state per scan instead of N.  None for a column without NULLs."""
        if self.nulls is None or not self.values.is_cuda:
            return None
        if self._null_bits is None:
            import ctypes as C

            from . import _native as N

            lib = N.load_library()
            n = len(self)
            # esc_pack_nulls writes every word, the padding words past the rows included
            bits = torch.empty(int(lib.esc_null_bits_words(n)), dtype=torch.int32, device=self.values.device)
            N.check(lib.esc_pack_nulls(C.c_void_p(self.nulls.data_ptr() if n else None), n, C.c_void_p(bits.data_ptr()),
                                       C.c_void_p(torch.cuda.current_stream(self.values.device).cuda_stream)),
                    "esc_pack_nulls")
            self._null_bits = bits
        return self._null_bits

    @classmethod
    def device_column(cls, name: str, kind: ColumnKind, values: torch.Tensor, nulls: torch.Tensor | None,
                      dictionary: "Dictionary | None") -> "Column":
        """Internal: wrap device tensors the kernels just produced (contiguous, native dtype, on
        the column's device) without re-validating them; a null mask still goes through the
        normal path (it is dropped when it holds no NULL)."""
        if nulls is not None or values.dtype == torch.bool:
            return cls(name, kind, values, nulls, dictionary)
        c = cls.__new__(cls)
        c.name, c.kind, c.values, c.nulls = name, kind, values, None
        c.dictionary = Dictionary() if kind.is_text and dictionary is None else dictionary
        c._zero_mask = None
        c._null_bits = None
        return c

    # -- reference-compatible surface ------------------------------------------------------
    @property
    def null_mask(self) -> torch.Tensor:
        """Bool mask (True = NULL); an all-False mask is materialised lazily on request."""
        if self.nulls is not None:
            return self.nulls
        if self._zero_mask is None:
            self._zero_mask = torch.zeros(len(self), dtype=torch.bool, device=self.values.device)
        return self._zero_mask

    @property
    def has_nulls(self) -> bool:
        return self.nulls is not None

    @property
    def device(self) -> torch.device:
        return self.values.device

    def __len__(self):
        return int(self.values.numel())

    def __repr__(self):
        return (f"Column({self.name!r}, {self.kind}, {self.values.dtype}, n={len(self)}, "
                f"nulls={'yes' if self.nulls is not None else 'no'}, device={self.device})")

    def take(self, indices) -> "Column":
        """Gather rows (device kernel ``esc_gather``); TEXT keeps the SAME dictionary object
        (reference ``storage.py:176-184``)."""
        from . import executor

        return executor.take_column(self, indices)

    def decode_value(self, i: int):
        """Python value of row ``i`` (None when NULL) — a host read, for tests and printing."""
        if self.nulls is not None and bool(self.nulls[i]):
            return None
        v = self.values[i].item()
        if self.kind.is_text:
            return self.dictionary.decode(int(v))
        if self.kind.name == DATE:
            return days_to_date(int(v))
        if self.kind.is_decimal:
            return format_decimal(int(v), self.kind.scale)
        return v

    def to_numpy(self) -> tuple[np.ndarray, np.ndarray]:
        """(values, null_mask) host copies in the reference's layout."""
        vals = self.values.cpu().numpy()
        mask = self.nulls.cpu().numpy() if self.nulls is not None else np.zeros(len(vals), bool)
        return vals, mask


@dataclass(frozen=True)
class ShardInfo:
    """Where a row-partitioned table's local rows sit in the global table.

    Rank ``rank`` of ``world`` holds global rows ``[offset, offset + counts[rank])``; ``counts``
    lists every rank's rows in rank order, so the ranks' slices concatenated in rank order are the
    global table in row order — the reference's chunk-order concatenation
    (``executor.py:500-504``).  ``group`` is the ``torch.distributed`` process group the ranks
    exchange counts over (None: the default group)."""

    rank: int
    world: int
    offset: int
    counts: tuple
    group: object = field(default=None, compare=False)

    @property
    def global_rows(self) -> int:
        return sum(self.counts)


class ColumnTable:
    """Immutable named relation of equal-length device columns (reference ``storage.py:206-244``).

    ``shard`` (multi-GPU extension): this object holds ONE rank's contiguous row range of a
    row-partitioned table; ``row_count`` is the local rows, :attr:`global_row_count` the table's."""

    def __init__(self, name: str, columns: Sequence[Column], is_temporary: bool = False,
                 shard: "ShardInfo | None" = None):
        columns = list(columns)
        if not columns:
            raise EmptySchema(f"table {name!r} must have at least one column")
        sizes = {len(c) for c in columns}
        if len(sizes) != 1:
            detail = ", ".join(f"{c.name}={len(c)}" for c in columns)
            raise LengthMismatch(f"table {name!r}: column lengths differ: {detail}")
        names = [c.name for c in columns]
        if len(set(names)) != len(names):
            raise StorageError(f"table {name!r}: duplicate column names")
        devices = {c.device for c in columns}
        if len(devices) != 1:
            raise StorageError(f"table {name!r}: columns live on different devices {devices}")
        self.name = name
        self.columns = columns
        self.row_count = sizes.pop()
        self.is_temporary = is_temporary
        self._by_name = {c.name: c for c in columns}
        if shard is not None and shard.counts[shard.rank] != self.row_count:
            raise LengthMismatch(f"table {name!r}: shard of rank {shard.rank} holds {self.row_count} rows, "
                                 f"its ShardInfo says {shard.counts[shard.rank]}")
        self.shard = shard

    @property
    def global_row_count(self) -> int:
        """Rows of the whole table (all ranks' shards); ``row_count`` when not sharded."""
        return self.shard.global_rows if self.shard is not None else self.row_count

    @classmethod
    def empty(cls, name: str, schema, device=None) -> "ColumnTable":
        if not schema:
            raise EmptySchema(f"table {name!r} must have at least one column")
        return cls(name, [Column(n, k, np.empty(0, dtype=_DEFAULT_DTYPE.get(k.name, np.int64)),
                                 device=device) for n, k in schema])

    @classmethod
    def from_arrays(cls, name: str, spec, device=None, is_temporary=False) -> "ColumnTable":
        """Build from ``[(col_name, kind, values[, null_mask[, dictionary]]), ...]``."""
        cols = []
        for item in spec:
            cname, kind, values = item[0], item[1], item[2]
            nulls = item[3] if len(item) > 3 else None
            dictionary = item[4] if len(item) > 4 else None
            cols.append(Column(cname, kind, values, nulls, dictionary, device=device))
        return cls(name, cols, is_temporary=is_temporary)

    @property
    def schema(self) -> list:
        return [(c.name, c.kind) for c in self.columns]

    @property
    def device(self) -> torch.device:
        return self.columns[0].device

    def column(self, name: str) -> Column:
        return self._by_name[name]

    def has_column(self, name: str) -> bool:
        return name in self._by_name

    def row(self, i: int) -> tuple:
        return tuple(c.decode_value(i) for c in self.columns)

    def nbytes(self) -> int:
        total = 0
        for c in self.columns:
            total += c.values.numel() * c.values.element_size()
            if c.nulls is not None:
                total += c.nulls.numel()
        return total


@dataclass(frozen=True)
class TempTableHandle:
    """Opaque handle of an optimizer temp table (reference ``storage.py:325-334``).

    For a sharded temp (multi-GPU) ``row_count`` is the GLOBAL row count — what the planner
    orders builds by — and every rank's handle has the same id (ranks plan in lockstep)."""

    id: int
    schema: tuple = field(compare=False)
    row_count: int = field(compare=False, default=0)

    def __str__(self):
        return f"temp#{self.id}"


class TempTableStore:
    """Live temp tables keyed by handle id; device buffers are released on drop/sweep
    (reference ``storage.py:337-375``)."""

    def __init__(self):
        self._next = 1
        self._tables: dict[int, ColumnTable] = {}

    def materialize(self, columns: Sequence[Column], shard: ShardInfo | None = None) -> TempTableHandle:
        """Register compacted columns as a temp.  ``shard``: they are this rank's slice of a
        row-partitioned temp (the slices of all ranks, in rank order, are the temp); the handle
        then carries the global row count."""
        tid = self._next
        self._next += 1
        table = ColumnTable(f"$temp{tid}", columns, is_temporary=True, shard=shard)
        self._tables[tid] = table
        return TempTableHandle(tid, tuple((c.name, c.kind) for c in table.columns), table.global_row_count)

    def resolve(self, handle: TempTableHandle) -> ColumnTable:
        try:
            return self._tables[handle.id]
        except KeyError:
            raise DeadHandle(f"{handle} is not live") from None

    def drop(self, handle: TempTableHandle):
        if self._tables.pop(handle.id, None) is None:
            raise DeadHandle(f"{handle} is not live")

    def is_live(self, handle: TempTableHandle) -> bool:
        return handle.id in self._tables

    def live_handles(self) -> list[int]:
        return sorted(self._tables)

    def sweep(self) -> int:
        n = len(self._tables)
        self._tables.clear()
        return n
