"""Hash joins over device-resident tables — the "next" rows f1/f2 of SURVEY §8(f).

Drop-in for the join half of the reference executor (``pkg/src/escdb/executor.py:253-531``) and
``optimizer.execute_plan`` (``optimizer.py:403-430``), with the same names, fields, statistics and
result order:

=======================  ================================================  ======================
name                     reference                                         device path
=======================  ================================================  ======================
``HashTableIndex``       ``executor.py:275-350`` (splitmix64, open          group build on device,
                         addressing, load 0.7, duplicate groups)            ``esc_hash_insert``
``probe_groups``         ``executor.py:327-346``                           ``esc_hash_probe``
``build_hash``           ``executor.py:353-358``                           K1 select + the above
``probe_joins``          ``executor.py:403-531``                           COUNT: ``esc_join_count``
                                                                            (one fused pass);
                                                                            rows: ``esc_expand``
``execute_plan``         ``optimizer.py:403-430``                          builds + probe_joins
=======================  ================================================  ======================

A build side is small (an ESC temp or a dimension): its rows come from the K1 scan, its keys are
grouped with a stable device sort, and its table is filled by ``esc_hash_insert``.  Group ids are
indices into the ascending unique keys exactly as in the reference, so ``probe_groups`` agrees
value for value.  The probe side is where the time goes (the fact table): a COUNT(*) plan runs as
ONE fused kernel over the probe table's key columns that never expands a tuple (see
``esc_join.cuh``); plans with a projection expand stage by stage on the device in the
reference's order (probe row, then each build's matches in group order).

There is no CPU fallback: every path needs the CUDA extension and device-resident tables.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import torch

from . import _native as N
from . import expr as ex
from . import executor
from .errors import ExecutionError
from .storage import Column, ColumnTable, TempTableHandle

LOAD_FACTOR = 0.7
_FLOAT_DTYPES = (torch.float32, torch.float64, torch.float16, torch.bfloat16)


def capacity_for(n: int) -> int:
    """Smallest power of two >= 8 with ``cap * 0.7 >= n`` (reference ``_capacity_for``)."""
    cap = 8
    while cap * LOAD_FACTOR < n:
        cap *= 2
    return cap


def _stream(dev):
    return executor._stream(dev)


def _as_device_keys(keys, dev) -> torch.Tensor:
    t = keys if isinstance(keys, torch.Tensor) else torch.as_tensor(keys)
    if t.dtype in _FLOAT_DTYPES or t.dtype == torch.bool:
        raise ExecutionError("hash join keys must be integer values")
    return t.to(device=dev).contiguous()


class HashTableIndex:
    """Open-addressed index from join-key value to build-row indices (reference
    ``executor.py:275-350``): slots hold ids of key groups; a group's row indices sit contiguously,
    ascending, in ``group_rows``.  All arrays are device tensors."""

    def __init__(self, table: ColumnTable, key: str, rows: torch.Tensor | None, _defer: bool = False):
        """``rows``: build-row ids (None = every row).  The grouping (stable sort by key, runs,
        offsets) is one ``esc_hash_build`` call; its statistics (distinct keys, key range,
        largest group) stay on the device until :meth:`_finish` reads them — ``build_indexes``
        reads every build of a plan at once."""
        self.table = table
        self.key = key
        col = table.column(key)
        if col.values.dtype in _FLOAT_DTYPES:
            raise ExecutionError(f"cannot hash-join on floating-point column {key!r}")
        dev = table.device
        if rows is not None:
            rows = rows.to(device=dev, dtype=torch.int64).contiguous()
        if col.nulls is not None and len(col):  # NULL keys never match: drop them first
            rows = torch.arange(len(col), device=dev) if rows is None else rows
            if rows.numel():
                rows = rows[~col.nulls[rows]].contiguous()
        n = len(col) if rows is None else int(rows.numel())
        self.n_entries = n
        lib = N.load_library()
        temp_bytes = C.c_size_t()
        N.check(lib.esc_hash_build_temp_bytes(n, C.byref(temp_bytes)), "esc_hash_build_temp_bytes")
        temp = torch.empty(max(temp_bytes.value, 1), dtype=torch.uint8, device=dev)
        self.group_rows = torch.empty(n, dtype=torch.int64, device=dev)
        self._uk = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        self._cnt = torch.empty(n + 1, dtype=torch.int64, device=dev)
        self._start = torch.empty(n + 1, dtype=torch.int64, device=dev)
        self._stats = torch.empty(4, dtype=torch.int64, device=dev)
        ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None and t.numel() else None  # noqa: E731
        N.check(lib.esc_hash_build(ptr(col.values), N.dtype_code(col.values), ptr(rows), n, ptr(self.group_rows),
                                   ptr(self._uk), ptr(self._cnt), ptr(self._start), ptr(self._stats), ptr(temp),
                                   temp_bytes.value, C.c_void_p(_stream(dev).cuda_stream)), "esc_hash_build")
        self._temp = temp  # alive until the queued kernels ran (freed in _finish, stream-ordered)
        if not _defer:
            self._finish(self._stats.tolist())

    def _finish(self, stats):
        """Second half of the build once (distinct, min, max, largest group) are on the host."""
        dev = self.table.device
        u, lo, hi, most = (int(x) for x in stats)
        self.key_range = (lo, hi, most) if u else None
        self.unique_keys = self._uk[:u]
        self.group_counts = self._cnt[:u]
        self.group_start = self._start[: u + 1]
        self._temp = self._stats = None
        self.capacity = capacity_for(u)
        self.slots = torch.empty(self.capacity, dtype=torch.int64, device=dev)
        lib = N.load_library()
        N.check(lib.esc_hash_insert(C.c_void_p(self.unique_keys.data_ptr()) if u else None, u,
                                    C.c_void_p(self.slots.data_ptr()), self.capacity,
                                    C.c_void_p(_stream(dev).cuda_stream)), "esc_hash_insert")

    @property
    def distinct_keys(self) -> int:
        return int(self.unique_keys.numel())

    def _probe(self, keys: torch.Tensor, nulls, rows, valid) -> torch.Tensor:
        dev = self.table.device
        n = int(rows.numel()) if rows is not None else int(keys.numel()) if valid is None else int(valid.numel())
        out = torch.empty(n, dtype=torch.int64, device=dev)
        if n == 0:
            return out
        lib = N.load_library()
        ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
        N.check(lib.esc_hash_probe(ptr(self.slots), self.capacity, ptr(self.unique_keys)
                                   if self.unique_keys.numel() else ptr(self.slots), ptr(keys),
                                   N.dtype_code(keys), ptr(nulls), ptr(rows), ptr(valid), n, ptr(out),
                                   C.c_void_p(_stream(dev).cuda_stream)), "esc_hash_probe")
        return out

    def probe_groups(self, keys, valid) -> torch.Tensor:
        """Group id per key (-1 when absent or the key slot is invalid)."""
        dev = self.table.device
        k = _as_device_keys(keys, dev)
        v = torch.as_tensor(valid).to(device=dev, dtype=torch.bool).contiguous()
        if k.numel() != v.numel():
            raise ExecutionError("keys and valid differ in length")
        if self.unique_keys.numel() == 0:
            return torch.full((k.numel(),), -1, dtype=torch.int64, device=dev)
        return self._probe(k, None, None, v.view(torch.uint8))

    def probe_column(self, col: Column, rows: torch.Tensor | None) -> torch.Tensor:
        """Group ids of ``col`` at ``rows`` (NULL keys miss) — the probe of one pipeline stage."""
        if col.values.dtype in _FLOAT_DTYPES:
            raise ExecutionError(f"cannot hash-join on floating-point column {col.name!r}")
        n = int(rows.numel()) if rows is not None else len(col)
        if self.unique_keys.numel() == 0 or n == 0:
            return torch.full((n,), -1, dtype=torch.int64, device=self.table.device)
        return self._probe(col.values, col.nulls.view(torch.uint8) if col.nulls is not None else None, rows, None)

    def lookup(self, key: int) -> torch.Tensor:
        """Build-row indices matching ``key`` (test/debug convenience)."""
        g = int(self.probe_groups(torch.tensor([int(key)], dtype=torch.int64), torch.ones(1, dtype=torch.bool))[0])
        if g < 0:
            return torch.empty(0, dtype=torch.int64, device=self.table.device)
        s, e = int(self.group_start[g]), int(self.group_start[g + 1])
        return self.group_rows[s:e]


def build_hash(table: ColumnTable, key: str, residual: ex.Expr | None = None) -> HashTableIndex:
    """Hash index over rows passing ``residual`` (NULL keys excluded) — reference
    ``executor.py:353-358``; the rows come from the K1 scan on the device."""
    return HashTableIndex(table, key, executor.eval_predicate(table, residual).indices)


def build_indexes(specs) -> list:
    """``build_hash`` for several (table, key, residual): every build's grouping is queued, then
    ONE host read of all their statistics finishes them (a plan's builds wait once together)."""
    idx = [HashTableIndex(t, k, executor.eval_predicate(t, r).indices, _defer=True) for t, k, r in specs]
    if idx:
        vals = torch.stack([i._stats for i in idx]).tolist()
        for i, v in zip(idx, vals):
            i._finish(v)
    return idx


@dataclass
class BuildStep:
    """One hash table plus the column (on the probe table or an earlier build) whose values
    probe it."""

    alias: str
    index: HashTableIndex
    probe_key: ex.ColumnRef


@dataclass
class ExecStats:
    build_cards: list = field(default_factory=list)
    build_distinct: list = field(default_factory=list)
    build_ms: list = field(default_factory=list)
    probe_out: list = field(default_factory=list)
    probe_in: int = 0
    result_rows: int = 0
    probe_ms: float = 0.0
    materialized_rows: int = 0

    @property
    def build_card_sum(self) -> int:
        return sum(self.build_cards)


# ------------------------------------------------------------------------------------------------
# COUNT pipeline: one fused pass
# ------------------------------------------------------------------------------------------------
# a key range is indexed directly (factor[key - min]) when that array is small: at most
# DENSE_MAX_BYTES, or no bigger than DENSE_VS_HASH x the hash table it replaces
DENSE_MAX_BYTES = 8 << 20
DENSE_VS_HASH = 4
DENSE_SPAN_MAX = 1 << 28


def _factor_array(index: HashTableIndex):
    """(dense_min, dense_len, tensor, bits) of the group sizes indexed by key - min, or None when
    the key range is too sparse for a direct array."""
    u = index.distinct_keys
    if u == 0:
        return None
    lo, hi, most = index.key_range  # read with the build's statistics (no extra wait)
    span = hi - lo + 1
    bits = 1 if most <= 1 else 8 if most < 256 else 16 if most < 65536 else 32 if most < (1 << 32) else 64
    nbytes = span * bits // 8
    hash_bytes = index.capacity * 8 + u * 16
    if span > DENSE_SPAN_MAX or nbytes > max(DENSE_MAX_BYTES, DENSE_VS_HASH * hash_bytes):
        return None
    dev = index.table.device
    # padded to 16 bytes (the probe kernels stage it with 16-byte copies); one native launch
    if most <= 1:
        bits, dt, n_el = 1, torch.int32, ((span + 31) // 32 + 3) // 4 * 4
    else:
        bits, dt = next((b, d) for b, d in ((8, torch.uint8), (16, torch.int16), (32, torch.int32), (64, torch.int64))
                        if most < (1 << b) or b == 64)
        pad = 16 * 8 // bits
        n_el = (span + pad - 1) // pad * pad
    arr = torch.empty(n_el, dtype=dt, device=dev)
    N.check(N.load_library().esc_factor_array(C.c_void_p(index.unique_keys.data_ptr()),
                                              C.c_void_p(index.group_counts.data_ptr()), u, lo, span, bits,
                                              C.c_void_p(arr.data_ptr()), arr.numel() * arr.element_size(),
                                              C.c_void_p(_stream(dev).cuda_stream)), "esc_factor_array")
    return lo, span, arr, bits


def _stage_weights(steps: list, probe_alias: str) -> dict:
    """weight[(t, s)] (device int64 per group of step t) for every stage s >= t: group size times
    the product of the weights, at stage s, of the later steps probed from step t's rows —
    the COUNT of a join tree folded bottom-up, per stage prefix."""
    S = len(steps)
    children = {t: [c for c in range(S) if steps[c].probe_key.table == steps[t].alias] for t in range(S)}
    out = {}
    for s in range(1, S + 1):
        for t in reversed(range(s)):
            idx = steps[t].index
            w = torch.ones(idx.n_entries, dtype=torch.int64, device=idx.table.device)
            for c in children[t]:
                if c >= s:
                    continue
                col = idx.table.column(steps[c].probe_key.name)
                g = steps[c].index.probe_column(col, idx.group_rows)
                wc = out[(c, s)]
                f = torch.where(g >= 0, wc[g.clamp(min=0)] if wc.numel() else torch.zeros_like(g),
                                torch.zeros_like(g))
                w = w * f
            cs = torch.zeros(idx.n_entries + 1, dtype=torch.int64, device=w.device)
            torch.cumsum(w, 0, out=cs[1:])
            out[(t, s)] = cs[idx.group_start[1:]] - cs[idx.group_start[:-1]]
    return out


def _count_pipeline(probe: ColumnTable, probe_alias: str, probe_pred, steps: list) -> list:
    """probe_out (S + 1 stage counts) of the pipeline, by ONE esc_join_count pass."""
    S = len(steps)
    if S > N.MAX_STEPS:
        raise ExecutionError(f"a probe pipeline supports at most {N.MAX_STEPS} build steps")
    keep = []
    lib = N.load_library()
    j = N.EscJoin()
    j.n_stages = S
    j.nrows = probe.row_count
    if probe_pred is not None:
        sel = executor.select(probe, probe_pred)
        keep.append(sel)
        j.bitmap = sel.buffers[0].data_ptr()
    probe_keyed = [t for t in range(S) if steps[t].probe_key.table == probe_alias]
    star = len(probe_keyed) == S
    j.star = 1 if star else 0
    weights = {} if star else _stage_weights(steps, probe_alias)
    for k, t in enumerate(probe_keyed):
        st = steps[t]
        col = probe.column(st.probe_key.name)
        if col.values.dtype in _FLOAT_DTYPES:
            raise ExecutionError(f"cannot hash-join on floating-point column {col.name!r}")
        d = j.steps[k]
        j.stage_of[k] = t + 1
        d.key_data = col.values.data_ptr() if len(col) else None
        d.key_nulls = col.nulls.data_ptr() if col.nulls is not None and len(col) else None
        d.key_dtype = N.dtype_code(col.values)
        idx = st.index
        fa = _factor_array(idx) if star else None
        if fa is not None:
            lo, span, arr, bits = fa
            keep.append(arr)
            d.mode = N.JOIN_DENSE
            d.dense_min, d.dense_len, d.factor, d.factor_bits = lo, span, arr.data_ptr(), bits
            continue
        if star:  # sparse key range: a (key, factor) pair table at load <= 1/4, one load per probe
            cap = 16
            while cap < 4 * max(idx.distinct_keys, 1):
                cap *= 2
            pairs = torch.empty((int(lib.esc_pairs_bytes(cap)) + 7) // 8, dtype=torch.int64, device=probe.device)
            keep.append(pairs)
            N.check(lib.esc_pairs_build(C.c_void_p(idx.unique_keys.data_ptr()) if idx.distinct_keys else None,
                                        C.c_void_p(idx.group_counts.data_ptr()) if idx.distinct_keys else None,
                                        idx.distinct_keys, C.c_void_p(pairs.data_ptr()), cap,
                                        C.c_void_p(_stream(probe.device).cuda_stream)), "esc_pairs_build")
            d.mode = N.JOIN_PAIRS
            d.slots, d.capacity = pairs.data_ptr(), cap
            continue
        d.mode = N.JOIN_HASH
        d.slots, d.capacity = idx.slots.data_ptr(), idx.capacity
        uk = idx.unique_keys if idx.unique_keys.numel() else idx.slots
        d.unique_keys = uk.data_ptr()
        for s in range(t + 1, S + 1):
            w = idx.group_counts if star else weights[(t, s)]
            if w.numel() == 0:
                w = torch.zeros(1, dtype=torch.int64, device=probe.device)
            keep.append(w)
            d.weight[s] = w.data_ptr()
    j.n_steps = len(probe_keyed)
    out = torch.empty(S + 1, dtype=torch.int64, device=probe.device)
    stream = _stream(probe.device)
    ev0 = executor._ev_start(stream)
    N.check(lib.esc_join_count(C.byref(j), C.c_void_p(out.data_ptr()), C.c_void_p(stream.cuda_stream)),
            "esc_join_count")
    executor._ev_end(stream, ev0, "join")
    counts = [int(x) for x in out.cpu().tolist()]
    del keep
    return counts


# ------------------------------------------------------------------------------------------------
# row pipeline: device expansion in the reference's order
# ------------------------------------------------------------------------------------------------
def _expand_pipeline(probe: ColumnTable, probe_alias: str, probe_pred, steps: list):
    prow = executor.eval_predicate(probe, probe_pred).to_indices()
    stage_out = [int(prow.numel())]
    brows: dict = {}
    tables = {probe_alias: probe}
    lib = N.load_library()
    stream = _stream(probe.device)
    for step in steps:
        src = step.probe_key.table
        rows_src = prow if src == probe_alias else brows[src]
        col = tables[src].column(step.probe_key.name)
        idx = step.index
        groups = idx.probe_column(col, rows_src)
        cnt = torch.where(groups >= 0, idx.group_counts[groups.clamp(min=0)] if idx.group_counts.numel()
                          else torch.zeros_like(groups), torch.zeros_like(groups))
        ends = torch.cumsum(cnt, 0)
        total = int(ends[-1]) if ends.numel() else 0
        out_tuple = torch.empty(total, dtype=torch.int64, device=probe.device)
        out_row = torch.empty(total, dtype=torch.int64, device=probe.device)
        if total:
            offsets = ends - cnt
            N.check(lib.esc_expand(C.c_void_p(groups.data_ptr()), C.c_void_p(offsets.data_ptr()),
                                   int(groups.numel()), C.c_void_p(idx.group_start.data_ptr()),
                                   C.c_void_p(idx.group_rows.data_ptr()), C.c_void_p(out_tuple.data_ptr()),
                                   C.c_void_p(out_row.data_ptr()), C.c_void_p(stream.cuda_stream)), "esc_expand")
        prow = prow[out_tuple]
        for a in brows:
            brows[a] = brows[a][out_tuple]
        brows[step.alias] = out_row
        tables[step.alias] = idx.table
        stage_out.append(total)
    return prow, brows, tables, stage_out


def probe_joins(probe: ColumnTable, probe_alias: str, probe_pred, steps: list, projection,
                workers: int = 1):
    """Stream the probe relation through every hash table in order (reference
    ``executor.py:478-531``).  ``projection`` is a tuple of resolved column refs; None means
    count only (no output materialization).  Output row order is the probe row order, then each
    build's matches in group order; ``workers`` is accepted for API parity (one device pass)."""
    del workers
    stats = ExecStats()
    for step in steps:
        stats.build_cards.append(step.index.n_entries)
        stats.build_distinct.append(step.index.distinct_keys)
    stats.probe_in = probe.row_count
    t0 = time.perf_counter()
    if projection is None:
        stats.probe_out = _count_pipeline(probe, probe_alias, probe_pred, steps)
        stats.result_rows = stats.probe_out[-1]
        stats.probe_ms = (time.perf_counter() - t0) * 1000.0
        return None, stats
    prow, brows, tables, stage_out = _expand_pipeline(probe, probe_alias, probe_pred, steps)
    stats.probe_out = stage_out
    stats.result_rows = int(prow.numel())
    stats.probe_ms = (time.perf_counter() - t0) * 1000.0
    rows_of = {probe_alias: prow, **brows}
    out_columns, used = [], set()
    for ref in projection:
        col = executor.take_column(tables[ref.table].column(ref.name), rows_of[ref.table])
        name = ref.name if ref.name not in used else f"{ref.table}.{ref.name}"
        used.add(name)
        out_columns.append(Column(name, col.kind, col.values, col.nulls, col.dictionary))
    result = ColumnTable("result", out_columns, is_temporary=True)
    stats.materialized_rows = result.row_count
    return result, stats


def execute_plan(plan_, catalog, workers: int = 1):
    """Run the pipeline of a PhysicalPlan; returns (result table or None, result count, stats)
    — reference ``optimizer.py:403-430``.  Pushed-down builds read their ESC temps in place."""
    probe_table = catalog.table(plan_.probe_source)
    specs = []
    for b in plan_.builds:
        table = catalog.resolve_temp(b.source) if isinstance(b.source, TempTableHandle) else catalog.table(b.source)
        specs.append((table, b.build_key.name, b.residual))
    t0 = time.perf_counter()
    indexes = build_indexes(specs)  # the builds share one host wait; their time is split evenly
    share = (time.perf_counter() - t0) * 1000.0 / max(len(specs), 1)
    build_ms = [share] * len(specs)
    steps = [BuildStep(b.alias, index, b.probe_key) for b, index in zip(plan_.builds, indexes)]
    result, stats = probe_joins(probe_table, plan_.probe_alias, plan_.probe_pred, steps, plan_.projection,
                                workers=workers)
    stats.build_ms = build_ms
    stats.build_cards = [b.input_rows for b in plan_.builds]
    return result, stats.result_rows, stats
