"""K3: row-range partitioning of tables across the GPUs of one box, the count/offset exchange,
sharded temps, and the planner / join pipeline over sharded tables.

The reference's only parallelism is a row-range split (``np.linspace`` bounds,
``executor.py:485-489``) whose fragments are concatenated in chunk order (``executor.py:500-504``).
Here one process drives one GPU (``torch.distributed``; NCCL over NVLink/NVSwitch on a GPU box,
gloo in the CPU tests); rank ``r`` holds rows ``[floor(r*N/G), floor((r+1)*N/G))`` of a sharded
table in its HBM (a :class:`~.storage.ColumnTable` whose ``shard`` is a
:class:`~.storage.ShardInfo`).

An ESC sub-query over a sharded table runs the same prepared device step as on one GPU, on the
rank's shard, with ONE exchange inserted between the scan and the compaction
(:class:`_CountExchange`): the scan leaves the local count in a device word, an ``all_gather`` of
that word (stream-ordered — no host round trip) gives every rank every rank's count, and
``esc_count_gate`` folds them on the device into the global count, this rank's exclusive offset
and the gate the queued compaction reads, so a table that does not qualify GLOBALLY is not
compacted anywhere.  The host waits once per planning batch.  The sharded temp is the ranks'
compacted slices; concatenated in rank order they ARE the reference's temp, row for row.  No
table data crosses NVLink for the ESC decision.

Joins over sharded tables (:func:`execute_plan_sharded`): each build's filtered input is gathered
to every rank (a broadcast hash join — builds are the small side), each rank probes its own rows
of the probe table, and the per-stage counts are summed with one ``all_reduce``; projected rows
stay sharded in probe order.
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass
from fractions import Fraction

import torch
import torch.distributed as dist

from . import _native as N
from . import executor
from .compiler import compile_predicate
from .errors import EscdbError, ExecutionError, NoPredicate
from .storage import Column, ColumnTable, ShardInfo, TempTableHandle

_NO_FAIL = (1 << 64) - 1


# ------------------------------------------------------------------------------------------------
# partitioning
# ------------------------------------------------------------------------------------------------
def shard_bounds(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous row range of every rank (balanced to within one row)."""
    return [((r * n) // world, ((r + 1) * n) // world) for r in range(world)]


def exclusive_offsets(counts) -> list[int]:
    out, acc = [], 0
    for c in counts:
        out.append(acc)
        acc += int(c)
    return out


def shard_info(n: int, rank: int, world: int, group=None) -> ShardInfo:
    """The ShardInfo of rank ``rank``'s row range of an ``n``-row table."""
    b = shard_bounds(n, world)
    return ShardInfo(rank, world, b[rank][0], tuple(hi - lo for lo, hi in b), group)


def shard_table(table: ColumnTable, rank: int, world: int, group=None) -> ColumnTable:
    """Rank ``rank``'s shard of a whole table (column views of its row range; tests and loaders
    that hold the whole table — a real deployment uploads only its shard)."""
    info = shard_info(table.row_count, rank, world, group)
    lo, hi = info.offset, info.offset + info.counts[rank]
    cols = [Column.device_column(c.name, c.kind, c.values[lo:hi], c.nulls[lo:hi] if c.nulls is not None else None,
                                 c.dictionary) for c in table.columns]
    return ColumnTable(table.name, cols, table.is_temporary, shard=info)


# ------------------------------------------------------------------------------------------------
# collectives (one process per GPU; NCCL on a GPU box, gloo in the CPU tests)
# ------------------------------------------------------------------------------------------------
def _backend(group=None) -> str:
    return dist.get_backend(group)


def _comm_device(group=None) -> torch.device:
    if _backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def all_gather_ints(values: list[int], group=None) -> list[list[int]]:
    """all_gather of an int64 vector (same length on every rank) -> one list per rank."""
    world = dist.get_world_size(group)
    dev = _comm_device(group)
    k = len(values)
    mine = torch.tensor(values if k else [0], dtype=torch.int64, device=dev)
    every = torch.empty(world * max(k, 1), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(every, mine, group=group)
    flat = every.cpu().tolist()
    m = max(k, 1)
    return [flat[r * m: r * m + k] for r in range(world)]


def exchange_counts(local: int, group=None) -> tuple[int, list[int], list[int]]:
    """all_gather of one int64 per rank -> (global count, per-rank counts, exclusive offsets)."""
    counts = [v[0] for v in all_gather_ints([int(local)], group)]
    return sum(counts), counts, exclusive_offsets(counts)


def allreduce_min(values: list[int], group=None) -> list[int]:
    """Element-wise minimum over ranks of unsigned 64-bit words (failure rows)."""
    if not values:
        return []
    dev = _comm_device(group)
    # map u64 -> i64 order-preservingly for the signed reduction
    t = torch.tensor([v - (1 << 63) for v in values], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return [int(v) + (1 << 63) for v in t.cpu().tolist()]


def allreduce_sum(values: list[int], group=None) -> list[int]:
    if not values:
        return []
    t = torch.tensor(values, dtype=torch.int64, device=_comm_device(group))
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return [int(v) for v in t.cpu().tolist()]


def _device_all_gather(out: torch.Tensor, inp: torch.Tensor, group=None):
    """all_gather of device tensors, stream-ordered.  NCCL reads and writes device memory on
    the stream; other backends (gloo: the CPU tests that run several ranks on one GPU) stage
    through host memory — the same exchange, a different transport."""
    if _backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp, group=group)
        return
    host = torch.empty(out.numel(), dtype=out.dtype)
    dist.all_gather_into_tensor(host, inp.cpu(), group=group)
    out.copy_(host.to(out.device))


def _ragged_all_gather(t: torch.Tensor, counts: list[int], group=None) -> torch.Tensor:
    """Rank-order concatenation of every rank's ``t`` (``counts[r]`` elements on rank r)."""
    world = len(counts)
    m = max(counts) if counts else 0
    if m == 0:
        return t.new_empty(0)
    dev = t.device if _backend(group) == "nccl" else torch.device("cpu")
    padded = torch.zeros(m, dtype=t.dtype, device=dev)
    padded[: t.numel()] = t.to(dev)
    every = torch.empty(world * m, dtype=t.dtype, device=dev)
    dist.all_gather_into_tensor(every, padded, group=group)
    pieces = [every[r * m: r * m + counts[r]] for r in range(world)]
    return torch.cat(pieces).to(t.device)


# ------------------------------------------------------------------------------------------------
# the sharded ESC step
# ------------------------------------------------------------------------------------------------
class _CountExchange:
    """``between`` of a queued step (executor.launch_step): all_gather of the ranks' device
    counts, then ``esc_count_gate`` -> [counts | global, offset, gate] in the plan's gate buffer,
    copied to pinned host memory behind it (read after the one host wait)."""

    def __init__(self, shard: ShardInfo, gcap: int):
        self.shard = shard
        self.gcap = gcap
        self.host = None

    def __call__(self, plan, stream):
        sh = self.shard
        dev = plan.sel.table.device
        dbuf, hbuf = executor.gate_buffers(plan, dev, sh.world)
        ws = N.workspace(dev, stream)
        _device_all_gather(dbuf[: sh.world], ws.dcount, sh.group)
        N.check(N.load_library().esc_count_gate(C.c_void_p(dbuf.data_ptr()), sh.world, sh.rank, self.gcap,
                                                C.c_void_p(dbuf.data_ptr() + 8 * sh.world),
                                                C.c_void_p(stream.cuda_stream)), "esc_count_gate")
        hbuf.copy_(dbuf, non_blocking=True)
        self.host = hbuf

    def after(self, plan, stream):
        """Ungated variant: the step ran as on one GPU (its compaction checked the LOCAL count
        against the local capacity); the counts are gathered behind it for the host."""
        sh = self.shard
        dbuf, hbuf = executor.gate_buffers(plan, plan.sel.table.device, sh.world)
        _device_all_gather(dbuf[: sh.world], N.workspace(plan.sel.table.device, stream).dcount, sh.group)
        hbuf.copy_(dbuf, non_blocking=True)
        self.host = hbuf

    def counts(self) -> list[int]:
        return [int(x) for x in self.host[: self.shard.world].tolist()]


@dataclass
class _Launched:
    alias: str
    table: ColumnTable
    predicate: object
    needed: list
    rc: int            # global rows
    fused: bool
    gcap: int          # global capacity: floor(max_selectivity * global rows)
    cap: int           # local capacity
    ps: object = None  # executor.PendingStep
    exchange: _CountExchange | None = None
    sync_sel: object = None   # (count, fails, Selection) of the synchronous large-output path


# Where the count exchange sits in the sharded step.  Default (ungated): the step runs as on one
# GPU — scan + compaction in one graph with the PDL overlap, the compaction testing the LOCAL
# count against the local capacity — and the all_gather of the counts is queued behind it; the
# host decides on the global count.  A rank whose table does not qualify globally may have
# compacted for nothing (bounded by its capacity).  Gated (ESC_MG_GATED=1): all_gather +
# esc_count_gate between the scan and the compaction, which then tests the GLOBAL count; it
# measured 5 us slower at the 8-GPU shard size on one GPU, and it puts the compaction after
# the cross-rank exchange (the slowest rank's scan) instead of before it.
GATED = os.environ.get("ESC_MG_GATED", "0") == "1"


def _launch(item: _Launched, slot: int):
    t = item.table
    n = t.row_count
    if item.fused and n > executor.ONEPASS_MAX_ROWS:
        row_bytes = sum(t.column(c).values.element_size() + (1 if t.column(c).nulls is not None else 0)
                        for c in item.needed)
        if not (0 < item.cap and item.cap * max(row_bytes, 1) <= executor.SPECULATE_BYTES):
            # outputs too large to queue speculatively: record the selection and wait (no local
            # UDF-error check here — the replay runs on GLOBAL failure rows once all ranks are in)
            cp = compile_predicate(t, item.predicate)
            count, fails, sel = executor.launch_select(cp, t, None, n, capture=item.needed)
            item.sync_sel = (count, fails, sel, cp)
            return
        item.exchange = _CountExchange(t.shard, item.gcap)
    gated = item.exchange is not None and GATED
    item.ps = executor.launch_step(t, item.predicate, item.needed, item.cap, materialize=item.fused, slot=slot,
                                   between=item.exchange if gated else None)
    if item.exchange is not None and item.ps.kind != "queued":
        item.exchange = None
    if item.exchange is not None and not gated:
        item.exchange.after(item.ps.plan, executor._stream(t.device))


def _global_replay(table: ColumnTable, cp, local_fails: list, n_global: int):
    """UDF error semantics over the GLOBAL table: first failing row = min over ranks (global row
    ids), short-circuit decisions from global prefix counts (every rank walks the same tree and
    issues the same collectives in the same order)."""
    sh = table.shard
    shifted = [(((f >> 3) + sh.offset) << 3) | (f & 7) if f != _NO_FAIL else _NO_FAIL for f in local_fails]
    fails = allreduce_min(shifted, sh.group)
    if not cp.unbound and all(f == _NO_FAIL for f in fails):
        return

    def global_count(sub):
        c, _ = executor.launch_count(compile_predicate(table, sub), table, None, table.row_count)
        return exchange_counts(c, sh.group)[0]

    executor.raise_udf_errors(table, cp, fails, None, n_global, count_fn=global_count)


def _finish(item: _Launched):
    """After the host wait: (local count, per-rank counts, local columns or None)."""
    t = item.table
    sh = t.shard
    if item.sync_sel is not None:
        count, fails, sel, cp = item.sync_sel
        if cp.unbound or cp.may_fail:
            _global_replay(t, cp, fails, item.rc)
        counts = [v[0] for v in all_gather_ints([count], sh.group)]
        cols = executor.materialize_selection(sel, item.needed) if sum(counts) <= item.gcap else None
        return count, counts, cols
    ps = item.ps
    if ps.kind == "done":  # (not reached for sharded tables: handled by sync_sel)
        raise ExecutionError("internal: unexpected synchronous step")
    ws = N.workspace(t.device, executor._stream(t.device))
    count, fails = ws.read_result(ps.cp.n_udfs, ps.slot)
    if ps.cp.unbound or ps.cp.may_fail:
        _global_replay(t, ps.cp, fails, item.rc)
    if item.exchange is not None:
        counts = item.exchange.counts()
    else:
        counts = [v[0] for v in all_gather_ints([count], sh.group)]
    if ps.kind == "count":
        return count, counts, None
    if sum(counts) <= item.gcap:
        # global count within the global capacity => local count <= min(gcap, local rows) = cap
        return count, counts, executor._take_outputs(ps, ws, count)
    executor._release(ps, ws)
    return count, counts, None


def esc_batch(catalog, prepared: list, config, register: bool = True) -> list:
    """ESC steps of several SHARDED tables (``prepared`` as optimizer.esc_subqueries builds it:
    (alias, table, predicate, needed, global rows, fused, global capacity)) — every step queued
    (scan, device count exchange, gated compaction), ONE host wait, then results in item order;
    qualifying temps are registered as sharded temps (this rank's slice + its global offset).
    Every rank must call this with the same items in the same order."""
    from .optimizer import EscDecision, decide_pushdown

    t0 = time.perf_counter()
    items, launch_error = [], None
    for i, (alias, base, predicate, needed, rc, fused, gcap) in enumerate(prepared):
        it = _Launched(alias, base, predicate, list(needed), rc, fused, gcap, max(0, min(gcap, base.row_count)))
        try:
            _launch(it, i + 1)
        except EscdbError as exc:
            launch_error = (ExecutionError(f"count sub-query on {alias!r} failed: {exc}"), exc)
            break
        items.append(it)
    for dev in {it.table.device for it in items}:
        executor._stream(dev).synchronize()
    share = (time.perf_counter() - t0) * 1000.0 / max(len(prepared), 1)
    decisions = []
    for it in items:
        t1 = time.perf_counter()
        try:
            local, counts, cols = _finish(it)
        except EscdbError as exc:
            raise ExecutionError(f"count sub-query on {it.alias!r} failed: {exc}") from exc
        sub_ms = share + (time.perf_counter() - t1) * 1000.0
        total = sum(counts)
        qualified = decide_pushdown(it.rc, total, config)
        temp, mat_ms = None, 0.0
        if qualified and config.materialize:
            if cols is None:
                raise ExecutionError(f"internal: qualified table {it.alias!r} overflowed its temp buffer")
            if register:
                t2 = time.perf_counter()
                sh = it.table.shard
                temp = catalog.materialize_temp(cols, ShardInfo(sh.rank, sh.world, exclusive_offsets(counts)[sh.rank],
                                                                tuple(counts), sh.group))
                mat_ms = (time.perf_counter() - t2) * 1000.0
        d = EscDecision(it.alias, it.predicate, total, it.rc, Fraction(total, it.rc) if it.rc else Fraction(0),
                        qualified, temp is not None, temp, sub_ms, mat_ms)
        d.local_count, d.counts = local, counts
        d.columns = cols if qualified and config.materialize else None
        decisions.append(d)
    if launch_error is not None:
        raise launch_error[0] from launch_error[1]
    return decisions


# ------------------------------------------------------------------------------------------------
# single-table API (kept from the first multi-GPU cut: bench and tests call it directly)
# ------------------------------------------------------------------------------------------------
@dataclass
class ShardedTable:
    """One rank's slice of a row-partitioned table (``local`` holds rows ``row_begin`` ..
    ``row_begin + local.row_count`` of ``global_rows``, the balanced split of shard_bounds)."""

    name: str
    local: ColumnTable
    global_rows: int
    row_begin: int
    rank: int
    world: int
    group: object = None

    @property
    def row_end(self) -> int:
        return self.row_begin + self.local.row_count

    def table(self) -> ColumnTable:
        """The shard as a ColumnTable carrying its ShardInfo (cached)."""
        t = getattr(self, "_table", None)
        if t is None:
            info = shard_info(self.global_rows, self.rank, self.world, self.group)
            if info.offset != self.row_begin or info.counts[self.rank] != self.local.row_count:
                raise ValueError(f"shard of rank {self.rank} is not the balanced row range of {self.global_rows} rows")
            t = ColumnTable(self.local.name, self.local.columns, self.local.is_temporary, shard=info)
            self._table = t
        return t


@dataclass
class ShardedDecision:
    table: str
    exact_count: int           # global
    row_count: int             # global
    selectivity: Fraction
    qualified: bool
    local_count: int
    offset: int                # global position of this rank's first compacted row
    counts: list               # per-rank counts
    columns: list | None       # this rank's compacted slice (None when not materialized)


def sharded_esc_subquery(st: ShardedTable, predicate, needed, config, group=None) -> ShardedDecision:
    """The ESC step of one sharded table: the scan on every rank's shard, one device count
    exchange, the gated compaction, one host wait.  The slice is returned, not registered."""
    from .optimizer import _ratio, _trivially_true

    if predicate is None or _trivially_true(predicate):
        raise NoPredicate(f"table {st.name!r} has no filtering predicate")
    if group is not None and st.group is None:
        st.group = group
    t = st.table()
    rc = st.global_rows
    fused = config.materialize and rc > 0 and rc >= config.min_table_size
    num, den = _ratio(config.max_selectivity)
    gcap = (num * rc) // den if fused else 0
    (d,) = esc_batch(None, [(st.name, t, predicate, list(needed), rc, fused, gcap)], config, register=False)
    return ShardedDecision(st.name, d.exact_count, rc, d.selectivity, d.qualified, d.local_count,
                           exclusive_offsets(d.counts)[st.rank], d.counts, d.columns)


# ------------------------------------------------------------------------------------------------
# gathering sharded data (builds of a join, tests)
# ------------------------------------------------------------------------------------------------
def gather_columns(cols: list, counts: list, group=None) -> list[Column]:
    """Every rank gets the rank-order concatenation of all ranks' slices of ``cols``."""
    out = []
    for c in cols:
        vals = _ragged_all_gather(c.values, counts, group)
        nulls = None
        if any(allreduce_sum([1 if c.nulls is not None else 0], group)):
            mine = c.nulls if c.nulls is not None else torch.zeros(len(c), dtype=torch.bool, device=c.device)
            nulls = _ragged_all_gather(mine.to(torch.uint8), counts, group).to(torch.bool)
        out.append(Column(c.name, c.kind, vals, nulls, c.dictionary, device=c.device))
    return out


def gather_table(table: ColumnTable, columns=None) -> ColumnTable:
    """The whole table (``columns`` of it) replicated on every rank, rows in global order."""
    sh = table.shard
    names = [c.name for c in table.columns] if columns is None else list(columns)
    cols = gather_columns([table.column(n) for n in names], list(sh.counts), sh.group)
    return ColumnTable(table.name, cols, table.is_temporary)


def gather_to_rank0(cols: list, counts: list, group=None) -> list | None:
    """The global, order-preserving temp on rank 0 (rank-order concatenation of the slices) —
    used by tests; the planner keeps temps sharded."""
    rank = dist.get_rank(group)
    out = [_ragged_all_gather(c.values, counts, group) for c in cols]
    return out if rank == 0 else None


# ------------------------------------------------------------------------------------------------
# joins over sharded tables: broadcast builds, sharded probe
# ------------------------------------------------------------------------------------------------
def execute_plan_sharded(plan_, catalog, workers: int = 1):
    """``join.execute_plan`` when tables are sharded: every build's filtered input (its ESC temp
    slices, or the base rows passing the residual) is gathered to every rank in global row order
    — so group ids and group row order are the reference's — each rank probes its own rows of the
    probe table, and the stage counts are summed over ranks (one all_reduce).  A projection's rows
    stay sharded: rank-order concatenation is the probe order.  Returns (local result table or
    None, GLOBAL result count, stats with global counts)."""
    from . import join

    probe_table = catalog.table(plan_.probe_source)
    group = probe_table.shard.group if probe_table.shard is not None else None
    needed = _build_columns(plan_)
    specs = []
    for b in plan_.builds:
        src = catalog.resolve_temp(b.source) if isinstance(b.source, TempTableHandle) else catalog.table(b.source)
        keep = [c.name for c in src.columns if c.name in needed[b.alias]]
        if src.shard is not None:
            if b.residual is not None:
                rows = executor.eval_predicate(src, b.residual).indices
                local = ColumnTable(src.name, [src.column(c).take(rows) for c in keep])
                counts = [v[0] for v in all_gather_ints([local.row_count], src.shard.group)]
                src = ColumnTable(src.name, gather_columns(local.columns, counts, src.shard.group))
            else:
                src = gather_table(src, keep)
            specs.append((src, b.build_key.name, None))
        else:
            specs.append((src, b.build_key.name, b.residual))
    t0 = time.perf_counter()
    indexes = join.build_indexes(specs)
    share = (time.perf_counter() - t0) * 1000.0 / max(len(specs), 1)
    steps = [join.BuildStep(b.alias, index, b.probe_key) for b, index in zip(plan_.builds, indexes)]
    result, stats = join.probe_joins(probe_table, plan_.probe_alias, plan_.probe_pred, steps, plan_.projection,
                                     workers=workers)
    if probe_table.shard is not None:
        total = allreduce_sum([*stats.probe_out, stats.materialized_rows], group)
        stats.probe_out, stats.materialized_rows = total[:-1], total[-1]
        stats.probe_in = probe_table.global_row_count
        stats.result_rows = stats.probe_out[-1] if stats.probe_out else stats.probe_in
        if result is not None:
            counts = [v[0] for v in all_gather_ints([result.row_count], group)]
            sh = probe_table.shard
            result = ColumnTable(result.name, result.columns, True,
                                 shard=ShardInfo(sh.rank, sh.world, exclusive_offsets(counts)[sh.rank],
                                                 tuple(counts), group))
            stats.result_rows = sum(counts)
    stats.build_ms = [share] * len(specs)
    stats.build_cards = [b.input_rows for b in plan_.builds]
    return result, stats.result_rows, stats


def _build_columns(plan_) -> dict:
    """Per build alias: the columns a replicated build needs (its key, the keys later steps probe
    with, and its projected columns)."""
    want = {b.alias: {b.build_key.name} for b in plan_.builds}
    for b in plan_.builds:
        if b.probe_key.table in want:
            want[b.probe_key.table].add(b.probe_key.name)
    for ref in plan_.projection or ():
        if ref.table in want:
            want[ref.table].add(ref.name)
    return want


def is_sharded(table: ColumnTable) -> bool:
    return getattr(table, "shard", None) is not None

