"""K3: row-range partitioning of a table across the GPUs of one box + the count/offset exchange.

The reference's only parallelism is a row-range split (``np.linspace`` bounds,
``executor.py:485-489``) whose fragments are concatenated in chunk order (``executor.py:500-504``).
Here one process drives one GPU (``torch.distributed``, NCCL over NVLink/NVSwitch); rank ``r``
holds rows ``[floor(r*N/G), floor((r+1)*N/G))`` of every table resident in its HBM.  An ESC
sub-query runs the fused scan/count/compaction kernel on each rank's shard, then a single
``all_gather`` of one int64 per rank yields the global count (for the push-down decision) and
the exclusive prefix offsets that place each rank's compacted slice in the global, order-
preserving result: the slices concatenated in rank order ARE the reference's row order.  No
table data crosses NVLink; the sharded temp stays where it was produced.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction

import torch
import torch.distributed as dist

from . import executor
from .compiler import compile_predicate
from .errors import EscdbError, ExecutionError, NoPredicate
from .optimizer import EscConfig, _trivially_true, decide_pushdown
from .storage import Column, ColumnTable

_NO_FAIL = (1 << 64) - 1


def shard_bounds(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous row range of every rank (balanced to within one row)."""
    return [((r * n) // world, ((r + 1) * n) // world) for r in range(world)]


def exclusive_offsets(counts) -> list[int]:
    out, acc = [], 0
    for c in counts:
        out.append(acc)
        acc += int(c)
    return out


def _comm_device(group=None) -> torch.device:
    backend = dist.get_backend(group)
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def exchange_counts(local: int, group=None) -> tuple[int, list[int], list[int]]:
    """all_gather of one int64 per rank -> (global count, per-rank counts, exclusive offsets)."""
    world = dist.get_world_size(group)
    dev = _comm_device(group)
    mine = torch.tensor([int(local)], dtype=torch.int64, device=dev)
    every = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(every, mine, group=group)
    counts = [int(x) for x in every.cpu().tolist()]
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


@dataclass
class ShardedTable:
    """One rank's slice of a row-partitioned table."""

    name: str
    local: ColumnTable
    global_rows: int
    row_begin: int
    rank: int
    world: int

    @property
    def row_end(self) -> int:
        return self.row_begin + self.local.row_count


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


def _global_replay(st: ShardedTable, cp, local_fails: list, group):
    """UDF error semantics over the GLOBAL table: first failing row = min over ranks (global row
    ids), short-circuit decisions from global prefix counts (all ranks walk the same tree)."""
    shifted = [(((f >> 3) + st.row_begin) << 3) | (f & 7) if f != _NO_FAIL else _NO_FAIL for f in local_fails]
    fails = allreduce_min(shifted, group)
    any_unbound = bool(cp.unbound)
    if not any_unbound and all(f == _NO_FAIL for f in fails):
        return

    class _GlobalCount:
        def __call__(self, sub):
            c, _ = executor.launch_count(compile_predicate(st.local, sub), st.local, None, st.local.row_count)
            total, _, _ = exchange_counts(c, group)
            return total

    executor.raise_udf_errors(st.local, cp, fails, None, st.global_rows, count_fn=_GlobalCount())


def _queued_sharded(st: ShardedTable, cp, needed, gcap: int, group):
    """Device-resident sharded ESC step, one host wait: K1 select writes the local count to the
    device; an NCCL all_gather of that word (stream-ordered, no host round trip) gives every rank
    the per-rank counts; a device flag = (global count <= global capacity) gates the compaction
    queued behind it.  Returns (local count, fails, per-rank counts, columns or None)."""
    import ctypes as C

    from . import _native as N

    lib = N.load_library()
    table = st.local
    n = table.row_count
    stream = executor._stream(table.device)
    ws = N.workspace(table.device, stream)
    ws_ptr, ws_bytes = ws.ensure(n, stream.cuda_stream)
    proj = [table.column(c) for c in needed]
    cap = min(gcap, n)
    plan = executor._step_plan(cp, table, proj, cap, ws)
    sp = C.c_void_p(stream.cuda_stream)
    res = C.c_void_p(ws.result_ptr(1))
    N.check(lib.esc_scan_select(C.byref(cp.program), cp.column_array(), cp.ncols, n, None, C.byref(plan.sel.desc),
                                res, C.c_void_p(ws_ptr), C.c_size_t(ws_bytes), sp), "esc_scan_select")
    every = torch.empty(dist.get_world_size(group), dtype=torch.int64, device=table.device)
    dist.all_gather_into_tensor(every, ws.dcount, group=group)
    if not hasattr(ws, "dflag"):
        ws.dflag = torch.zeros(1, dtype=torch.int64, device=table.device)
    # compaction gate: 0 (run) when the GLOBAL count fits the global capacity, else "over"
    ws.dflag.copy_(torch.where(every.sum(dim=0, keepdim=True) <= gcap, torch.zeros_like(ws.dflag),
                               torch.full_like(ws.dflag, 1 << 62)))
    gate = N.EscSelection.from_buffer_copy(plan.sel.desc)
    gate.d_count = ws.dflag.data_ptr()
    outs = N.EscOutputs.from_buffer_copy(plan.outs)
    outs.capacity = cap
    N.check(lib.esc_materialize_selection(C.byref(gate), n, plan.mat_cols, plan.mat_ncols, None, C.byref(outs),
                                          C.c_void_p(ws_ptr), C.c_size_t(ws_bytes), sp), "esc_materialize_selection")
    stream.synchronize()
    local, fails = ws.read_result(cp.n_udfs, 1)
    counts = [int(x) for x in every.cpu().tolist()]
    cols = None
    if sum(counts) <= gcap:
        ps = executor.PendingStep(table, cp, proj, cap, "queued", 1, plan)
        cols = executor._take_outputs(ps, ws, local)
    else:
        executor._plan_checkin(ws, plan)
    return local, fails, counts, cols


def sharded_esc_subquery(st: ShardedTable, predicate, needed, config: EscConfig, group=None) -> ShardedDecision:
    """The fused ESC step on every rank's shard + one count exchange."""
    if predicate is None or _trivially_true(predicate):
        raise NoPredicate(f"table {st.name!r} has no filtering predicate")
    rc = st.global_rows
    fused = config.materialize and rc > 0 and rc >= config.min_table_size
    cp = compile_predicate(st.local, predicate)
    n = st.local.row_count
    gcap = math.floor(Fraction(config.max_selectivity) * rc)
    proj_bytes = sum(st.local.column(c).values.element_size() + 1 for c in needed) if fused else 0
    if (fused and dist.get_backend(group) == "nccl" and st.local.device.type == "cuda" and n > 0
            and min(gcap, n) * max(proj_bytes, 1) <= executor.SPECULATE_BYTES):
        try:
            local, fails, counts, cols = _queued_sharded(st, cp, list(needed), gcap, group)
            if cp.unbound or cp.may_fail:
                _global_replay(st, cp, fails, group)
        except EscdbError as exc:
            raise ExecutionError(f"count sub-query on {st.name!r} failed: {exc}") from exc
        total = sum(counts)
        qualified = decide_pushdown(rc, total, config)
        return ShardedDecision(st.name, total, rc, Fraction(total, rc) if rc else Fraction(0), qualified, local,
                               exclusive_offsets(counts)[st.rank], counts, cols if qualified else None)
    try:
        if fused:
            local, fails, sel = executor.launch_select(cp, st.local, None, n, capture=needed)
        else:
            (local, fails), sel = executor.launch_count(cp, st.local, None, n), None
        if cp.unbound or cp.may_fail:
            _global_replay(st, cp, fails, group)
    except EscdbError as exc:
        raise ExecutionError(f"count sub-query on {st.name!r} failed: {exc}") from exc
    total, counts, offsets = exchange_counts(local, group)
    qualified = decide_pushdown(rc, total, config)
    cols = None
    if qualified and config.materialize and sel is not None:
        # every rank compacts its own slice from the selection it recorded; concatenated in rank
        # order the slices are the global, order-preserving temp (offset = this rank's position)
        cols = executor.materialize_selection(sel, list(needed))
    return ShardedDecision(st.name, total, rc, Fraction(total, rc) if rc else Fraction(0), qualified,
                           local, offsets[st.rank], counts, cols)


def gather_to_rank0(cols: list, counts: list, group=None) -> list | None:
    """Optional: assemble the global, order-preserving temp on rank 0 (rank-order concatenation
    of the slices) — used by tests; the planner keeps temps sharded."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    out = []
    for c in cols:
        pieces = [torch.empty(counts[r], dtype=c.values.dtype, device=c.values.device) for r in range(world)]
        if dist.get_backend(group) == "nccl":
            dist.all_gather(pieces, c.values.contiguous(), group=group) if len(set(counts)) == 1 else \
                _ragged_gather(pieces, c.values, counts, group)
        else:
            _ragged_gather(pieces, c.values, counts, group)
        if rank == 0:
            out.append(torch.cat(pieces))
    return out if rank == 0 else None


def _ragged_gather(pieces, mine, counts, group):
    """all_gather for unequal lengths: pad to the max count, then trim."""
    m = max(counts) if counts else 0
    dev = mine.device
    padded = torch.zeros(m, dtype=mine.dtype, device=dev)
    padded[: mine.numel()] = mine
    bufs = [torch.empty(m, dtype=mine.dtype, device=dev) for _ in counts]
    dist.all_gather(bufs, padded, group=group)
    for r, b in enumerate(bufs):
        pieces[r].copy_(b[: counts[r]])
