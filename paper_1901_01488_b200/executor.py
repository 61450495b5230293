"""Predicate evaluation on the GPU: exact counts, row selections, fused materialization.

Drop-in for the hot half of ``escdb.executor`` (reference ``pkg/src/escdb/executor.py:23-250``):

=====================  =============================================  ==========================
function               reference                                      device path
=====================  =============================================  ==========================
``count_star``         ``executor.py:218-224``                        K1 ``esc_scan_count``
``eval_predicate``     ``executor.py:202-215``                        K1 (size) + K2 row ids
``execute_count``      ``executor.py:232-250``                        host shim -> ``count_star``
``materialize``        ``optimizer.py:191-192`` (eval + take)         K2 ``esc_compact`` (1 pass)
``take_column``        ``storage.py:176-184``                         ``esc_gather``
=====================  =============================================  ==========================

UDF failures keep the reference's observable behaviour: the reference evaluates a UDF on every
row of the slice whenever the UDF is *reached* by its whole-slice short circuit
(``executor.py:183-196``: an AND stops once its running mask has no true row, an OR once it has
no false row) and reports ``ExecutionError("UDF 'f' failed at row i: <python message>")`` for
the first failing row (``executor.py:133-144``).  A UDF that can fail is evaluated densely by the
kernel, which records its first failing row; the host then replays the short-circuit decisions
with exact device counts of the sibling prefixes and raises exactly when the reference would.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

from . import _native as N
from . import expr as ex
from .compiler import CompiledPredicate, compile_predicate
from .errors import ExecutionError
from .ra import RaAggregate, RaProject, RaScan, RaSelect, RaTempScan
from .storage import Column, ColumnTable
from .udf import FAIL_MESSAGES

_NO_FAIL = (1 << 64) - 1

# bench/profiling hook: when a list, every kernel launch appends (start_event, end_event, kind)
# recorded on the launching stream around the launch (before any host synchronisation)
KERNEL_EVENTS: list | None = None


def _ev_start(stream):
    if KERNEL_EVENTS is None:
        return None
    ev = torch.cuda.Event(enable_timing=True)
    ev.record(stream)
    return ev


def _ev_end(stream, ev0, kind):
    if ev0 is not None and KERNEL_EVENTS is not None:
        ev1 = torch.cuda.Event(enable_timing=True)
        ev1.record(stream)
        KERNEL_EVENTS.append((ev0, ev1, kind))


@dataclass
class RowSelection:
    """Subset of a table's rows: ascending device row ids, or every row (``indices=None``)."""

    table: ColumnTable
    indices: torch.Tensor | None = None

    @property
    def count(self) -> int:
        return self.table.row_count if self.indices is None else int(self.indices.numel())

    def to_indices(self) -> torch.Tensor:
        if self.indices is None:
            return torch.arange(self.table.row_count, dtype=torch.int64, device=self.table.device)
        return self.indices


# ------------------------------------------------------------------------------------------------
# launches
# ------------------------------------------------------------------------------------------------
_STREAMS: dict = {}


def _stream(device: torch.device) -> torch.cuda.Stream:
    """The device's current stream; the Stream object is cached per (stream id, device) — the
    public ``torch.cuda.current_stream`` builds a new one per call (several microseconds, and
    an ESC step asks for it a few times)."""
    if device.type != "cuda":
        raise N.NativeUnavailable(f"table lives on {device}; the ESC kernels need a CUDA device")
    idx = device.index if device.index is not None else torch.cuda.current_device()
    key = torch._C._cuda_getCurrentStream(idx)
    s = _STREAMS.get(key)
    if s is None:
        s = _STREAMS[key] = torch.cuda.current_stream(idx)
    return s


def _row_ids(selection: RowSelection | None):
    if selection is None or selection.indices is None:
        return None, (selection.table.row_count if selection is not None else None)
    ids = selection.indices
    if ids.dtype != torch.int64 or not ids.is_contiguous():
        ids = ids.to(torch.int64).contiguous()
    return ids, int(ids.numel())


def launch_count(cp: CompiledPredicate, table: ColumnTable, ids: torch.Tensor | None, n: int,
                 sync: bool = True):
    """K1 over ``n`` logical rows; returns (count, [udf fail words]) after a stream sync."""
    lib = N.load_library()
    stream = _stream(table.device)
    ws = N.workspace(table.device, stream)
    ws_ptr, ws_bytes = ws.ensure(n, stream.cuda_stream)
    cols = cp.column_array()
    ev0 = _ev_start(stream)
    N.check(lib.esc_scan_count(C.byref(cp.program), cols, cp.ncols, n,
                               C.c_void_p(ids.data_ptr()) if ids is not None else None,
                               C.c_void_p(ws.result.data_ptr()), C.c_void_p(ws_ptr), C.c_size_t(ws_bytes),
                               C.c_void_p(stream.cuda_stream)), "esc_scan_count")
    _ev_end(stream, ev0, "count")
    if not sync:
        return None
    stream.synchronize()
    return ws.read_result(cp.n_udfs)


@dataclass
class Selection:
    """What the count sub-query recorded on the device: a bitmap over the slice's logical rows,
    the hits per warp segment and — for sparse segments — the hits' values of the captured
    projected columns; enough to materialise without re-evaluating (or, mostly, re-reading)."""

    table: ColumnTable
    count: int
    desc: object                 # N.EscSelection (device pointers)
    buffers: list                # tensors owning the device memory behind ``desc``
    captured: dict               # column name -> capture index
    cols: object                 # the esc_column_t array the scan used (slots of ``captured``)
    slot_of: dict                # column name -> slot in ``cols``
    nrows: int
    ids: torch.Tensor | None


# Scan-time capture of sparse segments' hits (ESC_CAPTURE=0 turns it off): the scan copies the
# hits' values of the projected PREDICATE columns — already staged in shared memory — into
# per-segment slots, so the materialisation copies them instead of re-gathering rows from HBM
# (DESIGN.md §4).  Projection-only columns are never captured: reading them would put HBM
# gathers inside the scan.
_CAPTURE = os.environ.get("ESC_CAPTURE", "1") == "1"
_CAPTURE_BYTES_LIMIT = 8 << 30


def set_capture(on: bool) -> bool:
    """Turn scan-time capture on/off; returns the previous setting (tests, tuning)."""
    global _CAPTURE
    prev, _CAPTURE = _CAPTURE, bool(on)
    return prev


def launch_select(cp: CompiledPredicate, table: ColumnTable, ids: torch.Tensor | None, n: int, capture=(),
                  sync: bool = True, d_count: torch.Tensor | None = None):
    """K1 + selection outputs (and capture of ``capture`` columns' sparse hits); returns
    (count, [udf fail words], Selection).  ``sync=False`` returns right after the launch with
    count/fails None (read them with :func:`finish_select`); ``d_count`` (device int64[1])
    receives the exact count on the device."""
    lib = N.load_library()
    stream = _stream(table.device)
    ws = N.workspace(table.device, stream)
    ws_ptr, ws_bytes = ws.ensure(n, stream.cuda_stream)
    slot_of = cp.slot_of
    capture = [table.column(c) for c in dict.fromkeys(capture) if c in slot_of] if _CAPTURE else []
    if capture and (ids is not None or cp.tile_rows() > 4096):
        capture = []  # no capture through row-id chains or with 32-row-per-lane (narrow) tiles
    capture = capture[: N.MAX_PROJ]
    words, segs, cap_entries = C.c_int64(), C.c_int64(), C.c_int64()
    lib.esc_selection_sizes(n, C.byref(words), C.byref(segs), C.byref(cap_entries))
    if sum(c.values.element_size() for c in capture) * cap_entries.value > _CAPTURE_BYTES_LIMIT:
        capture = []
    dev = table.device
    buffers = [torch.empty(max(words.value, 1), dtype=torch.int32, device=dev),
               torch.empty(max(segs.value, 1), dtype=torch.int32, device=dev)]
    for col in capture:
        buffers.append(torch.empty(max(cap_entries.value, 1), dtype=col.values.dtype, device=dev))
        buffers.append(torch.empty(max(cap_entries.value, 1), dtype=torch.uint8, device=dev)
                       if col.nulls is not None else None)
    desc = N.EscSelection()
    desc.bitmap = buffers[0].data_ptr()
    desc.seg_counts = buffers[1].data_ptr()
    captured = {}
    for k, col in enumerate(capture):
        desc.cap_slot[k] = slot_of[col.name]
        desc.cap_values[k] = buffers[2 + 2 * k].data_ptr()
        nb = buffers[3 + 2 * k]
        desc.cap_nulls[k] = nb.data_ptr() if nb is not None else None
        captured[col.name] = k
    desc.n_cap = len(captured)
    desc.d_count = d_count.data_ptr() if d_count is not None else None
    cols = cp.column_array()
    ev0 = _ev_start(stream)
    N.check(lib.esc_scan_select(C.byref(cp.program), cols, cp.ncols, n,
                                C.c_void_p(ids.data_ptr()) if ids is not None else None, C.byref(desc),
                                C.c_void_p(ws.result.data_ptr()), C.c_void_p(ws_ptr), C.c_size_t(ws_bytes),
                                C.c_void_p(stream.cuda_stream)), "esc_scan_select")
    _ev_end(stream, ev0, "select")
    sel = Selection(table, None, desc, [b for b in buffers if b is not None], captured, cols, dict(slot_of), n, ids)
    if not sync:
        return None, None, sel
    count, fails = finish_select(sel, cp)
    return count, fails, sel


def _plan_selection(cp: CompiledPredicate, table: ColumnTable, n: int, capture, ws):
    """Selection buffers + descriptor for a step plan (allocated, not launched)."""
    lib = N.load_library()
    slot_of = cp.slot_of
    cap_cols = [table.column(c) for c in dict.fromkeys(capture) if c in slot_of] if _CAPTURE else []
    if cp.tile_rows() > 4096:
        cap_cols = []
    cap_cols = cap_cols[: N.MAX_PROJ]
    words, segs, cap_entries = C.c_int64(), C.c_int64(), C.c_int64()
    lib.esc_selection_sizes(n, C.byref(words), C.byref(segs), C.byref(cap_entries))
    if sum(c.values.element_size() for c in cap_cols) * cap_entries.value > _CAPTURE_BYTES_LIMIT:
        cap_cols = []
    dev = table.device
    buffers = [torch.empty(max(words.value, 1), dtype=torch.int32, device=dev),
               torch.empty(max(segs.value, 1), dtype=torch.int32, device=dev)]
    desc = N.EscSelection()
    desc.bitmap = buffers[0].data_ptr()
    desc.seg_counts = buffers[1].data_ptr()
    captured = {}
    for k, col in enumerate(cap_cols):
        vals = torch.empty(max(cap_entries.value, 1), dtype=col.values.dtype, device=dev)
        buffers.append(vals)
        desc.cap_slot[k] = slot_of[col.name]
        desc.cap_values[k] = vals.data_ptr()
        if col.nulls is not None:
            nb = torch.empty(max(cap_entries.value, 1), dtype=torch.uint8, device=dev)
            buffers.append(nb)
            desc.cap_nulls[k] = nb.data_ptr()
        captured[col.name] = k
    desc.n_cap = len(captured)
    desc.d_count = ws.dcount.data_ptr()
    return None, None, Selection(table, None, desc, buffers, captured, cp.column_array(), dict(slot_of), n, None)



def finish_select(sel: Selection, cp: CompiledPredicate):
    """Wait for the scan of ``sel`` (and whatever was queued behind it) and read its result."""
    stream = _stream(sel.table.device)
    stream.synchronize()
    count, fails = N.workspace(sel.table.device, stream).read_result(cp.n_udfs)
    sel.count = count
    return count, fails


def launch_materialize_selection(sel: Selection, proj_cols: list, capacity: int, want_row_ids: bool,
                                 skip_over_capacity: bool = False, with_nulls: bool = True):
    """Order-preserving compaction of the selected rows of ``proj_cols`` (and/or their physical
    row ids) into fresh buffers of ``capacity`` rows.  ``skip_over_capacity``: the launch may be
    queued before the count is known; it does nothing when the count exceeds ``capacity``.
    ``with_nulls`` False: no NULL outputs (the caller's selection excludes NULLs)."""
    lib = N.load_library()
    table = sel.table
    stream = _stream(table.device)
    ws = N.workspace(table.device, stream)
    ws_ptr, ws_bytes = ws.ensure(sel.nrows, stream.cuda_stream)
    if len(proj_cols) > N.MAX_PROJ:
        raise ExecutionError("too many columns for one compaction")
    # projections the scan did not see go after its slots
    slot_of = dict(sel.slot_of)
    nscan = len(sel.cols)
    extra = []
    for col in proj_cols:
        if col.name not in slot_of:
            slot_of[col.name] = nscan + len(extra)
            extra.append(col)
    cols = (N.EscColumn * max(nscan + len(extra), 1))()
    for i in range(nscan):
        cols[i] = sel.cols[i]
    for j, col in enumerate(extra):
        N.require_cuda(col.values, f"column {col.name!r}")
        cols[nscan + j].data = col.values.data_ptr() if len(col) else None
        cols[nscan + j].nulls = col.nulls.data_ptr() if col.nulls is not None and len(col) else None
        cols[nscan + j].dtype = N.dtype_code(col.values)
    outs = N.EscOutputs()
    outs.n_proj = len(proj_cols)
    outs.capacity = capacity
    outs.flags = N.OUT_SKIP_OVER_CAPACITY if skip_over_capacity else 0
    values, nulls = [], []
    dev = table.device
    for k, col in enumerate(proj_cols):
        v = torch.empty(capacity, dtype=col.values.dtype, device=dev)
        m = torch.empty(capacity, dtype=torch.bool, device=dev) if col.nulls is not None and with_nulls else None
        values.append(v)
        nulls.append(m)
        outs.slot[k] = slot_of[col.name]
        outs.out_values[k] = v.data_ptr() if capacity else None
        outs.out_nulls[k] = m.data_ptr() if m is not None and capacity else None
    rows = torch.empty(capacity, dtype=torch.int64, device=dev) if want_row_ids else None
    outs.out_row_ids = rows.data_ptr() if rows is not None and capacity else None
    ev0 = _ev_start(stream)
    N.check(lib.esc_materialize_selection(C.byref(sel.desc), sel.nrows, cols, nscan + len(extra),
                                          C.c_void_p(sel.ids.data_ptr()) if sel.ids is not None else None,
                                          C.byref(outs), C.c_void_p(ws_ptr), C.c_size_t(ws_bytes),
                                          C.c_void_p(stream.cuda_stream)), "esc_materialize_selection")
    _ev_end(stream, ev0, "materialize")
    return values, nulls, rows


def launch_compact(cp: CompiledPredicate, table: ColumnTable, ids: torch.Tensor | None, n: int,
                   proj_cols: list, capacity: int, want_row_ids: bool, stage_proj: bool = False):
    """Single-pass predicate + count + order-preserving compaction with decoupled look-back
    (``esc_compact_onepass``) of ``proj_cols`` (and/or the physical row ids) into fresh buffers
    of ``capacity`` rows.  Bit-identical to select + materialize; kept as the one-pass variant."""
    lib = N.load_library()
    stream = _stream(table.device)
    ws = N.workspace(table.device, stream)
    ws_ptr, ws_bytes = ws.ensure(n, stream.cuda_stream)
    extra, slots = [], []
    for col in proj_cols:
        if col.name in cp.slot_of:
            slots.append(cp.slot_of[col.name])
        else:
            slots.append(cp.ncols + len(extra))
            extra.append(col)
    if cp.ncols + len(extra) > N.MAX_COLS or len(proj_cols) > N.MAX_PROJ:
        raise ExecutionError("too many columns for one compaction")
    cols = cp.column_array(extra)
    if stage_proj:
        staged = (N.EscColumn * len(cols))()
        C.memmove(staged, cols, C.sizeof(staged))
        for k in range(cp.ncols, cp.ncols + len(extra)):
            staged[k].flags |= N.COL_STAGE
        cols = staged
    outs = N.EscOutputs()
    outs.n_proj = len(proj_cols)
    outs.capacity = capacity
    values, nulls = [], []
    dev = table.device
    for k, col in enumerate(proj_cols):
        v = torch.empty(capacity, dtype=col.values.dtype, device=dev)
        m = torch.empty(capacity, dtype=torch.bool, device=dev) if col.nulls is not None and with_nulls else None
        values.append(v)
        nulls.append(m)
        outs.slot[k] = slots[k]
        outs.out_values[k] = v.data_ptr() if capacity else None
        outs.out_nulls[k] = m.data_ptr() if m is not None and capacity else None
    rows = torch.empty(capacity, dtype=torch.int64, device=dev) if want_row_ids else None
    outs.out_row_ids = rows.data_ptr() if rows is not None and capacity else None
    ev0 = _ev_start(stream)
    N.check(lib.esc_compact_onepass(C.byref(cp.program), cols, cp.ncols + len(extra), n,
                            C.c_void_p(ids.data_ptr()) if ids is not None else None, C.byref(outs),
                            C.c_void_p(ws.result.data_ptr()), C.c_void_p(ws_ptr), C.c_size_t(ws_bytes),
                            C.c_void_p(stream.cuda_stream)), "esc_compact_onepass")
    _ev_end(stream, ev0, "compact")
    stream.synchronize()
    count, fails = ws.read_result(cp.n_udfs)
    return count, fails, values, nulls, rows


# ------------------------------------------------------------------------------------------------
# UDF error replay (reference short-circuit semantics)
# ------------------------------------------------------------------------------------------------
def _contains(node, targets: set) -> bool:
    return any(id(a) in targets for a in ex.atoms(node))


def raise_udf_errors(table: ColumnTable, cp: CompiledPredicate, fails: list, ids, n: int, count_fn=None):
    """Raise the ExecutionError the reference would raise for this evaluation, if any.

    ``count_fn(sub_predicate) -> int`` counts a sibling prefix over the slice (default: a local
    device count; the multi-GPU path passes a global one)."""
    failing = {}
    for node_id, u in cp.udf_index.items():
        if u < len(fails) and fails[u] != _NO_FAIL:
            failing[node_id] = (fails[u] >> 3, fails[u] & 7)
    unbound = {id(a) for a in cp.unbound}
    targets = set(failing) | unbound
    if not targets:
        return

    def count(sub) -> int:
        if count_fn is not None:
            return count_fn(sub)
        scp = compile_predicate(table, sub)
        c, _ = launch_count(scp, table, ids, n)
        return c

    def check(node):
        if isinstance(node, ex.FnCall):
            if id(node) in unbound:
                raise ExecutionError(f"function {node.name!r} has no bound implementation")
            if id(node) in failing:
                row, code = failing[id(node)]
                raise ExecutionError(f"UDF {node.name!r} failed at row {row}: {FAIL_MESSAGES[code]}")
            return
        if isinstance(node, ex.ATOM_TYPES):
            return
        if isinstance(node, ex.Not):
            return check(node.child)
        items = node.items
        check(items[0])
        for k in range(1, len(items)):
            if not _contains(items[k], targets):
                continue
            prefix = type(node)(tuple(items[:k]))
            c = count(prefix)
            if isinstance(node, ex.And) and c == 0:
                return  # reference: `if not mask.any(): break`
            if isinstance(node, ex.Or) and c == n:
                return  # reference: `if mask.all(): break`
            check(items[k])

    check(cp.pred)


# ------------------------------------------------------------------------------------------------
# public API (reference names)
# ------------------------------------------------------------------------------------------------
def _count_with_errors(table, pred, selection=None) -> int:
    cp = compile_predicate(table, pred)
    ids, n = _row_ids(selection if selection is not None else RowSelection(table))
    count, fails = launch_count(cp, table, ids, n)
    if cp.unbound or cp.may_fail:
        raise_udf_errors(table, cp, fails, ids, n)
    return count


def select(table: ColumnTable, pred: ex.Expr, selection: RowSelection | None = None, capture=()) -> Selection:
    """The count sub-query that also records its selection on the device (one predicate pass;
    sparse segments' hits of the ``capture`` columns are captured on the way); raises the
    reference's UDF errors."""
    cp = compile_predicate(table, pred)
    ids, n = _row_ids(selection if selection is not None else RowSelection(table))
    count, fails, sel = launch_select(cp, table, ids, n, capture)
    if cp.unbound or cp.may_fail:
        raise_udf_errors(table, cp, fails, ids, n)
    return sel


def count_star(table: ColumnTable, pred: ex.Expr | None) -> int:
    """Exact number of rows satisfying ``pred`` (reference ``executor.py:218-224``); nothing is
    materialised — one fused scan over the predicate columns."""
    if pred is None:
        return table.row_count
    return _count_with_errors(table, pred)


def eval_predicate(table: ColumnTable, pred: ex.Expr | None,
                   selection: RowSelection | None = None) -> RowSelection:
    """Rows of ``selection`` (default: all) satisfying ``pred`` as ascending device row ids
    (reference ``executor.py:202-215``)."""
    if selection is None:
        selection = RowSelection(table)
    if pred is None:
        return selection
    n = table.row_count
    if selection.indices is None and 0 < n <= ONEPASS_MAX_ROWS:
        # small tables: ONE launch of the look-back kernel writes the row ids (select + the
        # compaction chain would be five launches and two waits)
        cp = compile_predicate(table, pred)
        count, fails, _, _, rows = launch_compact(cp, table, None, n, [], n, want_row_ids=True)
        if cp.unbound or cp.may_fail:
            raise_udf_errors(table, cp, fails, None, n)
        if count * 4 < n:  # don't pin an n-row buffer for a small selection: exact-size copy
            rows = _exact_copy(rows, count, _stream(table.device))
        return RowSelection(table, rows[:count])
    sel = select(table, pred, selection)
    _, _, rows = launch_materialize_selection(sel, [], sel.count, want_row_ids=True)
    return RowSelection(table, rows)


def materialize_selection(sel: Selection, needed, capacity: int | None = None) -> list[Column]:
    """Columns ``needed`` of the rows a Selection marks, in row order (no predicate re-scan)."""
    proj = [sel.table.column(name) for name in needed]
    cap = sel.count if capacity is None else min(int(capacity), sel.count)
    values, nulls, _ = launch_materialize_selection(sel, proj, cap, want_row_ids=False)
    return [Column(c.name, c.kind, v, m, c.dictionary) for c, v, m in zip(proj, values, nulls)]


def materialize(table: ColumnTable, pred: ex.Expr, needed, count: int | None = None,
                stage_proj: bool | None = None) -> list[Column]:
    """Qualifying rows of ``needed`` columns, in row order, as new device columns — the
    equivalent of ``eval_predicate(...).to_indices()`` + ``Column.take`` per column (reference
    ``optimizer.py:191-192``): one predicate pass recording the selection, one compaction pass
    over the selection.  ``count`` / ``stage_proj`` are accepted for API stability."""
    del count, stage_proj
    return materialize_selection(select(table, pred, capture=needed), needed)


# below this many rows the fused ESC step is ONE launch of the one-pass look-back kernel (a few
# tiles: the look-back is trivial and launch latency dominates); above, select + gather
ONEPASS_MAX_ROWS = int(os.environ.get("ESC_ONEPASS_MAX_ROWS", str(1 << 21)))

# the compaction is queued behind the scan (one host round trip per table) when its
# capacity-sized output buffers stay below this many bytes
SPECULATE_BYTES = int(os.environ.get("ESC_SPECULATE_BYTES", str(4 << 30)))
# capacity-sized outputs up to this size become the temp as views (no trim copy)
SMALL_OUTPUT_BYTES = int(os.environ.get("ESC_SMALL_OUTPUT_BYTES", str(1 << 20)))
# device bytes the cached step plans (selection + capacity-sized output buffers) may hold per stream
STEP_PLAN_BYTES = int(os.environ.get("ESC_STEP_PLAN_BYTES", str(8 << 30)))


def count_and_materialize(table: ColumnTable, pred: ex.Expr, needed, capacity: int):
    """The ESC step: one predicate pass (exact count + selection bitmap), then — only when the
    count fits ``capacity`` (the push-down threshold) — the compaction of ``needed`` from the
    recorded selection.  The compaction is queued right behind the scan and checks the count
    on the device (it does nothing for a table that does not qualify), so the host waits once;
    the qualifying rows are then trimmed out of the ``capacity``-row buffers.  Small tables take
    the single-launch one-pass kernel with the output bounded by ``capacity``.  Returns
    ``(count, columns or None)``."""
    ps = launch_step(table, pred, needed, capacity, slot=1)
    _stream(table.device).synchronize()
    return finish_step(ps)


@dataclass
class PendingStep:
    """An ESC step whose kernels are queued and whose result has not been read back yet
    (``launch_step`` / ``finish_step``): steps of independent tables share one host wait."""

    table: ColumnTable
    cp: CompiledPredicate | None
    proj: list
    capacity: int
    kind: str                   # "count" | "onepass" | "queued" | "done"
    slot: int = 0
    plan: object = None
    result: tuple | None = None


def launch_step(table: ColumnTable, pred: ex.Expr, needed, capacity: int, materialize: bool = True,
                slot: int = 1, between=None) -> PendingStep:
    """Queue one table's ESC step on the stream without waiting: K1 count (``materialize``
    False), the one-pass compaction (small tables) or K1 select + the queued compaction; the
    kernels' result block is the workspace's pinned ``slot`` (1 .. N.RESULT_SLOTS).

    ``between(plan, stream)`` (multi-GPU): on the queued path it is called after the scan and
    before the compaction — it queues the count exchange and the device gate
    (``plan.gate_buf``, :func:`gate_buffers`) that the compaction then reads instead of the local
    count.  ``PendingStep.kind`` tells the caller whether it ran (``"queued"``)."""
    cp = compile_predicate(table, pred)
    n = table.row_count
    lib = N.load_library()
    stream = _stream(table.device)
    ws = N.workspace(table.device, stream)
    ws_ptr, ws_bytes = ws.ensure(n, stream.cuda_stream)
    res = C.c_void_p(ws.result_ptr(slot))
    sp = C.c_void_p(stream.cuda_stream)
    if not materialize:
        ev0 = _ev_start(stream)
        N.check(lib.esc_scan_count(C.byref(cp.program), cp.column_array(), cp.ncols, n, None, res,
                                   C.c_void_p(ws_ptr), C.c_size_t(ws_bytes), sp), "esc_scan_count")
        _ev_end(stream, ev0, "count")
        return PendingStep(table, cp, [], capacity, "count", slot)
    proj = [table.column(name) for name in needed]
    cap = max(0, min(int(capacity), n))
    if n <= ONEPASS_MAX_ROWS:
        plan = _onepass_plan(cp, table, proj, cap, ws)
        # the prepared launch lives with the compiled predicate (same table, so same columns);
        # output buffers handed over as the temp are replaced by rebinding the new ones
        ckey = (plan.key[3:], n, slot, ws_ptr, N.TUNING[0])
        handle = cp.c_plans.get(ckey)
        if handle is None:
            h = C.c_void_p()
            N.check(lib.esc_step_plan_create(C.byref(cp.program), plan.mat_cols, plan.mat_ncols, n, None, None, 0,
                                             C.byref(plan.outs), res, C.c_void_p(ws_ptr), C.c_size_t(ws_bytes),
                                             C.byref(h)), "esc_step_plan_create")
            handle = cp.c_plans[ckey] = _CPlan(h.value, lib)
        else:
            N.check(lib.esc_step_plan_rebind(C.c_void_p(handle.ptr), C.byref(plan.outs)), "esc_step_plan_rebind")
        ev0 = _ev_start(stream)
        N.check(lib.esc_step_plan_launch(C.c_void_p(handle.ptr), 3, sp), "esc_step_plan_launch")
        _ev_end(stream, ev0, "compact")
        return PendingStep(table, cp, proj, cap, "onepass", slot, plan)
    row_bytes = sum(c.values.element_size() + (1 if c.nulls is not None else 0) for c in proj)
    if not (0 < cap and cap * max(row_bytes, 1) <= SPECULATE_BYTES):
        sel = select(table, pred, capture=needed)  # waits: the count sizes the output
        if sel.count > cap:
            return PendingStep(table, None, proj, cap, "done", result=(sel.count, None))
        return PendingStep(table, None, proj, cap, "done", result=(sel.count, materialize_selection(sel, needed)))
    plan = _step_plan(cp, table, proj, cap, ws)
    gated = between is not None
    ckey = (slot, ws_ptr, N.TUNING[0], gated)
    handle = plan.c_plans.get(ckey) if plan.c_plans is not None else None
    if handle is None:  # prepare the scan + compaction launches once (lowering, geometry, JIT lookup)
        h = C.c_void_p()
        if gated:  # the compaction's skip test reads the gate word the exchange step writes
            world = table.shard.world if table.shard is not None else None
            plan.sel.desc.d_gate = gate_buffers(plan, table.device, world)[0][-1:].data_ptr()
        try:
            N.check(lib.esc_step_plan_create(C.byref(cp.program), cp.column_array(), cp.ncols, n,
                                             C.byref(plan.sel.desc), plan.mat_cols, plan.mat_ncols, C.byref(plan.outs),
                                             res, C.c_void_p(ws_ptr), C.c_size_t(ws_bytes), C.byref(h)),
                    "esc_step_plan_create")
        finally:
            plan.sel.desc.d_gate = None
        handle = _CPlan(h.value, lib)
        if plan.c_plans is None:
            plan.c_plans = {}
        plan.c_plans[ckey] = handle
    if gated:
        for part, kind in ((1, "select"), (2, "materialize")):
            ev0 = _ev_start(stream)
            N.check(lib.esc_step_plan_launch(C.c_void_p(handle.ptr), part | N.PLAN_GRAPH, sp), "esc_step_plan_launch")
            _ev_end(stream, ev0, kind)
            if part == 1:
                between(plan, stream)
    elif KERNEL_EVENTS is None:
        N.check(lib.esc_step_plan_launch(C.c_void_p(handle.ptr), 3, sp), "esc_step_plan_launch")
    else:  # profiling: events between the scan and the compaction
        for part, kind in ((1, "select"), (2, "materialize")):
            ev0 = _ev_start(stream)
            N.check(lib.esc_step_plan_launch(C.c_void_p(handle.ptr), part, sp), "esc_step_plan_launch")
            _ev_end(stream, ev0, kind)
    return PendingStep(table, cp, proj, cap, "queued", slot, plan)


class _CPlan:
    """Owner of an esc_step_plan handle (destroyed with the Python plan that holds it)."""

    __slots__ = ("ptr", "lib")

    def __init__(self, ptr, lib):
        self.ptr, self.lib = ptr, lib

    def __del__(self):
        if self.ptr:
            try:
                self.lib.esc_step_plan_destroy(self.ptr)
            except Exception:  # noqa: BLE001 — interpreter shutdown: the process frees it
                pass
            self.ptr = None


def finish_step(ps: PendingStep):
    """Read back a launched step (after its stream has been synchronised): the reference's UDF
    errors, then ``(count, columns or None)`` — None when the count exceeds the capacity."""
    if ps.kind == "done":
        return ps.result
    table, cp = ps.table, ps.cp
    stream = _stream(table.device)
    ws = N.workspace(table.device, stream)
    count, fails = ws.read_result(cp.n_udfs, ps.slot)
    if cp.unbound or cp.may_fail:
        raise_udf_errors(table, cp, fails, None, table.row_count)
    if ps.kind == "count":
        return count, None
    return count, _take_outputs(ps, ws, count) if count <= ps.capacity else _release(ps, ws)


def _release(ps: PendingStep, ws):
    _plan_checkin(ws, ps.plan)
    return None


def _take_outputs(ps: PendingStep, ws, k: int) -> list[Column]:
    """The first ``k`` rows of a finished step's outputs as temp columns.  Small one-pass outputs
    are handed over as views (their plan is not cached again).  A queued step's outputs are lent:
    the temp columns are views of the plan's buffers, and the plan goes back to the cache only
    once no view of them is left (:func:`_step_plan` checks), so no trim copy runs on the step.
    Other outputs are trimmed by one copy."""
    plan = ps.plan
    if (ps.kind == "onepass" and plan.nbytes <= SMALL_OUTPUT_BYTES) or (ps.kind == "queued" and LEND_OUTPUTS):
        cols = [Column.device_column(c.name, c.kind, v[:k], m[:k] if m is not None else None, c.dictionary)
                for c, v, m in zip(ps.proj, plan.out_values, plan.out_nulls)]
        if ps.kind == "queued":
            _plan_lend(ws, plan)
        return cols
    if plan.trim_cache is None:
        plan.trim_cache = {}
    cols = _trim(ps.proj, plan.out_values, plan.out_nulls, k, _stream(ps.table.device), plan.trim_cache)
    _plan_checkin(ws, plan)
    return cols


@dataclass
class _StepPlan:
    """Everything one queued ESC step launches with, built once per (predicate, table, columns,
    capacity) and kept in the stream's workspace: the selection and its buffers, the
    capacity-sized compaction outputs and the argument structs (the host only re-issues)."""

    key: tuple
    cp: CompiledPredicate         # held: keeps id(cp) in ``key`` unique
    sel: Selection
    outs: object
    out_values: list
    out_nulls: list
    mat_cols: object
    mat_ncols: int
    nbytes: int = 0
    c_plans: dict | None = None   # (result slot, workspace, tuning, gated) -> prepared esc_step_plan
    trim_cache: dict | None = None  # _trim's ctypes arguments (sources are the fixed outputs)
    gate: tuple | None = None     # multi-GPU: (device int64[world + 3], pinned host copy)


def gate_buffers(plan: _StepPlan, device: torch.device, world: int | None = None) -> tuple:
    """The multi-GPU exchange buffers of a queued step plan: a device int64 vector
    ``[counts of every rank (world) | global count, this rank's offset, gate]`` (esc_count_gate's
    layout; the gate word is the last) and its pinned host copy.  The device buffer's address is
    captured by the gated C plan, so it lives as long as the plan."""
    if plan.gate is None:
        if world is None:
            import torch.distributed as dist

            world = dist.get_world_size() if dist.is_initialized() else 1
        dbuf = torch.zeros(world + 3, dtype=torch.int64, device=device)
        plan.gate = (dbuf, torch.zeros(world + 3, dtype=torch.int64, pin_memory=True))
    return plan.gate


def _step_plan(cp: CompiledPredicate, table: ColumnTable, proj: list, capacity: int, ws) -> _StepPlan:
    key = (id(cp), id(table), tuple(c.name for c in proj), capacity)
    plan = ws.scratch.setdefault("plans", {}).pop(key, None)  # checked out until finish_step
    if plan is not None:
        return plan
    lent = ws.scratch.get("lent")
    if lent:  # the latest plan whose lent outputs are no longer referenced (its temps were swept);
        # other free plans of the same key are dropped (their buffers go back to the allocator)
        free = [q for q in lent if q.key == key and _outputs_free(q)]
        if free:
            lent[:] = [q for q in lent if not any(q is f for f in free)]
            return free[-1]
        _reclaim_lent(ws)
    n = table.row_count
    _, _, sel = _plan_selection(cp, table, n, [c.name for c in proj], ws)
    slot_of = dict(sel.slot_of)
    nscan = len(sel.cols)
    extra = [c for c in proj if c.name not in slot_of]
    for j, c in enumerate(extra):
        slot_of[c.name] = nscan + j
    cols = (N.EscColumn * max(nscan + len(extra), 1))()
    for i in range(nscan):
        cols[i] = sel.cols[i]
    for j, col in enumerate(extra):
        cols[nscan + j].data = col.values.data_ptr() if len(col) else None
        cols[nscan + j].nulls = col.nulls.data_ptr() if col.nulls is not None and len(col) else None
        cols[nscan + j].dtype = N.dtype_code(col.values)
    outs = N.EscOutputs()
    outs.n_proj = len(proj)
    outs.capacity = capacity
    outs.flags = N.OUT_SKIP_OVER_CAPACITY
    values, nulls = [], []
    for k, col in enumerate(proj):
        v = torch.empty(capacity, dtype=col.values.dtype, device=table.device)
        m = torch.empty(capacity, dtype=torch.bool, device=table.device) if col.nulls is not None else None
        values.append(v)
        nulls.append(m)
        outs.slot[k] = slot_of[col.name]
        outs.out_values[k] = v.data_ptr()
        outs.out_nulls[k] = m.data_ptr() if m is not None else None
    plan = _StepPlan(key, cp, sel, outs, values, nulls, cols, nscan + len(extra))
    plan.nbytes = sum(b.numel() * b.element_size() for b in [*sel.buffers, *values, *[m for m in nulls if m is not None]])
    return plan


def _plan_checkin(ws, plan):
    """Return a finished step's plan to the stream's cache (most recently used last; least
    recently used plans are dropped beyond STEP_PLAN_BYTES)."""
    plans = ws.scratch.setdefault("plans", {})
    plans[plan.key] = plan
    while len(plans) > 1 and sum(p.nbytes for p in plans.values()) > STEP_PLAN_BYTES:
        plans.pop(next(iter(plans)))


# queued steps hand their capacity-sized outputs over as views (no trim copy on the step)
LEND_OUTPUTS = os.environ.get("ESC_LEND_OUTPUTS", "1") != "0"
LENT_PLANS = 8  # lent plans tracked per stream (older ones are forgotten: their views keep the outputs)


def _outputs_free(plan) -> bool:
    """No tensor besides the plan's own refers to its output buffers (one reference from the
    plan, one from the temporary storage object of the query)."""
    for t in (*plan.out_values, *[m for m in plan.out_nulls if m is not None]):
        if torch._C._storage_Use_Count(t.untyped_storage()._cdata) > 2:
            return False
    return True


def _plan_lend(ws, plan):
    """A step's outputs became temp columns (views): the plan is reusable once they are gone."""
    _reclaim_lent(ws)
    lent = ws.scratch.setdefault("lent", [])
    lent.append(plan)
    if len(lent) > LENT_PLANS:
        lent.pop(0)


def _reclaim_lent(ws):
    """Lent plans whose outputs are free again go back to the plan cache, where its byte budget
    (STEP_PLAN_BYTES, least recently used first) applies: plans of tables that are gone (a new
    table object per step) do not pile up with their capacity-sized buffers."""
    lent = ws.scratch.get("lent")
    if not lent:
        return
    keep = []
    for q in lent:
        if _outputs_free(q):
            _plan_checkin(ws, q)
        else:
            keep.append(q)
    lent[:] = keep


def release_step_plans(device: torch.device | None = None):
    """Drop the cached step plans (and their device buffers) of the current stream."""
    dev = device or torch.device("cuda", torch.cuda.current_device())
    scratch = N.workspace(dev, torch.cuda.current_stream(dev)).scratch
    scratch.pop("plans", None)
    scratch.pop("lent", None)


def materialize_onepass(table: ColumnTable, pred: ex.Expr, needed, capacity: int | None = None):
    """Single-pass variant (decoupled look-back kernel); same results as :func:`materialize`.
    Rows beyond ``capacity`` are counted, not written: returns ``(count, columns of the first
    min(count, capacity) qualifying rows)``."""
    n = table.row_count
    cap = n if capacity is None else max(0, min(int(capacity), n))
    ps = launch_step(table, pred, needed, cap, slot=1) if n <= ONEPASS_MAX_ROWS else None
    if ps is None:  # large tables: force the one-pass kernel anyway (tests, tuning)
        cp = compile_predicate(table, pred)
        proj = [table.column(name) for name in needed]
        count, fails, values, nulls, _ = launch_compact(cp, table, None, n, proj, cap, want_row_ids=False)
        if cp.unbound or cp.may_fail:
            raise_udf_errors(table, cp, fails, None, n)
        return count, _trim(proj, values, nulls, min(count, cap), _stream(table.device))
    _stream(table.device).synchronize()
    ws = N.workspace(table.device, _stream(table.device))
    count, fails = ws.read_result(ps.cp.n_udfs, ps.slot)
    if ps.cp.unbound or ps.cp.may_fail:
        raise_udf_errors(table, ps.cp, fails, None, n)
    return count, _take_outputs(ps, ws, min(count, cap))


def _onepass_plan(cp: CompiledPredicate, table: ColumnTable, proj: list, capacity: int, ws) -> _StepPlan:
    key = ("onepass", id(cp), id(table), tuple(c.name for c in proj), capacity)
    plan = ws.scratch.setdefault("plans", {}).pop(key, None)  # checked out until finished
    if plan is not None:
        return plan
    # the shape-only parts (slots, column array, outputs template) are kept with the compiled
    # predicate: a small table's outputs become its temp, so each step needs new buffers only
    shape = cp.shapes.get(key[3:])
    if shape is None:
        extra, slots = [], []
        for col in proj:
            if col.name in cp.slot_of:
                slots.append(cp.slot_of[col.name])
            else:
                slots.append(cp.ncols + len(extra))
                extra.append(col)
        if cp.ncols + len(extra) > N.MAX_COLS or len(proj) > N.MAX_PROJ:
            raise ExecutionError("too many columns for one compaction")
        tmpl = N.EscOutputs()
        tmpl.n_proj = len(proj)
        tmpl.capacity = capacity
        for k in range(len(proj)):
            tmpl.slot[k] = slots[k]
        shape = cp.shapes[key[3:]] = (tmpl, cp.column_array(extra), cp.ncols + len(extra))
    tmpl, mat_cols, mat_ncols = shape
    outs = N.EscOutputs.from_buffer_copy(tmpl)
    n_alloc = max(capacity, 1)
    dev = table.device
    values, nulls, nbytes = [], [], 0
    for k, col in enumerate(proj):
        v = torch.empty(n_alloc, dtype=col.values.dtype, device=dev)
        m = torch.empty(n_alloc, dtype=torch.bool, device=dev) if col.nulls is not None else None
        values.append(v)
        nulls.append(m)
        nbytes += n_alloc * (v.element_size() + (1 if m is not None else 0))
        if capacity:
            outs.out_values[k] = v.data_ptr()
            outs.out_nulls[k] = m.data_ptr() if m is not None else None
    plan = _StepPlan(key, cp, None, outs, values, nulls, mat_cols, mat_ncols)
    plan.nbytes = nbytes
    return plan


def _trim(proj: list, values: list, nulls: list, count: int, stream, cache: dict | None = None) -> list[Column]:
    """Exact-size temp columns: the first ``count`` rows of each capacity-sized output, copied
    by ONE batched launch (esc_copy_regions) into one caching-allocator tensor per column (a
    single allocation carved into views measured 7 us slower per step: each slice + view is a
    torch op of its own).  ``cache`` (a plan's dict) keeps the ctypes argument arrays — the
    sources are the plan's fixed buffers — so a step only fills in the destinations and sizes."""
    srcs = [t for v, m in zip(values, nulls) for t in ((v,) if m is None else (v, m))]
    k = len(srcs)
    if not k:
        return []
    dev = values[0].device
    outs = [torch.empty(count, dtype=t.dtype, device=dev) for t in srcs]
    if count:
        arrs = cache.get("trim") if cache is not None else None
        if arrs is None:
            arrs = ((C.c_void_p * k)(), (C.c_void_p * k)(*[t.data_ptr() for t in srcs]), (C.c_int64 * k)())
            if cache is not None:
                cache["trim"] = arrs
        dst, src, nbytes = arrs
        for i, t in enumerate(outs):
            dst[i] = t.data_ptr()
            nbytes[i] = count * t.element_size()
        N.check(N.load_library().esc_copy_regions(k, dst, src, nbytes, C.c_void_p(stream.cuda_stream)),
                "esc_copy_regions")
    out, r = [], 0
    for c, m in zip(proj, nulls):
        vv = outs[r]
        r += 1
        mm = None
        if m is not None:
            mm = outs[r]
            r += 1
        out.append(Column.device_column(c.name, c.kind, vv, mm, c.dictionary))
    return out


def _exact_copy(t: torch.Tensor, k: int, stream) -> torch.Tensor:
    """The first ``k`` elements of a device tensor in a new exact-size tensor (esc_copy_regions)."""
    out = torch.empty(k, dtype=t.dtype, device=t.device)
    if k:
        nbytes = k * t.element_size()
        N.check(N.load_library().esc_copy_regions(1, (C.c_void_p * 1)(out.data_ptr()),
                                                  (C.c_void_p * 1)(t.data_ptr()), (C.c_int64 * 1)(nbytes),
                                                  C.c_void_p(stream.cuda_stream)), "esc_copy_regions")
    return out


def take_column(col: Column, indices) -> Column:
    """``Column.take`` on the device (reference ``storage.py:176-184``)."""
    lib = N.load_library()
    dev = col.device
    stream = _stream(dev)
    idx = indices if isinstance(indices, torch.Tensor) else torch.as_tensor(indices)
    idx = idx.to(device=dev, dtype=torch.int64).contiguous()
    n = int(idx.numel())
    out = torch.empty(n, dtype=col.values.dtype, device=dev)
    nulls = torch.empty(n, dtype=torch.bool, device=dev) if col.nulls is not None else None
    desc = N.EscColumn()
    desc.data = col.values.data_ptr() if len(col) else None
    desc.nulls = col.nulls.data_ptr() if col.nulls is not None and len(col) else None
    desc.dtype = N.dtype_code(col.values)
    N.check(lib.esc_gather(C.byref(desc), C.c_void_p(idx.data_ptr()) if n else None, n,
                           C.c_void_p(out.data_ptr()) if n else None,
                           C.c_void_p(nulls.data_ptr()) if nulls is not None and n else None,
                           C.c_void_p(stream.cuda_stream)), "esc_gather")
    return Column(col.name, col.kind, out, nulls, col.dictionary)


def gather_values(values: torch.Tensor, indices: torch.Tensor) -> torch.Tensor:
    """values[indices] for a plain device tensor (esc_gather; no NULL mask)."""
    lib = N.load_library()
    dev = values.device
    idx = indices.to(device=dev, dtype=torch.int64).contiguous()
    n = int(idx.numel())
    out = torch.empty(n, dtype=values.dtype, device=dev)
    desc = N.EscColumn()
    desc.data = values.data_ptr() if values.numel() else None
    desc.nulls = None
    desc.dtype = N.dtype_code(values)
    N.check(lib.esc_gather(C.byref(desc), C.c_void_p(idx.data_ptr()) if n else None, n,
                           C.c_void_p(out.data_ptr()) if n else None, None, C.c_void_p(_stream(dev).cuda_stream)),
            "esc_gather")
    return out


def execute_count(ra, catalog) -> int:
    """Single-table COUNT tree: Aggregate over optional Select over optional Project over a
    Scan / TempScan (reference ``executor.py:232-250``)."""
    from .ra import adopt as adopt_ra

    ra = adopt_ra(ra)
    node = ra.child if isinstance(ra, RaAggregate) else ra
    pred = None
    if isinstance(node, RaSelect):
        pred, node = node.predicate, node.child
    if isinstance(node, RaProject):
        node = node.child
    if isinstance(node, RaScan):
        table = catalog.table(node.table)
    elif isinstance(node, RaTempScan):
        table = catalog.resolve_temp(node.handle)
    else:
        raise ExecutionError(f"cannot count over node {type(node).__name__}")
    return count_star(table, pred)
