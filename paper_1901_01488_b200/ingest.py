"""CSV ingestion straight into device-resident tables — SURVEY §8(f) row f3.

Drop-in for the reference loader (``pkg/src/escdb/storage.py:245-275, :385-425``):
``load_csv(text_or_file, name, schema, has_header)`` returns a :class:`ColumnTable` whose columns
already live in HBM, so a table crosses PCIe exactly once (the paper's PCIe note,
``PAPER.md:400``) and every later ESC sub-query scans it in place.

The bytes are copied to the device and parsed there (``csrc/esc_csv.cuh``): tokenisation with
quote-aware separators, record validation, and per-column conversion — INT64, DECIMAL(p,s) scaled
by 10**s, DATE as epoch days, TEXT dictionary-encoded in first-appearance order (the reference's
``Dictionary.encode`` order) from 64-bit content hashes that are then verified byte for byte.
Values, NULLs (``\\N``), dictionaries and the reference's error messages are identical for the
grammar below; the host only formats the message of the first failing cell.

Grammar (the reference accepts a few exotic forms beyond it; those raise a ``CsvError`` naming
the cell instead of being loaded):
* RFC 4180 quoting (a quote may only open/close a field, ``""`` inside) — Python's ``csv`` also
  tolerates stray quotes inside unquoted fields;
* INT64 ``[ws][+-]digits[ws]`` with single ``_`` between digits (ASCII) — Python's ``int`` also
  takes non-ASCII digits / whitespace;
* DATE ``YYYY-MM-DD`` or ``YYYYMMDD`` — ``date.fromisoformat`` also takes ISO week dates.
"""

from __future__ import annotations

import ctypes as C
import csv
import io
import warnings

import numpy as np
import torch

from . import _native as N
from . import executor, sorting
from .errors import CsvError, TypeMismatch
from .storage import (DATE, INT64, Column, ColumnKind, ColumnTable, Dictionary, date_to_days, default_device,
                      format_decimal)

NULL_TOKEN = r"\N"
_CODES = {"INT64": 0, "DECIMAL": 1, "DATE": 2, "TEXT": 3}
_ERR_QUOTE = 2
_ERR_OVERFLOW = 3


def parse_decimal_scaled(text: str, scale: int) -> int:
    """``"12.34"`` -> the scaled integer of a DECIMAL(p, scale) column; more fraction digits than
    the scale raise (the loader never rounds) — reference ``storage.py:100-118``."""
    t = text.strip()
    sign = -1 if t[:1] == "-" else 1
    if t[:1] in "+-":
        t = t[1:]
    whole, _, frac = t.partition(".")
    digits = whole + frac
    if not digits or not digits.isdigit():
        raise TypeMismatch(f"bad DECIMAL literal {text!r}")
    if len(frac) > scale:
        raise TypeMismatch(f"DECIMAL literal {text!r} exceeds scale {scale}")
    return sign * (int(whole or "0") * 10**scale + int(frac.ljust(scale, "0") or "0"))


def convert_cell(raw, kind: ColumnKind, dictionary: Dictionary | None) -> tuple[int, bool]:
    """One Python / text cell -> (int value, is_null) with the reference's rules and messages
    (``storage.py:245-274``); the host path of ``append_rows`` and the message of a failing cell."""
    if raw is None:
        return 0, True
    if kind.is_text:
        if not isinstance(raw, str):
            raise TypeMismatch(f"expected TEXT value, got {raw!r}")
        return dictionary.encode(raw), False
    if kind.name == DATE:
        if isinstance(raw, str):
            return date_to_days(raw), False
        if isinstance(raw, int):
            return raw, False
        raise TypeMismatch(f"expected DATE value, got {raw!r}")
    if kind.is_decimal:
        if isinstance(raw, str):
            return parse_decimal_scaled(raw, kind.scale), False
        if isinstance(raw, int):
            return raw, False  # already scaled
        raise TypeMismatch(f"expected DECIMAL value, got {raw!r}")
    if kind.name != INT64:
        raise TypeMismatch(f"column kind {kind} is not loadable from text")
    if isinstance(raw, (int, np.integer)) and not isinstance(raw, bool):
        return int(raw), False
    if isinstance(raw, str):
        try:
            return int(raw.strip()), False
        except ValueError:
            raise TypeMismatch(f"expected INT64 value, got {raw!r}") from None
    raise TypeMismatch(f"expected INT64 value, got {raw!r}")


def _check_int64(v: int):
    if not -(2**63) <= v < 2**63:
        raise OverflowError("Python int too large to convert to C long")


def append_rows(table: ColumnTable, rows, first_row_number: int = 1) -> ColumnTable:
    """A new table with Python ``rows`` appended (reference ``storage.py:277-320``): TEXT cells
    are dictionary-encoded on insert, strings parse per kind, bad rows raise ArityMismatch /
    TypeMismatch citing the row number.  The rows are host objects, so they are converted on the
    host and uploaded once; bulk text goes through :func:`load_csv` on the device."""
    from .errors import ArityMismatch

    rows = list(rows)
    width = len(table.columns)
    fresh = [(np.empty(len(rows), dtype=np.int64), np.zeros(len(rows), dtype=bool)) for _ in table.columns]
    for rix, row in enumerate(rows):
        if len(row) != width:
            raise ArityMismatch(f"table {table.name!r}: row {first_row_number + rix}: "
                                f"has {len(row)} values, expected {width}")
        for cix, col in enumerate(table.columns):
            try:
                value, is_null = convert_cell(row[cix], col.kind, col.dictionary)
            except TypeMismatch as exc:
                raise TypeMismatch(f"table {table.name!r}: row {first_row_number + rix}, "
                                   f"column {col.name!r}: {exc}") from None
            _check_int64(value)
            fresh[cix][0][rix] = value
            fresh[cix][1][rix] = is_null
    cols = []
    for (vals, nulls), c in zip(fresh, table.columns):
        dev = c.device
        old_v, old_m = c.values, c.null_mask
        new_v = torch.cat([old_v, torch.from_numpy(vals).to(device=dev, dtype=old_v.dtype)])
        new_m = torch.cat([old_m, torch.from_numpy(nulls).to(dev)])
        cols.append(Column(c.name, c.kind, new_v, new_m, c.dictionary))
    return ColumnTable(table.name, cols, table.is_temporary)


def _raw_bytes(text_or_file) -> bytes:
    if isinstance(text_or_file, (bytes, bytearray, memoryview)):
        return bytes(text_or_file)
    if isinstance(text_or_file, str):
        return text_or_file.encode("utf-8")
    data = text_or_file.read()
    return data.encode("utf-8") if isinstance(data, str) else bytes(data)


def _cell_text(data: bytes, start: int, end: int) -> tuple[str, bool]:
    """The reference's cell string of a field (RFC 4180 unquoting) and whether it was well-formed."""
    raw = data[start:end]
    if raw[:1] == b'"':
        ok = len(raw) >= 2 and raw[-1:] == b'"' and b'"' not in raw[1:-1].replace(b'""', b"")
        return raw[1:-1].replace(b'""', b'"').decode("utf-8", "replace"), ok
    return raw.decode("utf-8", "replace"), b'"' not in raw


_STAGE_BYTES = 8 << 20
_staging: dict = {}


def _upload(host: torch.Tensor, dev: torch.device, stream) -> torch.Tensor:
    """The CSV bytes to HBM through two reused pinned staging buffers: the host copy of chunk
    i + 1 overlaps the DMA of chunk i (pinning the whole text first, then copying it, serialised
    the two)."""
    n = int(host.numel())
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    if n <= _STAGE_BYTES:
        out.copy_(host.pin_memory(), non_blocking=True)
        return out
    bufs = _staging.get(dev)
    if bufs is None:
        bufs = _staging[dev] = [(torch.empty(_STAGE_BYTES, dtype=torch.uint8).pin_memory(),
                                 torch.cuda.Event()) for _ in range(2)]
    for i, off in enumerate(range(0, n, _STAGE_BYTES)):
        ln = min(_STAGE_BYTES, n - off)
        buf, ev = bufs[i % 2]
        ev.synchronize()  # the DMA that last read this buffer is done
        buf[:ln].copy_(host[off:off + ln])
        with torch.cuda.stream(stream):
            out[off:off + ln].copy_(buf[:ln], non_blocking=True)
            ev.record(stream)
    return out


def load_csv(text_or_file, name: str, schema, has_header: bool = False, device=None) -> ColumnTable:
    """Build a device table from RFC-4180 CSV text (``\\N`` = NULL, ISO dates) — reference
    ``storage.load_csv``; errors are the reference's ``CsvError`` / ``OverflowError`` text."""
    schema = [(n, k) for n, k in schema]
    for cname, kind in schema:
        if not (kind.is_text or kind.is_decimal or kind.name in (INT64, DATE)):
            raise TypeMismatch(f"column kind {kind} is not loadable from CSV")
    ncols = len(schema)
    dev = torch.device(device) if device is not None else default_device()
    data = _raw_bytes(text_or_file)
    n = len(data)
    lib = N.load_library()
    if dev.type != "cuda":
        raise N.NativeUnavailable(f"load_csv needs a CUDA device, got {dev}")
    stream = torch.cuda.current_stream(dev)
    sp = C.c_void_p(stream.cuda_stream)
    if n:
        with warnings.catch_warnings():  # read-only view of the caller's bytes; only copied from
            warnings.simplefilter("ignore", UserWarning)
            host = torch.frombuffer(data, dtype=torch.uint8)
        d_bytes = _upload(host, dev, stream)
    else:
        d_bytes = torch.zeros(1, dtype=torch.uint8, device=dev)
    ws_bytes = int(lib.esc_csv_workspace_bytes(n))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    # small device words are initialised by a host copy, not a fill kernel
    totals = torch.tensor([0, 0, 0], dtype=torch.int64, device=dev)
    N.check(lib.esc_csv_count(C.c_void_p(d_bytes.data_ptr()), n, C.c_void_p(totals.data_ptr()),
                              C.c_void_p(ws.data_ptr()), C.c_size_t(ws_bytes), sp), "esc_csv_count")
    nsep, nrec, open_quote = (int(x) for x in totals.cpu().tolist())
    if open_quote:
        raise CsvError(f"{name}: unexpected end of data (unterminated quoted field)")
    trailing = n > 0 and data[-1:] not in (b"\n", b"\r")
    field_end = torch.empty(nsep + 1, dtype=torch.int64, device=dev)
    field_kind = torch.empty(nsep + 1, dtype=torch.uint8, device=dev)
    rec_end = torch.empty(nrec + 1, dtype=torch.int64, device=dev)
    N.check(lib.esc_csv_fields(C.c_void_p(d_bytes.data_ptr()), n, C.c_void_p(field_end.data_ptr()),
                               C.c_void_p(field_kind.data_ptr()), C.c_void_p(rec_end.data_ptr()),
                               C.c_void_p(ws.data_ptr()), C.c_size_t(ws_bytes), sp), "esc_csv_fields")
    if trailing:  # the last record ends at the end of the text
        field_end[nsep] = n
        field_kind[nsep] = 2
        rec_end[nrec] = nsep
        nsep += 1
        nrec += 1
    field_end, field_kind, rec_end = field_end[:nsep], field_kind[:nsep], rec_end[:nrec]
    first_rec = 1 if has_header and nrec > 0 else 0
    nrows = nrec - first_rec
    # records must hold exactly ncols fields (an empty line is a record of 0 fields), and Python's
    # csv (text without newline translation) rejects a lone '\r' that is followed by more data on
    # its line; records of earlier lines are still checked first — one device pass (esc_csv_check)
    first_field = 0
    if first_rec:
        first_field = int(rec_end[0].item()) + 1
    chk = torch.empty(2, dtype=torch.int64, device=dev)
    N.check(lib.esc_csv_check(C.c_void_p(d_bytes.data_ptr()), n, C.c_void_p(field_end.data_ptr()) if nsep else None,
                              C.c_void_p(field_kind.data_ptr()) if nsep else None, nsep,
                              C.c_void_p(rec_end.data_ptr() + 8 * first_rec) if nrows else None, nrows, first_field,
                              ncols, C.c_void_p(chk.data_ptr()), sp), "esc_csv_check")
    bad_word, cr_word = (int(x) & ((1 << 64) - 1) for x in chk.cpu().tolist())
    lone_cr = -1 if cr_word == (1 << 64) - 1 else cr_word
    if bad_word != (1 << 64) - 1:
        r, got = bad_word >> 32, bad_word & 0xFFFFFFFF
        if got >= 1 << 31:
            got -= 1 << 32
        last_field = int(rec_end[first_rec + r].item())
        if lone_cr < 0 or int(field_end[last_field].item()) < data.rfind(b"\n", 0, lone_cr) + 1:
            raise CsvError(f"{name}: row {first_rec + r + 1}: expected {ncols} fields, got {got}")
    if lone_cr >= 0:
        raise csv.Error("new-line character seen in unquoted field - do you need to open the file with newline=''?")

    first_error = torch.tensor([-1], dtype=torch.int64, device=dev)  # all ones = none
    # which columns hold a NULL at all (the parse kernel flags them): one read for every column (a
    # column without NULLs keeps no mask, as the Column constructor would decide)
    null_seen = torch.tensor([0] * max(ncols, 1), dtype=torch.int32, device=dev)
    out = []
    for c, (cname, kind) in enumerate(schema):
        code = _CODES["TEXT" if kind.is_text else "DECIMAL" if kind.is_decimal else kind.name]
        vals = torch.empty(max(nrows, 1), dtype=torch.int64, device=dev)
        lens = torch.empty(max(nrows, 1), dtype=torch.int64, device=dev) if kind.is_text else None
        nulls = torch.empty(max(nrows, 1), dtype=torch.uint8, device=dev)
        N.check(lib.esc_csv_parse(C.c_void_p(d_bytes.data_ptr()), C.c_void_p(field_end.data_ptr()) if nsep else None,
                                  C.c_void_p(field_kind.data_ptr()) if nsep else None, first_field, nrows, ncols, c,
                                  code, kind.scale if kind.is_decimal else 0, C.c_void_p(vals.data_ptr()),
                                  C.c_void_p(lens.data_ptr()) if lens is not None else None,
                                  C.c_void_p(nulls.data_ptr()), C.c_void_p(first_error.data_ptr()),
                                  C.c_void_p(null_seen.data_ptr() + 4 * c), sp),
                "esc_csv_parse")
        out.append((vals[:nrows], nulls[:nrows].view(torch.bool), lens))  # bytes are 0 / 1
    err = int(first_error.item()) & ((1 << 64) - 1)
    if err != (1 << 64) - 1:
        _raise_cell_error(data, field_end, field_kind, first_field, ncols, schema, name,
                          2 if has_header else 1, err >> 4, err & 15)
    has_null = [bool(x) for x in null_seen.tolist()[:len(out)]] if out and nrows else [False] * len(out)
    cols = []
    for (cname, kind), (vals, nulls, _), hn in zip(schema, out, has_null):
        mask = nulls if hn else None
        if kind.is_text:
            codes, dictionary = _encode_text(data, d_bytes, field_end, field_kind, first_field, nrows, ncols,
                                             schema.index((cname, kind)), vals, nulls, sp, name)
            cols.append(Column.device_column(cname, kind, codes, mask, dictionary) if mask is None
                        else Column(cname, kind, codes, mask, dictionary))
        elif kind.name == DATE:
            v = vals.to(torch.int32)
            cols.append(Column.device_column(cname, kind, v, None, None) if mask is None else Column(cname, kind, v, mask))
        else:
            cols.append(Column.device_column(cname, kind, vals, None, None) if mask is None
                        else Column(cname, kind, vals, mask))
    return ColumnTable(name, cols)


def _raise_cell_error(data, field_end, field_kind, first_field, ncols, schema, name, first_row_number, idx, code):
    r, c = divmod(idx, ncols)
    f = first_field + idx
    end = int(field_end[f])
    start = 0 if f == 0 else int(field_end[f - 1]) + (2 if int(field_kind[f - 1]) == 3 else 1)
    text, well_formed = _cell_text(data, start, end)
    cname, kind = schema[c]
    where = f"table {name!r}: row {first_row_number + r}, column {cname!r}"
    if code == _ERR_QUOTE or not well_formed:
        raise CsvError(f"{name}: row {first_row_number + r}: quoting outside RFC 4180 is not supported "
                       f"by the device loader (column {cname!r})")
    raw = None if text == NULL_TOKEN else text
    try:
        value, _ = convert_cell(raw, kind, Dictionary())
    except TypeMismatch as exc:
        raise CsvError(f"{where}: {exc}") from None
    _check_int64(value)  # the reference's numpy store raises OverflowError
    raise CsvError(f"{where}: literal {text!r} is valid Python but outside the device loader's grammar")


def _encode_text(data, d_bytes, field_end, field_kind, first_field, nrows, ncols, col, hashes, nulls, sp, name):
    """First-appearance dictionary codes from the device content hashes, verified byte for byte."""
    dev = hashes.device
    if nrows == 0:
        return torch.empty(0, dtype=torch.int32, device=dev), Dictionary()
    # codes in first-appearance order by the framework's own device sort (esc_dict_encode: cells
    # grouped by content hash with a stable radix sort, groups ordered by their first row)
    codes, rep, first, u = sorting.dict_encode(hashes, nulls)
    words = []
    if u:
        bad = torch.tensor([0], dtype=torch.int32, device=dev)
        N.check(N.load_library().esc_csv_verify_text(C.c_void_p(d_bytes.data_ptr()), C.c_void_p(field_end.data_ptr()),
                                                    C.c_void_p(field_kind.data_ptr()), first_field, nrows, ncols, col,
                                                    C.c_void_p(rep.data_ptr()), C.c_void_p(bad.data_ptr()), sp),
                "esc_csv_verify_text")
        if int(bad.item()):
            raise CsvError(f"{name}: TEXT content hash collision in column {col}; the device loader cannot "
                           "encode this file")
        reps = first.cpu().numpy()
        f = first_field + reps * ncols + col  # the representative cells' field numbers (host)
        fi = torch.as_tensor(np.concatenate([f, np.maximum(f - 1, 0)]), device=dev)
        ends = executor.gather_values(field_end, fi).cpu().numpy()  # esc_gather, one launch
        fe, prev = ends[:u], ends[u:]
        pk = executor.gather_values(field_kind, fi[u:]).cpu().numpy()
        for fi_, e, p_, k in zip(f.tolist(), fe.tolist(), prev.tolist(), pk.tolist()):
            s = 0 if fi_ == 0 else p_ + (2 if k == 3 else 1)
            words.append(_cell_text(data, s, e)[0])
    d = Dictionary()
    for w in words:
        d.encode(w)
    return codes, d


def dump_csv(table: ColumnTable, include_header: bool = False) -> str:
    """Serialize a table back to the loader's CSV format (reference ``storage.py:412-425``)."""
    out = io.StringIO()
    writer = csv.writer(out, lineterminator="\n")
    if include_header:
        writer.writerow([c.name for c in table.columns])
    host = [c.to_numpy() for c in table.columns]
    for i in range(table.row_count):
        row = []
        for c, (vals, nulls) in zip(table.columns, host):
            if nulls[i]:
                row.append(NULL_TOKEN)
                continue
            v = int(vals[i]) if not c.kind.is_float else float(vals[i])
            if c.kind.is_text:
                row.append(c.dictionary.decode(v))
            elif c.kind.name == DATE:
                from .storage import days_to_date

                row.append(days_to_date(v))
            elif c.kind.is_decimal:
                row.append(format_decimal(v, c.kind.scale))
            else:
                row.append(str(v))
        writer.writerow(row)
    return out.getvalue()
