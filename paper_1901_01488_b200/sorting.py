"""Device sort and grouping through the framework's own kernels (``csrc/esc_sort.cuh``).

The planner's neighbours need numpy's ``np.sort`` / stable ``argsort`` / ``np.unique`` in three
places — the hash build's grouping (f1, reference ``executor.py:275-303``), the CSV loader's TEXT
dictionary in first-appearance order (f3, ``storage.py:127-153, :247-275``) and the histogram
arm's value sort (f4, ``catalog.py:178-223``).  These wrappers run them on the device: a stable
LSD radix sort of 32/64-bit unsigned keys with 64-bit values carried along, and the runs of a
sorted key array.  Equal keys keep their input order, so results match numpy's stable sorts
element for element.  No library kernels, no CPU fallback.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from . import executor

KEY_RAW, KEY_U32, KEY_I32, KEY_I64 = 0, 1, 2, 3  # esc_runs decodings of the stored keys


def _temp(n: int, key_bytes: int, with_values: bool, dev) -> torch.Tensor:
    nb = int(N.load_library().esc_sort_temp_bytes(max(n, 1), key_bytes, 1 if with_values else 0))
    return torch.empty(max(nb, 1), dtype=torch.uint8, device=dev)


def ordered_keys(values: torch.Tensor) -> tuple[torch.Tensor, int, int]:
    """Order-preserving unsigned sort keys of an integer column (esc_order_keys): int8/16/32 ->
    uint32 ^ 2^31, uint8 -> uint32, int64 -> uint64 ^ 2^63.  Returns (keys as an int32/int64
    tensor holding the unsigned bits, key bytes, the esc_runs decoding)."""
    N.require_cuda(values, "sort keys")
    code = N.dtype_code(values)
    if values.dtype == torch.int64:
        kb, dec = 8, KEY_I64
    elif values.dtype == torch.uint8:
        kb, dec = 4, KEY_U32
    elif values.dtype in (torch.int8, torch.int16, torch.int32):
        kb, dec = 4, KEY_I32
    else:
        raise TypeError(f"cannot radix-sort {values.dtype}")
    n = int(values.numel())
    out = torch.empty(max(n, 1), dtype=torch.int64 if kb == 8 else torch.int32, device=values.device)
    if n:
        N.check(N.load_library().esc_order_keys(C.c_void_p(values.contiguous().data_ptr()), code, n,
                                                C.c_void_p(out.data_ptr()),
                                                C.c_void_p(executor._stream(values.device).cuda_stream)),
                "esc_order_keys")
    return out[:n], kb, dec


def sort_pairs(keys: torch.Tensor, values: torch.Tensor | None = None, key_bits: int | None = None):
    """Stable device sort of unsigned keys (int32 / int64 tensors holding the unsigned bit
    patterns) by their low ``key_bits`` bits, with int64 ``values`` carried along.  Returns
    (sorted keys, sorted values or None)."""
    N.require_cuda(keys, "sort keys")
    kb = keys.element_size()
    if kb not in (4, 8):
        raise TypeError("sort keys must be 4- or 8-byte integers")
    n = int(keys.numel())
    dev = keys.device
    keys = keys.contiguous()
    out_k = torch.empty_like(keys)
    out_v = None
    if values is not None:
        values = values.to(torch.int64).contiguous()
        out_v = torch.empty_like(values)
    if n == 0:
        return out_k, out_v
    bits = key_bits if key_bits is not None else 8 * kb
    tmp = _temp(n, kb, values is not None, dev)
    stream = executor._stream(dev)
    N.check(N.load_library().esc_sort_pairs(C.c_void_p(keys.data_ptr()),
                                            C.c_void_p(values.data_ptr()) if values is not None else None,
                                            C.c_void_p(out_k.data_ptr()),
                                            C.c_void_p(out_v.data_ptr()) if out_v is not None else None,
                                            n, kb, 0, bits, C.c_void_p(tmp.data_ptr()), C.c_size_t(tmp.numel()),
                                            C.c_void_p(stream.cuda_stream)), "esc_sort_pairs")
    return out_k, out_v


def runs(sorted_keys: torch.Tensor, decode: int = KEY_RAW, want_run_of: bool = False, want_counts: bool = True):
    """Runs of a sorted key array (device): (unique keys int64, starts int64[runs+1], counts or
    None, run_of int64[n] or None, stats int64[4] = runs, first, last, largest run).  The arrays
    are sized for n runs; slice them by stats[0] after reading it."""
    n = int(sorted_keys.numel())
    dev = sorted_keys.device
    kb = sorted_keys.element_size()
    uk = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    starts = torch.empty(n + 1, dtype=torch.int64, device=dev)
    counts = torch.empty(max(n, 1), dtype=torch.int64, device=dev) if want_counts else None
    run_of = torch.empty(max(n, 1), dtype=torch.int64, device=dev) if want_run_of else None
    stats = torch.empty(4, dtype=torch.int64, device=dev)
    tmp = _temp(n, kb, False, dev)
    stream = executor._stream(dev)
    N.check(N.load_library().esc_runs(C.c_void_p(sorted_keys.contiguous().data_ptr()), kb, decode, n,
                                      C.c_void_p(uk.data_ptr()), C.c_void_p(starts.data_ptr()),
                                      C.c_void_p(counts.data_ptr()) if counts is not None else None,
                                      C.c_void_p(run_of.data_ptr()) if run_of is not None else None,
                                      C.c_void_p(stats.data_ptr()), C.c_void_p(tmp.data_ptr()),
                                      C.c_size_t(tmp.numel()), C.c_void_p(stream.cuda_stream)), "esc_runs")
    return uk, starts, counts, run_of, stats


def rank_values(unique_keys, starts, stats, ranks: torch.Tensor) -> torch.Tensor:
    """Values of a column given as runs at sorted positions ``ranks`` (device int64)."""
    k = int(ranks.numel())
    out = torch.empty(max(k, 1), dtype=torch.int64, device=ranks.device)
    N.check(N.load_library().esc_rank_values(C.c_void_p(unique_keys.data_ptr()), C.c_void_p(starts.data_ptr()),
                                             C.c_void_p(stats.data_ptr()), C.c_void_p(ranks.data_ptr()), k,
                                             C.c_void_p(out.data_ptr()),
                                             C.c_void_p(executor._stream(ranks.device).cuda_stream)),
            "esc_rank_values")
    return out[:k]


def hist_buckets(unique_keys, starts, stats, n: int, bounds: torch.Tensor):
    """(hi, distinct) per equi-depth bucket over a column given as runs (esc_hist_buckets)."""
    nb = int(bounds.numel()) - 1
    dev = bounds.device
    hi = torch.empty(max(nb, 1), dtype=torch.int64, device=dev)
    distinct = torch.empty(max(nb, 1), dtype=torch.int64, device=dev)
    N.check(N.load_library().esc_hist_buckets(C.c_void_p(unique_keys.data_ptr()), C.c_void_p(starts.data_ptr()),
                                              C.c_void_p(stats.data_ptr()), n, C.c_void_p(bounds.data_ptr()), nb,
                                              C.c_void_p(hi.data_ptr()), C.c_void_p(distinct.data_ptr()),
                                              C.c_void_p(executor._stream(dev).cuda_stream)), "esc_hist_buckets")
    return hi[:nb], distinct[:nb]


def dict_encode(hashes: torch.Tensor, nulls: torch.Tensor | None):
    """First-appearance dictionary codes of TEXT cells from their content hashes (esc_dict_encode):
    (codes int32[n], representative row int64[n] (-1 for NULL), first row of every code
    int64[n_codes], n_codes)."""
    n = int(hashes.numel())
    dev = hashes.device
    lib = N.load_library()
    codes = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    rep = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    first = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    n_codes = torch.tensor([0], dtype=torch.int64, device=dev)  # a host copy, not a fill kernel
    tmp = torch.empty(max(int(lib.esc_dict_temp_bytes(n)), 1), dtype=torch.uint8, device=dev)
    nl = None
    if nulls is not None:  # bool bytes are 0 / 1: viewed, not converted
        nl = (nulls.view(torch.uint8) if nulls.dtype == torch.bool else nulls.to(torch.uint8)).contiguous()
    N.check(lib.esc_dict_encode(C.c_void_p(hashes.contiguous().data_ptr()),
                                C.c_void_p(nl.data_ptr()) if nl is not None else None, n,
                                C.c_void_p(codes.data_ptr()), C.c_void_p(rep.data_ptr()), C.c_void_p(first.data_ptr()),
                                C.c_void_p(n_codes.data_ptr()), C.c_void_p(tmp.data_ptr()), C.c_size_t(tmp.numel()),
                                C.c_void_p(executor._stream(dev).cuda_stream)), "esc_dict_encode")
    u = int(n_codes.item())
    return codes[:n], rep[:n], first[:u], u
