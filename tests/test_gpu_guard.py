"""Out-of-bounds write checks of the C ABI (the pool forbids compute-sanitizer: runs under it
left GPUs needing a reset).  Every output, scratch and workspace buffer handed to an entry point
is an exact-size window into a larger allocation whose guard bands are filled with a canary
pattern; after the call the bands must be intact and the results must equal the oracle / numpy.
Sizes sweep the tile boundaries (128-row chunks, 1024/4096/8192-row tiles, the 2048-key sort
tile), the one-pass / mid-size / chained thresholds and capacities below, at and above the
count — where an off-by-one in a kernel's bounds would write past a buffer."""

import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

PAD = 4096
CANARY = 0xA5


class Guarded:
    """``nbytes`` usable bytes between two PAD-byte canary bands (device)."""

    def __init__(self, nbytes: int, dev, align: int = 256):
        self.nbytes = int(nbytes)
        self.buf = torch.full((PAD + max(self.nbytes, 1) + PAD + align,), CANARY, dtype=torch.uint8, device=dev)
        base = self.buf.data_ptr()
        self.off = PAD + (-(base + PAD) % align)
        self.ptr = base + self.off

    def view(self, dtype, count):
        return self.buf[self.off:self.off + count * torch.tensor([], dtype=dtype).element_size()].view(dtype)

    def intact(self) -> bool:
        torch.cuda.synchronize()
        b = self.buf.cpu().numpy()
        return bool((b[: self.off] == CANARY).all() and (b[self.off + self.nbytes:] == CANARY).all())


def _result():
    """A kernel result block in pinned host memory (the last CTA writes it through UVA)."""
    from paper_1901_01488_b200 import _native as N

    t = torch.zeros(C.sizeof(N.EscResult), dtype=torch.uint8, pin_memory=True)
    return t, N.EscResult.from_address(t.data_ptr())


def _check(*bufs):
    for i, g in enumerate(bufs):
        assert g.intact(), f"guard band {i} overwritten"


def _table(n, dev, seed=1):
    from paper_1901_01488_b200.storage import KIND_INT32, KIND_INT64, Column, ColumnTable

    g = np.random.default_rng(seed)
    a = g.integers(0, 1000, n).astype(np.int32)
    b = g.integers(-(1 << 40), 1 << 40, n).astype(np.int64)
    bn = g.random(n) < 0.1
    t = ColumnTable("t", [Column("a", KIND_INT32, a, device=dev), Column("b", KIND_INT64, b, bn, device=dev)])
    return t, a, b, bn


SIZES = [1, 127, 128, 1025, 4097, 8193, 65_537, (1 << 21) + 3, 3_000_005]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("route", ["chain", "mid", "stream", "hitlist"])
def test_select_and_materialize_stay_in_bounds(cuda, n, route):
    from paper_1901_01488_b200 import _native as N, expr as ex
    from paper_1901_01488_b200.compiler import compile_predicate

    lib = N.load_library()
    prev_mid = N.set_mid_max_rows(1 << 40 if route == "mid" else 0)
    prev_div = N.set_stream_div(1 << 30 if route == "stream" else 32)
    prev_hl = N.set_hit_lists(2 if route == "hitlist" else 1)
    try:
        t, a, b, bn = _table(n, cuda)
        for hi in (9, 499, 999):  # ~1%, 50%, 100% of the rows
            pred = ex.Range(ex.ColumnRef("t", "a"), 0, hi)
            want = np.flatnonzero(a <= hi)
            cp = compile_predicate(t, pred)
            words, segs, cap_entries = C.c_int64(), C.c_int64(), C.c_int64()
            lib.esc_selection_sizes(n, C.byref(words), C.byref(segs), C.byref(cap_entries))
            ws = Guarded(lib.esc_workspace_bytes(n), cuda)
            N.check(lib.esc_workspace_init(C.c_void_p(ws.ptr), C.c_size_t(ws.nbytes), None), "init")
            bm, sc = Guarded(words.value * 4, cuda), Guarded(segs.value * 4, cuda)
            capv = Guarded(cap_entries.value * 4, cuda)
            sel = N.EscSelection()
            sel.bitmap, sel.seg_counts = bm.ptr, sc.ptr
            sel.n_cap = 1
            sel.cap_slot[0] = cp.slot_of["a"]
            sel.cap_values[0] = capv.ptr
            res_t, res = _result()
            stream = torch.cuda.current_stream().cuda_stream
            N.check(lib.esc_scan_select(C.byref(cp.program), cp.column_array(), cp.ncols, n, None, C.byref(sel),
                                        C.c_void_p(res_t.data_ptr()), C.c_void_p(ws.ptr), C.c_size_t(ws.nbytes), C.c_void_p(stream)),
                    "esc_scan_select")
            torch.cuda.synchronize()
            assert res.count == want.size
            cols = (N.EscColumn * 2)()
            for i, c in enumerate(("a", "b")):
                col = t.column(c)
                cols[i].data = col.values.data_ptr()
                cols[i].nulls = col.nulls.data_ptr() if col.nulls is not None else None
                cols[i].dtype = N.dtype_code(col.values)
            # the scan's own column array decides slot numbering: map a/b onto it when present
            scan_cols = cp.column_array()
            slot_a = cp.slot_of["a"]
            for cap in (max(want.size - 3, 0), want.size, want.size + 5):
                mcols = (N.EscColumn * (cp.ncols + 1))()
                for i in range(cp.ncols):
                    mcols[i] = scan_cols[i]
                mcols[cp.ncols] = cols[1]
                va, vb, nb, rid = (Guarded(cap * 4, cuda), Guarded(cap * 8, cuda), Guarded(cap, cuda),
                                   Guarded(cap * 8, cuda))
                outs = N.EscOutputs()
                outs.n_proj = 2
                outs.capacity = cap
                outs.slot[0], outs.slot[1] = slot_a, cp.ncols
                outs.out_values[0], outs.out_values[1] = va.ptr, vb.ptr
                outs.out_nulls[1] = nb.ptr
                outs.out_row_ids = rid.ptr
                N.check(lib.esc_materialize_selection(C.byref(sel), n, mcols, cp.ncols + 1, None, C.byref(outs),
                                                      C.c_void_p(ws.ptr), C.c_size_t(ws.nbytes), C.c_void_p(stream)),
                        "esc_materialize_selection")
                _check(va, vb, nb, rid, ws, bm, sc, capv)
                k = min(cap, want.size)
                assert np.array_equal(rid.view(torch.int64, k).cpu().numpy(), want[:k])
                assert np.array_equal(va.view(torch.int32, k).cpu().numpy(), a[want[:k]])
                assert np.array_equal(nb.view(torch.uint8, k).cpu().numpy().astype(bool), bn[want[:k]])
                vv = vb.view(torch.int64, k).cpu().numpy()
                assert np.array_equal(vv[~bn[want[:k]]], b[want[:k]][~bn[want[:k]]])
    finally:
        N.set_mid_max_rows(prev_mid)
        N.set_stream_div(prev_div)
        N.set_hit_lists(prev_hl)


@pytest.mark.parametrize("n", [1, 127, 4097, 65_537, 300_001])
def test_onepass_stays_in_bounds(cuda, n):
    from paper_1901_01488_b200 import _native as N, expr as ex
    from paper_1901_01488_b200.compiler import compile_predicate

    lib = N.load_library()
    t, a, _, _ = _table(n, cuda, seed=2)
    pred = ex.Range(ex.ColumnRef("t", "a"), 100, 349)
    want = np.flatnonzero((a >= 100) & (a <= 349))
    cp = compile_predicate(t, pred)
    ws = Guarded(lib.esc_workspace_bytes(n), cuda)
    N.check(lib.esc_workspace_init(C.c_void_p(ws.ptr), C.c_size_t(ws.nbytes), None), "init")
    for cap in (0, max(want.size // 2, 1), want.size, want.size + 1):
        va, rid = Guarded(cap * 4, cuda), Guarded(cap * 8, cuda)
        outs = N.EscOutputs()
        outs.n_proj = 1
        outs.capacity = cap
        outs.slot[0] = cp.slot_of["a"]
        outs.out_values[0] = va.ptr if cap else None
        outs.out_row_ids = rid.ptr if cap else None
        res_t, res = _result()
        N.check(lib.esc_compact_onepass(C.byref(cp.program), cp.column_array(), cp.ncols, n, None, C.byref(outs),
                                        C.c_void_p(res_t.data_ptr()), C.c_void_p(ws.ptr), C.c_size_t(ws.nbytes),
                                        C.c_void_p(torch.cuda.current_stream().cuda_stream)), "esc_compact_onepass")
        _check(va, rid, ws)
        torch.cuda.synchronize()
        k = min(cap, want.size)
        assert res.count == want.size
        assert np.array_equal(rid.view(torch.int64, k).cpu().numpy(), want[:k])


@pytest.mark.parametrize("n", [1, 2047, 2048, 2049, 100_003])
@pytest.mark.parametrize("kb", [4, 8])
def test_sort_and_runs_stay_in_bounds(cuda, n, kb):
    from paper_1901_01488_b200 import _native as N

    lib = N.load_library()
    g = np.random.default_rng(n + kb)
    k = g.integers(0, 50, n).astype(np.uint32 if kb == 4 else np.uint64)
    v = np.arange(n, dtype=np.int64)
    kin = torch.from_numpy(k.view(np.int32 if kb == 4 else np.int64)).to(cuda)
    vin = torch.from_numpy(v).to(cuda)
    ko, vo = Guarded(n * kb, cuda), Guarded(n * 8, cuda)
    tmp = Guarded(lib.esc_sort_temp_bytes(n, kb, 1), cuda)
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    N.check(lib.esc_sort_pairs(C.c_void_p(kin.data_ptr()), C.c_void_p(vin.data_ptr()), C.c_void_p(ko.ptr),
                               C.c_void_p(vo.ptr), n, kb, 0, 8 * kb, C.c_void_p(tmp.ptr), C.c_size_t(tmp.nbytes), stream),
            "esc_sort_pairs")
    _check(ko, vo, tmp)
    order = np.argsort(k, kind="stable")
    assert np.array_equal(vo.view(torch.int64, n).cpu().numpy(), order)
    uk, st, ct, ro, stats = (Guarded(n * 8, cuda), Guarded((n + 1) * 8, cuda), Guarded(n * 8, cuda),
                             Guarded(n * 8, cuda), Guarded(32, cuda))
    tmp2 = Guarded(lib.esc_sort_temp_bytes(n, kb, 0), cuda)
    N.check(lib.esc_runs(C.c_void_p(ko.ptr), kb, 0, n, C.c_void_p(uk.ptr), C.c_void_p(st.ptr), C.c_void_p(ct.ptr),
                         C.c_void_p(ro.ptr), C.c_void_p(stats.ptr), C.c_void_p(tmp2.ptr), C.c_size_t(tmp2.nbytes), stream),
            "esc_runs")
    _check(uk, st, ct, ro, stats, tmp2)
    u = int(stats.view(torch.int64, 4)[0])
    assert u == np.unique(k).size


@pytest.mark.parametrize("n", [1, 1000, 16_384, 16_385, 70_001])
def test_hash_build_stays_in_bounds(cuda, n):
    from paper_1901_01488_b200 import _native as N

    lib = N.load_library()
    g = np.random.default_rng(n)
    keys = torch.from_numpy(g.integers(-500, 500, n).astype(np.int32)).to(cuda)
    tb = C.c_size_t()
    N.check(lib.esc_hash_build_temp_bytes(n, C.byref(tb)), "temp bytes")
    rows, uk, cnt, start, stats, tmp = (Guarded(n * 8, cuda), Guarded(n * 8, cuda), Guarded((n + 1) * 8, cuda),
                                        Guarded((n + 1) * 8, cuda), Guarded(32, cuda), Guarded(tb.value, cuda))
    N.check(lib.esc_hash_build(C.c_void_p(keys.data_ptr()), N.dtype_code(keys), None, n, C.c_void_p(rows.ptr),
                               C.c_void_p(uk.ptr), C.c_void_p(cnt.ptr), C.c_void_p(start.ptr), C.c_void_p(stats.ptr),
                               C.c_void_p(tmp.ptr), C.c_size_t(tmp.nbytes),
                               C.c_void_p(torch.cuda.current_stream().cuda_stream)), "esc_hash_build")
    _check(rows, uk, cnt, start, stats, tmp)
    u = int(stats.view(torch.int64, 4)[0])
    kn = keys.cpu().numpy()
    assert u == np.unique(kn).size
    assert np.array_equal(rows.view(torch.int64, n).cpu().numpy(), np.argsort(kn, kind="stable"))
