"""The framework's own device sort and grouping (csrc/esc_sort.cuh) against numpy: stable radix
sort of 32/64-bit keys with values (== np.argsort(kind="stable")), the runs of a sorted array
(== np.unique with first indices and counts), order-preserving key encodings, the first-appearance
dictionary codes of the CSV loader, and the large-build path of esc_hash_build (== the
reference's np.unique + stable argsort grouping, via the oracle)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SIZES = [1, 2, 2047, 2048, 2049, 5 * 2048 + 7, 100_003, 1_000_000]


def _keys(kind, n, g, kb):
    hi = (1 << 32) if kb == 4 else (1 << 63)
    if kind == "uniform":
        return g.integers(0, hi, n, dtype=np.uint64 if kb == 8 else np.int64)
    if kind == "few":
        return g.choice(np.array([7, 3, hi - 1, 0], dtype=np.uint64), n)
    if kind == "equal":
        return np.full(n, 12345, dtype=np.uint64)
    return np.sort(g.integers(0, 1 << 20, n))[::-1].copy()  # descending


@pytest.mark.parametrize("kb", [4, 8])
@pytest.mark.parametrize("kind", ["uniform", "few", "equal", "descending"])
def test_sort_pairs_is_stable_argsort(cuda, kb, kind):
    from paper_1901_01488_b200 import sorting

    g = np.random.default_rng(kb * 31 + len(kind))
    for n in SIZES:
        k = _keys(kind, n, g, kb).astype(np.uint32 if kb == 4 else np.uint64)
        v = g.integers(-(1 << 62), 1 << 62, n)
        kt = torch.from_numpy(k.view(np.int32 if kb == 4 else np.int64)).to(cuda)
        sk, sv = sorting.sort_pairs(kt, torch.from_numpy(v).to(cuda))
        order = np.argsort(k, kind="stable")
        assert np.array_equal(sk.cpu().numpy().view(k.dtype), k[order]), (kind, n)
        assert np.array_equal(sv.cpu().numpy(), v[order]), (kind, n)
        sk2, none = sorting.sort_pairs(kt)  # keys only
        assert none is None and np.array_equal(sk2.cpu().numpy().view(k.dtype), k[order])


def test_sort_partial_bits(cuda):
    """Sorting by the low bits only (the dictionary's second sort uses 32 of 32, the hash build 32
    of 32; a 20-bit range must still be stable by those bits)."""
    from paper_1901_01488_b200 import sorting

    g = np.random.default_rng(4)
    k = g.integers(0, 1 << 20, 300_001).astype(np.uint32)
    v = np.arange(k.size, dtype=np.int64)
    sk, sv = sorting.sort_pairs(torch.from_numpy(k.view(np.int32)).to(cuda), torch.from_numpy(v).to(cuda), key_bits=20)
    order = np.argsort(k, kind="stable")
    assert np.array_equal(sv.cpu().numpy(), v[order])


@pytest.mark.parametrize("kb", [4, 8])
def test_runs_match_numpy_unique(cuda, kb):
    from paper_1901_01488_b200 import sorting

    g = np.random.default_rng(9 + kb)
    for n in SIZES:
        for card in (1, 5, 1000, n):
            k = np.sort(g.integers(0, card, n).astype(np.uint32 if kb == 4 else np.uint64))
            uk, starts, counts, run_of, stats = sorting.runs(torch.from_numpy(k.view(np.int32 if kb == 4 else np.int64)).to(cuda),
                                                             sorting.KEY_RAW, want_run_of=True)
            u_np, first_np, inv_np, cnt_np = np.unique(k, return_index=True, return_inverse=True, return_counts=True)
            s = stats.cpu().tolist()
            u = s[0]
            assert u == u_np.size and s[1] == int(u_np[0]) and s[2] == int(u_np[-1]) and s[3] == int(cnt_np.max())
            assert np.array_equal(uk[:u].cpu().numpy(), u_np.astype(np.int64))
            assert np.array_equal(starts[:u + 1].cpu().numpy(), np.append(first_np, n))
            assert np.array_equal(counts[:u].cpu().numpy(), cnt_np)
            assert np.array_equal(run_of[:n].cpu().numpy(), inv_np)


@pytest.mark.parametrize("dtype", [np.int8, np.int16, np.int32, np.int64, np.uint8])
def test_ordered_keys_round_trip(cuda, dtype):
    from paper_1901_01488_b200 import sorting

    info = np.iinfo(dtype)
    g = np.random.default_rng(2)
    x = g.integers(info.min, int(info.max) + 1, 70_001, dtype=np.int64).astype(dtype)
    x[:4] = [info.min, info.max, 0, info.min + 1] if info.min < 0 else [0, info.max, 1, 2]
    keys, kb, dec = sorting.ordered_keys(torch.from_numpy(x).to(cuda))
    sk, _ = sorting.sort_pairs(keys)
    uk, starts, counts, _, stats = sorting.runs(sk, dec)
    u = int(stats[0])
    want = np.unique(x.astype(np.int64))
    assert np.array_equal(uk[:u].cpu().numpy(), want)


@pytest.mark.parametrize("null_fraction", [0.0, 0.2, 1.0])
def test_dict_encode_first_appearance(cuda, null_fraction):
    """Codes in first-appearance order, representatives = first rows, NULLs coded 0 / rep -1 —
    the reference's Dictionary.encode over the cells in row order."""
    from paper_1901_01488_b200 import sorting

    g = np.random.default_rng(17)
    for n in (1, 2049, 200_001):
        h = g.choice(g.integers(-(1 << 63), (1 << 63) - 1, 40, dtype=np.int64), n)
        nulls = g.random(n) < null_fraction
        codes, rep, first, u = sorting.dict_encode(torch.from_numpy(h).to(cuda), torch.from_numpy(nulls).to(cuda))
        seen, want_codes, want_rep, firsts = {}, [], [], []
        for i, (x, nl) in enumerate(zip(h.tolist(), nulls.tolist())):
            if nl:
                want_codes.append(0)
                want_rep.append(-1)
                continue
            key = x >> 1 if x >= 0 else (x + (1 << 64)) >> 1  # the device groups by hash >> 1
            if key not in seen:
                seen[key] = (len(firsts), i)
                firsts.append(i)
            want_codes.append(seen[key][0])
            want_rep.append(seen[key][1])
        assert u == len(firsts)
        assert codes.cpu().tolist() == want_codes
        assert rep.cpu().tolist() == want_rep
        assert first.cpu().tolist() == firsts


@pytest.mark.parametrize("dtype", ["INT64", "INT32", "INT8", "INT16"])
def test_large_hash_build_grouping(cuda, dtype):
    """esc_hash_build above the one-block size (the device-wide sort path) == the oracle's
    np.unique + stable argsort grouping: unique keys, group rows in ascending row order,
    statistics; with negative keys, duplicates and a row-id subset."""
    from oracle import esc_oracle as O
    from paper_1901_01488_b200 import join
    from paper_1901_01488_b200.storage import Column, ColumnTable, parse_kind

    np_dt = {"INT64": np.int64, "INT32": np.int32, "INT8": np.int8, "INT16": np.int16}[dtype]
    info = np.iinfo(np_dt)
    g = np.random.default_rng(23)
    n = 300_007
    keys = g.integers(max(info.min, -50_000), min(int(info.max), 50_000) + 1, n).astype(np_dt)
    keys[:3] = [info.min, info.max, 0]
    t = ColumnTable("b", [Column("k", parse_kind(dtype), keys, device=cuda)])
    rows = np.sort(g.choice(n, n // 2, replace=False)).astype(np.int64)
    for sel in (None, rows):
        idx = join.HashTableIndex(t, "k", torch.from_numpy(sel).to(cuda) if sel is not None else None)
        ot = O.OTable("b", {"k": O.OColumn(keys.astype(np.int64), np.zeros(n, bool))})
        oi = O.build_index(ot, "k", sel if sel is not None else np.arange(n))
        assert np.array_equal(idx.unique_keys.cpu().numpy(), oi.unique_keys)
        assert np.array_equal(idx.group_rows.cpu().numpy(), oi.group_rows)
        assert np.array_equal(idx.group_start.cpu().numpy()[: len(oi.group_start)], oi.group_start)


@pytest.mark.parametrize("dtype", ["uint8", "uint16", "uint32", "int8", "int16", "int32"])
def test_one_block_hash_build_matches_numpy(cuda, dtype):
    """The one-block build (<= 8K rows, keys <= 4 bytes; larger ones take the device-wide sort)
    against numpy's unique + stable argsort,
    for unsigned keys (bias 0) and keys equal to the 32-bit padding sentinel (0xFFFFFFFF after
    the bias: INT32_MAX, UINT32_MAX), with duplicates and a row subset."""
    from paper_1901_01488_b200 import join
    from paper_1901_01488_b200.storage import Column, ColumnKind, ColumnTable

    np_dt = np.dtype(dtype)
    info = np.iinfo(np_dt)
    g = np.random.default_rng(5)
    for n in (1, 100, 8192, 8193, 16_384):
        keys = g.integers(int(info.min), int(info.max) + 1, n, dtype=np.int64).astype(np_dt)
        keys[: min(n, 3)] = info.max  # the sentinel after biasing, and duplicates of it
        if n > 10:
            keys[5:9] = info.min
        t = ColumnTable("b", [Column("k", ColumnKind("INT64"), keys, device=cuda)])
        rows = np.sort(g.choice(n, max(n // 2, 1), replace=False)).astype(np.int64)
        for sel in (None, rows):
            idx = join.HashTableIndex(t, "k", torch.from_numpy(sel).to(cuda) if sel is not None else None)
            sub = keys.astype(np.int64) if sel is None else keys.astype(np.int64)[sel]
            base = np.arange(n) if sel is None else sel
            u = np.unique(sub)
            order = np.argsort(sub, kind="stable")
            assert np.array_equal(idx.unique_keys.cpu().numpy(), u), (dtype, n)
            assert np.array_equal(idx.group_rows.cpu().numpy(), base[order]), (dtype, n)
