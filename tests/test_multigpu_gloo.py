"""The multi-GPU row partitioner's host logic at world_size 2 over gloo (CPU): contiguous row
ranges, the count/offset all_gather, the global UDF-failure reduction, and the rank-order
assembly of compacted slices — with each rank's local counts / slices computed by the oracle
(kernels need a GPU), checked against the oracle on the whole table."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import esc_oracle as O


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch

    from paper_1901_01488_b200 import multigpu

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 10_007
        g = np.random.default_rng(5)
        a = g.integers(0, 1000, n)
        b = g.integers(-50, 50, n)
        pred = ["or", [["range", ["a", None], 100, 299], ["cmp", ["b", None], ">", 40]]]
        lo, hi = multigpu.shard_bounds(n, world)[rank]
        local = O.OTable("t", {"a": O.OColumn(a[lo:hi], np.zeros(hi - lo, bool)),
                               "b": O.OColumn(b[lo:hi], np.zeros(hi - lo, bool))})
        rows = O.eval_predicate(local, pred)
        total, counts, offsets = multigpu.exchange_counts(int(rows.size))
        # slices concatenated in rank order (the sharded temp)
        sl = torch.from_numpy(a[lo:hi][rows].astype(np.int64))
        from types import SimpleNamespace

        cols = multigpu.gather_to_rank0([SimpleNamespace(values=sl)], counts)
        # global first-failing-row reduction (u64 words, ~0 = none)
        fail_local = [((int(rows[0]) + lo) << 3) | 1 if rows.size else (1 << 64) - 1, (1 << 64) - 1]
        fails = multigpu.allreduce_min(fail_local)
        if rank == 0:
            q.put((total, counts, offsets, cols[0].numpy().tolist(), fails))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_partition_exchange_and_assembly(world):
    n = 10_007
    g = np.random.default_rng(5)
    a = g.integers(0, 1000, n)
    b = g.integers(-50, 50, n)
    pred = ["or", [["range", ["a", None], 100, 299], ["cmp", ["b", None], ">", 40]]]
    whole = O.OTable("t", {"a": O.OColumn(a, np.zeros(n, bool)), "b": O.OColumn(b, np.zeros(n, bool))})
    want_rows = O.eval_predicate(whole, pred)

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    total, counts, offsets, assembled, fails = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    from paper_1901_01488_b200.multigpu import exclusive_offsets, shard_bounds

    assert total == want_rows.size and sum(counts) == total
    assert offsets == exclusive_offsets(counts) and offsets[0] == 0
    assert assembled == a[want_rows].tolist()          # rank-order concatenation == global row order
    assert fails[0] >> 3 == int(want_rows[0]) and fails[1] == (1 << 64) - 1
    b0 = shard_bounds(n, world)
    assert b0[0][0] == 0 and b0[-1][1] == n and all(b0[i][1] == b0[i + 1][0] for i in range(world - 1))


def _worker_shards(rank, world, port, q):
    """Sharded-table plumbing over gloo on CPU tensors: ShardInfo of shard_table, the int
    vector exchanges, and gather_columns (ragged slices with NULLs) == the whole table."""
    import traceback

    try:
        from paper_1901_01488_b200 import multigpu
        from paper_1901_01488_b200.storage import KIND_INT32, KIND_INT64, Column, ColumnTable

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        try:
            n = 1_003
            g = np.random.default_rng(3)
            a = g.integers(-50, 50, n).astype(np.int64)
            an = g.random(n) < 0.1
            b = g.integers(0, 9, n).astype(np.int32)
            full = ColumnTable("t", [Column("a", KIND_INT64, a, an, device="cpu"),
                                     Column("b", KIND_INT32, b, device="cpu")])
            sh = multigpu.shard_table(full, rank, world)
            info = sh.shard
            vec = multigpu.all_gather_ints([rank, 10 * rank + 1, -rank])
            tot = multigpu.allreduce_sum([rank + 1, 2])
            # ragged: keep a different number of rows on every rank
            keep = np.arange(sh.row_count) % (rank + 2) == 0
            loc = [Column(c.name, c.kind, c.values[torch.from_numpy(keep)],
                          c.nulls[torch.from_numpy(keep)] if c.nulls is not None else None, device="cpu")
                   for c in sh.columns]
            counts = [v[0] for v in multigpu.all_gather_ints([int(keep.sum())])]
            got = multigpu.gather_columns(loc, counts)
            q.put((rank, (info.offset, info.counts, sh.global_row_count, vec, tot, counts,
                          [c.to_numpy() for c in got], keep.tolist()), None))
        finally:
            dist.destroy_process_group()
    except BaseException:  # noqa: BLE001
        q.put((rank, None, traceback.format_exc()))


def test_sharded_tables_and_gathers():
    import torch  # noqa: F401

    from paper_1901_01488_b200.multigpu import shard_bounds

    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_shards, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, val, err = q.get(timeout=180)
        assert err is None, err
        res[rank] = val
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    n = 1_003
    g = np.random.default_rng(3)
    a = g.integers(-50, 50, n).astype(np.int64)
    an = g.random(n) < 0.1
    b = g.integers(0, 9, n).astype(np.int32)
    bounds = shard_bounds(n, world)
    keep_all = np.concatenate([np.array(res[r][7], bool) for r in range(world)])
    for r in range(world):
        off, counts, total, vec, tot, kept, cols, _ = res[r]
        assert off == bounds[r][0] and list(counts) == [hi - lo for lo, hi in bounds] and total == n
        assert vec == [[q_, 10 * q_ + 1, -q_] for q_ in range(world)]
        assert tot == [sum(range(1, world + 1)), 2 * world]
        assert kept == [int(np.array(res[x][7], bool).sum()) for x in range(world)]
        (va, ma), (vb, mb) = cols
        assert np.array_equal(ma, an[keep_all]) and np.array_equal(va[~ma], a[keep_all][~an[keep_all]])
        assert np.array_equal(vb, b[keep_all]) and not mb.any()
