"""The sharded ESC step (K3) on a real device: NCCL process group of one rank on cuda:0 (this
box has one GPU; NCCL refuses two ranks on one device, and ranks whose kernels wait on each other
must not share a GPU).  The device-resident path — K1 select, NCCL all_gather of the device
count, device-gated compaction, one host wait — must equal the single-GPU ESC step exactly; the
N-rank host logic is covered over gloo in test_multigpu_gloo.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group(cuda):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    yield
    dist.destroy_process_group()


def test_sharded_step_equals_single_gpu(cuda, nccl_group):
    from paper_1901_01488_b200 import Catalog, ColumnTable, expr as ex, multigpu, optimizer
    from paper_1901_01488_b200.errors import ExecutionError
    from paper_1901_01488_b200.storage import KIND_INT32, KIND_INT64, Column

    n = 3_000_003
    g = np.random.default_rng(8)
    x = g.integers(0, 100_000, n).astype(np.int32)
    y = g.integers(-(1 << 40), 1 << 40, n).astype(np.int64)
    yn = g.random(n) < 0.05
    t = ColumnTable("t", [Column("x", KIND_INT32, x, device=cuda), Column("y", KIND_INT64, y, yn, device=cuda)])
    cat = Catalog()
    cat.register(t)
    st = multigpu.ShardedTable("t", t, n, 0, 0, 1)
    cfg = optimizer.EscConfig()
    for hi in (99, 9_999, 29_999):  # qualifies, qualifies, over the 20% threshold
        p = ex.Range(ex.ColumnRef("t", "x"), 0, hi)
        d = multigpu.sharded_esc_subquery(st, p, ["y", "x"], cfg)
        ref = optimizer.esc_subquery(cat, "t", p, ["y", "x"], cfg)
        assert (d.exact_count, d.qualified, d.counts, d.offset) == (ref.exact_count, ref.qualified, [ref.exact_count], 0)
        if ref.pushed_down:
            want = cat.resolve_temp(ref.temp).columns
            for a, b in zip(d.columns, want):
                va, ma = a.to_numpy()
                vb, mb = b.to_numpy()
                assert (ma == mb).all() and (va[~ma] == vb[~mb]).all()
        else:
            assert d.columns is None
        cat.temps.sweep()
    bad = ex.FnCall("inv", (ex.ColumnRef("t", "x"),), ">", 0.5, lambda v: 1.0 / v)
    with pytest.raises(ExecutionError) as err:
        multigpu.sharded_esc_subquery(st, bad, ["x"], cfg)
    with pytest.raises(ExecutionError) as err2:
        optimizer.esc_subquery(cat, "t", bad, ["x"], cfg)
    assert str(err.value) == str(err2.value)
