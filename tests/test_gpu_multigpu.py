"""The sharded ESC step and the planner over row-partitioned tables, at world size 2 and 3.

This box has one GPU, so the ranks are processes sharing cuda:0 and exchange over gloo: the
collectives go through host memory, but every kernel, the device count gate and the code path
from ``optimizer.plan`` / ``Engine.run`` down to the gated compaction are the ones NCCL ranks
run (no rank's kernel waits on another's).  Every result must equal the single-GPU path on the
whole table: global counts, decisions, rank-order concatenation of the sharded temps, join order,
join counts and rows, and the reference's UDF error text.  A one-rank NCCL group checks the NCCL
transport of the same step."""

import os
import socket
import traceback

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# ------------------------------------------------------------------------------------------------
# scenarios (run in every rank; return picklable results)
# ------------------------------------------------------------------------------------------------
def _esc_scenario(rank, world, dev):
    from paper_1901_01488_b200 import Catalog, ColumnTable, expr as ex, multigpu, optimizer
    from paper_1901_01488_b200.errors import ExecutionError
    from paper_1901_01488_b200.storage import KIND_INT32, KIND_INT64, Column

    out = []
    for n in (1_000_003, 40_001):  # queued path (ESC_ONEPASS_MAX_ROWS lowered) / one-pass path
        g = np.random.default_rng(8 + n)
        x = g.integers(0, 100_000, n).astype(np.int32)
        if n < 100_000:  # the only zero (UDF failure) in the LAST rank's rows
            x[x == 0] = 1
            x[n - 7] = 0
        y = g.integers(-(1 << 40), 1 << 40, n).astype(np.int64)
        yn = g.random(n) < 0.05
        full = ColumnTable("t", [Column("x", KIND_INT32, x, device=dev), Column("y", KIND_INT64, y, yn, device=dev)])
        cat = Catalog()
        cat.register(full)
        lo, hi = multigpu.shard_bounds(n, world)[rank]
        st = multigpu.ShardedTable("t", ColumnTable("t", [Column("x", KIND_INT32, x[lo:hi], device=dev),
                                                          Column("y", KIND_INT64, y[lo:hi], yn[lo:hi], device=dev)]),
                                   n, lo, rank, world)
        cfg = optimizer.EscConfig()
        for hi_x in (99, 9_999, 29_999):  # qualifies, qualifies, over the 20% threshold
            p = ex.Range(ex.ColumnRef("t", "x"), 0, hi_x)
            d = multigpu.sharded_esc_subquery(st, p, ["y", "x"], cfg)
            ref = optimizer.esc_subquery(cat, "t", p, ["y", "x"], cfg)
            want = None
            if ref.pushed_down:
                want = [c.to_numpy() for c in cat.resolve_temp(ref.temp).columns]
            got = [c.to_numpy() for c in d.columns] if d.columns is not None else None
            out.append({"n": n, "hi": hi_x, "count": d.exact_count, "qualified": d.qualified, "counts": d.counts,
                        "offset": d.offset, "local": d.local_count, "slice": got,
                        "ref": (ref.exact_count, ref.qualified, want)})
            cat.temps.sweep()
        # a UDF that fails on one row only (x == 0 somewhere): the first failing GLOBAL row and
        # the reference's message, on every rank
        bad = ex.FnCall("inv", (ex.ColumnRef("t", "x"),), ">", 0.5, lambda v: 1.0 / v)
        msgs = []
        for fn in (lambda: multigpu.sharded_esc_subquery(st, bad, ["x"], cfg),
                   lambda: optimizer.esc_subquery(cat, "t", bad, ["x"], cfg)):
            try:
                fn()
                msgs.append(None)
            except ExecutionError as exc:
                msgs.append(str(exc))
        out.append({"n": n, "errors": msgs})
    return out


def _star_tables(dev, fact_rows):
    from paper_1901_01488_b200 import datagen
    from paper_1901_01488_b200.storage import Column, ColumnTable, Dictionary, parse_kind

    g = datagen.config3(fact_rows=fact_rows)
    names = {"date": "dates"}
    return {names.get(t, t): ColumnTable(names.get(t, t), [
        Column(c, parse_kind(s[0]), s[1], None, Dictionary(s[2]) if len(s) > 2 else None, device=dev)
        for c, s in cols.items()]) for t, cols in g.items()}


def _star_query(cat):
    from paper_1901_01488_b200 import datagen, expr as ex, ra, serde

    names = {"date": "dates"}
    r = ex.ColumnRef
    conj = [ex.ColumnCompare(r("fact", a), "=", r(names.get(d, d), b)) for _, a, d, b in datagen.CONFIG3_EDGES]
    conj += [serde.from_json(j, names.get(d, d)) for d, j in datagen.CONFIG3_WHERE.items()]
    return ra.query(cat, ["fact", "dates", "customer", "supplier", "part"], ex.And(tuple(conj)))


def _star_scenario(rank, world, dev):
    """Config 3 (exact dimension recipes, 2M-row fact): every table row-partitioned; Engine.run
    on the shards vs Engine.run on the whole tables."""
    from paper_1901_01488_b200 import Engine, multigpu

    full = _star_tables(dev, 2_000_000)
    single = Engine()
    sharded = Engine()
    for t in full.values():
        single.catalog.register(t)
        sharded.catalog.register(multigpu.shard_table(t, rank, world))
    q1, q2 = _star_query(single.catalog), _star_query(sharded.catalog)
    r1 = single.run(q1)
    r2 = sharded.run(q2)
    dec = lambda p: [(d.table, d.exact_count, d.row_count, d.qualified, d.pushed_down) for d in p.decisions]
    return {"single": (dec(r1.plan), r1.plan.build_order, r1.plan.build_card_sum, r1.count, r1.stats.probe_out),
            "sharded": (dec(r2.plan), r2.plan.build_order, r2.plan.build_card_sum, r2.count, r2.stats.probe_out),
            "live_temps": sharded.catalog.temps.live_handles()}


def _rows_scenario(rank, world, dev):
    """A projection over a 2-step join (duplicate and NULL keys, a pushed-down dimension and a
    base build with a residual): the ranks' result slices in rank order == the single-GPU rows."""
    from paper_1901_01488_b200 import Engine, expr as ex, multigpu, ra
    from paper_1901_01488_b200.storage import KIND_INT32, KIND_INT64, Column, ColumnTable

    g = np.random.default_rng(77)
    nf, nd, ne = 300_001, 5_000, 3_000
    fk = g.integers(0, 6_000, nf).astype(np.int64)
    fk_n = g.random(nf) < 0.03
    fe = g.integers(0, 4_000, nf).astype(np.int32)
    fv = g.integers(-10**9, 10**9, nf).astype(np.int64)
    dk = g.integers(0, 6_000, nd).astype(np.int64)     # duplicate keys
    dv = g.integers(0, 100, nd).astype(np.int32)
    ek = np.arange(ne, dtype=np.int32)
    ew = g.integers(0, 1000, ne).astype(np.int32)
    tabs = [ColumnTable("f", [Column("fk", KIND_INT64, fk, fk_n, device=dev), Column("fe", KIND_INT32, fe, device=dev),
                              Column("fv", KIND_INT64, fv, device=dev)]),
            ColumnTable("d", [Column("dk", KIND_INT64, dk, device=dev), Column("dv", KIND_INT32, dv, device=dev)]),
            ColumnTable("e", [Column("ek", KIND_INT32, ek, device=dev), Column("ew", KIND_INT32, ew, device=dev)])]
    r = ex.ColumnRef
    pred = ex.And((ex.ColumnCompare(r("f", "fk"), "=", r("d", "dk")), ex.ColumnCompare(r("f", "fe"), "=", r("e", "ek")),
                   ex.Comparison(r("d", "dv"), "<", 10), ex.Range(r("e", "ew"), 100, 700)))
    proj = [r("f", "fv"), r("d", "dv"), r("e", "ew")]
    out = {}
    for name, shard in (("single", False), ("sharded", True)):
        eng = Engine()
        for t in tabs:
            eng.catalog.register(multigpu.shard_table(t, rank, world) if shard else t)
        res = eng.run(ra.query(eng.catalog, ["f", "d", "e"], pred, proj))
        out[name] = {"count": res.count, "probe_out": res.stats.probe_out,
                     "order": res.plan.build_order,
                     "rows": [c.to_numpy()[0] for c in res.rows.columns]}
    return out


SCENARIOS = {"esc": _esc_scenario, "star": _star_scenario, "rows": _rows_scenario}


def _rank_main(rank, world, port, scenario, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), ESC_ONEPASS_MAX_ROWS="100000")
    try:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        try:
            q.put((rank, SCENARIOS[scenario](rank, world, torch.device("cuda", 0)), None))
        finally:
            dist.destroy_process_group()
    except BaseException:  # noqa: BLE001 — report to the parent instead of hanging it
        q.put((rank, None, traceback.format_exc()))


def _run(scenario, world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, scenario, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            rank, val, err = q.get(timeout=600)
            assert err is None, f"rank {rank}:\n{err}"
            res[rank] = val
    finally:
        for p in procs:
            p.join(60)
            if p.exitcode is None:
                p.kill()
    return [res[r] for r in range(world)]


@pytest.mark.parametrize("world,gated", [(2, "0"), (3, "0"), (2, "1")])
def test_sharded_esc_step_equals_single_gpu(cuda, world, gated, monkeypatch):
    """Both placements of the count exchange (multigpu.GATED): behind the step, or between the
    scan and the gated compaction."""
    monkeypatch.setenv("ESC_MG_GATED", gated)  # the spawned ranks read it when they import
    ranks = _run("esc", world)
    for i, first in enumerate(ranks[0]):
        if "errors" in first:
            msgs = {tuple(r[i]["errors"]) for r in ranks}
            assert len(msgs) == 1
            (sharded_msg, single_msg), = msgs
            assert single_msg is not None and sharded_msg == single_msg
            continue
        ref_count, ref_q, ref_cols = first["ref"]
        assert all(r[i]["count"] == ref_count and r[i]["qualified"] == ref_q for r in ranks)
        counts = first["counts"]
        assert sum(counts) == ref_count and all(r[i]["counts"] == counts for r in ranks)
        assert [r[i]["local"] for r in ranks] == counts
        assert [r[i]["offset"] for r in ranks] == list(np.cumsum([0] + counts[:-1]))
        if ref_q:
            for k, (want_v, want_m) in enumerate(ref_cols):
                got_v = np.concatenate([r[i]["slice"][k][0] for r in ranks])
                got_m = np.concatenate([r[i]["slice"][k][1] for r in ranks])
                assert np.array_equal(got_m, want_m)
                assert np.array_equal(got_v[~got_m], want_v[~want_m])
        else:
            assert all(r[i]["slice"] is None for r in ranks)


def test_sharded_star_plan_and_query(cuda):
    import golden_io as G

    ranks = _run("star", 2)
    want = G.known()["star"]
    for r in ranks:
        assert r["sharded"] == r["single"]
        decisions, order, card_sum, _, _ = r["sharded"]
        assert {d[0]: list(d[:4]) + [d[4]] for d in decisions} == {d[0]: d for d in want["decisions"]}
        assert order == want["order"] and card_sum == want["build_card_sum"]
        assert r["live_temps"] == []  # Engine.run swept every rank's sharded temps


def test_sharded_projection_rows(cuda):
    ranks = _run("rows", 2)
    single = ranks[0]["single"]
    for r in ranks:
        assert r["single"]["count"] == single["count"]
        assert r["sharded"]["count"] == single["count"] and r["sharded"]["probe_out"] == single["probe_out"]
        assert r["sharded"]["order"] == single["order"]
    for k in range(len(single["rows"])):
        got = np.concatenate([r["sharded"]["rows"][k] for r in ranks])
        assert np.array_equal(got, single["rows"][k])


def test_nccl_transport_one_rank(cuda):
    """The same sharded step over an NCCL group (one rank: this box has one GPU; NCCL refuses two
    ranks on one device): the all_gather runs on the stream, device to device."""
    import torch
    import torch.distributed as dist

    from paper_1901_01488_b200 import Catalog, ColumnTable, expr as ex, multigpu, optimizer
    from paper_1901_01488_b200.storage import KIND_INT32, Column

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    try:
        n = 3_000_003
        x = np.random.default_rng(8).integers(0, 100_000, n).astype(np.int32)
        t = ColumnTable("t", [Column("x", KIND_INT32, x, device=cuda)])
        cat = Catalog()
        cat.register(t)
        st = multigpu.ShardedTable("t", t, n, 0, 0, 1)
        cfg = optimizer.EscConfig()
        for hi in (99, 29_999):
            p = ex.Range(ex.ColumnRef("t", "x"), 0, hi)
            d = multigpu.sharded_esc_subquery(st, p, ["x"], cfg)
            ref = optimizer.esc_subquery(cat, "t", p, ["x"], cfg)
            assert (d.exact_count, d.qualified, d.counts, d.offset) == (ref.exact_count, ref.qualified,
                                                                         [ref.exact_count], 0)
            if ref.pushed_down:
                assert torch.equal(d.columns[0].values, cat.resolve_temp(ref.temp).columns[0].values)
            cat.temps.sweep()
    finally:
        dist.destroy_process_group()
