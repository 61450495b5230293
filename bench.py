#!/usr/bin/env python
"""ESC selectivity sub-query benchmark (B200).

One *step* = the per-table ESC sub-query on config 4 of BASELINE.json (600M rows: Zipf A,
correlated B, float32 C, uniform D; predicate ``A = 0 AND C BETWEEN -0.5 AND 1.0 AND (D = 17 OR
D > 900) AND (B*3 + D) % 7 > 3`` with the last term a Python UDF): exact count + push-down
decision + order-preserving materialization of (A, C, D) — one fused kernel pass per GPU, plus
one NCCL count/offset exchange when the table is row-partitioned over N > 1 GPUs (strong
scaling: the 600M rows are split across the ranks).

Prints ONE JSON line (rank 0).  ``--impl reference`` times the reference algorithm's CPU
implementation (the numpy port in ``oracle/``) on the host cores instead.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback, used only when MEASURED_PEAKS.json is absent
L2_BYTES = 126 * 2**20
# ONE metric string for both arms (the driver divides the arms' values only when metric, unit and
# direction agree); "fused" vs "reference" is in each line's `impl` / `config`
METRIC = "rows/s (ESC sub-query: scan+count+compaction)"
PARITY_CHUNK = 2_500_000  # rows per reference-port task (np.frompyfunc object arrays stay ~200 MB)


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--rows", type=int, default=600_000_000)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-extras", action="store_true")
    p.add_argument("--sweep", default="", help="write the config-5 selectivity sweep JSON here")
    p.add_argument("--cpu-sample-rows", type=int, default=0)
    p.add_argument("--no-parity", action="store_true", help="skip the full-shard parity check")
    return p.parse_args()


def peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def recorded_traffic(kind: str, rows: int, profiled_rows: int = 600_000_000):
    """DRAM bytes per launch from the committed ncu capture (profiles/traffic.json, one launch
    over ``profiled_rows`` rows), scaled to a launch over ``rows`` rows (a rank's shard); None
    when absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            v = json.load(fh).get(kind)
    except (OSError, ValueError):
        return None
    return None if v is None else v * rows / profiled_rows


# ------------------------------------------------------------------------------------------------
# clocks sampled during the timed region
# ------------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    @classmethod
    def snapshot(cls, index: int) -> list:
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(index), f"--query-gpu={cls.FIELDS}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20)
            return [ln.strip() for ln in out.stdout.splitlines() if ln.strip()]
        except (OSError, subprocess.SubprocessError):
            return []

    def summary(self):
        rows = []
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[2:6], float(parts[6])))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "note": "nvidia-smi returned no samples"}
        loaded = [r for r in rows if r[3] > 0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded)}


# ------------------------------------------------------------------------------------------------
# CPU side: the reference algorithm (numpy port) over row-range chunks in a process pool
# ------------------------------------------------------------------------------------------------
_CPU_STATE = {}


def _cpu_chunk(bounds):
    from oracle import esc_oracle as O

    lo, hi = bounds
    st = _CPU_STATE
    t = O.OTable("t", {k: O.OColumn(v[lo:hi], np.zeros(hi - lo, bool)) for k, v in st["cols"].items()})
    count = O.count_star(t, st["pred"], st["udfs"])
    mat = O.materialize(t, st["pred"], st["project"], st["udfs"])  # reference re-scans
    return count, [mat[c].values for c in st["project"]]


def cpu_reference_run(cols: dict, pred, project, udfs, rows: int, procs: int, reps: int = 1,
                      row_begin: int = 0, chunk: int = 0):
    """Run the reference algorithm (count sub-query + materialization; the numpy port of
    executor.count_star + optimizer.materialize_pushdown) over rows [row_begin, row_begin+rows)
    in a pool of ``procs`` processes.  The range is cut into ``procs`` contiguous chunks, or into
    ``chunk``-row tasks when given (the reference's own row-range concept, executor.py:485-504:
    counts add up, chunk results concatenate in row order).  Returns (seconds per rep, count);
    ``cpu_reference_run.last_columns`` holds the materialised columns of the last rep."""
    import multiprocessing as mp

    _CPU_STATE.update(cols=cols, pred=pred, project=project, udfs=udfs)
    hi = row_begin + rows
    if chunk:
        bounds = [(lo, min(lo + chunk, hi)) for lo in range(row_begin, hi, chunk)]
    else:
        bounds = [(row_begin + (i * rows) // procs, row_begin + ((i + 1) * rows) // procs) for i in range(procs)]
    ctx = mp.get_context("fork")
    times, count = [], 0
    with ctx.Pool(procs) as pool:
        for _ in range(reps):
            t0 = time.perf_counter()
            res = pool.map(_cpu_chunk, bounds, chunksize=1)
            times.append(time.perf_counter() - t0)
            count = sum(r[0] for r in res)
    # the materialised columns, chunks concatenated in row order (parity digest)
    cpu_reference_run.last_columns = [np.concatenate([r[1][k] for r in res]) for k in range(len(project))]
    return times, count


def full_parity_reference(cols: dict, pred, project, udfs, rows: int, procs: int):
    """The reference port over EVERY row of this rank's shard (2.5M-row tasks in ``procs``
    processes, outside any timed region): (count, digest of the materialised columns, seconds)."""
    t0 = time.perf_counter()
    _, count = cpu_reference_run(cols, pred, project, udfs, rows, procs, reps=1, chunk=PARITY_CHUNK)
    return count, columns_digest(cpu_reference_run.last_columns), time.perf_counter() - t0


def columns_digest(arrays) -> str:
    import hashlib

    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def default_cpu_rows(procs: int) -> int:
    # config 4 through the reference costs ~0.4 us/row/core (Python UDF via np.frompyfunc, twice):
    # ~1.2M rows per core keeps one rep near 1 s, a bounded sample of the 600M-row workload
    return 1_200_000 * procs


# ------------------------------------------------------------------------------------------------
def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    args = parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        # `bench.py --gpus N` on its own: re-launch as N ranks, one process per GPU (what the
        # driver's torchrun launch does), each rank reading RANK/LOCAL_RANK/WORLD_SIZE
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
               *sys.argv[1:]]
        return subprocess.call(cmd)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU"}),
              flush=True)
        return 2
    if args.impl == "reference":
        return run_reference(args, rank, max(world, args.gpus))
    return run_ours(args, rank, world, local_rank)


def run_reference(args, rank, world):
    """The reference arm: the reference's CPU algorithm for this path (the numpy port in oracle/,
    pinned to the reference's own outputs) on the host cores, on our arm's workload, metric and
    unit.  Each step = the count sub-query + materialization over a bounded sample of config 4's
    rows in every host core (contiguous row ranges, one process each); the single-core figure
    (the reference as it ships: single-threaded numpy) is timed beside it."""
    if rank != 0:
        return 0
    from paper_1901_01488_b200 import datagen

    procs = os.cpu_count() or 1
    rows = args.cpu_sample_rows or default_cpu_rows(procs)
    w = datagen.config4_blocked(args.rows, 0, rows)
    cols = {k: v[1] for k, v in w.columns.items()}
    times, count = cpu_reference_run(cols, w.pred, w.project, w.udfs, rows, procs, reps=args.warmup + args.steps)
    timed = times[args.warmup:]
    per_step = sum(timed) / len(timed)
    value = rows / per_step
    one_rows = rows // procs
    t1, _ = cpu_reference_run(cols, w.pred, w.project, w.udfs, one_rows, 1, reps=2)
    single = {"value": one_rows / min(t1), "unit": "rows/s", "cores": 1, "kind": "port",
              "sample": f"first {one_rows} rows of config 4 in ONE process (the reference ships single-threaded)"}
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "rows/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "i32+f32+f64", "data": "synthetic (block-seeded Appendix B config-4 recipe)",
        "config": {"workload": CONFIG4_WORKLOAD, "rows_total": args.rows, "sample_rows": rows,
                   "sample_count": count},
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": procs, "kind": "port",
                         "sample": f"first {rows} rows of config 4, {procs} processes x contiguous row ranges; "
                                   "numpy port of executor.count_star + optimizer.materialize_pushdown "
                                   "(Python UDF via np.frompyfunc)",
                         "single_core": single},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


CONFIG4_WORKLOAD = ("config4: 600M-row table, A=x AND C BETWEEN -0.5 AND 1.0 AND (D=17 OR D>900) AND udf(B,D)>3; "
                    "count + compaction of (A,C,D)")


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_1901_01488_b200 import datagen

    n = args.rows
    bounds = [((r * n) // world, ((r + 1) * n) // world) for r in range(world)]
    lo, hi = bounds[rank]
    m = hi - lo

    # host shard, generated straight into pinned buffers (they feed both the resident table and
    # the end-to-end leg's host->device copies)
    threads = max(1, (os.cpu_count() or 1) // world)
    pinned = {k: torch.empty(m, dtype=torch.float32 if k == "C" else torch.int32, pin_memory=True) for k in "ABCD"}
    t0 = time.perf_counter()
    w = datagen.config4_blocked(n, lo, hi, out={k: v.numpy() for k, v in pinned.items()}, threads=threads)
    gen_s = time.perf_counter() - t0

    # CPU work BEFORE any CUDA context exists (the pools fork): the baseline on a bounded sample
    # (rank 0, N = 1) and the parity reference over EVERY row of this rank's shard
    cpu_baseline, cpu_parity = None, None
    cols = {k: v[1] for k, v in w.columns.items()}
    procs = max(1, (os.cpu_count() or 1) // world)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rows = min(m, args.cpu_sample_rows or default_cpu_rows(procs))
        times, _ = cpu_reference_run(cols, w.pred, w.project, w.udfs, rows, procs, reps=2)
        per = min(times[1:]) if len(times) > 1 else times[0]
        one_rows = rows // procs
        t1, _ = cpu_reference_run(cols, w.pred, w.project, w.udfs, one_rows, 1, reps=2)
        cpu_baseline = {"value": rows / per, "unit": "rows/s", "cores": procs, "kind": "port",
                        "sample": f"first {rows} rows of this config-4 shard; numpy port of the reference "
                                  f"(count sub-query + materialization) in {procs} processes",
                        "single_core": {"value": one_rows / min(t1), "unit": "rows/s", "cores": 1, "kind": "port",
                                        "sample": f"first {one_rows} rows in ONE process (the reference ships "
                                                  "single-threaded)"}}
    if not args.no_parity:
        cpu_parity = full_parity_reference(cols, w.pred, w.project, w.udfs, m, procs)

    import torch.distributed as dist

    from paper_1901_01488_b200 import executor, multigpu, optimizer, serde
    from paper_1901_01488_b200.catalog import Catalog
    from paper_1901_01488_b200.storage import Column, ColumnTable, parse_kind

    # ESC_BENCH_BACKEND=gloo (plumbing checks on a one-GPU box only): every rank on cuda:0,
    # counts exchanged through host memory — never a measurement configuration
    backend = os.environ.get("ESC_BENCH_BACKEND", "nccl")
    gpu = local_rank if backend == "nccl" else local_rank % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    # ESC_BENCH_SHARDED=1 runs the multi-GPU step (device count exchange + gated compaction) even
    # at N = 1 (a one-rank group): its fixed per-step cost against the single-GPU step
    sharded = world > 1 or os.environ.get("ESC_BENCH_SHARDED") == "1"
    if sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None, rank=rank, world_size=world)
    pred = serde.from_json(w.pred, "t", w.udfs)
    cfg = optimizer.EscConfig()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def make_table():
        return ColumnTable("t", [Column(k, parse_kind(w.columns[k][0]), pinned[k].to(dev, non_blocking=True))
                                 for k in "ABCD"])

    table = make_table()
    torch.cuda.synchronize()
    cat = Catalog()
    cat.register(table)
    st = multigpu.ShardedTable("t", table, n, lo, rank, world)

    def step(keep: bool = False):
        if sharded:
            d = multigpu.sharded_esc_subquery(st, pred, w.project, cfg)
            return d.exact_count, d.local_count, d.columns
        d = optimizer.esc_subquery(cat, "t", pred, w.project, cfg)
        cols_ = cat.resolve_temp(d.temp).columns if keep and d.temp is not None else None
        cat.temps.sweep()
        return d.exact_count, d.exact_count, cols_

    parity = None
    if cpu_parity is not None:
        # the device step over the WHOLE shard vs the reference port over the whole shard: the
        # count and the digest of the materialised (A, C, D) slice; counts are additive and the
        # ranks' slices concatenate in rank order, so per-rank equality is global equality
        scount, sdigest, ssec = cpu_parity
        _, dcount, dcols = step(keep=True)
        ddigest = columns_digest([c.values.cpu().numpy() for c in dcols]) if dcols is not None else None
        ok = dcount == scount and ddigest == sdigest
        all_ok = ok if world == 1 else bool(max_over_ranks(0.0 if ok else 1.0) == 0.0)
        parity = {"sample_rows": m, "rows": m, "count_reference_port": scount, "count_device": dcount,
                  "rows_digest_equal": ddigest == sdigest, "bit_exact": ok, "all_ranks_bit_exact": all_ok,
                  "reference_s": round(ssec, 1), "reference_procs": procs,
                  "note": "every row of this rank's shard through the reference port (2.5M-row tasks), "
                          "outside the timed region"}

    for _ in range(args.warmup):
        step()
    barrier()
    stream = torch.cuda.current_stream()
    from paper_1901_01488_b200 import _native

    launches0 = _native.load_library().esc_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(gpu).__enter__()  # sampled across every timed region below
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        total, local, _ = step()
    e1.record(stream)
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    launches = _native.load_library().esc_launch_count() - launches0  # the library's own counter
    # per-kernel breakdown (roofline): the same steps again with CUDA events around each launch —
    # a separate loop, so the event records do not weigh on the timed steps above
    executor.KERNEL_EVENTS = []
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    events = executor.KERNEL_EVENTS
    executor.KERNEL_EVENTS = None
    sel_ms = [a.elapsed_time(b) for a, b, k in events if k == "select"]
    mat_ms = [a.elapsed_time(b) for a, b, k in events if k == "materialize"]
    kern_avg = statistics.mean(sel_ms)
    mat_avg = statistics.mean(mat_ms) if mat_ms else 0.0
    k_local = local
    proj_w = sum(w.columns[c][1].itemsize for c in w.project)
    algo_bytes = m * w.pred_bytes_per_row()               # K1 (select): predicate columns, read once
    step_bytes = algo_bytes + k_local * proj_w            # + the temp table written (proj within pred)
    peak, peak_src = peak_hbm()
    achieved = algo_bytes / (kern_avg * 1e-3) / 1e9
    value = n / (ms * 1e-3)

    # ---- end to end through the public API with host buffers ----------------------------------
    e2e = None
    if not args.no_e2e:
        proj_bytes = sum(w.columns[c][1].itemsize for c in w.project)

        def e2e_step():
            t = make_table()                                    # H2D of this rank's shard
            c2 = Catalog()
            c2.register(t)
            if sharded:
                d = multigpu.sharded_esc_subquery(multigpu.ShardedTable("t", t, n, lo, rank, world), pred,
                                                  w.project, cfg)
                outs = d.columns or []
                kk = d.local_count
            else:
                d = optimizer.esc_subquery(c2, "t", pred, w.project, cfg)
                outs = c2.resolve_temp(d.temp).columns if d.temp is not None else []
                kk = d.exact_count
            host = [c.values.to("cpu") for c in outs]            # D2H of the result
            c2.temps.sweep()
            return kk, host

        for _ in range(max(1, args.warmup)):
            e2e_step()
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.steps):
            kk, _ = e2e_step()
        s1.record(stream)
        barrier()
        ems = max_over_ranks(s0.elapsed_time(s1)) / args.steps
        e2e = {"value": n / (ems * 1e-3), "unit": "rows/s", "ms_per_step": ems,
               "h2d_bytes_per_step": m * 16, "d2h_bytes_per_step": kk * proj_bytes,
               "path": "ColumnTable from pinned host tensors -> optimizer.esc_subquery -> temp columns .to('cpu')"}

    clocks.__exit__(None, None, None)
    if not clocks.lines:  # the device-timed region is ~20 ms: take one reading right after it
        clocks.lines = ClockSampler.snapshot(gpu)
    extras = {}
    if not args.no_extras and world == 1:
        extras = run_extras(table, w, pred, cfg, dev, peak)
    if args.sweep and world == 1:
        del table, cat, st
        torch.cuda.empty_cache()
        sweep = run_sweep(args, dev, peak)
        with open(args.sweep, "w") as fh:
            json.dump(sweep, fh, indent=1)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "i32+f32+f64", "data": "synthetic (block-seeded Appendix B config-4 recipe)",
            "config": {"workload": CONFIG4_WORKLOAD, "impl_note": "fused device scan+count+compaction",
                       "rows": n, "rows_per_gpu": m, "count": total, "selectivity": total / n,
                       "l2": f"inputs {m * 16 / 1e9:.1f} GB per GPU >> L2 (126 MB): no flush needed",
                       "parallelism": (f"row-partitioned x{world}, {backend.upper()} all_gather of counts" if sharded
                                       else "1 GPU"),
                       "host_gen_s": round(gen_s, 1)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": recorded_traffic("select_config4", m),
                         "peak_source": peak_src,
                         "kernel": "esc_scan_kernel<C, false, JitPred> (K1: predicate + count + selection bitmap)",
                         "kernel_ms": kern_avg, "algorithmic_bytes": algo_bytes,
                         "bytes_note": "N x (A,B,C,D: 16 B) predicate columns per launch; the N/8 bitmap write "
                                       "is overhead, not counted"},
            "step": {"select_ms": kern_avg, "materialize_ms": mat_avg,
                     "algorithmic_bytes": step_bytes,
                     "GBps": step_bytes / (ms * 1e-3) / 1e9, "frac_of_peak": step_bytes / (ms * 1e-3) / 1e9 / peak,
                     "note": "one predicate pass (count + selection bitmap) + one gather pass over the "
                             "selection (only the hit rows of the projected columns)"},
            "cpu_baseline": cpu_baseline,
            "parity": parity,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "extras": extras,
        }
        print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()
    return 0


def _flush_l2(dev, clean: bool = False):
    """Evict L2 with a buffer twice its size: written (``clean`` False — L2 is left full of DIRTY
    lines, so the next kernel's first 126 MB of reads also pay their write-backs), or read
    (``clean`` True — L2 left holding clean lines, what a scan meets after other reads)."""
    import torch

    buf = getattr(_flush_l2, "buf", None)
    if buf is None:
        buf = _flush_l2.buf = torch.zeros(2 * L2_BYTES, dtype=torch.uint8, device=dev)
    if clean:
        buf.view(torch.int64).max()
    else:
        buf.zero_()


def _time_kernels(fn, reps, dev, flush=False):
    import torch

    from paper_1901_01488_b200 import executor

    executor.KERNEL_EVENTS = []
    for _ in range(reps):
        if flush:
            _flush_l2(dev)
        fn()
    torch.cuda.synchronize()
    ev = executor.KERNEL_EVENTS
    executor.KERNEL_EVENTS = None
    return [(a.elapsed_time(b), k) for a, b, k in ev]


def _device_step_ms(launch, finish, reps, dev, flush=True, clean=False) -> float:
    """Median device time of ``launch()`` (kernels queued, no host wait inside): L2 flushed, then
    a ~1 ms sleep kernel holds the stream while the host enqueues the events and the launches, so
    the events bracket device work only; ``finish(result)`` after each rep."""
    import torch

    for _ in range(3):
        r = launch()
        torch.cuda.synchronize()
        finish(r)
    ts = []
    for _ in range(reps):
        if flush:
            _flush_l2(dev, clean)
        torch.cuda._sleep(2_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = launch()
        e1.record()
        torch.cuda.synchronize()
        finish(r)
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def run_extras(table, w, pred, cfg, dev, peak):
    """Secondary numbers: count-only K1 on config 4, config 2 (L2 flushed), config 3 ESC overhead."""
    import torch

    from paper_1901_01488_b200 import count_star, datagen, executor, optimizer, ra, serde
    from paper_1901_01488_b200.catalog import Catalog
    from paper_1901_01488_b200.storage import Column, ColumnTable, Dictionary, parse_kind

    out = {}
    n = table.row_count
    for _ in range(2):
        count_star(table, pred)
    t = _time_kernels(lambda: count_star(table, pred), 5, dev)
    kms = statistics.mean(x for x, k in t if k == "count")
    gbs = n * w.pred_bytes_per_row() / (kms * 1e-3) / 1e9
    out["config4_count_only"] = {"kernel_ms": kms, "rows_per_s": n / (kms * 1e-3), "GBps": gbs, "frac": gbs / peak}

    # config 2: exact recipe, 6M rows (72 MB of predicate columns < L2: flush between reps)
    w2 = datagen.config2()
    t2 = ColumnTable("lineitem", [Column(k, parse_kind(v[0]), v[1], None, Dictionary(v[2]) if len(v) > 2 else None,
                                         device=dev) for k, v in w2.columns.items()])
    c2 = Catalog()
    c2.register(t2)
    p2 = serde.from_json(w2.pred, "lineitem")
    d = optimizer.esc_subquery(c2, "lineitem", p2, w2.project, cfg)
    c2.temps.sweep()
    cap2 = (d.row_count * 1) // 5  # floor(0.2 * rows): the queued step's capacity
    kms = _device_step_ms(lambda: executor.launch_step(t2, p2, w2.project, cap2), executor.finish_step, 15, dev)
    kms_clean = _device_step_ms(lambda: executor.launch_step(t2, p2, w2.project, cap2), executor.finish_step, 15,
                                dev, clean=True)
    b2 = w2.algorithmic_bytes(d.exact_count)
    out["config2_fused"] = {"count": d.exact_count, "kernel_ms": kms, "rows_per_s": w2.nrows / (kms * 1e-3),
                            "GBps": b2 / (kms * 1e-3) / 1e9, "frac": b2 / (kms * 1e-3) / 1e9 / peak,
                            "kernel_ms_clean_l2": kms_clean, "frac_clean_l2": b2 / (kms_clean * 1e-3) / 1e9 / peak,
                            "note": "device time of the queued step (K1 select + one-kernel mid-size compaction), "
                                    "L2 flushed before every rep by WRITING 252 MB (kernel_ms: the scan's first reads "
                                    "also pay the flush's dirty write-backs) or by READING it (kernel_ms_clean_l2); "
                                    "a sleep kernel holds the stream while the step is enqueued, so no host launch "
                                    "latency is inside the events"}

    # config 3: the 4-dimension star query — ESC overhead (reference definition, engine.py:69) and
    # the query executed end to end (Engine.run: ESC + hash builds over the temps + the fused
    # COUNT probe of the 60M-row fact, exact Appendix B recipe)
    g = datagen.config3(fact_rows=60_000_000)
    from paper_1901_01488_b200 import Engine, expr as ex

    eng = Engine(cfg)
    names = {"date": "dates"}
    for name, cols in g.items():
        eng.catalog.register(ColumnTable(names.get(name, name), [
            Column(k, parse_kind(v[0]), v[1], None, Dictionary(v[2]) if len(v) > 2 else None, device=dev)
            for k, v in cols.items()]))
    del g
    conj = [ex.ColumnCompare(ex.ColumnRef("fact", a), "=", ex.ColumnRef(names.get(dim, dim), b))
            for _, a, dim, b in datagen.CONFIG3_EDGES]
    conj += [serde.from_json(j, names.get(dim, dim)) for dim, j in datagen.CONFIG3_WHERE.items()]
    q = ra.query(eng.catalog, ["fact", "dates", "customer", "supplier", "part"], ex.And(tuple(conj)))
    overheads, walls, plan_ = [], [], None
    for i in range(12):
        t0 = time.perf_counter()
        plan_ = optimizer.plan(q, eng.catalog, cfg)
        wall = (time.perf_counter() - t0) * 1e3
        if i >= 2:
            overheads.append(optimizer.esc_overhead_ms(plan_))
            walls.append(wall)
        eng.catalog.temps.sweep()
    out["config3_esc"] = {
        "overhead_ms_median": statistics.median(overheads), "plan_wall_ms_median": statistics.median(walls),
        "decisions": [(d.table, d.exact_count, d.row_count, d.pushed_down) for d in plan_.decisions],
        "build_order": plan_.build_order, "build_card_sum": plan_.build_card_sum,
        "target_ms": 5.0, "reference_cpu_ms": 0.66,
    }
    try:
        out["ingest_csv"] = _ingest_extra(dev)
    except Exception as exc:  # noqa: BLE001 — a secondary number must not sink the bench line
        out["ingest_csv"] = {"error": f"{type(exc).__name__}: {exc}"}
    runs, res = [], None
    for i in range(8):
        executor.KERNEL_EVENTS = [] if i >= 3 else None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = eng.run(q)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        if i >= 3:
            ev = executor.KERNEL_EVENTS
            runs.append((wall, sum(a.elapsed_time(b) for a, b, k in ev if k == "join")))
    executor.KERNEL_EVENTS = None
    jms = statistics.median(r[1] for r in runs)
    fact_bytes = 60_000_000 * 4 * 4
    out["config3_query"] = {
        "count": res.count, "probe_out": res.stats.probe_out, "expected_count": datagen.CONFIG3_STAR_COUNT,
        "parity": res.stats.probe_out == datagen.CONFIG3_STAR_PROBE_OUT,
        "query_wall_ms_median": statistics.median(r[0] for r in runs), "join_kernel_ms": jms,
        "join_GBps": fact_bytes / (jms * 1e-3) / 1e9, "join_frac": fact_bytes / (jms * 1e-3) / 1e9 / peak,
        "join_bytes_note": "60M fact rows x 4 int32 foreign keys read once; dimension factors in shared memory",
        "cpu_baseline": _star_cpu_baseline(eng, plan_, res),
    }
    return out


def _ingest_extra(dev, rows: int = 1_000_000):
    """Device CSV ingestion (row f3): a seeded 4-column file (INT64, DECIMAL(12,2), DATE, TEXT with
    quoting) loaded through ingest.load_csv, H2D included; reference-equivalent host parsing
    (csv module + the reference's cell conversion) timed on a 100K-row slice for comparison."""
    import csv as _csv
    import io as _io

    import numpy as np
    import torch

    from paper_1901_01488_b200 import Dictionary
    from paper_1901_01488_b200.engine import parse_schema_spec
    from paper_1901_01488_b200.ingest import convert_cell, load_csv

    g = np.random.default_rng(2026)
    ints = g.integers(-10**12, 10**12, rows)
    cents = g.integers(0, 10**8, rows)
    days = g.integers(0, 20000, rows)
    words = np.array(["alpha", "beta", '"gamma, delta"', "epsilon", '"say ""hi"""', "zeta"])
    w = words[g.integers(0, len(words), rows)]
    import datetime as _dt

    base = _dt.date(1970, 1, 1).toordinal()
    date_txt = np.array([_dt.date.fromordinal(base + int(d)).isoformat() for d in range(20000)])[days]
    text = "\n".join(f"{a},{c // 100}.{c % 100:02d},{d},{s}" for a, c, d, s in zip(ints.tolist(), cents.tolist(),
                                                                                   date_txt.tolist(), w.tolist()))
    data = (text + "\n").encode()
    schema = parse_schema_spec("i:int64,d:decimal(12,2),t:date,s:text")
    load_csv(data, "t", schema, device=dev)  # warm-up (pinned staging, allocator)
    times = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        t = load_csv(data, "t", schema, device=dev)
        torch.cuda.synchronize()
        times.append((time.perf_counter() - t0) * 1e3)
    ms = statistics.median(times)
    sample = "\n".join(text.split("\n", 100_000)[:100_000])
    t1 = time.perf_counter()
    kinds = [k for _, k in schema]
    dicts = [Dictionary() for _ in kinds]
    for rec in _csv.reader(_io.StringIO(sample)):
        for raw, k, dct in zip(rec, kinds, dicts):
            convert_cell(None if raw == "\\N" else raw, k, dct)
    cpu_s = time.perf_counter() - t1
    return {"rows": rows, "bytes": len(data), "device_ms": ms, "device_MBps": len(data) / ms / 1e3,
            "rows_per_s": rows / (ms * 1e-3), "check_rows": t.row_count,
            "cpu_baseline": {"value": 100_000 / cpu_s, "unit": "rows/s", "cores": 1, "kind": "port",
                             "sample": "100K rows: Python csv.reader + the reference's per-cell conversion"},
            "note": "wall time of ingest.load_csv incl. the H2D copy of the text and the dictionary build"}


def _star_cpu_baseline(eng, plan_, res, sample_rows: int = 6_000_000):
    """The reference's probe pipeline (oracle port of executor.probe_joins, numpy, 1 core) over
    the first ``sample_rows`` fact rows with the plan's builds: rows/s of the CPU path."""
    import numpy as np

    from oracle import esc_oracle as O
    from paper_1901_01488_b200 import serde

    def otable(t, rows=None):
        cols = {}
        for c in t.columns:
            v, m = c.to_numpy()
            if rows is not None:
                v, m = v[:rows], m[:rows]
            cols[c.name] = O.OColumn(np.asarray(v).astype(np.int64), np.asarray(m))
        return O.OTable(t.name, cols)

    steps = []
    for b in plan_.builds:
        t = eng.catalog.table(b.source if isinstance(b.source, str) else plan_.graph.source[b.alias])
        res_j = serde.to_json(b.residual) if b.residual is not None else None
        if not isinstance(b.source, str):  # pushed-down build: the reference filters the same rows
            d = next(d for d in plan_.decisions if d.table == b.alias)
            res_j = serde.to_json(d.predicate)
        steps.append((b.alias, O.build_hash(otable(t), b.build_key.name, res_j), (b.probe_key.table, b.probe_key.name)))
    fact = otable(eng.catalog.table(plan_.probe_source), sample_rows)
    t0 = time.perf_counter()
    stage, _ = O.probe_joins(fact, plan_.probe_alias, None, steps)
    s = time.perf_counter() - t0
    return {"value": sample_rows / s, "unit": "fact rows/s", "cores": 1, "kind": "port",
            "sample": f"first {sample_rows} fact rows through the plan's 4 hash tables (oracle port of "
                      f"executor.probe_joins, numpy); sample COUNT {stage[-1]}"}


def _port_digest_threads(cols: dict, pred, names: list) -> tuple:
    """The reference port's selection over every row (2.5M-row chunks on the host threads): its
    count and, per column of ``names``, an order-sensitive digest of the selected values in row
    order — (sum v, sum position * v), both mod 2**64 — the full-size pin of a sweep point's
    compacted columns."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import esc_oracle as O

    n = len(next(iter(cols.values())))

    def one(lo):
        hi = min(lo + PARITY_CHUNK, n)
        t = O.OTable("t", {k: O.OColumn(v[lo:hi], np.zeros(hi - lo, bool)) for k, v in cols.items()})
        idx = O.eval_predicate(t, pred, None, {})
        j = np.arange(idx.size, dtype=np.uint64)
        parts = []
        for c in names:
            v = cols[c][lo:hi][idx].astype(np.int64).view(np.uint64)
            parts.append((int(v.sum(dtype=np.uint64)), int((j * v).sum(dtype=np.uint64))))
        return idx.size, parts

    with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
        res = list(ex.map(one, range(0, n, PARITY_CHUNK)))
    mask = (1 << 64) - 1
    total, dig = 0, [[0, 0] for _ in names]
    for k, parts in res:  # positions continue across chunks in row order
        for d, (s0, s1) in zip(dig, parts):
            d[0] = (d[0] + s0) & mask
            d[1] = (d[1] + total * s0 + s1) & mask
        total += k
    return total, [tuple(d) for d in dig]


def _values_digest(v: np.ndarray) -> tuple:
    """(sum v, sum position * v) mod 2**64 of a compacted column, in its order."""
    u = v.astype(np.int64).view(np.uint64)
    j = np.arange(u.size, dtype=np.uint64)
    return int(u.sum(dtype=np.uint64)), int((j * u).sum(dtype=np.uint64))


def run_sweep(args, dev, peak):
    """Config 5: single-range and 4-column conjunctive predicates at six selectivities, count-only
    vs fused count+compaction of (c0, c1, c4, c5); HBM GB/s vs selectivity."""
    import torch

    from paper_1901_01488_b200 import count_star, datagen, executor, optimizer, serde
    from paper_1901_01488_b200.catalog import Catalog
    from paper_1901_01488_b200.storage import Column, ColumnTable, parse_kind

    n = args.rows
    w = datagen.config5_blocked(n, 0.01)
    t = ColumnTable("t", [Column(k, parse_kind(v[0]), v[1], device=dev) for k, v in w.columns.items()])
    host = {k: v[1] for k, v in w.columns.items() if int(k[1]) < 4}  # the predicate columns (parity)
    del w
    res = []
    for conj4 in (False, True):
        for s in datagen.CONFIG5_SELECTIVITIES:
            wl = datagen.config5(8, s, conj4)
            wl.columns = {k: (("INT32" if int(k[1]) < 4 else "INT64"), np.empty(n, np.int32 if int(k[1]) < 4 else np.int64))
                          for k in t._by_name}
            p = serde.from_json(wl.pred, "t")
            cat = Catalog()
            cat.register(t)
            cfg = optimizer.EscConfig(max_selectivity=1.0)
            count_star(t, p)
            executor.materialize(t, p, wl.project)  # warm-up (JIT compile of the selection shape)
            tc = _time_kernels(lambda: count_star(t, p), 3, dev)
            cms = statistics.mean(x for x, k in tc if k == "count")
            k = count_star(t, p)
            tm = _time_kernels(lambda: executor.materialize(t, p, wl.project, count=k), 3, dev)
            mms = sum(x for x, kk in tm if kk in ("select", "materialize")) / 3
            bc = wl.algorithmic_bytes(k, materialize=False)
            bm = wl.algorithmic_bytes(k, materialize=True)
            # DRAM floor at 128-byte-line granularity (what a scattered hit really costs: ncu shows
            # one line fetched per gathered value): the scan's columns + bitmap write and read +
            # every projected column's lines that hold a hit + the output
            se = k / n
            pw = [t.column(c).values.element_size() for c in wl.project]
            lines = sum(n * w * (1.0 - (1.0 - se) ** (128 // w)) for w in pw)
            floor = bc + n / 4 + lines + k * sum(pw)
            # full-size pin: the count AND the compacted (c0, c1) columns (c1 is gathered for the
            # single-range predicate) against the reference port over all rows, outside the timing
            names = [c for c in ("c0", "c1") if c in wl.project]
            ref_k, ref_dig = _port_digest_threads(host, wl.pred, names)
            got = executor.materialize(t, p, names, count=k)
            dev_dig = [_values_digest(c.values.cpu().numpy()) for c in got]
            del got
            res.append({"pred": "conj4" if conj4 else "single", "s": s, "count": k, "count_ms": cms,
                        "count_reference_port": ref_k, "rows_digest_equal": dev_dig == ref_dig,
                        "bit_exact": ref_k == k and dev_dig == ref_dig,
                        "count_GBps": bc / cms / 1e6, "count_frac": bc / cms / 1e6 / peak,
                        "compact_ms": mms, "compact_GBps": bm / mms / 1e6, "compact_frac": bm / mms / 1e6 / peak,
                        "line_floor_ms": floor / peak / 1e6, "line_floor_frac": floor / peak / 1e6 / mms})
            torch.cuda.empty_cache()
    return {"rows": n, "peak_GBps": peak, "results": res}


if __name__ == "__main__":
    sys.exit(main())
