"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every ESC kernel
family at small and tile-boundary sizes, each result checked against the oracle so a sanitizer
run is also a correctness run.

    compute-sanitizer --tool memcheck python tools/sanitize.py

Covers K1 count / select (+ capture) in the interpreter and JIT tiers, the selection compaction
chain (partials, apply, stream, compact) through the queued step and the capacity skip, the
one-pass decoupled look-back kernel, the multi-GPU count gate, the hash build (one-block and
large), probe and expansion kernels, the star COUNT probe, and CSV ingestion."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import helpers as H  # noqa: E402
from oracle import esc_oracle as O  # noqa: E402
from paper_1901_01488_b200 import _native as N  # noqa: E402
from paper_1901_01488_b200 import count_star, executor, expr as ex, serde  # noqa: E402
from paper_1901_01488_b200.storage import KIND_INT32, KIND_INT64, Column, ColumnTable  # noqa: E402

dev = torch.device("cuda", 0)
quick = "--quick" in sys.argv
SIZES = [1, 127, 128 * 16 + 3, 65_536, 100_003] if not quick else [128 * 16 + 3, 65_536]


def check(a, b, what):
    if a != b:
        raise SystemExit(f"MISMATCH {what}: {a} != {b}")


def k1_and_compaction():
    for tier in (0, 2):  # interpreter, JIT
        N.set_jit(tier, 0)
        for n in SIZES:
            arrays = H.mixed_arrays(n, 11)
            t = H.device_table("data", arrays, device=dev)
            ot = H.oracle_table("data", arrays)
            for j in (["and", [["range", ["a", None], 100, 600], ["cmp", ["b", None], "<", 300]]],
                      ["or", [["eq", ["tag", None], 3], ["fn", "mixy", [["a", None], ["b", None]], ">", 6.0]]]):
                pred = serde.from_json(j, "data", H.UDFS)
                want = O.eval_predicate(ot, j, udfs=H.UDFS)
                check(count_star(t, pred), int(want.size), f"count n={n}")
                cols = executor.materialize(t, pred, ["id", "b"])
                check(cols[0].values.cpu().numpy().tolist(), (want + 1).tolist(), f"materialize n={n}")
                k, cols1 = executor.materialize_onepass(t, pred, ["id"])
                check(cols1[0].values.cpu().numpy().tolist(), (want + 1).tolist(), f"onepass n={n}")
                k2, cols2 = executor.count_and_materialize(t, pred, ["id", "a"], max(1, n // 5))
                check(k2, int(want.size), f"queued count n={n}")
                if cols2 is not None:
                    check(cols2[0].values.cpu().numpy().tolist(), (want + 1).tolist(), f"queued n={n}")
                rows = executor.eval_predicate(t, pred).indices
                check(rows.cpu().numpy().tolist(), want.tolist(), f"eval_predicate n={n}")
    N.set_jit(1, 1 << 22)


def gate_and_joins():
    lib = N.load_library()
    counts = torch.tensor([5, 7, 11], dtype=torch.int64, device=dev)
    out = torch.zeros(3, dtype=torch.int64, device=dev)
    import ctypes as C

    N.check(lib.esc_count_gate(C.c_void_p(counts.data_ptr()), 3, 1, 20, C.c_void_p(out.data_ptr()),
                               C.c_void_p(torch.cuda.current_stream().cuda_stream)), "esc_count_gate")
    check(out.cpu().tolist(), [23, 5, 1 << 62], "count gate")
    from paper_1901_01488_b200 import join

    g = np.random.default_rng(5)
    for nb in (100, 20_000):
        keys = g.integers(0, nb // 2 + 1, nb).astype(np.int64)
        d = ColumnTable("d", [Column("k", KIND_INT64, keys, device=dev)])
        idx = join.build_hash(d, "k")
        probe = g.integers(0, nb, 50_001).astype(np.int32)
        f = ColumnTable("f", [Column("fk", KIND_INT32, probe, device=dev)])
        _, st = join.probe_joins(f, "f", None, [join.BuildStep("d", idx, ex.ColumnRef("f", "fk"))], None)
        oidx = O.build_index(O.OTable("d", {"k": O.OColumn(keys, np.zeros(nb, bool))}), "k", np.arange(nb))
        want, _ = O.probe_joins(O.OTable("f", {"fk": O.OColumn(probe.astype(np.int64), np.zeros(probe.size, bool))}),
                                "f", None, [("d", oidx, ("f", "fk"))])
        check(st.probe_out, want, f"join count nb={nb}")
        res, st2 = join.probe_joins(f, "f", None, [join.BuildStep("d", idx, ex.ColumnRef("f", "fk"))],
                                    (ex.ColumnRef("f", "fk"),))
        check(st2.probe_out, want, f"join rows nb={nb}")


def csv():
    from paper_1901_01488_b200.ingest import load_csv
    from paper_1901_01488_b200.storage import parse_kind

    text = "".join(f'{i},"w{i % 7}",{i * 3}.5\n' for i in range(5000))
    t = load_csv(text, "c", [("i", parse_kind("int64")), ("s", parse_kind("text")),
                             ("d", parse_kind("decimal(9,1)"))], device=dev)
    check(t.row_count, 5000, "csv rows")


k1_and_compaction()
gate_and_joins()
csv()
torch.cuda.synchronize()
print("sanitize workload ok")
