"""Seeded synthetic inputs for the BASELINE configurations.

Every recipe draws from ``np.random.default_rng(np.random.SeedSequence([seed, stream]))`` — the
reference harness's per-table stream convention (``pkg/src/escdb/bench.py:83-85``) — in the listed
column order, with numpy's default int64 ``integers`` then a cast to the physical width.  No
public dataset is involved: these recipes ARE the benchmark inputs (BASELINE.json names none).

Each config returns numpy arrays (host) plus the predicate (JSON form, see :mod:`.serde`) and the
projection, so the same inputs feed the GPU path, the oracle and the CPU baseline.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEED = 42


def rng(stream: int, seed: int = SEED) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([seed, stream]))


@dataclass
class Workload:
    name: str
    columns: dict                  # name -> (kind_name, np.ndarray[, words])
    pred: list                     # JSON predicate
    project: list                  # projected column names (materialization)
    udfs: dict = field(default_factory=dict)
    note: str = ""

    @property
    def nrows(self) -> int:
        return len(next(iter(self.columns.values()))[1])

    def pred_bytes_per_row(self) -> int:
        names = set()

        def walk(j):
            tag = j[0]
            if tag in ("and", "or"):
                for i in j[1]:
                    walk(i)
            elif tag == "not":
                walk(j[1])
            elif tag == "colcmp":
                names.update((j[1][0], j[3][0]))
            elif tag == "fn":
                names.update(a[0] for a in j[2])
            else:
                names.add(j[1][0])

        walk(self.pred)
        return sum(self.columns[n][1].itemsize for n in names)

    def algorithmic_bytes(self, k: int, materialize: bool = True) -> int:
        """N*sum(w_pred) [+ K*sum(w_proj \\ pred) + K*sum(w_proj)]."""
        b = self.nrows * self.pred_bytes_per_row()
        if materialize:
            pred_cols = self._pred_cols()
            for n in self.project:
                w = self.columns[n][1].itemsize
                b += k * w * (1 if n in pred_cols else 2)
        return b

    def _pred_cols(self) -> set:
        out = set()

        def walk(j):
            tag = j[0]
            if tag in ("and", "or"):
                for i in j[1]:
                    walk(i)
            elif tag == "not":
                walk(j[1])
            elif tag == "colcmp":
                out.update((j[1][0], j[3][0]))
            elif tag == "fn":
                out.update(a[0] for a in j[2])
            else:
                out.add(j[1][0])

        walk(self.pred)
        return out


def udf_b3d(b, d):
    """Config 4's UDF: (B*3 + D) % 7 in CPython float arithmetic."""
    return (b * 3.0 + d) % 7.0


def config1(n: int = 1_000_000) -> Workload:
    g = rng(1)
    a = g.integers(0, 10000, n).astype(np.int32)
    b = g.integers(0, 100, n).astype(np.int32)
    pred = ["and", [["range", ["a", None], 2000, 4999], ["eq", ["b", None], 7]]]
    return Workload("config1", {"a": ("INT32", a), "b": ("INT32", b)}, pred, ["a"])


def config2(n: int = 6_000_000) -> Workload:
    g = rng(2)
    lines = g.integers(1, 8, n)
    orderkey = np.repeat(np.arange(1, n + 1, dtype=np.int64), lines)[:n]
    date = g.integers(8035, 8035 + 2557, n).astype(np.int32)
    quantity = g.integers(1, 51, n).astype(np.int32)
    price = g.integers(90000, 10500000, n).astype(np.int64)
    discount = g.integers(0, 11, n).astype(np.int32)
    tax = g.integers(0, 9, n).astype(np.int32)
    flag = g.integers(0, 3, n).astype(np.int8)
    cols = {
        "orderkey": ("INT64", orderkey), "date": ("DATE", date), "quantity": ("INT32", quantity),
        "price": ("DECIMAL(15,2)", price), "discount": ("INT32", discount), "tax": ("INT32", tax),
        "flag": ("TEXT", flag, ["A", "N", "R"]),
    }
    pred = ["and", [["range", ["date", None], 8766, 9130], ["range", ["discount", None], 5, 7],
                    ["cmp", ["quantity", None], "<", 24]]]
    return Workload("config2", cols, pred, ["orderkey", "price", "discount"])


def config4(n: int = 600_000_000, x: int = 0, chunk: int = 50_000_000) -> Workload:
    """Zipf A, correlated B, float32 C, uniform D; Eq ∧ f32 range ∧ OR ∧ UDF."""
    g = rng(4)
    a = ((g.zipf(1.1, n) - 1) % 1_000_000).astype(np.int32)
    b = (a % 1000 + g.integers(-5, 6, n)).astype(np.int32)
    c = np.empty(n, dtype=np.float32)
    for s in range(0, n, chunk):  # standard_normal streams identically in chunks
        c[s:s + chunk] = g.standard_normal(min(chunk, n - s)).astype(np.float32)
    d = g.integers(0, 1000, n).astype(np.int32)
    pred = ["and", [["eq", ["A", None], x], ["range", ["C", None], -0.5, 1.0],
                    ["or", [["eq", ["D", None], 17], ["cmp", ["D", None], ">", 900]]],
                    ["fn", "b3d", [["B", None], ["D", None]], ">", 3.0]]]
    cols = {"A": ("INT32", a), "B": ("INT32", b), "C": ("FLOAT32", c), "D": ("INT32", d)}
    return Workload("config4", cols, pred, ["A", "C", "D"], {"b3d": udf_b3d})


CONFIG5_SELECTIVITIES = (1e-4, 1e-3, 1e-2, 0.1, 0.5, 0.9)


def config5(n: int = 600_000_000, s: float = 0.01, conj4: bool = False) -> Workload:
    g = rng(5)
    cols = {}
    for i in range(4):
        cols[f"c{i}"] = ("INT32", g.integers(0, 1_000_000, n).astype(np.int32))
    for i in range(4, 8):
        cols[f"c{i}"] = ("INT64", g.integers(0, 10**12, n).astype(np.int64))
    if conj4:
        hi = round(s ** 0.25 * 1e6) - 1
        pred = ["and", [["range", [f"c{i}", None], 0, hi] for i in range(4)]]
    else:
        pred = ["range", ["c0", None], 0, round(s * 1e6) - 1]
    return Workload(f"config5_s{s}{'_conj4' if conj4 else ''}", cols, pred, ["c0", "c1", "c4", "c5"])


# ---- config 3: star schema --------------------------------------------------------------------
DIM_SIZES = {"date": 2556, "customer": 30000, "supplier": 2000, "part": 200000}


def _calendar_years(ndays: int) -> np.ndarray:
    import datetime as _dt

    base = _dt.date(1992, 1, 1)
    return np.array([(base + _dt.timedelta(days=k)).year for k in range(ndays)], dtype=np.int32)


def config3(fact_rows: int = 60_000_000) -> dict:
    """Dimension tables + fact FKs; predicates per dimension (Appendix B)."""
    out = {}
    gd = rng(31)
    nd = DIM_SIZES["date"]
    out["date"] = {
        "d_datekey": ("INT32", np.arange(1, nd + 1, dtype=np.int32)),
        "d_year": ("INT32", _calendar_years(nd)),
        "d_dow": ("TEXT", gd.integers(0, 7, nd).astype(np.int8), [f"D{i}" for i in range(7)]),
    }
    gc = rng(32)
    nc = DIM_SIZES["customer"]
    out["customer"] = {
        "c_custkey": ("INT32", np.arange(1, nc + 1, dtype=np.int32)),
        "c_region": ("TEXT", gc.integers(0, 5, nc).astype(np.int8), [f"R{i}" for i in range(5)]),
    }
    gs = rng(33)
    ns = DIM_SIZES["supplier"]
    out["supplier"] = {
        "s_suppkey": ("INT32", np.arange(1, ns + 1, dtype=np.int32)),
        "s_nation": ("TEXT", gs.integers(0, 25, ns).astype(np.int8), [f"N{i:02d}" for i in range(25)]),
    }
    gp = rng(34)
    npart = DIM_SIZES["part"]
    out["part"] = {
        "p_partkey": ("INT32", np.arange(1, npart + 1, dtype=np.int32)),
        "p_category": ("TEXT", gp.integers(0, 25, npart).astype(np.int8), [f"C{i:02d}" for i in range(25)]),
    }
    gf = rng(30)
    out["fact"] = {
        "f_datekey": ("INT32", gf.integers(1, nd + 1, fact_rows).astype(np.int32)),
        "f_custkey": ("INT32", gf.integers(1, nc + 1, fact_rows).astype(np.int32)),
        "f_suppkey": ("INT32", gf.integers(1, ns + 1, fact_rows).astype(np.int32)),
        "f_partkey": ("INT32", gf.integers(1, npart + 1, fact_rows).astype(np.int32)),
    }
    return out


# predicates in storage units (TEXT codes: word index in the dictionary)
CONFIG3_WHERE = {
    "customer": ["eq", ["c_region", None], 1],                                     # c_region = 'R1'
    "part": ["or", [["eq", ["p_category", None], 3], ["eq", ["p_category", None], 7]]],  # IN ('C03','C07')
    "date": ["range", ["d_year", None], 1993, 1994],
    "supplier": ["or", [["eq", ["s_nation", None], 2], ["eq", ["s_nation", None], 5]]],
}
CONFIG3_EDGES = [("fact", "f_datekey", "date", "d_datekey"), ("fact", "f_custkey", "customer", "c_custkey"),
                 ("fact", "f_suppkey", "supplier", "s_suppkey"), ("fact", "f_partkey", "part", "p_partkey")]

# the reference's answer for the config-3 star query over the 60M-row fact (COUNT and stage
# counts of execute_plan), pinned in tests/golden/known.json["star_execute"]
CONFIG3_STAR_COUNT = 21105
CONFIG3_STAR_PROBE_OUT = [60_000_000, 4_559_813, 1_303_361, 260_088, 21_105]


# ---- block-seeded variants for the 600M-row benchmarks ----------------------------------------
# The exact Appendix B recipes above draw each column from one sequential stream, which takes
# ~2 minutes single-threaded at 600M rows and cannot be split by rank.  The benchmark therefore
# uses the SAME per-row distributions drawn in independent blocks of BLOCK_ROWS rows, block b
# seeded with SeedSequence([42, stream, b]): any row range (one rank's shard) is generated alone,
# in parallel threads (numpy releases the GIL), directly into caller-provided (pinned) buffers.
BLOCK_ROWS = 2_500_000


def _blocked(n: int, row_begin: int, row_end: int, out: dict, fill_block, threads: int | None = None):
    import os
    from concurrent.futures import ThreadPoolExecutor

    b0, b1 = row_begin // BLOCK_ROWS, (row_end + BLOCK_ROWS - 1) // BLOCK_ROWS

    def work(b):
        lo, hi = b * BLOCK_ROWS, min(n, (b + 1) * BLOCK_ROWS)
        block = fill_block(b, hi - lo)
        s, e = max(lo, row_begin), min(hi, row_end)
        for name, arr in block.items():
            out[name][s - row_begin:e - row_begin] = arr[s - lo:e - lo]

    with ThreadPoolExecutor(threads or min(32, os.cpu_count() or 1)) as pool:
        list(pool.map(work, range(b0, b1)))
    return out


def config4_blocked(n: int = 600_000_000, row_begin: int = 0, row_end: int | None = None,
                    out: dict | None = None, threads: int | None = None) -> Workload:
    row_end = n if row_end is None else row_end
    m = row_end - row_begin
    out = out or {k: np.empty(m, dtype=np.float32 if k == "C" else np.int32) for k in "ABCD"}

    def fill(b, k):
        g = np.random.default_rng(np.random.SeedSequence([SEED, 4, b]))
        a = ((g.zipf(1.1, k) - 1) % 1_000_000).astype(np.int32)
        return {"A": a, "B": (a % 1000 + g.integers(-5, 6, k)).astype(np.int32),
                "C": g.standard_normal(k).astype(np.float32), "D": g.integers(0, 1000, k).astype(np.int32)}

    _blocked(n, row_begin, row_end, out, fill, threads)
    w = config4(8)  # predicate / projection / UDF of the config (tiny throwaway data)
    w.columns = {"A": ("INT32", out["A"]), "B": ("INT32", out["B"]), "C": ("FLOAT32", out["C"]),
                 "D": ("INT32", out["D"])}
    w.note = f"block-seeded config-4 recipe, rows [{row_begin}, {row_end}) of {n}"
    return w


def config5_blocked(n: int = 600_000_000, s: float = 0.01, conj4: bool = False, row_begin: int = 0,
                    row_end: int | None = None, out: dict | None = None, threads: int | None = None) -> Workload:
    row_end = n if row_end is None else row_end
    m = row_end - row_begin
    out = out or {f"c{i}": np.empty(m, dtype=np.int32 if i < 4 else np.int64) for i in range(8)}

    def fill(b, k):
        g = np.random.default_rng(np.random.SeedSequence([SEED, 5, b]))
        d = {f"c{i}": g.integers(0, 1_000_000, k).astype(np.int32) for i in range(4)}
        d.update({f"c{i}": g.integers(0, 10**12, k).astype(np.int64) for i in range(4, 8)})
        return d

    _blocked(n, row_begin, row_end, out, fill, threads)
    w = config5(8, s, conj4)
    w.columns = {k: ("INT32" if int(k[1]) < 4 else "INT64", v) for k, v in out.items()}
    w.note = f"block-seeded config-5 recipe, rows [{row_begin}, {row_end}) of {n}"
    return w
