"""Test helpers: seeded mixed-kind tables (same numpy arrays feed the device table and the
oracle) and a random predicate corpus in the JSON form both sides understand."""

from __future__ import annotations

import random

import numpy as np

from oracle import esc_oracle as O

WORDS = ["apple", "Banana", "cherry", "date", "elder", "fig", "grape", "honeydew", "kiwi",
         "lemon", "mango", "nectarine"]

UDFS = {
    "mixy": lambda x, y: (x * 7.0 + y) % 13.0,
    "lin": lambda x: x * 0.5 - 3.0,
    "fdiv": lambda x, y: (x - y) // 3.0,
    "nabs": lambda x: -abs(x) + 2.0,
    "sq": lambda x: x**2 - 10.0 * x,
    "inv": lambda x: 100.0 / x,
    "rmod": lambda x, y: x % (y - 500.0),
}


def mixed_arrays(n: int, seed: int, null_fraction: float = 0.08) -> dict:
    """name -> (kind, values, nulls or None, words or None)."""
    g = np.random.default_rng(np.random.SeedSequence([seed, 99]))

    def nulls():
        return (g.random(n) < null_fraction) if null_fraction > 0 else None

    def zero_at(v, m):
        if m is not None:
            v = np.where(m, 0, v).astype(v.dtype)
        return v

    cols = {}
    cols["id"] = ("INT64", np.arange(1, n + 1, dtype=np.int64), None, None)
    m = nulls()
    cols["a"] = ("INT64", zero_at(g.integers(0, 1000, n), m), m, None)
    m = nulls()
    cols["b"] = ("INT32", zero_at(g.integers(-500, 1000, n).astype(np.int32), m), m, None)
    m = nulls()
    cols["val"] = ("DECIMAL(15,2)", zero_at(g.integers(0, 1_000_001, n), m), m, None)
    m = nulls()
    cols["when"] = ("DATE", zero_at(g.integers(8035, 8035 + 2400, n).astype(np.int32), m), m, None)
    m = nulls()
    cols["tag"] = ("TEXT", zero_at(g.integers(0, len(WORDS), n).astype(np.int8), m), m, WORDS)
    m = nulls()
    cols["f"] = ("FLOAT32", zero_at(g.standard_normal(n).astype(np.float32), m), m, None)
    cols["big"] = ("INT64", (2**53 + g.integers(-8, 8, n)).astype(np.int64), None, None)
    cols["g8"] = ("INT8", g.integers(-100, 100, n).astype(np.int8), None, None)
    cols["u8"] = ("INT16", g.integers(-3000, 3000, n).astype(np.int16), None, None)
    return cols


def device_table(name: str, arrays: dict, device=None):
    from paper_1901_01488_b200.storage import Column, ColumnTable, Dictionary, parse_kind

    cols = []
    for cname, (kind, vals, nulls, words) in arrays.items():
        cols.append(Column(cname, parse_kind(kind), vals, nulls,
                           Dictionary(words) if words is not None else None, device=device))
    return ColumnTable(name, cols)


def oracle_table(name: str, arrays: dict) -> O.OTable:
    t = O.OTable(name)
    for cname, (kind, vals, nulls, words) in arrays.items():
        scale = int(kind[8:-1].split(",")[1]) if kind.startswith("DECIMAL") else 0
        t.columns[cname] = O.OColumn(vals, nulls if nulls is not None else np.zeros(len(vals), bool),
                                     kind, scale, words)
    return t


class Corpus:
    """Random resolved predicates over ``mixed_arrays`` columns; constants sampled from stored
    values so atoms have non-trivial selectivity."""

    NUM = ["a", "b", "val", "when", "id", "g8", "u8", "big"]
    OPS = ["<", "<=", ">", ">=", "<>", "="]

    def __init__(self, arrays: dict, rng: random.Random, udfs=("mixy", "lin", "fdiv", "nabs")):
        self.arrays = arrays
        self.rng = rng
        self.udfs = list(udfs)

    def _ref(self, c):
        kind = self.arrays[c][0]
        scale = int(kind[8:-1].split(",")[1]) if kind.startswith("DECIMAL") else None
        return [c, scale]

    def _stored(self, c):
        vals = self.arrays[c][1]
        return vals[self.rng.randrange(len(vals))].item()

    def atom(self):
        r = self.rng.random()
        R = self.rng
        if r < 0.07:
            a, b = R.sample(["a", "b", "id", "g8", "u8"], 2)
            return ["colcmp", self._ref(a), R.choice(self.OPS), self._ref(b)]
        if r < 0.10:
            return ["colcmp", self._ref("f"), R.choice(self.OPS), self._ref(R.choice(["b", "g8"]))]
        if r < 0.18:
            name = R.choice(self.udfs)
            nargs = 2 if name in ("mixy", "fdiv") else 1
            args = [self._ref(c) for c in R.sample(["a", "b", "val", "when", "g8", "f"], nargs)]
            return ["fn", name, args, R.choice(["<", ">=", ">", "="]), float(R.randrange(-3, 13))]
        if r < 0.30:  # TEXT
            if R.random() < 0.5:
                return ["eq", self._ref("tag"), R.randrange(len(WORDS) + 1)]
            if R.random() < 0.5:
                return ["cmp", self._ref("tag"), R.choice(["<", "<=", ">", ">="]), R.choice(WORDS + ["c", "zzz"])]
            lo, hi = sorted(R.sample(WORDS, 2))
            return ["range", self._ref("tag"), lo, hi]
        if r < 0.38:  # float32 column: python floats compare in f32 (NEP 50)
            k = R.choice([0.1, -0.5, 1.0, 0.3333333333333333, 2.5, 1e-8, 3])
            if R.random() < 0.3:
                return ["range", self._ref("f"), -abs(k), abs(k)]
            return ["cmp", self._ref("f"), R.choice(self.OPS), k]
        c = R.choice(self.NUM)
        if r < 0.52:
            return ["eq", self._ref(c), self._stored(c)]
        if r < 0.70:
            return ["cmp", self._ref(c), R.choice(self.OPS), self._stored(c)]
        if r < 0.76:  # fractional constant on an integer column -> float64 compare
            return ["cmp", self._ref(c), R.choice(self.OPS), self._stored(c) + 0.5]
        if r < 0.79:  # out-of-range python ints compare mathematically
            return ["cmp", self._ref(c), R.choice(self.OPS), R.choice([2**40, -(2**40), 2**70, -(2**70)])]
        if r < 0.93:
            lo, hi = sorted((self._stored(c), self._stored(c)))
            if R.random() < 0.15:
                lo, hi = hi, lo
            if R.random() < 0.15:
                hi = hi + 0.25
            return ["range", self._ref(c), lo, hi]
        return ["folded", self._ref(R.choice(list(self.arrays))), R.random() < 0.5]

    def pred(self, depth=0):
        r = self.rng.random()
        if depth >= 3 or r < 0.4:
            return self.atom()
        if r < 0.65:
            return ["and", [self.pred(depth + 1) for _ in range(self.rng.choice([2, 2, 3]))]]
        if r < 0.88:
            return ["or", [self.pred(depth + 1) for _ in range(self.rng.choice([2, 2, 3]))]]
        return ["not", self.pred(depth + 1)]
