"""CSV ingestion scenarios: (name, text, schema spec, has_header).  Shared by
make_golden.py (reference load_csv outputs or errors) and the tests."""

from __future__ import annotations

import numpy as np


def _big(seed: int, n: int) -> str:
    g = np.random.default_rng(seed)
    words = ["alpha", "beta", "gamma, delta", 'say "hi"', "", "x\ny", "Ünïcödé", "zeta"]
    lines = []
    for i in range(n):
        cells = [str(int(g.integers(-10**12, 10**12))) if g.random() > 0.05 else r"\N",
                 f"{int(g.integers(0, 10**6))}.{int(g.integers(0, 100)):02d}" if g.random() > 0.05 else r"\N",
                 f"{int(g.integers(1990, 2030))}-{int(g.integers(1, 13)):02d}-{int(g.integers(1, 29)):02d}",
                 words[int(g.integers(0, len(words)))]]
        out = []
        for k, c in enumerate(cells):
            if k == 3 and (any(ch in c for ch in ',"\n') or g.random() < 0.2):
                out.append('"' + c.replace('"', '""') + '"')
            else:
                out.append(c)
        lines.append(",".join(out))
    term = "\r\n" if seed % 2 else "\n"
    return term.join(lines) + (term if seed % 3 else "")


SPEC4 = "i:int64,d:decimal(12,2),t:date,s:text"

CASES = [
    ("basic", "1,2.5,2020-01-31,a\n-3,0.01,1970-01-01,b\n4,\\N,\\N,a\n", SPEC4, False),
    ("header", "i,d,t,s\n7,1,19991231,zz\n8,2.10,2000-02-29,\"q\"\n", SPEC4, True),
    ("quoted", '5,"3.25","2001-01-01","a,b"\n6,4,2001-01-02,"he said ""no"""\n9,1,2001-01-03,"line\nbreak"\n', SPEC4, False),
    ("crlf_no_trailing", "1,1,2020-01-01,x\r\n2,2,2020-01-02,y\r\n3,3,2020-01-03,x", SPEC4, False),
    ("lone_cr", "1,1,2020-01-01,x\r2,2,2020-01-02,y\r", SPEC4, False),
    ("spaces_signs", " 12 ,+1.5,2020-12-31,  padded  \n-0,-0.5,2020-06-15,\\N\n1_000,7.,2020-06-16,\"\\N\"\n", SPEC4, False),
    ("empty_text", '1,1,2020-01-01,\n2,2,2020-01-02,""\n', SPEC4, False),
    ("empty_file", "", SPEC4, False),
    ("header_only", "i,d,t,s\n", SPEC4, True),
    ("int_only", "\n".join(str(v) for v in range(-50, 50)) + "\n", "v:int64", False),
    ("big_lf", _big(2, 3000), SPEC4, False),
    ("big_crlf", _big(3, 3000), SPEC4, False),
    ("big_notrail", _big(4, 2500), SPEC4, False),
    # errors (first failing cell / record in the reference's order)
    ("err_fields", "1,1,2020-01-01,a\n2,2,2020-01-02\n", SPEC4, False),
    ("err_empty_line", "1,1,2020-01-01,a\n\n2,2,2020-01-02,b\n", SPEC4, False),
    ("err_int", "1,1,2020-01-01,a\n2x,2,2020-01-02,b\n", SPEC4, False),
    ("err_decimal", "1,1.5.5,2020-01-01,a\n", SPEC4, False),
    ("err_scale", "1,1.555,2020-01-01,a\n", SPEC4, False),
    ("err_date", "1,1,2020-02-30,a\n", SPEC4, False),
    ("err_date_format", "1,1,2020/01/01,a\n", SPEC4, False),
    ("err_float_int", "1.0,1,2020-01-01,a\n", SPEC4, False),
    ("err_overflow", "9223372036854775808,1,2020-01-01,a\n", SPEC4, False),
    ("err_order", "1,bad,2020-01-01,a\nalso_bad,1,2020-01-01,a\n", SPEC4, False),
    ("err_header_row_numbers", "i,d,t,s\n1,1,2020-01-01,a\n2,2,2020-13-01,b\n", SPEC4, True),
]
