"""Generate tests/golden/tns.json from the REAL reference's read_tns<float>
(P/src/io.cpp:42-120, compiled into oracle/_ref by oracle/Makefile):

    python tests/golden/make_tns_golden.py

Cases: the files of the reference's own tests (P/tests/test_io.cpp:40-150,
the malformed list of P/tests/acceptance.cpp:490-500), the format's edge
cases (CRLF, tabs, leading blanks, no final newline, comment-only, dims
override), and value tokens at the edges of std::from_chars(float): the
denormal and overflow boundaries, exact float midpoints (ties to even),
long digit strings, inf / nan spellings, rejected spellings. Each record is
{body (latin-1 text), dims (or null), and either result {dims, idx, bits}
(values as u32 bit patterns) or error {type, msg} with the file path
replaced by "{path}"}.
"""
from __future__ import annotations

import json
import os
import sys
import tempfile
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Ref  # noqa: E402


def value_tokens():
    toks = ["1e-45", "7.006492321624085e-46", "7.006492321624086e-46", "7e-46", "1e-46",
            "1e-50", "1.1754942e-38", "1.17549435e-38", "3.4028234e38",
            "3.4028235677973366e38", "340282356779733661637539395458142568448",
            "340282356779733661637539395458142568447", "3.5e38", "1e39", "inf", "-inf",
            "INF", "Infinity", "-infinity", "nan", "-nan", "NaN(abc_12)", "nan()", "nan(a-b)",
            "infin", "+1", "1.", "1.e5", ".5", "-.5", "-0", "0", "0.0", "0e999999999",
            "00000", "-00.000e-5", "1e", "1e+", "1e-", "0x1p3", "1_0", "4..5", "--4", "-", ".",
            "e5", "1.5E-3", "1e-0038", "1e+38", "1.0000000596046448",
            "1.00000005960464477539062500000001", "1.0000000596046447753906250",
            "16777217", "16777219", "33554435", "0.1", "0.2", "0.3", "3.14159265358979",
            "1" * 39, "1" * 40, "1" * 150, "0." + "0" * 200 + "1e200",
            "0." + "0" * 44 + "14", "123456789012345678901234567890",
            "9999999999999999999999999999999999999e1", "4.5", "-1.25", "1/3", "1,5", "\xa0"]
    # exact midpoints between neighbouring floats (ties to even) and their
    # one-ulp-of-decimal neighbours, across binades and into the denormals
    rng = np.random.default_rng(2024)
    for e in (-149, -140, -126, -125, -20, -1, 0, 1, 23, 24, 60, 100, 126, 127):
        f = np.float32(2.0 ** e) * np.float32(1 + rng.random())
        g = np.nextafter(f, np.float32(np.inf))
        if not np.isfinite(g):
            continue
        m = (Fraction(float(f)) + Fraction(float(g))) / 2
        # m = p / 2^k exactly: m * 10^k is an integer
        k = max(0, (m.denominator).bit_length() - 1)
        n = m.numerator * 10 ** k // m.denominator
        s = str(n)
        toks.append(f"{s}e-{k}" if k else s)
        toks.append(f"{n - 1}e-{k}" if k else str(n - 1))
        toks.append(f"{n + 1}e-{k}" if k else str(n + 1))
    for _ in range(120):
        toks.append(repr(float(np.float32(rng.standard_normal() * 10.0 ** rng.integers(-45, 39)))))
        toks.append("%.*e" % (int(rng.integers(0, 25)),
                              rng.standard_normal() * 10.0 ** rng.integers(-47, 40)))
    return toks


def files():
    out = []
    # P/tests/test_io.cpp:40-80
    out.append(("# a comment\n\n1 2 3 4.5\n2 1 1 -1.25\n", None))
    out.append(("1 1 1 2.0\n2 2 2 3.0\n", [4, 4, 4]))
    out.append(("1 1 1 2.0\n5 1 1 3.0\n", [4, 4, 4]))
    out.append(("# nothing\n# here\n", None))
    out.append(("# nothing\n# here\n", [3, 2]))
    # P/tests/test_io.cpp:130-150 and acceptance.cpp:490-500
    for bad in ("1 2 1.0", "1 2 3 4 1.0", "x 2 3 1.0", "0 2 3 1.0", "-1 2 3 1.0",
                "5000000000 2 3 1.0", "1 2 3", "1 2 3 4..5", "1 2 3 1e999", "1 2 3 --4"):
        out.append((f"1 2 3 1.0\n{bad}\n", None))
    # format edges
    out += [("", None), ("", [2, 2]), ("\n", None), ("\n\n\n", [1]),
            ("1 2 3 4.5\r\n2 1 1 -1.25\r\n", None), ("1 2 3 4.5\n2 1 1 -1.25", None),
            ("  \t1\t2 \t 3   4.5 \t\n", None), ("1 1\n\r\r\n", None), ("1 1\r", None),
            ("0005 1\n00000000000000000000000000005000000000 1\n", None),
            ("18446744073709551615 1\n", None), ("18446744073709551616 1\n", None),
            ("4294967295 1\n", None), ("4294967296 1\n", None), ("1 1\n1\t 2   \t3\n", [4, 4]),
            ("5\n", None), ("x 5\n", None), ("1 1 1 1 1 1 1 1 1\n", None),
            ("1 1 1 1 1 1 1 1 1 1\n", None), ("2 3 0.5\n", None), ("1 1\n2 2 2\n", None),
            ("1 1 1\n", [2]), ("1 1\n#\n  # x\n2 2\n", None), ("3 1\n1 2\n", [2]),
            ("1 2 3 1.0\n1 2 3 1.0 \n1 2 3 1.0\t\n", None), ("1 2 3 1.0\n\x0b1 2 3 1.0\n", None)]
    # value tokens, one per line of one file each
    for t in value_tokens():
        out.append((f"7 {t}\n", None))
    # one larger file: many lines, mixed spacing, comments
    rng = np.random.default_rng(7)
    lines = []
    for i in range(3000):
        if i % 97 == 0:
            lines.append("# comment " + str(i))
        elif i % 89 == 0:
            lines.append("")
        else:
            ix = rng.integers(1, 40, size=3)
            v = float(np.float32(rng.standard_normal()))
            sep = " " if i % 3 else "\t "
            lines.append(sep.join(str(int(a)) for a in ix) + sep + repr(v))
    out.append(("\n".join(lines) + "\n", None))
    return out


def main():
    ref = Ref()
    recs = []
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "case.tns")
        for body, dims in files():
            with open(path, "wb") as f:
                f.write(body.encode("latin-1"))
            rec = {"body": body, "dims": dims}
            try:
                t = ref.read_tns(path, dims)
                rec["result"] = {"dims": [int(e) for e in t.dims],
                                 "idx": [ix.tolist() for ix in t.indices],
                                 "bits": t.values.view(np.uint32).tolist()}
            except Exception as e:  # noqa: BLE001 -- the reference's error is the record
                rec["error"] = {"type": type(e).__name__, "msg": str(e).replace(path, "{path}")}
            recs.append(rec)
    out = os.path.join(HERE, "tns.json")
    with open(out, "w") as f:
        json.dump(recs, f, separators=(",", ":"))
    print(f"{len(recs)} cases -> {out}")


if __name__ == "__main__":
    main()
