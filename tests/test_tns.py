""".tns ingest: read_tns<float>, P/src/io.cpp:42-120.

Pinning: tests/golden/tns.json holds the REAL reference's result or error
for every case (tests/golden/make_tns_golden.py: the files of
P/tests/test_io.cpp and the malformed list of P/tests/acceptance.cpp, the
format's edge cases, std::from_chars(float) boundary tokens). The CPU tests
check the Python restatement (oracle.read_tns_py) against it, and against
the live reference library where oracle/_ref is built; the GPU tests check
the device parser (paper_1902_03317_b200.tns, through the C-ABI) against the
same records bit for bit -- indices, value bits, dims, error line and text --
and on larger files against the reference run here.
"""
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "tns.json")
MAX_ORDER = 8  # SPT_MAX_ORDER: the device path's order limit (the reference has none)


def _cases():
    with open(GOLDEN) as f:
        return json.load(f)


def _ref():
    from oracle.oracle import REF_SO, Ref
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    return Ref()


def _same_bits(a, b):
    """float32 bit patterns equal, NaN payloads included."""
    return np.array_equal(np.asarray(a, np.uint32), np.asarray(b, np.uint32))


# ---- CPU: the restatement against the reference ------------------------------

def test_oracle_matches_golden():
    from oracle.oracle import read_tns_py
    n = 0
    for rec in _cases():
        body = rec["body"].encode("latin-1")
        if "error" in rec:
            with pytest.raises((RuntimeError, ValueError)) as ei:
                read_tns_py(body, rec["dims"], "{path}")
            assert str(ei.value) == rec["error"]["msg"], rec["body"][:60]
        else:
            dims, idx, vals = read_tns_py(body, rec["dims"], "{path}")
            r = rec["result"]
            assert dims == r["dims"]
            assert [i.tolist() for i in idx] == r["idx"]
            assert _same_bits(vals.view(np.uint32), r["bits"]), rec["body"][:60]
        n += 1
    assert n > 300


def test_oracle_matches_live_reference(tmp_path):
    """Random value spellings near float boundaries, against the reference
    library itself (beyond the committed records)."""
    from fractions import Fraction

    from oracle.oracle import read_tns_py
    ref = _ref()
    rng = np.random.default_rng(11)
    lines = []
    for k in range(600):
        if k % 3 == 0:
            f = max(np.float32(abs(rng.standard_normal()) * 10.0 ** rng.integers(-44, 38)), np.float32(3e-45))
            g = np.nextafter(f, np.float32(np.inf))
            m = (Fraction(float(f)) + Fraction(float(g))) / 2
            s = str(m.numerator * 10 ** 70 // m.denominator + int(rng.integers(-1, 2))) + "e-70"
        elif k % 3 == 1:
            s = "%.*e" % (int(rng.integers(0, 20)), rng.standard_normal() * 10.0 ** rng.integers(-44, 38))
        else:
            s = repr(float(np.float32(rng.standard_normal() * 10.0 ** rng.integers(-40, 38))))
        lines.append(f"{k + 1} {s}")
    body = ("\n".join(lines) + "\n").encode()
    p = tmp_path / "r.tns"
    p.write_bytes(body)
    t = ref.read_tns(str(p))
    dims, idx, vals = read_tns_py(body, None, str(p))
    assert dims == list(t.dims)
    assert _same_bits(vals.view(np.uint32), t.values.view(np.uint32))


# ---- GPU: the device parser ---------------------------------------------------

gpu = pytest.mark.gpu


@pytest.fixture(scope="module")
def tns():
    pytest.importorskip("torch")
    from paper_1902_03317_b200 import _lib, tns as mod
    return _lib, mod


def _host(z):
    return ([int(e) for e in z.dims], [ix.cpu().numpy().view(np.uint32).tolist() for ix in z.indices],
            z.values.cpu().numpy().view(np.uint32))


@gpu
def test_device_matches_golden(tns, tmp_path):
    _lib, mod = tns
    p = str(tmp_path / "case.tns")
    checked = 0
    for rec in _cases():
        with open(p, "wb") as f:
            f.write(rec["body"].encode("latin-1"))
        if "error" in rec:
            with pytest.raises((RuntimeError, ValueError)) as ei:
                mod.read_tns(p, rec["dims"])
            assert str(ei.value) == rec["error"]["msg"].replace("{path}", p), rec["body"][:60]
            assert isinstance(ei.value, _lib.DeviceRuntimeError) == (rec["error"]["type"] ==
                                                                     "RuntimeError")
        elif len(rec["result"]["dims"]) > MAX_ORDER:
            with pytest.raises(_lib.IndexOverflow):
                mod.read_tns(p, rec["dims"])
        else:
            z = mod.read_tns(p, rec["dims"])
            dims, idx, bits = _host(z)
            r = rec["result"]
            assert dims == r["dims"] and idx == r["idx"], rec["body"][:60]
            assert _same_bits(bits, r["bits"]), rec["body"][:60]
            assert z.sort_order is None and not z.coalesced
        checked += 1
    assert checked > 300


@gpu
def test_device_write_read_round_trip(tns, tmp_path):
    """write_tns -> read_tns bit-exact (P/tests/test_io.cpp:84-110,
    acceptance.cpp:440-470), including 0, denorm_min and 1/3."""
    _lib, mod = tns
    ref = _ref()
    from oracle.oracle import HostTensor
    rng = np.random.default_rng(8000)
    for i in range(12):
        order = 1 + i % 4
        dims = [int(rng.integers(1, 40)) for _ in range(order)]
        t = ref.gen_synthetic(dims, max(1, int(np.prod(dims) * 0.2)), int(rng.integers(1 << 30)))
        if i % 3 == 0:
            t.values[:] = rng.uniform(-5, 5, t.nnz).astype(np.float32)
        t.values[0] = 0.0
        if t.nnz > 1:
            t.values[1] = np.float32(1.4e-45)
        if t.nnz > 2:
            t.values[2] = np.float32(1.0) / np.float32(3.0)
        p = str(tmp_path / f"rt{i}.tns")
        ref.write_tns(HostTensor(t.dims, t.indices, t.values), p)
        z = mod.read_tns(p, t.dims)
        dims, idx, bits = _host(z)
        assert dims == list(t.dims)
        assert idx == [ix.tolist() for ix in t.indices]
        assert _same_bits(bits, t.values.view(np.uint32))
        z2 = mod.read_tns(p)
        r2 = ref.read_tns(p)
        assert [int(e) for e in z2.dims] == list(r2.dims)


@gpu
def test_device_large_file_matches_reference(tns, tmp_path):
    """A 2M-line file (comments, blank lines, CRLF, tabs, every value form)
    against the reference's parse of the same bytes."""
    _lib, mod = tns
    ref = _ref()
    rng = np.random.default_rng(5)
    n = 2_000_000
    i0 = rng.integers(1, 100_000, n)
    i1 = rng.integers(1, 3_000, n)
    i2 = rng.integers(1, 70, n)
    v = (rng.standard_normal(n) * 10.0 ** rng.integers(-6, 6, n)).astype(np.float32)
    parts = []
    for k in range(0, n, 100_000):
        sl = slice(k, k + 100_000)
        vs = [repr(float(x)) if j % 4 else "%.9g" % x for j, x in enumerate(v[sl])]
        rows = [f"{a} {b}\t{c} {s}" for a, b, c, s in zip(i0[sl], i1[sl], i2[sl], vs)]
        rows[::1000] = [r + "\r" for r in rows[::1000]]
        parts.append("\n".join(rows))
        parts.append("# block %d\n" % k)
    body = "\n".join(parts).encode()
    p = str(tmp_path / "big.tns")
    with open(p, "wb") as f:
        f.write(body)
    t = ref.read_tns(p)
    z = mod.read_tns(p)
    dims, idx, bits = _host(z)
    assert dims == list(t.dims)
    for a, b in zip(idx, t.indices):
        assert np.array_equal(np.asarray(a, np.uint32), b)
    assert _same_bits(bits, t.values.view(np.uint32))


@gpu
def test_device_first_error_in_file_order(tns, tmp_path):
    """Many bad lines: the error names the first one (the reference stops
    there), whichever thread found its own first."""
    _lib, mod = tns
    rows = ["1 1 1.0"] * 50_000
    for k in (40_001, 7_777, 123, 49_999):
        rows[k] = "1 0 1.0" if k % 2 else "1 1 x"
    p = str(tmp_path / "bad.tns")
    with open(p, "w") as f:
        f.write("\n".join(rows) + "\n")
    with pytest.raises(_lib.DeviceRuntimeError) as ei:
        mod.read_tns(p)
    assert str(ei.value) == f"{p}:124: indices are 1-based; got 0"


@gpu
def test_device_errors(tns, tmp_path):
    _lib, mod = tns
    with pytest.raises(_lib.DeviceRuntimeError, match="cannot open"):
        mod.read_tns(str(tmp_path / "missing.tns"))
    p = str(tmp_path / "a.tns")
    with open(p, "w") as f:
        f.write("1 1 1.0\n")
    with pytest.raises(_lib.InvalidArgument, match="must not be empty"):
        mod.read_tns(p, [])
    with pytest.raises(_lib.IndexOverflow):
        mod.read_tns(p, [1] * (MAX_ORDER + 1))
