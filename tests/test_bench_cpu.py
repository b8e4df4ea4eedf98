"""bench.py's CPU legs (the reference arm and the cpu_baseline) on small host
arrays: the reference library only, both MTTKRP strategies timed, the
BASELINE.md section 3 record, and no torch / repo library in the process."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import REF_SO  # noqa: E402

pytestmark = pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference library not built")


def _coo(rng, dims, nnz, prefix, order):
    cap = int(np.prod(dims))
    lin = np.sort(rng.choice(cap, size=nnz, replace=False))
    idx, rest = [], lin
    for d in reversed(dims):
        idx.append((rest % d).astype(np.uint32))
        rest = rest // d
    idx = idx[::-1]
    keys = np.lexsort([idx[d] for d in reversed(order)])
    out = {f"{prefix}i{d}": idx[d][keys] for d in range(len(dims))}
    out[f"{prefix}val"] = rng.uniform(0.5, 1.5, nnz).astype(np.float32)
    return out


def test_c5_leg_strategies_and_record():
    import bench
    rng = np.random.default_rng(0)
    dims, n, R = [300, 200, 100], 20000, 32
    arrays = {}
    orders = []
    for m in range(3):
        o = [m] + [d for d in range(3) if d != m]
        orders.append(o)
        arrays.update(_coo(rng, dims, n, f"m{m}_", o))
    arrays.update(_coo(rng, dims, n, "eq_", [0, 1, 2]))
    arrays["eq_yval"] = rng.uniform(0.5, 1.5, n).astype(np.float32)
    for d in range(3):
        arrays[f"f{d}"] = rng.uniform(0, 1, (dims[d], R)).astype(np.float32)
    meta = {"dims": dims, "sample_nnz": n, "sort_orders": orders, "eq_sort_order": [0, 1, 2],
            "sample": "test"}
    res = bench.run_cpu_leg("c5", arrays, meta, steps=2, warmup=1)
    assert res["value"] > 0 and res["kind"] == "reference" and res["cores"] >= 1
    assert set(res["mttkrp_strategy"]) == {"mttkrp_m0", "mttkrp_m1", "mttkrp_m2"}
    for v in res["mttkrp_strategy"].values():
        assert v["chosen"] in ("privatize", "atomic") and v["privatize_s"] > 0
    assert res["seq"]["cores"] == 1 and res["seq"]["value"] > 0
    assert res["host"]["nproc"] >= 1
    assert res["host"]["omp"]["OMP_PROC_BIND"] == "close"
    assert res["step_s_median"] > 0 and res["value_median"] > 0


def test_c2_leg_and_files_roundtrip(tmp_path):
    import bench
    rng = np.random.default_rng(1)
    dims, n = [50, 40, 30], 3000
    arrays = _coo(rng, dims, n, "x_", [0, 1, 2])
    arrays["yval"] = rng.uniform(0.5, 1.5, n).astype(np.float32)
    arrays.update(_coo(rng, dims, n, "y2_", [0, 1, 2]))
    meta = {"dims": dims, "sort_order": [0, 1, 2], "sample_nnz": n, "sample": "t",
            "config": {"workload": "c2-tew_eq-tew"}}
    bench.save_arrays(str(tmp_path), arrays, meta)
    a2, m2 = bench.load_arrays(str(tmp_path))
    assert m2 == meta and set(a2) == set(arrays)
    res = bench.run_cpu_leg("c2", a2, m2, steps=1, warmup=0)
    assert res["value"] > 0


def test_reference_process_loads_no_repo_library():
    """The reference arm's process imports bench (and runs the reference
    library) without torch or libspten_b200 (the GPU inputs come from a
    separate --prep-cpu process)."""
    code = ("import sys, bench; import oracle.oracle as o; o.Ref();"
            "mods = [m for m in sys.modules if m.startswith(('torch', 'paper_1902_03317_b200'))];"
            "maps = open('/proc/self/maps').read();"
            "print(mods, 'libspten_b200' in maps, 'libspten_ref' in maps)")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         check=True).stdout.strip()
    assert out == "[] False True", out


def test_default_workload_is_c5():
    import bench
    assert bench.DEFAULT_WORKLOAD == "c5"
    assert json.dumps(bench.host_record())


def test_tns_leg_reads_the_sample_file():
    import bench
    rng = np.random.default_rng(2)
    lines = [f"{a} {b} {c} {v:.6f}" for a, b, c, v in
             zip(rng.integers(1, 50, 5000), rng.integers(1, 40, 5000), rng.integers(1, 30, 5000),
                 rng.uniform(0.5, 1.5, 5000))]
    text = np.frombuffer(("\n".join(lines) + "\n").encode(), np.uint8)
    meta = {"dims": [49, 39, 29], "sample_nnz": 5000, "sample": "t"}
    res = bench.run_cpu_leg("tns", {"text": text}, meta, steps=2, warmup=1)
    assert res["value"] > 0 and "seq" not in res
