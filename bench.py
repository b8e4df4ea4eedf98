#!/usr/bin/env python
"""Benchmark of the B200 COO sparse-tensor kernels on the BASELINE.json configs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5]
                    [--impl ours|reference] [--mttkrp plan|seg]

A step is one pass of the workload's ops over its seeded synthetic inputs
(already resident in HBM). Default workload = the largest single-GPU config,
BASELINE.json configs[4] (C5): MTTKRP modes 0/1/2 (R=32) + TEW-eq mul on a
1B-nnz order-3 tensor with Zipf(1.1) modes. MTTKRP runs on plans (csrc/
mttkrp_plan.cu) built once per mode as preprocessing, timed apart like the
reference's sort_s (P/src/bench.cpp:363-368). `value` is nonzeros/s over all
ranks, each op timed with CUDA events on its stream after an L2 flush (inputs
are also > L2). `roofline` is for the op with the largest time share:
algorithmic bytes per launch / mean event duration vs
MEASURED_PEAKS.json hbm_gbs. `e2e` times the same ops through the public API
(ops.* -> C-ABI) from pinned host buffers: every step uploads the tensors and
factors, builds the plans, runs the ops and downloads every result.
`cpu_baseline` is the reference's own OpenMP path (oracle/_ref, compiled from
the reference sources) on this host, BASELINE.md section 3 protocol.

--impl reference runs only that CPU path. Its inputs are made by a separate
process (`bench.py --prep-cpu DIR`, the GPU generator) and read from files,
so the reference process loads no library of this repository.

Multi-GPU (torchrun): C5 shards ONE tensor (strong scaling, row-aligned
MTTKRP shards + one all-gather, TEW-eq nnz shards); the other workloads run
an independent instance per rank (weak scaling). Timing = max over ranks.
"""
from __future__ import annotations

import os

# the reference's OpenMP threads close-bound to cores.
# Set before any OpenMP runtime is loaded (torch and the reference library
# both bring libgomp, which reads these once at load).
os.environ.setdefault("OMP_PROC_BIND", "close")
os.environ.setdefault("OMP_PLACES", "cores")

import argparse  # noqa: E402
import json  # noqa: E402
import shutil  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import tempfile  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "nonzeros/sec per COO op (MTTKRP/TTM/TTV/TEW/TS) & achieved HBM GB/s vs peak"
DEFAULT_WORKLOAD = "c5"


def _measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def peaks():
    d = _measured_peaks()
    if "hbm_gbs" in d:
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
# clocks sampler


class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (driver attach, several 100 ms) stalls CUDA
            # calls of this process: let it deliver its first sample before the
            # timed region begins; it keeps sampling every 100 ms through it
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [s.strip() for s in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def tensor_bytes(nnz, order):
    return nnz * (4 * order + 4)


# ===========================================================================
# CPU legs: the reference library's own kernels (oracle/_ref/libspten_ref.so)
# on host arrays. Nothing here imports torch or loads a library of this repo.


def host_record() -> dict:
    """nproc, lscpu model, free -g."""
    rec = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                rec["cpu_model"] = ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    try:
        out = subprocess.run(["free", "-g"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Mem:"):
                rec["mem_total_gb"] = int(ln.split()[1])
    except (OSError, subprocess.SubprocessError, ValueError, IndexError):
        pass
    rec["omp"] = {k: os.environ.get(k) for k in ("OMP_PROC_BIND", "OMP_PLACES")}
    return rec


def _host_tensor(arrays, prefix, dims, sort_order, n=None):
    from oracle.oracle import HostTensor
    N = len(dims)
    idx = [arrays[f"{prefix}i{d}"][:n] for d in range(N)]
    return HostTensor(list(dims), [np.ascontiguousarray(a, dtype=np.uint32) for a in idx],
                      np.ascontiguousarray(arrays[f"{prefix}val"][:n], dtype=np.float32),
                      None if sort_order is None else list(sort_order), True)


class CpuLeg:
    """A bounded sample of one workload on the reference's par:: kernels.
    MTTKRP calls time both strategies once and keep
    the faster; `seq()` runs the same ops with seq:: on one core."""

    def __init__(self, ref, nthreads):
        import ctypes
        self.ref, self.lib, self.ct, self.nt = ref, ref.lib, ctypes, nthreads
        self.keep, self.calls, self.strategy = [], [], {}

    # handles
    def coo(self, ht):
        h = self.ref.coo(ht)
        self.keep.append(h)
        return h

    def matrix(self, a):
        a = np.ascontiguousarray(a, dtype=np.float32)
        self.keep.append(a)
        return self.lib.ref_matrix_new(a.ctypes.data_as(self.ct.POINTER(self.ct.c_float)),
                                       a.shape[0], a.shape[1])

    def vector(self, a):
        a = np.ascontiguousarray(a, dtype=np.float32)
        self.keep.append(a)
        return self.lib.ref_vector_new(a.ctypes.data_as(self.ct.POINTER(self.ct.c_float)),
                                       a.shape[0])

    def factors(self, hx, mats):
        """One reference factor vector (matrices copied in; the temporaries go
        at once -- C5's factors are 1.28 GB each)."""
        f32p = self.ct.POINTER(self.ct.c_float)
        hs = (self.ct.c_void_p * len(mats))()
        for d, m in enumerate(mats):
            a = np.ascontiguousarray(m, dtype=np.float32)
            hs[d] = self.lib.ref_matrix_new(a.ctypes.data_as(f32p), a.shape[0], a.shape[1])
        fv = self.lib.ref_factors_new(hx, hs)
        for h in hs:
            self.lib.ref_matrix_free(h)
        return fv

    def _run(self, fn, *args, kind="coo"):
        out = self.ct.c_void_p()
        self.ref._check(fn(*args, self.ct.byref(out)))
        (self.lib.ref_matrix_free if kind == "matrix" else self.lib.ref_coo_free)(out.value)

    # op builders: each call is (name, units, fn(variant, nthreads))
    def add(self, name, units, fn):
        self.calls.append((name, units, fn))

    def add_mttkrp(self, name, units, hx, fv, mode):
        def fn(variant, nt, strat=None):
            s = self.strategy.get(name, 0) if strat is None else strat
            self._run(self.lib.ref_mttkrp_fv, hx, fv, mode, variant, nt, s, kind="matrix")
        self.calls.append((name, units, fn))

    def calibrate(self) -> dict:
        """Time privatize and atomic once per MTTKRP call; keep the faster."""
        rec = {}
        for name, _, fn in self.calls:
            if not name.startswith("mttkrp"):
                continue
            t = {}
            for s, sname in ((0, "privatize"), (1, "atomic")):
                t0 = time.perf_counter()
                fn(1, self.nt, s)
                t[sname] = time.perf_counter() - t0
            best = min(t, key=t.get)
            self.strategy[name] = 0 if best == "privatize" else 1
            rec[name] = {"privatize_s": round(t["privatize"], 4), "atomic_s": round(t["atomic"], 4),
                         "chosen": best}
        return rec

    def units(self) -> int:
        return sum(u for _, u, _ in self.calls)

    def step(self) -> int:
        for _, _, fn in self.calls:
            fn(1, self.nt)
        return self.units()


def _cpu_leg(name, ref, arrays, meta, nthreads):
    """Build the CpuLeg of workload `name` from host arrays (CPU-only)."""
    leg = CpuLeg(ref, nthreads)
    dims = meta["dims"]
    N = len(dims)
    if name == "c1":
        hx = leg.coo(_host_tensor(arrays, "x_", dims, meta["sort_order"]))
        fv = leg.factors(hx, [arrays[f"f{d}"] for d in range(N)])
        n = meta["sample_nnz"]
        leg.add_mttkrp("mttkrp_m0", n, hx, fv, 0)
        for op, nm in ((0, "ts_add"), (1, "ts_mul")):
            leg.add(nm, n, lambda v, nt, op=op: leg._run(leg.lib.ref_ts, hx, 2.5, op, v, nt))
    elif name == "c2":
        hx = leg.coo(_host_tensor(arrays, "x_", dims, meta["sort_order"]))
        from oracle.oracle import HostTensor
        hxt = _host_tensor(arrays, "x_", dims, meta["sort_order"])
        hy = leg.coo(HostTensor(hxt.dims, hxt.indices, np.ascontiguousarray(arrays["yval"]),
                                hxt.sort_order, True))
        hy2 = leg.coo(_host_tensor(arrays, "y2_", dims, meta["sort_order"]))
        n = meta["sample_nnz"]
        for op, nm in ((0, "tew_eq_add"), (1, "tew_eq_sub"), (2, "tew_eq_mul"), (3, "tew_eq_div")):
            leg.add(nm, n, lambda v, nt, op=op: leg._run(leg.lib.ref_tew_eq, hx, hy, op, v, nt))
        for op, nm in ((0, "tew_add"), (2, "tew_mul")):
            leg.add(nm, 2 * n, lambda v, nt, op=op: leg._run(leg.lib.ref_tew, hx, hy2, op, v, nt))
    elif name == "c3":
        for m in range(N):
            hx = leg.coo(_host_tensor(arrays, f"m{m}_", dims, meta["sort_orders"][m]))
            fib = leg.lib.ref_fiber_new(hx, m)  # preprocessing, untimed (P/src/bench.cpp:363-368)
            leg.keep.append(("fib", fib))
            hv, hu = leg.vector(arrays[f"v{m}"]), leg.matrix(arrays[f"u{m}"])
            n = meta["sample_nnz"]
            leg.add(f"ttv_m{m}", n, lambda v, nt, hx=hx, hv=hv, m=m, fib=fib:
                    leg._run(leg.lib.ref_ttv_fib, hx, hv, m, fib, v, nt))
            leg.add(f"ttm_m{m}", n, lambda v, nt, hx=hx, hu=hu, m=m, fib=fib:
                    leg._run(leg.lib.ref_ttm_fib, hx, hu, m, fib, v, nt))
    elif name in ("c4", "c5"):
        fv = None
        for m in range(N):
            hx = leg.coo(_host_tensor(arrays, f"m{m}_", dims, meta["sort_orders"][m]))
            if fv is None:
                fv = leg.factors(hx, [arrays[f"f{d}"] for d in range(N)])
                leg.keep.append(("fv", fv))
            leg.add_mttkrp(f"mttkrp_m{m}", meta["sample_nnz"], hx, fv, m)
        if name == "c5":
            from oracle.oracle import HostTensor
            hxt = _host_tensor(arrays, "eq_", dims, meta["eq_sort_order"])
            hx = leg.coo(hxt)
            hy = leg.coo(HostTensor(hxt.dims, hxt.indices, np.ascontiguousarray(arrays["eq_yval"]),
                                    hxt.sort_order, True))
            leg.add("tew_eq_mul", meta["sample_nnz"],
                    lambda v, nt: leg._run(leg.lib.ref_tew_eq, hx, hy, 2, v, nt))
    elif name == "tns":
        base = "/dev/shm" if os.path.isdir("/dev/shm") else None
        fd, path = tempfile.mkstemp(suffix=".tns", dir=base)
        with os.fdopen(fd, "wb") as fh:
            fh.write(arrays["text"].tobytes())
        leg.keep.append(("file", path))
        leg.add("read_tns", meta["sample_nnz"], lambda v, nt: leg.ref.read_tns(path))
    elif name == "pre":
        from oracle.oracle import HostTensor
        t = _host_tensor(arrays, "x_", dims, None)
        n = meta["sample_nnz"]

        def sort_once(v, nt):
            leg.ref.sort_lexicographic(HostTensor(t.dims, [a.copy() for a in t.indices],
                                                  t.values.copy(), None, True), [0, 1, 2])
        leg.add("sort_lexicographic", n, sort_once)
    else:
        raise ValueError(name)
    return leg


def run_cpu_leg(name, arrays, meta, steps, warmup, seq=True) -> dict:
    """par:: with every host thread, both MTTKRP
    strategies, `warmup` untimed + `steps` timed runs (mean and median), and
    one seq:: pass on one core."""
    from oracle.oracle import Ref
    ref = Ref()
    nthreads = os.cpu_count() or 1
    leg = _cpu_leg(name, ref, arrays, meta, nthreads)
    strategies = leg.calibrate()
    for _ in range(warmup):
        leg.step()
    t = []
    for _ in range(steps):
        t0 = time.perf_counter()
        leg.step()
        t.append(time.perf_counter() - t0)
    units = leg.units()
    for item in leg.keep:
        if isinstance(item, tuple) and item[0] == "file":
            os.remove(item[1])
    res = {"value": units / statistics.mean(t), "unit": "nnz/s", "cores": nthreads,
           "kind": "reference", "sample": meta["sample"], "step_s_mean": statistics.mean(t),
           "step_s_median": statistics.median(t), "value_median": units / statistics.median(t),
           "protocol": f"{warmup} untimed warm-up + {steps} timed runs, mean (P/src/bench.cpp:"
                       f"199-209) and median; par:: with nthreads={nthreads}",
           "mttkrp_strategy": strategies, "host": host_record()}
    if seq and name not in ("pre", "tns"):
        # seq:: on one core over the same calls (one pass; long calls on a
        # prefix of the sample when the par:: step is heavy)
        t0 = time.perf_counter()
        for nm, _, fn in leg.calls:
            fn(0, 1) if not nm.startswith("mttkrp") else fn(0, 1, 0)
        dt = time.perf_counter() - t0
        res["seq"] = {"value": units / dt, "unit": "nnz/s", "cores": 1,
                      "note": "spten::seq:: over the same sample, one pass"}
    return res


def crosscheck(name, arrays, meta, k=200_000) -> dict:
    """The reference bench's crosscheck (P/src/bench.cpp:226-229, :346-443)
    for the GPU rows: each op of the workload on the first k entries of the
    CPU sample, GPU (this library) against the reference's seq:: kernels,
    with the reference's own rules -- bit-identical outputs, MTTKRP
    max_rel_diff <= 1e-4 at f32 (P/src/bench.cpp:282). Returns op -> pass/fail."""
    import torch
    from oracle.oracle import HostTensor, Ref
    from paper_1902_03317_b200 import ops
    from paper_1902_03317_b200.coo import HostCOO
    ref = Ref()
    dims = meta["dims"]
    N = len(dims)

    def dev(t):
        return HostCOO(t.dims, t.indices, t.values, t.sort_order, t.coalesced).to_device(0)

    def same(g, r):
        g = g.to_host()
        return (list(g.dims) == list(r.dims) and
                all(np.array_equal(a, b) for a, b in zip(g.indices, r.indices)) and
                np.array_equal(g.values.view(np.uint32), r.values.view(np.uint32)))

    def rel(a, b):
        den = np.maximum(np.abs(a), np.abs(b))
        return float(np.max(np.where(den > 0, np.abs(a - b) / np.where(den > 0, den, 1), 0)))

    out = {}
    if name in ("c1", "c2"):
        x = _host_tensor(arrays, "x_", dims, meta["sort_order"], k)
        dx = dev(x)
        if name == "c1":
            for op, nm in ((0, "ts_add"), (1, "ts_mul")):
                out[nm] = "pass" if same(ops.ts(dx, 2.5, op), ref.ts(x, 2.5, op)) else "fail"
            fs = [arrays[f"f{d}"] for d in range(N)]
            g = ops.mttkrp(dx, [torch.from_numpy(f).cuda() for f in fs], 0).cpu().numpy()
            out["mttkrp_m0"] = "pass" if rel(g, ref.mttkrp(x, fs, 0)) <= 1e-4 else "fail"
        else:
            y = HostTensor(x.dims, x.indices, np.ascontiguousarray(arrays["yval"][:k]),
                           x.sort_order, True)
            dy = dev(y)
            for op, nm in ((0, "tew_eq_add"), (1, "tew_eq_sub"), (2, "tew_eq_mul"),
                           (3, "tew_eq_div")):
                out[nm] = "pass" if same(ops.tew_eq(dx, dy, op), ref.tew_eq(x, y, op)) else "fail"
            y2 = _host_tensor(arrays, "y2_", dims, meta["sort_order"], k)
            for op, nm in ((0, "tew_add"), (2, "tew_mul")):
                z, _, _, _ = ref.tew(x.copy(), y2.copy(), op)
                out[nm] = "pass" if same(ops.tew(dev(x), dev(y2), op), z) else "fail"
    elif name == "tns":
        from paper_1902_03317_b200 import tns
        base = "/dev/shm" if os.path.isdir("/dev/shm") else None
        fd, path = tempfile.mkstemp(suffix=".tns", dir=base)
        try:
            with os.fdopen(fd, "wb") as fh:
                fh.write(arrays["text"].tobytes())
            g, r = tns.read_tns(path), ref.read_tns(path)
            out["read_tns"] = "pass" if same(g, r) else "fail"
        finally:
            os.remove(path)
    elif name in ("c4", "c5"):
        fs = [arrays[f"f{d}"] for d in range(N)]
        tf = [torch.from_numpy(f).cuda() for f in fs]
        for m in range(N):
            x = _host_tensor(arrays, f"m{m}_", dims, meta["sort_orders"][m], k)
            g = ops.mttkrp(dev(x), tf, m).cpu().numpy()
            out[f"mttkrp_m{m}"] = "pass" if rel(g, ref.mttkrp(x, fs, m)) <= 1e-4 else "fail"
        if name == "c5":
            x = _host_tensor(arrays, "eq_", dims, meta["eq_sort_order"], k)
            y = HostTensor(x.dims, x.indices, np.ascontiguousarray(arrays["eq_yval"][:k]),
                           x.sort_order, True)
            out["tew_eq_mul"] = ("pass" if same(ops.tew_eq(dev(x), dev(y), 2),
                                                ref.tew_eq(x, y, 2)) else "fail")
    return out


def save_arrays(d, arrays, meta):
    os.makedirs(d, exist_ok=True)
    for k, a in arrays.items():
        np.save(os.path.join(d, k + ".npy"), a)
    with open(os.path.join(d, "meta.json"), "w") as fh:
        json.dump(meta, fh)


def load_arrays(d):
    meta = json.load(open(os.path.join(d, "meta.json")))
    arrays = {f[:-4]: np.load(os.path.join(d, f)) for f in os.listdir(d) if f.endswith(".npy")}
    return arrays, meta


# ===========================================================================
# GPU workloads (torch + the C-ABI library)


class _OpRecord:
    """An Op's name and timings without its closures (which hold device state)."""

    def __init__(self, op):
        self.name, self.times, self.units = op.name, list(op.times), op.units


class Op:
    def __init__(self, name, fn, units, bytes_fn, prep=None):
        self.name, self.fn, self.units, self.bytes_fn = name, fn, units, bytes_fn
        self.prep = prep  # untimed setup before each call (e.g. restore an unsorted input)
        self.times = []
        self.launches = 0


DIST = None  # torch.distributed when running under torchrun with N > 1


def allreduce(t):
    """MTTKRP's exchange for the weak-scaled workloads: every
    rank holds the dims[n] x R partial of its own instance; NCCL all-reduce."""
    if DIST is not None:
        DIST.all_reduce(t, op=DIST.ReduceOp.SUM)
    return t


def _np(t):
    return t.cpu().numpy()


def _idx_np(t):
    return t.cpu().numpy().view(np.uint32)


def _strided(n, k):
    """Positions of a uniform strided sample of k of n entries (sorted order
    kept, so a sample of a sorted coalesced tensor is sorted and coalesced)."""
    s = max(1, n // max(1, k))
    return slice(0, s * min(k, n), s)


class Workload:
    name = ""
    STRONG = False
    preprocess = {}

    def config(self):
        return {}


class C1(Workload):
    """BASELINE configs[0]: MTTKRP mode 0 (R=16) + TS add/mul by 2.5, 1M nnz."""

    name = "c1-mttkrp-ts"
    MTTKRP = "seg"

    def __init__(self, seed, device, scale=1.0, mttkrp=None):
        import torch
        from paper_1902_03317_b200 import generate, ops
        from paper_1902_03317_b200.coo import DeviceCOO
        c = generate.CONFIGS["c1"]
        self.dims, self.R = c["dims"], c["R"]
        self.nnz = int(c["nnz"] * scale)
        self.impl = mttkrp or self.MTTKRP
        self.x = generate.coo(self.dims, self.nnz, seed, c["zipf"], 0.0, 1.0, [0, 1, 2], device)
        self.f = [generate.uniform((d, self.R), seed, 100 + k, 0.0, 1.0, device)
                  for k, d in enumerate(self.dims)]
        self.out = torch.empty((self.dims[0], self.R), dtype=torch.float32, device=f"cuda:{device}")
        self.z = DeviceCOO.empty(self.dims, self.nnz, device)
        n, N, R = self.nnz, 3, self.R
        if self.impl == "plan":
            t0 = time.perf_counter()
            self.plan = ops.mttkrp_plan(self.x, 0, R)
            self.preprocess = {"mttkrp_m0_plan_s": time.perf_counter() - t0}
            mt = lambda: ops.mttkrp(self.plan, self.f, 0, out=self.out, sync=False)  # noqa: E731
        else:
            mt = lambda: ops.mttkrp(self.x, self.f, 0, ops.MTTKRP_SEGMENTED,  # noqa: E731
                                    out=self.out, sync=False)
        self.ops = [
            Op("mttkrp_m0", lambda: allreduce(mt()), n,
               lambda: tensor_bytes(n, N) + 4 * R * sum(self.dims)),
            Op("ts_add", lambda: ops.ts(self.x, 2.5, ops.SCALAR_ADD, out=self.z, sync=False), n,
               lambda: 2 * tensor_bytes(n, N)),
            Op("ts_mul", lambda: ops.ts(self.x, 2.5, ops.SCALAR_MUL, out=self.z, sync=False), n,
               lambda: 2 * tensor_bytes(n, N)),
        ]

    def config(self):
        return {"workload": self.name, "baseline_config": "configs[0] (C1)", "dims": self.dims,
                "nnz": self.nnz, "R": self.R, "mttkrp": self.impl,
                "mttkrp_input": "sorted (0,1,2) (mode-0 leading)"}

    def cpu_arrays(self):
        arrays = {f"x_i{d}": _idx_np(self.x.indices[d]) for d in range(3)}
        arrays["x_val"] = _np(self.x.values)
        arrays.update({f"f{d}": _np(f) for d, f in enumerate(self.f)})
        return arrays, {"dims": self.dims, "sort_order": [0, 1, 2], "sample_nnz": self.nnz,
                        "sample": f"full C1 workload: mttkrp mode 0 (R={self.R}, faster "
                                  f"strategy) + ts add/mul on {self.nnz} nnz"}

    def e2e_arrays(self):
        """The full workload as host arrays for the C++ drop-in leg."""
        return self.cpu_arrays()

    # e2e through the C-ABI with host buffers
    E2E_CHUNKS = 4
    E2E_PATH = ("ops.* -> C-ABI; pinned host buffers; x uploaded in 4 chunks (TS of each chunk "
                "and its download overlap the next chunk's upload), factors up, MTTKRP on the "
                "whole tensor, its I x R result and both TS outputs down")

    def e2e_host(self, device=0):
        import torch
        from paper_1902_03317_b200.coo import DeviceCOO
        from paper_1902_03317_b200.staging import PinnedCOO, Pipeline
        dev = torch.device("cuda", device)
        n = self.nnz
        return {"pipe": Pipeline(dev),
                "px": PinnedCOO.from_host(self.x.to_host()),
                "pf": [f.cpu().pin_memory() for f in self.f],
                "dx": DeviceCOO(list(self.dims), [torch.empty(n, dtype=torch.int32, device=dev)
                                                  for _ in self.dims],
                                torch.empty(n, dtype=torch.float32, device=dev), [0, 1, 2], True),
                "df": [torch.empty_like(f) for f in self.f],
                "dz": [DeviceCOO.empty(self.dims, n, dev) for _ in range(2)],
                "dout": torch.empty((self.dims[0], self.R), dtype=torch.float32, device=dev),
                "out_ts": [PinnedCOO(self.dims, n) for _ in range(2)],
                "out_m": torch.empty((self.dims[0], self.R), dtype=torch.float32).pin_memory()}

    def e2e_step(self, host):
        """Pinned host inputs -> MTTKRP + TS add/mul -> pinned host outputs.
        Returns (h2d, d2h) bytes."""
        import torch
        from paper_1902_03317_b200 import ops
        from paper_1902_03317_b200.staging import Pipeline, chunk_bounds, view
        pl, px, dx = host["pipe"], host["px"], host["dx"]
        h2d = d2h = 0
        pl.begin()
        with torch.cuda.stream(pl.h2d):
            for a, b in zip(host["df"], host["pf"]):
                a.copy_(b, non_blocking=True)
                h2d += b.numel() * 4
        b = chunk_bounds(self.nnz, self.E2E_CHUNKS)
        ev_in = []
        for lo, hi in zip(b[:-1], b[1:]):
            h2d += px.upload(dx, lo, hi, pl.h2d)
            ev_in.append(Pipeline.mark(pl.h2d))
        with torch.cuda.stream(pl.cmp):
            for c, (lo, hi) in enumerate(zip(b[:-1], b[1:])):
                pl.cmp.wait_event(ev_in[c])
                for k, op in enumerate((ops.SCALAR_ADD, ops.SCALAR_MUL)):
                    z = ops.ts(view(dx, lo, hi), 2.5, op, out=view(host["dz"][k], lo, hi),
                               sync=False)
                    pl.d2h.wait_event(Pipeline.mark(pl.cmp))
                    d2h += host["out_ts"][k].download(z, pl.d2h, at=lo)
            ops.mttkrp(dx, host["df"], 0, ops.MTTKRP_SEGMENTED, out=host["dout"], sync=False)
            pl.d2h.wait_event(Pipeline.mark(pl.cmp))
        with torch.cuda.stream(pl.d2h):
            host["out_m"].copy_(host["dout"], non_blocking=True)
            d2h += host["out_m"].numel() * 4
        pl.end()
        return h2d, d2h


class C2(Workload):
    """BASELINE configs[1]: TEW-eq x4 (shared pattern) + TEW add/mul (independent)."""

    name = "c2-tew_eq-tew"

    def __init__(self, seed, device, scale=1.0, mttkrp=None):
        import torch
        from paper_1902_03317_b200 import generate, ops
        from paper_1902_03317_b200.coo import DeviceCOO
        c = generate.CONFIGS["c2"]
        self.dims = c["dims"]
        self.nnz = int(c["nnz"] * scale)
        self.x = generate.coo(self.dims, self.nnz, seed, c["zipf"], 0.5, 1.5, [0, 1, 2], device)
        self.y = DeviceCOO(list(self.dims), [i.clone() for i in self.x.indices],
                           generate.uniform(self.nnz, seed, 77, 0.5, 1.5, device), [0, 1, 2],
                           True)
        self.y2 = generate.coo(self.dims, self.nnz, seed + 7919, c["zipf"], 0.5, 1.5, [0, 1, 2],
                               device)
        self.z = DeviceCOO.empty(self.dims, self.nnz, device)
        self.zu = DeviceCOO.empty(self.dims, 2 * self.nnz, device)
        self.cnt = torch.zeros(2, dtype=torch.int64, device=f"cuda:{device}")
        nz_add = ops.tew(self.x, self.y2, ops.ADD).nnz
        nz_mul = ops.tew(self.x, self.y2, ops.MUL).nnz
        self.nz = {"add": nz_add, "mul": nz_mul}
        n, N = self.nnz, 3
        self.ops = []
        for opn, op in (("add", ops.ADD), ("sub", ops.SUB), ("mul", ops.MUL), ("div", ops.DIV)):
            self.ops.append(Op(f"tew_eq_{opn}",
                               (lambda op=op: ops.tew_eq(self.x, self.y, op, out=self.z,
                                                         sync=False)),
                               n, lambda: 3 * tensor_bytes(n, N)))
        for opn, op, k in (("add", ops.ADD, 0), ("mul", ops.MUL, 1)):
            nz = self.nz[opn]
            self.ops.append(Op(f"tew_{opn}",
                               (lambda op=op, k=k: ops.tew_device(self.x, self.y2, op, self.zu,
                                                                  self.cnt[k:k + 1])),
                               2 * n, (lambda nz=nz: tensor_bytes(2 * n + nz, N))))

    def config(self):
        return {"workload": self.name, "baseline_config": "configs[1] (C2)", "dims": self.dims,
                "nnz": self.nnz, "order": 3, "values": "U[0.5,1.5)",
                "pattern": "uniform distinct tuples, sorted (0,1,2)",
                "tew_second_pattern_nnz": self.nnz, "tew_union": self.nz["add"],
                "tew_intersection": self.nz["mul"]}

    def cpu_arrays(self):
        arrays = {f"x_i{d}": _idx_np(self.x.indices[d]) for d in range(3)}
        arrays["x_val"] = _np(self.x.values)
        arrays["yval"] = _np(self.y.values)
        arrays.update({f"y2_i{d}": _idx_np(self.y2.indices[d]) for d in range(3)})
        arrays["y2_val"] = _np(self.y2.values)
        return arrays, {"dims": self.dims, "sort_order": [0, 1, 2], "sample_nnz": self.nnz,
                        "sample": f"full C2 workload (4 x tew_eq on {self.nnz} nnz + tew "
                                  f"add/mul on {self.nnz} + {self.nnz} nnz)"}

    def host_inputs(self):
        return [self.x.to_host(), self.y.to_host(), self.y2.to_host()]

    def e2e_arrays(self):
        """The full workload as host arrays for the C++ drop-in leg."""
        return self.cpu_arrays()

    E2E_CHUNKS = 8
    E2E_PATH = ("ops.* -> C-ABI; pinned host buffers; H2D / kernels / D2H overlapped on three "
                "streams (staging.Pipeline), x/y uploaded in 8 chunks")

    def e2e_host(self, device=0):
        import torch
        from paper_1902_03317_b200.coo import DeviceCOO
        from paper_1902_03317_b200.staging import PinnedCOO, Pipeline
        dev = torch.device("cuda", device)
        n = self.nnz
        return {"pipe": Pipeline(dev),
                "pinned": [PinnedCOO.from_host(h) for h in self.host_inputs()],
                "dev": [DeviceCOO(list(self.dims), [torch.empty(n, dtype=torch.int32, device=dev)
                                                    for _ in self.dims],
                                  torch.empty(n, dtype=torch.float32, device=dev), [0, 1, 2],
                                  True) for _ in range(3)],
                "dz": [DeviceCOO.empty(self.dims, n, dev) for _ in range(4)],
                "dzu": [DeviceCOO.empty(self.dims, 2 * n, dev),
                        DeviceCOO.empty(self.dims, n, dev)],
                "out_eq": [PinnedCOO(self.dims, n) for _ in range(4)],
                "out_tew": [PinnedCOO(self.dims, 2 * n), PinnedCOO(self.dims, n)]}

    def e2e_step(self, host):
        import torch
        from paper_1902_03317_b200 import ops
        from paper_1902_03317_b200.staging import Pipeline, chunk_bounds, view
        pl = host["pipe"]
        (px, py, py2), (dx, dy, dy2) = host["pinned"], host["dev"]
        h2d = d2h = 0
        pl.begin()
        b = chunk_bounds(self.nnz, self.E2E_CHUNKS)
        ev_in = []
        for lo, hi in zip(b[:-1], b[1:]):
            h2d += px.upload(dx, lo, hi, pl.h2d) + py.upload(dy, lo, hi, pl.h2d)
            ev_in.append(Pipeline.mark(pl.h2d))
        h2d += py2.upload(dy2, 0, self.nnz, pl.h2d)
        ev_y2 = Pipeline.mark(pl.h2d)
        with torch.cuda.stream(pl.cmp):
            for c, (lo, hi) in enumerate(zip(b[:-1], b[1:])):
                pl.cmp.wait_event(ev_in[c])
                for k, op in enumerate((ops.ADD, ops.SUB, ops.MUL, ops.DIV)):
                    z = ops.tew_eq(view(dx, lo, hi), view(dy, lo, hi), op,
                                   out=view(host["dz"][k], lo, hi), sync=False)
                    pl.d2h.wait_event(Pipeline.mark(pl.cmp))
                    d2h += host["out_eq"][k].download(z, pl.d2h, at=lo)
            pl.cmp.wait_event(ev_y2)
            for k, op in enumerate((ops.ADD, ops.MUL)):
                zu = host["dzu"][k]
                z = ops.tew(dx, dy2, op, out=view(zu, 0, zu.nnz))
                pl.d2h.wait_event(Pipeline.mark(pl.cmp))
                d2h += host["out_tew"][k].download(z, pl.d2h)
        pl.end()
        return h2d, d2h


class C3(Workload):
    """configs[2]: TTV and TTM (R=16) along every mode, 50M nnz, mode-0 Zipf(1.1)."""

    name = "c3-ttv-ttm"
    CPU_SAMPLE = 2_000_000

    def __init__(self, seed, device, scale=1.0, mttkrp=None):
        from paper_1902_03317_b200 import generate, ops
        from paper_1902_03317_b200.coo import DeviceCOO
        c = generate.CONFIGS["c3"]
        self.dims, self.R = c["dims"], c["R"]
        self.nnz = int(c["nnz"] * scale)
        base = generate.coo(self.dims, self.nnz, seed, c["zipf"], 0.0, 1.0, None, device)
        self.xs, self.fib, self.v, self.u = [], [], [], []
        n, N, R = self.nnz, 3, self.R
        self.ops = []
        max_nf = 0
        for mode in range(3):
            xs = base.clone()
            ops.sort_lexicographic(xs, ops.mode_last_order(3, mode))
            fib = ops.build_fiber_index(xs, mode)
            self.xs.append(xs)
            self.fib.append(fib)
            self.v.append(generate.uniform(self.dims[mode], seed, 200 + mode, -1.0, 1.0, device))
            self.u.append(generate.uniform((self.dims[mode], R), seed, 300 + mode, -1.0, 1.0,
                                           device))
            max_nf = max(max_nf, fib.nfibs)
        self.host_x = base.to_host()  # e2e: the caller's copy (draw order, unsorted)
        del base
        self.max_nf = max_nf
        self.zv = DeviceCOO.empty([1, 1], max_nf, device)
        self.zm = DeviceCOO.empty([1, 1, 1], max_nf * R, device)
        for mode in range(3):
            nf, I = self.fib[mode].nfibs, self.dims[mode]
            self.ops.append(Op(
                f"ttv_m{mode}",
                lambda m=mode: ops.ttv(self.xs[m], self.v[m], m, self.fib[m],
                                       out=DeviceCOO([1, 1], [a[:self.fib[m].nfibs] for a in
                                                              self.zv.indices[:2]],
                                                     self.zv.values[:self.fib[m].nfibs])),
                n, lambda nf=nf, I=I: 8 * n + nf * (4 + 8 * (N - 1) + 4) + 4 * I))
            self.ops.append(Op(
                f"ttm_m{mode}",
                lambda m=mode: ops.ttm(self.xs[m], self.u[m], m, self.fib[m],
                                       out=DeviceCOO([1, 1, 1], [a[:self.fib[m].nfibs * R] for a
                                                                 in self.zm.indices],
                                                     self.zm.values[:self.fib[m].nfibs * R])),
                n, lambda nf=nf, I=I: 8 * n + nf * (4 + 4 * (N - 1)) + nf * R * (4 * N + 4)
                + 4 * I * R))

    def config(self):
        return {"workload": self.name, "baseline_config": "configs[2] (C3)", "dims": self.dims,
                "nnz": self.nnz, "R": self.R, "nfibs": [f.nfibs for f in self.fib],
                "mode0": "Zipf(1.1) over a seeded id permutation; modes 1,2 uniform"}

    # e2e through the public API from host buffers (the full workload)
    E2E_PATH = ("ops.* -> C-ABI from pinned host buffers, every step: x (draw order, 0.8 GB), "
                "the three vectors and matrices uploaded; per mode x sorted mode-last and its "
                "fiber index built on the device (the preprocessing a host caller pays), TTV and "
                "TTM run and their full outputs (indices + values; TTM's is nfibs x R entries) "
                "downloaded -- 24 GB down per step, which bounds it")

    def e2e_host(self, device=0):
        import torch
        from paper_1902_03317_b200.coo import DeviceCOO
        from paper_1902_03317_b200.staging import PinnedCOO, Pipeline
        dev = torch.device("cuda", device)
        n = self.nnz
        host = {"pipe": Pipeline(dev), "px": PinnedCOO.from_host(self.host_x),
                "pv": [v.cpu().pin_memory() for v in self.v],
                "pu": [u.cpu().pin_memory() for u in self.u]}
        self.xs, self.fib, self.ops = [], [], []
        torch.cuda.synchronize()
        torch.cuda.empty_cache()

        def coo():
            return DeviceCOO(list(self.dims), [torch.empty(n, dtype=torch.int32, device=dev)
                                               for _ in self.dims],
                             torch.empty(n, dtype=torch.float32, device=dev), None, True)
        host["dx"], host["work"] = coo(), coo()
        host["dv"] = [torch.empty_like(v, device=dev) for v in host["pv"]]
        host["du"] = [torch.empty_like(u, device=dev) for u in host["pu"]]
        host["out_v"] = PinnedCOO([1, 1], self.max_nf)
        host["out_m"] = PinnedCOO([1, 1, 1], self.max_nf * self.R)
        return host

    def e2e_step(self, host):
        import torch
        from paper_1902_03317_b200 import ops
        from paper_1902_03317_b200.coo import DeviceCOO
        from paper_1902_03317_b200.staging import Pipeline, chunk_bounds
        pl, R = host["pipe"], self.R
        h2d = d2h = 0
        pl.begin()
        b = chunk_bounds(self.nnz, 4)
        for lo, hi in zip(b[:-1], b[1:]):
            h2d += host["px"].upload(host["dx"], lo, hi, pl.h2d)
        with torch.cuda.stream(pl.h2d):
            for d_, p_ in zip(host["dv"] + host["du"], host["pv"] + host["pu"]):
                d_.copy_(p_, non_blocking=True)
                h2d += p_.numel() * 4
        ev_in = Pipeline.mark(pl.h2d)
        with torch.cuda.stream(pl.cmp):
            pl.cmp.wait_event(ev_in)
            work = host["work"]
            for m in range(3):
                for a, s_ in zip(work.indices, host["dx"].indices):
                    a.copy_(s_, non_blocking=True)
                work.values.copy_(host["dx"].values, non_blocking=True)
                work.sort_order = None
                ops.sort_lexicographic(work, ops.mode_last_order(3, m), sync=False)
                fib = ops.build_fiber_index(work, m)
                nf = fib.nfibs
                # the output buffers are shared by the modes: the previous
                # download must have left them
                pl.cmp.wait_event(Pipeline.mark(pl.d2h))
                zv = ops.ttv(work, host["dv"][m], m, fib,
                             out=DeviceCOO([1, 1], [a[:nf] for a in self.zv.indices[:2]],
                                           self.zv.values[:nf]))
                pl.d2h.wait_event(Pipeline.mark(pl.cmp))
                d2h += host["out_v"].download(zv, pl.d2h)
                zm = ops.ttm(work, host["du"][m], m, fib,
                             out=DeviceCOO([1, 1, 1], [a[:nf * R] for a in self.zm.indices],
                                           self.zm.values[:nf * R]))
                pl.d2h.wait_event(Pipeline.mark(pl.cmp))
                d2h += host["out_m"].download(zm, pl.d2h)
        pl.end()
        return h2d, d2h

    def cpu_arrays(self):
        # the first k entries of each mode-last sorted copy: whole fibers but
        # the last
        k = min(self.CPU_SAMPLE, self.nnz)
        arrays = {}
        for m in range(3):
            for d in range(3):
                arrays[f"m{m}_i{d}"] = _idx_np(self.xs[m].indices[d][:k])
            arrays[f"m{m}_val"] = _np(self.xs[m].values[:k])
            arrays[f"v{m}"] = _np(self.v[m])
            arrays[f"u{m}"] = _np(self.u[m])
        return arrays, {"dims": self.dims, "sample_nnz": k,
                        "sort_orders": [list(x.sort_order) for x in self.xs],
                        "sample": f"ttv + ttm (R={self.R}) along every mode on the first {k} "
                                  "entries of each mode-last sorted copy"}


class C4(Workload):
    """configs[3]: MTTKRP every mode, R=32, 4th order, 100M nnz, Zipf(1.2) modes."""

    name = "c4-mttkrp"
    MTTKRP = "plan"
    CPU_SAMPLE = 4_000_000

    def __init__(self, seed, device, scale=1.0, mttkrp=None):
        import torch
        from paper_1902_03317_b200 import generate, ops
        c = generate.CONFIGS["c4"]
        self.dims, self.R = c["dims"], c["R"]
        self.nnz = int(c["nnz"] * scale)
        self.impl = mttkrp or self.MTTKRP
        base = generate.coo(self.dims, self.nnz, seed, c["zipf"], 0.0, 1.0, None, device)
        self.f = [generate.uniform((d, self.R), seed, 100 + k, 0.0, 1.0, device)
                  for k, d in enumerate(self.dims)]
        idx = torch.arange(0, self.nnz, max(1, self.nnz // self.CPU_SAMPLE),
                           device=base.values.device)[: self.CPU_SAMPLE]
        from paper_1902_03317_b200.coo import DeviceCOO
        self.sample = DeviceCOO(list(self.dims), [i[idx] for i in base.indices], base.values[idx],
                                None, True)
        self.xs, self.plans, self.preprocess = [], [], {}
        for mode in range(4):
            if self.impl == "plan":
                t0 = time.perf_counter()
                self.plans.append(ops.mttkrp_plan(base, mode, self.R))
                self.preprocess[f"mttkrp_m{mode}_plan_s"] = time.perf_counter() - t0
            else:
                xs = base.clone()
                ops.sort_lexicographic(xs, [mode] + [d for d in range(4) if d != mode])
                self.xs.append(xs)
        self.host_x = base.to_host()  # e2e: the caller's copy (draw order, unsorted)
        del base
        self.out = [torch.empty((d, self.R), dtype=torch.float32, device=f"cuda:{device}")
                    for d in self.dims]
        n, N, R = self.nnz, 4, self.R
        src = self.plans if self.impl == "plan" else self.xs
        strat = {} if self.impl == "plan" else {"strategy": ops.MTTKRP_SEGMENTED}
        self.ops = [Op(f"mttkrp_m{m}",
                       lambda m=m: allreduce(ops.mttkrp(src[m], self.f, m, out=self.out[m],
                                                        sync=False, **strat)),
                       n, lambda: tensor_bytes(n, N) + 4 * R * sum(self.dims))
                    for m in range(4)]

    def config(self):
        return {"workload": self.name, "baseline_config": "configs[3] (C4)", "dims": self.dims,
                "nnz": self.nnz, "R": self.R, "dist": "every mode Zipf(1.2), shuffled ids",
                "mttkrp": self.impl,
                "mttkrp_input": ("one plan per mode (preprocessing)" if self.impl == "plan" else
                                 "one mode-leading sorted copy per mode (preprocessing)")}

    def cpu_arrays(self):
        from paper_1902_03317_b200 import ops
        return _mode_sorted_sample_arrays(self, ops, 4)

    # e2e through the public API from host buffers (the full workload)
    E2E_PATH = ("ops.* -> C-ABI from pinned host buffers, every step: x (draw order, 2 GB) and "
                "the four factors uploaded; per mode an MTTKRP plan built (a 67-bit key sort, the "
                "preprocessing a host caller pays) and executed, its I x R result downloaded "
                "while the next plan builds")

    def e2e_host(self, device=0):
        import torch
        from paper_1902_03317_b200.coo import DeviceCOO
        from paper_1902_03317_b200.staging import PinnedCOO, Pipeline
        dev = torch.device("cuda", device)
        n = self.nnz
        hf = [f.cpu().pin_memory() for f in self.f]
        for p_ in self.plans:
            p_.close()
        self.plans, self.xs, self.ops = [], [], []
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        host = {"pipe": Pipeline(dev), "px": PinnedCOO.from_host(self.host_x), "pf": hf}
        host["dx"] = DeviceCOO(list(self.dims), [torch.empty(n, dtype=torch.int32, device=dev)
                                                 for _ in self.dims],
                               torch.empty(n, dtype=torch.float32, device=dev), None, True)
        host["df"] = [torch.empty(tuple(f.shape), dtype=torch.float32, device=dev) for f in hf]
        host["dout"] = self.out
        host["out_m"] = [torch.empty((d, self.R), dtype=torch.float32).pin_memory()
                         for d in self.dims]
        return host

    def e2e_step(self, host):
        import torch
        from paper_1902_03317_b200 import ops
        from paper_1902_03317_b200.staging import Pipeline, chunk_bounds
        pl = host["pipe"]
        h2d = d2h = 0
        pl.begin()
        b = chunk_bounds(self.nnz, 4)
        for lo, hi in zip(b[:-1], b[1:]):
            h2d += host["px"].upload(host["dx"], lo, hi, pl.h2d)
        ev_x = Pipeline.mark(pl.h2d)  # the plan builds start here
        with torch.cuda.stream(pl.h2d):
            for a, f in zip(host["df"], host["pf"]):
                a.copy_(f, non_blocking=True)
                h2d += f.numel() * 4
        ev_f = Pipeline.mark(pl.h2d)
        with torch.cuda.stream(pl.cmp):
            pl.cmp.wait_event(ev_x)
            for m in range(4):
                plan = ops.mttkrp_plan(host["dx"], m, self.R)
                pl.cmp.wait_event(ev_f)
                ops.mttkrp(plan, host["df"], m, out=host["dout"][m], sync=False)
                pl.d2h.wait_event(Pipeline.mark(pl.cmp))
                with torch.cuda.stream(pl.d2h):
                    host["out_m"][m].copy_(host["dout"][m], non_blocking=True)
                d2h += host["out_m"][m].numel() * 4
                plan.close()  # stream-ordered release: no device synchronisation
        pl.end()
        return h2d, d2h


def _mode_sorted_sample_arrays(wl, ops, N):
    """Uniform strided sample of the tensor (wl.sample, taken on the device),
    sorted with each mode leading (the order the GPU kernels get), plus the
    full factors."""
    arrays, orders = {}, []
    for m in range(N):
        s = wl.sample.clone()
        order = [m] + [d for d in range(N) if d != m]
        ops.sort_lexicographic(s, order)
        orders.append(order)
        for d in range(N):
            arrays[f"m{m}_i{d}"] = _idx_np(s.indices[d])
        arrays[f"m{m}_val"] = _np(s.values)
        del s
    arrays.update({f"f{d}": _np(f) for d, f in enumerate(wl.f)})
    k = wl.sample.nnz
    return arrays, {"dims": wl.dims, "sample_nnz": k, "sort_orders": orders,
                    "sample": f"mttkrp (R={wl.R}, faster strategy per mode) along every mode "
                              f"on a uniform strided sample of {k} of the {wl.nnz} entries, "
                              "sorted with the mode leading, full-size factors"}


class C5(Workload):
    """BASELINE configs[4] (C5): MTTKRP modes 0-2 (R=32) + TEW-eq mul on a
    1B-nnz order-3 tensor, every mode Zipf(1.1). One GPU holds the tensor
    (16 GB), one MTTKRP plan per mode (16 GB each) and the TEW-eq operand and
    output. Under torchrun the tensor is sharded (strong scaling)."""

    name = "c5-mttkrp-tew_eq"
    STRONG = True
    MTTKRP = "plan"
    CPU_SAMPLE = 16_000_000

    def __init__(self, seed, device, scale=1.0, mttkrp=None):
        import torch
        from paper_1902_03317_b200 import generate, ops
        from paper_1902_03317_b200.coo import DeviceCOO
        c = generate.CONFIGS["c5"]
        self.dims, self.R = c["dims"], c["R"]
        self.nnz = int(c["nnz"] * scale)
        self.impl = mttkrp or self.MTTKRP
        self.seed, self.device = seed, device
        dev = f"cuda:{device}"
        x = generate.coo(self.dims, self.nnz, seed, c["zipf"], 0.0, 1.0, [0, 1, 2], device)
        self.f = [generate.uniform((d, self.R), seed, 100 + k, 0.0, 1.0, device)
                  for k, d in enumerate(self.dims)]
        # TEW-eq operand: same pattern in its own buffers (as SURVEY 8(d) counts
        # the bytes), values U[0.5,1.5)
        self.y = DeviceCOO(list(self.dims), [i.clone() for i in x.indices],
                           generate.uniform(self.nnz, seed, 77, 0.5, 1.5, device), [0, 1, 2], True)
        sl = _strided(self.nnz, self.CPU_SAMPLE)
        self.sample = DeviceCOO(list(self.dims), [i[sl].clone() for i in x.indices],
                                x.values[sl].clone(), [0, 1, 2], True)
        self.sample_y = self.y.values[sl].clone()
        self.out = [torch.empty((d, self.R), dtype=torch.float32, device=dev) for d in self.dims]
        n, N, R = self.nnz, 3, self.R
        world = DIST.get_world_size() if DIST is not None else 1
        me = DIST.get_rank() if DIST is not None else 0
        self.preprocess = {}
        self.x = x
        if world == 1:
            src = self._mttkrp_inputs(x, None)
            self.z = DeviceCOO.empty(self.dims, self.nnz, device)
            self.ops = [Op(f"mttkrp_m{m}", lambda m=m: self._mttkrp(src[m], m), n,
                           lambda: tensor_bytes(n, N) + 4 * R * sum(self.dims))
                        for m in range(3)]
            self.ops.append(Op("tew_eq_mul",
                               lambda: ops.tew_eq(self.x, self.y, ops.MUL, out=self.z, sync=False),
                               n, lambda: 3 * tensor_bytes(n, N)))
            return
        # N > 1: MTTKRP on row-aligned nnz shards of each
        # mode-leading order, the owned row blocks all-gathered over NCCL (half
        # the all-reduce's volume); TEW-eq on contiguous nnz shards, no exchange.
        # Units per rank = nnz / world, so `value` is the whole tensor's nnz/s.
        from paper_1902_03317_b200 import parallel
        self.blocks = []
        lo, hi = parallel.shard_range(self.nnz, world, me)
        xe = parallel.slice_coo(x, lo, hi).clone()
        self.ye = parallel.slice_coo(self.y, lo, hi).clone()
        del self.y
        shards = []
        for m in range(3):
            xs = x.clone()
            if m:
                ops.sort_lexicographic(xs, [m] + [d for d in range(3) if d != m])
            rr = parallel.row_aligned_ranges(xs.indices[m], world)
            self.blocks.append(parallel.row_blocks(xs.indices[m], rr, self.dims[m]))
            shards.append(parallel.slice_coo(xs, *rr[me]).clone())
            del xs
            torch.cuda.empty_cache()
        del x
        self.x = xe
        src = self._mttkrp_inputs(None, shards)
        del shards
        torch.cuda.empty_cache()
        self.z = DeviceCOO.empty(self.dims, hi - lo, device)
        share = n / world

        def mt(m):
            part = lambda s, f, mm: self._mttkrp(s, mm)  # noqa: E731
            return parallel.mttkrp_row_allgather(src[m], self.f, m, self.dims[m], R,
                                                 self.blocks[m], part)
        self.ops = [Op(f"mttkrp_m{m}", lambda m=m: mt(m), share,
                       lambda: (tensor_bytes(n, N) + 4 * R * sum(self.dims)) / world)
                    for m in range(3)]
        self.ops.append(Op("tew_eq_mul",
                           lambda: ops.tew_eq(self.x, self.ye, ops.MUL, out=self.z, sync=False),
                           share, lambda: 3 * tensor_bytes(n, N) / world))

    def _mttkrp_inputs(self, x, shards):
        """Plans (or mode-leading sorted copies for --mttkrp seg) per mode;
        building them is preprocessing, timed apart."""
        import torch
        from paper_1902_03317_b200 import ops
        src = []
        for m in range(3):
            t = x if shards is None else shards[m]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if self.impl == "plan":
                src.append(ops.mttkrp_plan(t, m, self.R))
            else:
                xs = t.clone() if shards is None else t
                if shards is None or m:
                    ops.sort_lexicographic(xs, [m] + [d for d in range(3) if d != m])
                src.append(xs)
            torch.cuda.synchronize()
            self.preprocess[f"mttkrp_m{m}_{'plan' if self.impl == 'plan' else 'sort'}_s"] = \
                round(time.perf_counter() - t0, 4)
        return src

    def _mttkrp(self, src, m):
        from paper_1902_03317_b200 import ops
        if self.impl == "plan":
            return ops.mttkrp(src, self.f, m, out=self.out[m], sync=False)
        return ops.mttkrp(src, self.f, m, ops.MTTKRP_SEGMENTED, out=self.out[m], sync=False)

    def config(self):
        return {"workload": self.name, "baseline_config": "configs[4] (C5)", "dims": self.dims,
                "nnz": self.nnz, "R": self.R, "dist": "every mode Zipf(1.1), shuffled ids",
                "mttkrp": self.impl,
                "mttkrp_input": ("one plan per mode (mode-leading blocked copy + hot rows; "
                                 "preprocessing)" if self.impl == "plan" else
                                 "one mode-leading sorted copy per mode (preprocessing)"),
                "tew_eq": "mul against the same pattern, y U[0.5,1.5)"}

    def cpu_arrays(self):
        from paper_1902_03317_b200 import ops
        arrays, meta = _mode_sorted_sample_arrays(self, ops, 3)
        for d in range(3):
            arrays[f"eq_i{d}"] = _idx_np(self.sample.indices[d])
        arrays["eq_val"] = _np(self.sample.values)
        arrays["eq_yval"] = _np(self.sample_y)
        meta["eq_sort_order"] = [0, 1, 2]
        meta["sample"] += f" + tew_eq mul on the same {meta['sample_nnz']} entries"
        return arrays, meta

    # e2e through the public API from host buffers (the full workload)
    E2E_PATH = ("ops.* -> C-ABI from pinned host buffers, every step: x (mode-0 sorted, 16 GB), "
                "y and the three factors uploaded; per mode an MTTKRP plan built (sort + hot "
                "rows, the preprocessing a host caller pays) and executed, its I x R result "
                "downloaded while the next plan builds; TEW-eq mul per 1/16 chunk of y as it "
                "arrives (second kernel stream), each chunk of its output (indices + values) "
                "downloaded under the remaining uploads and the plan builds")

    def e2e_arrays(self):
        """The full workload as host arrays for the C++ drop-in leg (x in its
        mode-0 order, y's values, the factors)."""
        arrays = {f"x_i{d}": _idx_np(self.x.indices[d]) for d in range(3)}
        arrays["x_val"] = _np(self.x.values)
        arrays["yval"] = _np(self.y.values)
        arrays.update({f"f{d}": _np(f) for d, f in enumerate(self.f)})
        return arrays, {"dims": self.dims}

    def e2e_release(self):
        """Free the device-timed state (e2e needs the memory)."""
        import torch
        for k in ("x", "y", "z", "ye", "sample", "sample_y", "ops", "out"):
            if hasattr(self, k):
                delattr(self, k)
        torch.cuda.synchronize()
        torch.cuda.empty_cache()

    def e2e_host(self, device=0):
        import torch
        from paper_1902_03317_b200 import generate
        from paper_1902_03317_b200.coo import DeviceCOO
        from paper_1902_03317_b200.staging import PinnedCOO, Pipeline
        dev = torch.device("cuda", device)
        n = self.nnz
        hx = self.x.to_host()
        hy = self.y.to_host()
        hf = [f.cpu().pin_memory() for f in self.f]
        self.e2e_release()
        host = {"pipe": Pipeline(dev), "px": PinnedCOO.from_host(hx), "py": PinnedCOO.from_host(hy),
                "pf": hf}
        del hx, hy
        host["dx"] = DeviceCOO(list(self.dims), [torch.empty(n, dtype=torch.int32, device=dev)
                                                 for _ in self.dims],
                               torch.empty(n, dtype=torch.float32, device=dev), [0, 1, 2], True)
        host["dy"] = DeviceCOO(list(self.dims), [torch.empty(n, dtype=torch.int32, device=dev)
                                                 for _ in self.dims],
                               torch.empty(n, dtype=torch.float32, device=dev), [0, 1, 2], True)
        host["df"] = [torch.empty(tuple(f.shape), dtype=torch.float32, device=dev) for f in hf]
        host["dz"] = DeviceCOO.empty(self.dims, n, dev)
        host["dout"] = [torch.empty((d, self.R), dtype=torch.float32, device=dev)
                        for d in self.dims]
        host["out_m"] = [torch.empty((d, self.R), dtype=torch.float32).pin_memory()
                         for d in self.dims]
        host["out_eq"] = PinnedCOO(self.dims, n)
        return host

    def e2e_step(self, host):
        import torch
        from paper_1902_03317_b200 import ops
        from paper_1902_03317_b200.staging import Pipeline, chunk_bounds, view
        pl = host["pipe"]
        h2d = d2h = 0
        pl.begin()
        b = chunk_bounds(self.nnz, 8)
        for lo, hi in zip(b[:-1], b[1:]):
            h2d += host["px"].upload(host["dx"], lo, hi, pl.h2d)
        ev_x = Pipeline.mark(pl.h2d)  # the plan builds start here
        with torch.cuda.stream(pl.h2d):
            for a, b in zip(host["df"], host["pf"]):
                a.copy_(b, non_blocking=True)
                h2d += b.numel() * 4
        ev_f = Pipeline.mark(pl.h2d)
        # y arrives in chunks behind x; TEW-eq runs per chunk on the second
        # kernel stream (it does not depend on the plans) and each z chunk
        # goes back while later chunks still come up: PCIe both ways at once,
        # under the plan builds.
        by = chunk_bounds(self.nnz, 16)
        for lo, hi in zip(by[:-1], by[1:]):
            h2d += host["py"].upload(host["dy"], lo, hi, pl.h2d)
            ev = Pipeline.mark(pl.h2d)
            with torch.cuda.stream(pl.cmp2):
                pl.cmp2.wait_event(ev)
                z = ops.tew_eq(view(host["dx"], lo, hi), view(host["dy"], lo, hi), ops.MUL,
                               out=view(host["dz"], lo, hi), sync=False)
                pl.d2h.wait_event(Pipeline.mark(pl.cmp2))
            d2h += host["out_eq"].download(z, pl.d2h, at=lo)
        with torch.cuda.stream(pl.cmp):
            pl.cmp.wait_event(ev_x)
            for m in range(3):
                plan = ops.mttkrp_plan(host["dx"], m, self.R)
                pl.cmp.wait_event(ev_f)
                ops.mttkrp(plan, host["df"], m, out=host["dout"][m], sync=False)
                pl.d2h.wait_event(Pipeline.mark(pl.cmp))
                with torch.cuda.stream(pl.d2h):
                    host["out_m"][m].copy_(host["dout"][m], non_blocking=True)
                d2h += host["out_m"][m].numel() * 4
                plan.close()  # stream-ordered release: no device synchronisation
        pl.end()
        return h2d, d2h


class Pre(Workload):
    """SURVEY 8(f) "next" row 1: GPU preprocessing at parity and speed --
    sort_lexicographic (P/src/tensor.cpp:54-64) and build_fiber_index
    (:92-120), on C2's 10M tensor in draw (unsorted) order."""

    name = "pre-sort-fiber"
    CPU_SAMPLE = 2_000_000

    def __init__(self, seed, device, scale=1.0, mttkrp=None):
        from paper_1902_03317_b200 import generate, ops
        c = generate.CONFIGS["c2"]
        self.dims = c["dims"]
        self.nnz = int(c["nnz"] * scale)
        self.src = generate.coo(self.dims, self.nnz, seed, c["zipf"], 0.5, 1.5, None, device)
        self.work = self.src.clone()
        self.sorted = self.src.clone()
        ops.sort_lexicographic(self.sorted, [0, 1, 2])
        self.fib = ops.build_fiber_index(self.sorted, 2)
        n, N = self.nnz, 3

        def restore():
            for a, b in zip(self.work.indices, self.src.indices):
                a.copy_(b)
            self.work.values.copy_(self.src.values)
            self.work.sort_order = None

        self.ops = [
            Op("sort_lexicographic", lambda: ops.sort_lexicographic(self.work, [0, 1, 2],
                                                                    sync=False),
               n, lambda: 2 * tensor_bytes(n, N), prep=restore),
            Op("build_fiber_index", lambda: ops.build_fiber_index(self.sorted, 2),
               n, lambda: 8 * n + 4 * (self.fib.nfibs + 1)),
        ]

    def config(self):
        return {"workload": self.name, "dims": self.dims, "nnz": self.nnz,
                "sort": "draw order -> (0,1,2), stable LSD radix, bit-exact vs std::stable_sort",
                "fiber_index": "mode 2 on the (0,1,2)-sorted tensor",
                "note": "preprocessing, timed separately like the reference's sort_s"}

    def cpu_arrays(self):
        k = min(self.CPU_SAMPLE, self.nnz)
        arrays = {f"x_i{d}": _idx_np(self.src.indices[d][:k]) for d in range(3)}
        arrays["x_val"] = _np(self.src.values[:k])
        return arrays, {"dims": self.dims, "sample_nnz": k,
                        "sample": f"sort_lexicographic (0,1,2) of the first {k} entries "
                                  "(the reference's sort is serial)"}


class Tns(Workload):
    """.tns ingest (read_tns<float>, P/src/io.cpp:42-120)
    on C2's 10M-entry tensor written as text (1-based indices, values with 6
    decimals, one entry per line): the device parse of text already in HBM
    (spt_tns_scan + spt_tns_parse); e2e = read_tns(path) from the page cache
    (file -> pinned -> H2D -> parse)."""

    name = "tns-read"
    CPU_SAMPLE = 2_000_000

    def __init__(self, seed, device, scale=1.0, mttkrp=None):
        from paper_1902_03317_b200 import generate, tns
        c = generate.CONFIGS["c2"]
        self.dims = c["dims"]
        self.nnz = int(c["nnz"] * scale)
        x = generate.coo(self.dims, self.nnz, seed, c["zipf"], 0.5, 1.5, None, device)
        self.text = generate.tns_text(x)
        del x
        self.bytes = int(self.text.numel())
        n, N = self.nnz, 3
        self.ops = [Op("read_tns", lambda: tns.read_tns_bytes(self.text, None, device), n,
                       lambda: self.bytes + 4 * (N + 1) * n)]
        self.device = device

    def config(self):
        return {"workload": self.name, "dims": self.dims, "nnz": self.nnz,
                "text_bytes": self.bytes,
                "text": "C2's tensor (draw order) as .tns: 1-based indices, values %.6f, "
                        "single spaces, one entry per line",
                "note": "value: text resident in HBM; e2e: read_tns(path) from the page cache"}

    def cpu_arrays(self):
        t = self.text[: min(self.bytes, 64 << 20)].cpu().numpy()
        nl = np.flatnonzero(t == 10)
        k = min(self.CPU_SAMPLE, len(nl))
        t = np.ascontiguousarray(t[: nl[k - 1] + 1])
        return {"text": t}, {"dims": self.dims, "sample_nnz": k,
                             "sample": f"read_tns<float> of the first {k} lines "
                                       f"({t.size} bytes) from the page cache "
                                       "(the reference's reader is serial)"}

    E2E_PATH = ("tns.read_tns(path): file (page cache) -> pinned host buffer -> H2D -> "
                "device scan + parse; dims read back")

    def e2e_host(self, device=0):
        base = "/dev/shm" if os.path.isdir("/dev/shm") else None
        d = tempfile.mkdtemp(prefix="spt_tns_", dir=base)
        path = os.path.join(d, "x.tns")
        self.text.cpu().numpy().tofile(path)
        self._tmpdir = d
        return {"path": path}

    def e2e_step(self, host):
        from paper_1902_03317_b200 import tns
        z = tns.read_tns(host["path"], None, self.device)
        return self.bytes, 4 * len(z.dims)

    def e2e_done(self):
        d = getattr(self, "_tmpdir", None)
        if d:
            shutil.rmtree(d, ignore_errors=True)


WORKLOADS = {"c1": C1, "c2": C2, "c3": C3, "c4": C4, "c5": C5, "pre": Pre, "tns": Tns}


def report_rows(wl, ops_list):
    """Reference-schema rows (variant "gpu") for --report; flops are the
    sequential reference's counts (P/src/kernels_seq.cpp:37,51,65,99,144,172)."""
    from paper_1902_03317_b200 import report
    rows = []
    N = len(wl.dims)
    R = getattr(wl, "R", 0)
    pre = getattr(wl, "preprocess", {}) or {}
    for op in ops_list:
        name = op.name
        mode = opn = None
        if name.startswith("tew_eq"):
            kernel, opn = "tew_eq", name.split("_")[-1]
            fl = wl.nnz
        elif name.startswith("tew_"):
            kernel, opn = "tew", name.split("_")[1]
            nz = wl.nz[opn]
            fl = 2 * wl.nnz - nz if opn == "add" else nz
        elif name.startswith("ts_"):
            kernel, opn, fl = "ts", name.split("_")[1], wl.nnz
        elif name.startswith(("ttv", "ttm", "mttkrp")):
            kernel, _, mode = name.partition("_m")
            fl = {"ttv": 2 * wl.nnz, "ttm": 2 * R * wl.nnz, "mttkrp": N * R * wl.nnz}[kernel]
        else:
            kernel, fl = name, 0
        sort_s = sum(v for k, v in pre.items() if k.startswith(f"{name}_"))
        rows.append(report.bench_report(wl.name, wl.dims, wl.nnz, kernel,
                                        [t / 1e3 for t in op.times], fl, op=opn, mode=mode,
                                        rank=R if kernel in ("ttm", "mttkrp") else 0,
                                        sort_s=sort_s, preprocess_s=sort_s,
                                        crosscheck=getattr(wl, "crosscheck", {}).get(name)))
    return rows


# ===========================================================================
# entry points


def prep_cpu_inputs(args):
    """Separate process: build the workload on the GPU and write the CPU leg's
    host arrays (numpy files) for --impl reference."""
    import torch
    torch.cuda.set_device(0)
    W = WORKLOADS[args.workload]
    wl = W(args.seed, 0, args.scale, getattr(args, "mttkrp", None))
    arrays, meta = wl.cpu_arrays()
    meta["config"] = wl.config()  # the reference arm reports the same config
    save_arrays(args.prep_cpu, arrays, meta)


def main_reference(args, world, rank):
    """The reference's own CPU path on this host, on the workload's bounded
    sample; inputs from a separate prep process (no repo library loaded here)."""
    if rank != 0:
        return  # the reference arm runs on rank 0 only (CPU path)
    base = "/dev/shm" if os.path.isdir("/dev/shm") else None
    d = tempfile.mkdtemp(prefix="spt_ref_inputs_", dir=base)
    try:
        env = dict(os.environ)
        for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "LOCAL_WORLD_SIZE", "GROUP_RANK",
                  "ROLE_RANK", "TORCHELASTIC_RUN_ID"):
            env.pop(k, None)
        cmd = [sys.executable, os.path.abspath(__file__), "--prep-cpu", d, "--workload",
               args.workload, "--seed", str(args.seed), "--scale", str(args.scale)]
        subprocess.run(cmd, check=True, env=env)
        arrays, meta = load_arrays(d)
    finally:
        shutil.rmtree(d, ignore_errors=True)
    cb = run_cpu_leg(args.workload, arrays, meta, args.steps, args.warmup)
    cfg = meta["config"]
    line = {"metric": METRIC, "value": cb["value"], "unit": "nnz/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["step_s_mean"] * 1e3,
            "higher_is_better": True,
            "scaling": "strong" if WORKLOADS[args.workload].STRONG else "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Philox, BASELINE config shapes)", "impl": "reference",
            "config": cfg,
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "cpu_detail": {k: cb[k] for k in cb if k not in ("value", "unit", "cores", "kind",
                                                             "sample")},
            "e2e": {"value": cb["value"], "unit": "nnz/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def main_ours(args, world, rank, local):
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        global DIST
        DIST = dist

    from paper_1902_03317_b200 import _lib
    W = WORKLOADS[args.workload]
    # weak scaling: an independent instance per rank; strong (C5): one tensor
    wl = W(args.seed if W.STRONG else args.seed + 1009 * rank, local, args.scale, args.mttkrp)
    hbm, peak_src = peaks()
    ctx = _lib.Context.get(local)
    lib = _lib.load()
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream

    def run_op(op, timed):
        if op.prep is not None:
            op.prep()
        lib.spt_l2_flush(ctx.handle, sh)
        l0 = ctx.launches()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        op.fn()
        b.record(stream)
        if timed:
            op.launches += ctx.launches() - l0
        return a, b

    for _ in range(args.warmup):
        for op in wl.ops:
            run_op(op, False)
    torch.cuda.synchronize()
    _lib.check(lib.spt_ctx_check(ctx.handle, sh))

    clocks = Clocks(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev = []
    for _ in range(args.steps):
        ev.append([(op, *run_op(op, True)) for op in wl.ops])
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    _lib.check(lib.spt_ctx_check(ctx.handle, sh))
    step_ms = []
    for st in ev:
        tot = 0.0
        for op, a, b in st:
            ms = a.elapsed_time(b)
            op.times.append(ms)
            tot += ms
        step_ms.append(tot)
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    units_per_step = sum(op.units for op in wl.ops)
    value = world * units_per_step * args.steps / (total_ms / 1e3)

    ops_out = {}
    for op in wl.ops:
        mean_ms = statistics.mean(op.times)
        by = op.bytes_fn()
        gbs = by / (mean_ms / 1e3) / 1e9
        ops_out[op.name] = {"ms": round(mean_ms, 5),
                            "ms_median": round(statistics.median(op.times), 5),
                            "ms_max": round(max(op.times), 5),
                            "alg_bytes": int(by), "GB_s": round(gbs, 1),
                            "frac": round(gbs / hbm, 4), "nnz_s": op.units / (mean_ms / 1e3),
                            "launches_per_call": op.launches / args.steps}
    # MTTKRP's second floor: every gathered factor row costs at least one L1
    # wavefront (<= 128 B) per SM-cycle whether it hits L1, L2 or smem
    # ("Gather floor"); per rank's own units
    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    sm_hz = float(_measured_peaks().get("sm_max_mhz", 1965.0)) * 1e6
    for op in wl.ops:
        if op.name.startswith("mttkrp"):
            N, R = len(wl.dims), wl.R
            wf = op.units * (N - 1) * -(-4 * R // 128)
            floor_ms = wf / (props.multi_processor_count * sm_hz) * 1e3
            ops_out[op.name]["gather_floor_ms"] = round(floor_ms, 5)
            ops_out[op.name]["gather_floor_frac"] = round(floor_ms / ops_out[op.name]["ms"], 4)
    dom = max(wl.ops, key=lambda o: sum(o.times))
    d = ops_out[dom.name]
    roofline = {"bound": "hbm", "achieved": d["GB_s"], "peak": hbm, "unit": "GB/s",
                "frac": d["frac"], "traffic": None, "kernel": dom.name,
                "alg_bytes_per_launch": d["alg_bytes"], "peak_source": peak_src,
                "time_share": round(sum(dom.times) / sum(step_ms), 3)}
    if "gather_floor_ms" in d:
        roofline["gather_floor"] = {"ms": d["gather_floor_ms"], "frac": d["gather_floor_frac"],
                                    "model": "nnz*(N-1)*ceil(4R/128) L1 wavefronts / "
                                             "(SMs * SM clock)"}
    tr = os.path.join(ROOT, "profiles", f"traffic_{args.workload}.json")
    if os.path.exists(tr):
        t = json.load(open(tr))
        if t.get("mttkrp_impl", "seg") == getattr(wl, "impl", "seg") or \
                not dom.name.startswith("mttkrp"):
            roofline["traffic"] = t.get(dom.name)
            roofline["traffic_source"] = t.get("source", os.path.relpath(tr, ROOT))

    # everything that needs the device-timed state before e2e may release it
    gpu_launches = int(sum(op.launches for op in wl.ops))
    ops_snapshot = [_OpRecord(op) for op in wl.ops]  # the ops' timings outlive the device state
    rows = report_rows(wl, ops_snapshot) if (args.report and rank == 0) else None
    cpu_in = None
    if not args.no_cpu and rank == 0 and world == 1 and hasattr(wl, "cpu_arrays"):
        cpu_in = wl.cpu_arrays()

    e2e = e2e_dropin = None
    dropin = os.path.join(ROOT, "paper_1902_03317_b200", "host", "dropin_bench")
    dropin_dir = None
    if (not args.no_e2e and world == 1 and hasattr(wl, "e2e_arrays")
            and os.path.exists(dropin)):
        # inputs of the C++ drop-in leg (run after the pipeline, in its own process)
        arrays, meta = wl.e2e_arrays()
        base = "/dev/shm" if os.path.isdir("/dev/shm") else None
        dropin_dir = tempfile.mkdtemp(prefix="spt_e2e_", dir=base)
        save_arrays(dropin_dir, arrays, meta)
        del arrays
    if not args.no_e2e and hasattr(wl, "e2e_step"):
        # every rank runs its own host-buffer pipeline (its own PCIe link);
        # whole-job throughput over the slowest rank, like `value`
        host = wl.e2e_host(local)
        wl.e2e_step(host)
        torch.cuda.synchronize()
        times = []
        for _ in range(max(2, min(args.steps, 5))):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            a.record(stream)
            h2d, d2h = wl.e2e_step(host)
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        ms = statistics.mean(times)
        if dist:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        e2e = {"value": world * units_per_step / (ms / 1e3), "unit": "nnz/s",
               "h2d_bytes_per_step": world * h2d, "d2h_bytes_per_step": world * d2h,
               "ms_per_step": ms, "ms_each": [round(t, 3) for t in times],
               "path": getattr(wl, "E2E_PATH", "ops.* -> C-ABI")}
        del host
        if hasattr(wl, "e2e_done"):
            wl.e2e_done()
    if dropin_dir is not None:
        # the C++ drop-in (spten::gpu::*) on host SparseTensorCOO data in its own
        # process: every call uploads its operands from pageable std::vectors,
        # computes and returns its result by value (the reference API's contract)
        if hasattr(wl, "e2e_release"):
            wl.e2e_release()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        ctx.trim()
        try:
            key = {"c1-mttkrp-ts": "c1", "c2-tew_eq-tew": "c2", "c5-mttkrp-tew_eq": "c5"}[wl.name]
            env = {k: v for k, v in os.environ.items() if k not in ("OMP_PROC_BIND", "OMP_PLACES")}
            r = subprocess.run([dropin, dropin_dir, key, str(max(2, min(args.steps, 3))), "1"],
                               capture_output=True, text=True, env=env)
            res = json.loads(r.stdout.strip().splitlines()[-1])
            if "error" in res:
                e2e_dropin = {"value": None, "error": res["error"]}
            else:
                e2e_dropin = {"value": res["units_per_step"] / (res["ms_per_step"] / 1e3),
                              "unit": "nnz/s",
                              "h2d_bytes_per_step": int(res["h2d_bytes_per_step"]),
                              "d2h_bytes_per_step": int(res["d2h_bytes_per_step"]),
                              "ms_per_step": res["ms_per_step"], "ms_median": res["ms_median"],
                              "path": res["path"] + " (paper_1902_03317_b200/host/dropin_bench)",
                              "timing": "host wall clock per step; one call per op, operands "
                                        "uploaded from pageable vectors, results by value"}
        except (OSError, ValueError, IndexError, KeyError) as err:
            e2e_dropin = {"value": None, "error": str(err)}
        finally:
            shutil.rmtree(dropin_dir, ignore_errors=True)

    if cpu_in is not None:
        try:
            wl.crosscheck = crosscheck(args.workload, cpu_in[0], cpu_in[1])
        except Exception as e:  # reported, never silently replaced
            wl.crosscheck = {"error": str(e)}
        if args.report and rank == 0:
            rows = report_rows(wl, ops_snapshot)
    cpu = None
    if cpu_in is not None:
        try:
            cb = run_cpu_leg(args.workload, cpu_in[0], cpu_in[1], steps=5, warmup=1)
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            cpu["detail"] = {k: cb[k] for k in cb if k not in cpu}
        except Exception as e:  # reported, never silently replaced
            cpu = {"value": None, "unit": "nnz/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "strong" if W.STRONG else "weak",
                "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded Philox, BASELINE config shapes; public datasets "
                        "unavailable offline)",
                "config": wl.config(),
                "timing": {"l2": "inputs > L2 and L2 flushed before every op",
                           "clock": "CUDA events per op on the launch stream, max over ranks"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "e2e_dropin": e2e_dropin,
                "gpu_launches": gpu_launches,
                "clocks": clk, "ops": ops_out,
                "crosscheck": getattr(wl, "crosscheck", None),
                "preprocess_s": getattr(wl, "preprocess", {})}
        print(json.dumps(line))
        if rows is not None:
            from paper_1902_03317_b200 import report
            with open(args.report, "w") as fh:
                fh.write(report.emit_csv(rows) if args.report.endswith(".csv")
                         else report.emit_json(rows))
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mttkrp", default=None, choices=["plan", "seg"],
                    help="MTTKRP kernel (default per workload: C4/C5 plan, C1 seg)")
    ap.add_argument("--seed", type=int, default=20190210)
    ap.add_argument("--scale", type=float, default=1.0, help="nnz scale (testing only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--prep-cpu", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--report", default=None,
                    help="also write per-op rows in the reference's BenchReport schema "
                         "(.json or .csv, P/include/spten/report.hpp)")
    args = ap.parse_args()
    if args.prep_cpu:
        prep_cpu_inputs(args)
        return
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        main_reference(args, world, rank)
    else:
        main_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
