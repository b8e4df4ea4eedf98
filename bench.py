#!/usr/bin/env python
"""Benchmark of the B200 COO sparse-tensor kernels on the BASELINE.json configs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2]
                    [--impl ours|reference]

A step is one pass of the workload's ops over its seeded synthetic inputs
(already resident in HBM). Default workload = BASELINE.json configs[1] (C2):
TEW-eq add/sub/mul/div on two 10M-nnz tensors sharing a pattern, plus TEW
add/mul against an independent 10M-nnz pattern. `value` is nonzeros/s over
all ranks (TEW merge counts nnz_x + nnz_y), each op timed with CUDA events
on its stream after an L2 flush (inputs are also > L2). `roofline` is for the
op with the largest time share: algorithmic bytes per launch
/ mean event duration vs MEASURED_PEAKS.json hbm_gbs. `e2e` times the same ops
through the C-ABI with pinned host buffers, H2D of the inputs and D2H of the
outputs inside the timed region. `cpu_baseline` is the reference's own OpenMP
path (oracle/_ref, compiled from the reference sources) on this host.

Multi-GPU (torchrun): every rank runs its own instance of the workload (the
ops shard with no communication, "weak" scaling), timing = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "nonzeros/sec per COO op (MTTKRP/TTM/TTV/TEW/TS) & achieved HBM GB/s vs peak"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p)) if os.path.exists(p) else {}


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


# ---------------------------------------------------------------------------
# workloads


class Op:
    def __init__(self, name, fn, units, bytes_fn, e2e=None, prep=None):
        self.name, self.fn, self.units, self.bytes_fn = name, fn, units, bytes_fn
        self.prep = prep  # untimed setup before each call (e.g. restore an unsorted input)
        self.times = []
        self.launches = 0


def report_rows(wl, ops_list):
    """Reference-schema rows (variant "gpu") for --report; flops are the
    sequential reference's counts (P/src/kernels_seq.cpp:37,51,65,99,144,172)."""
    from paper_1902_03317_b200 import report
    rows = []
    N = len(wl.dims)
    R = getattr(wl, "R", 0)
    for op in ops_list:
        name = op.name
        kind, _, rest = name.rpartition("_") if name.startswith("tew_eq") else name.partition("_")
        mode = opn = None
        if name.startswith("tew_eq"):
            kernel, opn = "tew_eq", name.split("_")[-1]
            fl = wl.nnz
        elif name.startswith("tew_"):
            kernel, opn = "tew", rest
            nz = wl.nz[opn]
            fl = 2 * wl.nnz - nz if opn == "add" else nz
        elif name.startswith("ts_"):
            kernel, opn, fl = "ts", rest, wl.nnz
        else:
            kernel, mode = kind, rest.lstrip("m")
            fl = {"ttv": 2 * wl.nnz, "ttm": 2 * R * wl.nnz, "mttkrp": N * R * wl.nnz}[kernel]
        rows.append(report.bench_report(wl.name, wl.dims, wl.nnz, kernel,
                                        [t / 1e3 for t in op.times], fl, op=opn, mode=mode,
                                        rank=R if kernel in ("ttm", "mttkrp") else 0))
    return rows


def tensor_bytes(nnz, order):
    return nnz * (4 * order + 4)


DIST = None  # torch.distributed when running under torchrun with N > 1


def allreduce(t):
    """MTTKRP's one exchange step: every rank holds the
    dims[n] x R partial of its own nnz shard; NCCL all-reduce over NVLink."""
    if DIST is not None:
        DIST.all_reduce(t, op=DIST.ReduceOp.SUM)
    return t


class Workload:
    name = ""
    desc = ""

    def config(self):
        return {}


class C2(Workload):
    """BASELINE configs[1]: TEW-eq x4 (shared pattern) + TEW add/mul (independent)."""

    name = "c2-tew_eq-tew"

    def __init__(self, seed, device, scale=1.0):
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
        # union / intersection sizes (for the algorithmic byte count)
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

    # e2e through the C-ABI with host buffers
    def host_inputs(self):
        hx, hy, hy2 = self.x.to_host(), self.y.to_host(), self.y2.to_host()
        return [hx, hy, hy2]

    E2E_CHUNKS = 8
    E2E_PATH = ("ops.* -> C-ABI; pinned host buffers; H2D / kernels / D2H overlapped on three "
                "streams (staging.Pipeline), x/y uploaded in 8 chunks")

    def e2e_step(self, host, device):
        """Pinned host inputs -> the 6 ops -> pinned host outputs, pipelined on
        three streams (staging.Pipeline): x/y go up in chunks and each chunk's
        four tew_eq results go down while the next chunk computes, y2 goes up
        under the tew_eq downloads, then the two merges run and their
        outputs come down. Returns (h2d, d2h) bytes."""
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
                z = ops.tew(dx, dy2, op, out=view(zu, 0, zu.nnz))  # syncs pl.cmp only; raises
                # any deferred tew_eq error (sticky device error words)
                pl.d2h.wait_event(Pipeline.mark(pl.cmp))
                d2h += host["out_tew"][k].download(z, pl.d2h)
        pl.end()
        return h2d, d2h

    def e2e_host(self, device=0):
        from paper_1902_03317_b200.coo import DeviceCOO
        from paper_1902_03317_b200.staging import PinnedCOO, Pipeline
        dev = torch.device(device) if not isinstance(device, int) else torch.device("cuda", device)
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

    # reference CPU path (oracle/_ref = the reference library)
    def cpu_setup(self, ref, sample_nnz=None):
        from oracle.oracle import HostTensor
        hx, hy, hy2 = self.host_inputs()
        T = lambda h: HostTensor(h.dims, h.indices, h.values, h.sort_order, h.coalesced)
        self.h = [ref.coo(T(hx)), ref.coo(T(hy)), ref.coo(T(hy2))]
        self.cpu_units = 4 * self.nnz + 2 * 2 * self.nnz
        return f"full C2 workload (4 x tew_eq on {self.nnz} nnz + tew add/mul on " \
               f"{self.nnz} + {self.nnz} nnz), par:: kernels"

    def cpu_step(self, ref, nthreads):
        import ctypes
        hx, hy, hy2 = self.h
        lib = ref.lib
        out = ctypes.c_void_p()
        for op in range(4):
            ref._check(lib.ref_tew_eq(hx, hy, op, 1, nthreads, ctypes.byref(out)))
            lib.ref_coo_free(out.value)
        for op in (0, 2):
            ref._check(lib.ref_tew(hx, hy2, op, 1, nthreads, ctypes.byref(out)))
            lib.ref_coo_free(out.value)
        return self.cpu_units


# ---------------------------------------------------------------------------
# Reference CPU legs (oracle/_ref = the reference library, par:: kernels with
# every host thread) shared by the workloads' cpu_setup / cpu_step.


def _host_sample(t, k):
    """The first k entries of a device tensor as a HostTensor (a prefix of a
    sorted, coalesced tensor is sorted and coalesced, and its fibers are whole
    except possibly the last)."""
    from oracle.oracle import HostTensor
    k = min(k, t.nnz)
    return HostTensor(list(t.dims), [ix[:k].cpu().numpy().view(np.uint32).copy()
                                     for ix in t.indices],
                      t.values[:k].cpu().numpy().copy(),
                      None if t.sort_order is None else list(t.sort_order), t.coalesced)


class _RefCalls:
    """Handles for the reference's par:: kernels on fixed inputs."""

    def __init__(self, ref):
        import ctypes
        self.ref, self.lib, self.ct = ref, ref.lib, ctypes
        self.keep = []

    def coo(self, ht):
        h = self.ref.coo(ht)
        self.keep.append(("coo", h))
        return h

    def matrix(self, a):
        import numpy as np
        a = np.ascontiguousarray(a, dtype=np.float32)
        self.keep.append(("arr", a))
        f32p = self.ct.POINTER(self.ct.c_float)
        return self.lib.ref_matrix_new(a.ctypes.data_as(f32p), a.shape[0], a.shape[1])

    def vector(self, a):
        import numpy as np
        a = np.ascontiguousarray(a, dtype=np.float32)
        self.keep.append(("arr", a))
        f32p = self.ct.POINTER(self.ct.c_float)
        return self.lib.ref_vector_new(a.ctypes.data_as(f32p), a.shape[0])

    def factors(self, hx, mats):
        """One reference factor vector (the matrices are copied into it, so the
        temporaries go at once -- C5's factors are 1.28 GB each)."""
        import numpy as np
        f32p = self.ct.POINTER(self.ct.c_float)
        hs = (self.ct.c_void_p * len(mats))()
        for d, m in enumerate(mats):
            a = np.ascontiguousarray(m, dtype=np.float32)
            hs[d] = self.lib.ref_matrix_new(a.ctypes.data_as(f32p), a.shape[0], a.shape[1])
        fv = self.lib.ref_factors_new(hx, hs)
        for h in hs:
            self.lib.ref_matrix_free(h)
        return fv

    def run(self, fn, *args, kind="coo"):
        out = self.ct.c_void_p()
        self.ref._check(fn(*args, self.ct.byref(out)))
        (self.lib.ref_matrix_free if kind == "matrix" else self.lib.ref_coo_free)(out.value)

    def mttkrp(self, hx, fv, mode, nt):  # privatize: the strategy the paper reports
        self.run(self.lib.ref_mttkrp_fv, hx, fv, mode, 1, nt, 0, kind="matrix")


class C1(Workload):
    """BASELINE configs[0]: MTTKRP mode 0 (R=16) + TS add/mul by 2.5, 1M nnz."""

    name = "c1-mttkrp-ts"

    def __init__(self, seed, device, scale=1.0):
        from paper_1902_03317_b200 import generate, ops
        from paper_1902_03317_b200.coo import DeviceCOO
        c = generate.CONFIGS["c1"]
        self.dims, self.R = c["dims"], c["R"]
        self.nnz = int(c["nnz"] * scale)
        self.x = generate.coo(self.dims, self.nnz, seed, c["zipf"], 0.0, 1.0, [0, 1, 2], device)
        self.f = [generate.uniform((d, self.R), seed, 100 + k, 0.0, 1.0, device)
                  for k, d in enumerate(self.dims)]
        self.out = torch.empty((self.dims[0], self.R), dtype=torch.float32, device=f"cuda:{device}")
        self.z = DeviceCOO.empty(self.dims, self.nnz, device)
        n, N, R = self.nnz, 3, self.R
        self.ops = [
            Op("mttkrp_m0", lambda: allreduce(ops.mttkrp(self.x, self.f, 0, ops.MTTKRP_SEGMENTED,
                                                         out=self.out, sync=False)),
               n, lambda: tensor_bytes(n, N) + 4 * R * sum(self.dims)),
            Op("ts_add", lambda: ops.ts(self.x, 2.5, ops.SCALAR_ADD, out=self.z, sync=False), n,
               lambda: 2 * tensor_bytes(n, N)),
            Op("ts_mul", lambda: ops.ts(self.x, 2.5, ops.SCALAR_MUL, out=self.z, sync=False), n,
               lambda: 2 * tensor_bytes(n, N)),
        ]

    def config(self):
        return {"workload": self.name, "baseline_config": "configs[0] (C1)", "dims": self.dims,
                "nnz": self.nnz, "R": self.R, "mttkrp_input": "sorted (0,1,2) (mode-0 leading)"}

    # e2e through the C-ABI with host buffers
    E2E_CHUNKS = 4
    E2E_PATH = ("ops.* -> C-ABI; pinned host buffers; x uploaded in 4 chunks (TS of each chunk "
                "and its download overlap the next chunk's upload), factors up, MTTKRP on the "
                "whole tensor, its I x R result and both TS outputs down")

    def e2e_host(self, device=0):
        from paper_1902_03317_b200.coo import DeviceCOO
        from paper_1902_03317_b200.staging import PinnedCOO, Pipeline
        dev = torch.device(device) if not isinstance(device, int) else torch.device("cuda", device)
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

    def e2e_step(self, host, device):
        """Pinned host inputs -> MTTKRP + TS add/mul -> pinned host outputs.
        Returns (h2d, d2h) bytes."""
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

    def cpu_setup(self, ref, sample_nnz=None):
        c = self.cr = _RefCalls(ref)
        self.hx = c.coo(_host_sample(self.x, self.nnz))
        self.fv = c.factors(self.hx, [f.cpu().numpy() for f in self.f])
        self.cpu_units = 3 * self.nnz
        return f"full C1 workload: mttkrp mode 0 (privatize) + ts add/mul on {self.nnz} nnz, par::"

    def cpu_step(self, ref, nthreads):
        c = self.cr
        c.mttkrp(self.hx, self.fv, 0, nthreads)
        for op in (0, 1):
            c.run(c.lib.ref_ts, self.hx, 2.5, op, 1, nthreads)
        return self.cpu_units


class C3(Workload):
    """configs[2]: TTV and TTM (R=16) along every mode, 50M nnz, mode-0 Zipf(1.1)."""

    name = "c3-ttv-ttm"

    def __init__(self, seed, device, scale=1.0):
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
        del base
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

    def cpu_setup(self, ref, sample_nnz=1_000_000):
        c = self.cr = _RefCalls(ref)
        self.cpu_in = []
        k = min(sample_nnz, self.nnz)
        for m in range(3):
            hx = c.coo(_host_sample(self.xs[m], k))
            fib = ref.lib.ref_fiber_new(hx, m)  # preprocessing, untimed (P/src/bench.cpp:363-368)
            c.keep.append(("fib", fib))
            self.cpu_in.append((hx, fib, c.vector(self.v[m].cpu().numpy()),
                                c.matrix(self.u[m].cpu().numpy())))
        self.cpu_units = 6 * k
        return f"ttv + ttm (R={self.R}) along every mode on the first {k} entries of each " \
               "mode-last sorted copy, par::"

    def cpu_step(self, ref, nthreads):
        c = self.cr
        for m, (hx, fib, hv, hu) in enumerate(self.cpu_in):
            c.run(c.lib.ref_ttv_fib, hx, hv, m, fib, 1, nthreads)
            c.run(c.lib.ref_ttm_fib, hx, hu, m, fib, 1, nthreads)
        return self.cpu_units


class C4(Workload):
    """configs[3]: MTTKRP every mode, R=32, 4th order, 100M nnz, Zipf(1.2) modes."""

    name = "c4-mttkrp"

    def __init__(self, seed, device, scale=1.0):
        from paper_1902_03317_b200 import generate, ops
        c = generate.CONFIGS["c4"]
        self.dims, self.R = c["dims"], c["R"]
        self.nnz = int(c["nnz"] * scale)
        base = generate.coo(self.dims, self.nnz, seed, c["zipf"], 0.0, 1.0, None, device)
        self.f = [generate.uniform((d, self.R), seed, 100 + k, 0.0, 1.0, device)
                  for k, d in enumerate(self.dims)]
        self.xs = []
        for mode in range(4):
            xs = base.clone()
            ops.sort_lexicographic(xs, [mode] + [d for d in range(4) if d != mode])
            self.xs.append(xs)
        del base
        self.out = [torch.empty((d, self.R), dtype=torch.float32, device=f"cuda:{device}")
                    for d in self.dims]
        n, N, R = self.nnz, 4, self.R
        self.ops = [Op(f"mttkrp_m{m}",
                       lambda m=m: allreduce(ops.mttkrp(self.xs[m], self.f, m,
                                                        ops.MTTKRP_SEGMENTED, out=self.out[m],
                                                        sync=False)),
                       n, lambda: tensor_bytes(n, N) + 4 * R * sum(self.dims))
                    for m in range(4)]

    def config(self):
        return {"workload": self.name, "baseline_config": "configs[3] (C4)", "dims": self.dims,
                "nnz": self.nnz, "R": self.R, "dist": "every mode Zipf(1.2), shuffled ids",
                "mttkrp_input": "one mode-leading sorted copy per mode (preprocessing)"}

    def cpu_setup(self, ref, sample_nnz=1_000_000):
        c = self.cr = _RefCalls(ref)
        k = min(sample_nnz, self.nnz)
        self.cpu_in = []
        for m in range(4):
            self.cpu_in.append((c.coo(_host_sample(self.xs[m], k)), None))
        fv = c.factors(self.cpu_in[0][0], [f.cpu().numpy() for f in self.f])
        self.cpu_in = [(hx, fv) for hx, _ in self.cpu_in]
        self.cpu_units = 4 * k
        return f"mttkrp (R={self.R}, privatize) along every mode on the first {k} entries of " \
               "each mode-leading sorted copy (full-size factors), par::"

    def cpu_step(self, ref, nthreads):
        for m, (hx, fv) in enumerate(self.cpu_in):
            self.cr.mttkrp(hx, fv, m, nthreads)
        return self.cpu_units


class C5(Workload):
    """BASELINE configs[4] (C5): MTTKRP modes 0-2 (R=32) + TEW-eq mul on a
    1B-nnz order-3 tensor, every mode Zipf(1.1). One GPU holds the tensor
    (16 GB), one mode-leading copy per mode and the TEW-eq operand/output;
    under torchrun every rank runs its own instance and MTTKRP adds the NCCL
    all-reduce of the I_n x R partials."""

    name = "c5-mttkrp-tew_eq"
    # BASELINE configs[4] shards ONE 1B-nnz tensor over the GPUs: every rank
    # builds the same tensor (same seed) and keeps its shards
    STRONG = True

    def __init__(self, seed, device, scale=1.0):
        from paper_1902_03317_b200 import generate, ops
        from paper_1902_03317_b200.coo import DeviceCOO
        c = generate.CONFIGS["c5"]
        self.dims, self.R = c["dims"], c["R"]
        self.nnz = int(c["nnz"] * scale)
        dev = f"cuda:{device}"
        base = generate.coo(self.dims, self.nnz, seed, c["zipf"], 0.0, 1.0, None, device)
        self.f = [generate.uniform((d, self.R), seed, 100 + k, 0.0, 1.0, device)
                  for k, d in enumerate(self.dims)]
        self.xs = []
        for mode in range(3):
            xs = base if mode == 2 else base.clone()
            ops.sort_lexicographic(xs, [mode] + [d for d in range(3) if d != mode])
            self.xs.append(xs)
        del base
        torch.cuda.empty_cache()
        x = self.xs[0]
        # TEW-eq operand: same pattern in its own buffers (as SURVEY 8(d) counts
        # the bytes), values U[0.5,1.5)
        self.y = DeviceCOO(list(self.dims), [i.clone() for i in x.indices],
                           generate.uniform(self.nnz, seed, 77, 0.5, 1.5, device),
                           list(x.sort_order), x.coalesced)
        self.out = [torch.empty((d, self.R), dtype=torch.float32, device=dev) for d in self.dims]
        n, N, R = self.nnz, 3, self.R
        world = DIST.get_world_size() if DIST is not None else 1
        if world == 1:
            self.z = DeviceCOO.empty(self.dims, self.nnz, device)
            self.ops = [Op(f"mttkrp_m{m}",
                           lambda m=m: ops.mttkrp(self.xs[m], self.f, m, ops.MTTKRP_SEGMENTED,
                                                  out=self.out[m], sync=False),
                           n, lambda: tensor_bytes(n, N) + 4 * R * sum(self.dims))
                        for m in range(3)]
            self.ops.append(Op("tew_eq_mul",
                               lambda: ops.tew_eq(x, self.y, ops.MUL, out=self.z, sync=False),
                               n, lambda: 3 * tensor_bytes(n, N)))
            return
        # N > 1: MTTKRP on row-aligned nnz shards of each
        # mode-leading copy, the owned row blocks all-gathered over NCCL (half
        # the all-reduce's volume); TEW-eq on contiguous nnz shards, no exchange.
        # Units per rank = nnz / world, so `value` is the whole tensor's nnz/s.
        from paper_1902_03317_b200 import parallel
        me = DIST.get_rank()
        self.blocks = []
        # shards are cloned into their own (16-byte aligned) buffers, so the
        # kernels keep their vector paths, and the full copies are released
        lo, hi = parallel.shard_range(self.nnz, world, me)
        xe = parallel.slice_coo(x, lo, hi).clone()
        self.y = parallel.slice_coo(self.y, lo, hi).clone()
        del x
        for m in range(3):
            rr = parallel.row_aligned_ranges(self.xs[m].indices[m], world)
            self.blocks.append(parallel.row_blocks(self.xs[m].indices[m], rr, self.dims[m]))
            self.xs[m] = parallel.slice_coo(self.xs[m], *rr[me]).clone()
            torch.cuda.empty_cache()
        self.z = DeviceCOO.empty(self.dims, hi - lo, device)
        share = n / world

        def mt(m):
            part = lambda s, f, mm: ops.mttkrp(s, f, mm, ops.MTTKRP_SEGMENTED, out=self.out[mm],
                                               sync=False)
            return parallel.mttkrp_row_allgather(self.xs[m], self.f, m, self.dims[m], R,
                                                 self.blocks[m], part)
        self.ops = [Op(f"mttkrp_m{m}", lambda m=m: mt(m), share,
                       lambda: (tensor_bytes(n, N) + 4 * R * sum(self.dims)) / world)
                    for m in range(3)]
        self.ops.append(Op("tew_eq_mul",
                           lambda: ops.tew_eq(xe, self.y, ops.MUL, out=self.z, sync=False),
                           share, lambda: 3 * tensor_bytes(n, N) / world))

    def config(self):
        return {"workload": self.name, "baseline_config": "configs[4] (C5)", "dims": self.dims,
                "nnz": self.nnz, "R": self.R, "dist": "every mode Zipf(1.1), shuffled ids",
                "mttkrp_input": "one mode-leading sorted copy per mode (preprocessing)",
                "tew_eq": "mul against the same pattern, y U[0.5,1.5)"}

    def cpu_setup(self, ref, sample_nnz=1_000_000):
        c = self.cr = _RefCalls(ref)
        k = min(sample_nnz, self.nnz)
        self.cpu_in = []
        for m in range(3):
            self.cpu_in.append((c.coo(_host_sample(self.xs[m], k)), None))
        fv = c.factors(self.cpu_in[0][0], [f.cpu().numpy() for f in self.f])
        self.cpu_in = [(hx, fv) for hx, _ in self.cpu_in]
        from oracle.oracle import HostTensor
        hx0 = _host_sample(self.xs[0], k)
        hy = HostTensor(hx0.dims, hx0.indices, self.y.values[:k].cpu().numpy(), hx0.sort_order,
                        hx0.coalesced)
        self.eq = (c.coo(hx0), c.coo(hy))
        self.cpu_units = 4 * k
        return f"mttkrp (R={self.R}, privatize) modes 0-2 on the first {k} entries of each " \
               f"mode-leading copy (full 10M-row factors) + tew_eq mul on {k} entries, par::"

    def cpu_step(self, ref, nthreads):
        c = self.cr
        for m, (hx, fv) in enumerate(self.cpu_in):
            c.mttkrp(hx, fv, m, nthreads)
        c.run(c.lib.ref_tew_eq, self.eq[0], self.eq[1], 2, 1, nthreads)
        return self.cpu_units


class Pre(Workload):
    """SURVEY 8(f) "next" row 1: GPU preprocessing at parity and speed --
    sort_lexicographic (P/src/tensor.cpp:54-64; 4.56 s for 10M on the
    reference here) and build_fiber_index (:92-120), on C2's 10M tensor in
    draw (unsorted) order and C3's order for the fiber index."""

    name = "pre-sort-fiber"

    def __init__(self, seed, device, scale=1.0):
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

    def cpu_setup(self, ref, sample_nnz=2_000_000):
        from oracle.oracle import HostTensor
        h = self.src.to_host()
        k = min(sample_nnz, self.nnz)
        self.cpu_t = HostTensor(h.dims, [a[:k] for a in h.indices], h.values[:k], None, True)
        self.cpu_units = k
        return f"sort_lexicographic (0,1,2) of the first {k} entries (reference, serial)"

    def cpu_step(self, ref, nthreads):
        ref.sort_lexicographic(self.cpu_t, [0, 1, 2])
        return self.cpu_units


WORKLOADS = {"c1": C1, "c2": C2, "c3": C3, "c4": C4, "c5": C5, "pre": Pre}


# ---------------------------------------------------------------------------


def run_cpu_reference(wl, steps, warmup, sample_note=True):
    from oracle.oracle import Ref
    ref = Ref()
    nthreads = os.cpu_count() or 1
    os.environ.setdefault("OMP_PROC_BIND", "close")
    sample = wl.cpu_setup(ref)
    for _ in range(warmup):
        wl.cpu_step(ref, nthreads)
    t = []
    units = 0
    for _ in range(steps):
        t0 = time.perf_counter()
        units = wl.cpu_step(ref, nthreads)
        t.append(time.perf_counter() - t0)
    return {"value": units / statistics.mean(t), "unit": "nnz/s", "cores": nthreads,
            "kind": "reference", "sample": sample, "step_s_mean": statistics.mean(t),
            "step_s_median": statistics.median(t),
            "protocol": f"{warmup} untimed warm-up + {steps} timed (mean), as P/src/bench.cpp:199-209"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=20190210)
    ap.add_argument("--scale", type=float, default=1.0, help="nnz scale (testing only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--report", default=None,
                    help="also write per-op rows in the reference's BenchReport schema "
                         "(.json or .csv, P/include/spten/report.hpp)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference" and rank != 0:
        return  # the reference arm runs on rank 0 only (CPU path)
    torch.cuda.set_device(local)
    dist = None
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        global DIST
        DIST = dist

    from paper_1902_03317_b200 import _lib
    W = WORKLOADS[args.workload]
    # weak scaling: an independent instance per rank; strong (C5): one tensor
    wl = W(args.seed if getattr(W, "STRONG", False) else args.seed + 1009 * rank, local,
           args.scale)
    hbm, peak_src = peaks()

    if args.impl == "reference":
        cb = run_cpu_reference(wl, args.steps, args.warmup)
        line = {"metric": METRIC, "value": cb["value"], "unit": "nnz/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": cb["step_s_mean"] * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded Philox, BASELINE config shapes)", "impl": "reference",
                "config": wl.config(),
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": cb["value"], "unit": "nnz/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

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
        ops_out[op.name] = {"ms": round(mean_ms, 5), "ms_median": round(statistics.median(op.times), 5),
                            "alg_bytes": int(by), "GB_s": round(gbs, 1),
                            "frac": round(gbs / hbm, 4), "nnz_s": op.units / (mean_ms / 1e3),
                            "launches_per_call": op.launches / args.steps}
    # MTTKRP's second floor: every gathered factor row costs at least one L1
    # wavefront (<= 128 B) per SM-cycle whether it hits L1, L2 or smem
    # ("Gather floor")
    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    sm_hz = float(_measured_peaks().get("sm_max_mhz", 1965.0)) * 1e6
    for op in wl.ops:
        if op.name.startswith("mttkrp"):
            N, R = len(wl.dims), wl.R
            wf = wl.nnz * (N - 1) * -(-4 * R // 128)
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
                                    "model": "nnz*(N-1)*ceil(4R/128) L1 wavefronts / (SMs * SM clock)"}
    tr = os.path.join(ROOT, "profiles", f"traffic_{args.workload}.json")
    if os.path.exists(tr):
        roofline["traffic"] = json.load(open(tr)).get(dom.name)

    e2e = None
    if not args.no_e2e and hasattr(wl, "e2e_step"):
        # every rank runs its own host-buffer pipeline (its own PCIe link);
        # whole-job throughput over the slowest rank, like `value`
        host = wl.e2e_host(local)
        wl.e2e_step(host, f"cuda:{local}")
        torch.cuda.synchronize()
        times = []
        for _ in range(max(2, min(args.steps, 5))):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            a.record(stream)
            h2d, d2h = wl.e2e_step(host, f"cuda:{local}")
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
               "ms_per_step": ms,
               "path": getattr(wl, "E2E_PATH", "ops.* -> C-ABI with pinned host buffers")}
        del host

    cpu = None
    if not args.no_cpu and rank == 0 and world == 1 and hasattr(wl, "cpu_setup"):
        try:
            cb = run_cpu_reference(wl, steps=3, warmup=1)
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # reported, never silently replaced
            cpu = {"value": None, "unit": "nnz/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "strong" if getattr(wl, "STRONG", False) else "weak",
                "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded Philox, BASELINE config shapes; public datasets "
                        "unavailable offline)",
                "config": {**wl.config(), "l2": "inputs > L2 and L2 flushed before every op",
                           "timing": "CUDA events per op on the launch stream, max over ranks"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(sum(op.launches for op in wl.ops)),
                "clocks": clk, "ops": ops_out}
        print(json.dumps(line))
        if args.report:
            from paper_1902_03317_b200 import report
            rows = report_rows(wl, wl.ops)
            with open(args.report, "w") as fh:
                fh.write(report.emit_csv(rows) if args.report.endswith(".csv")
                         else report.emit_json(rows))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
