"""Where the C5 pinned-pipeline e2e step spends its time: the copies alone
(same buffers, same streams, no kernels) against the full step."""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1902_03317_b200.staging import Pipeline, chunk_bounds, view
wl = bench.C5(20190210, 0)
host = wl.e2e_host(0)
pl = host["pipe"]
def copies_only(up=True, down=True):
    pl.begin()
    if up:
        with torch.cuda.stream(pl.h2d):
            for a, b in zip(host["df"], host["pf"]):
                a.copy_(b, non_blocking=True)
        for lo, hi in zip(*(lambda b: (b[:-1], b[1:]))(chunk_bounds(wl.nnz, 8))):
            host["px"].upload(host["dx"], lo, hi, pl.h2d)
        for lo, hi in zip(*(lambda b: (b[:-1], b[1:]))(chunk_bounds(wl.nnz, 16))):
            host["py"].upload(host["dy"], lo, hi, pl.h2d)
    if down:
        host["out_eq"].download(host["dz"], pl.d2h)
        with torch.cuda.stream(pl.d2h):
            for m in range(3):
                host["out_m"][m].copy_(host["dout"][m], non_blocking=True)
    pl.end()
def t(fn, n=3):
    r = []
    for _ in range(n):
        torch.cuda.synchronize(); a = time.perf_counter(); fn(); torch.cuda.synchronize()
        r.append((time.perf_counter() - a) * 1e3)
    return [round(x) for x in r]
print("h2d only (35.84 GB)", t(lambda: copies_only(True, False)))
print("d2h only (19.84 GB)", t(lambda: copies_only(False, True)))
print("both directions    ", t(lambda: copies_only(True, True)))
print("full e2e step      ", t(lambda: wl.e2e_step(host)))
from paper_1902_03317_b200 import ops
def tm(fn):
    torch.cuda.synchronize(); a = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    return r, round((time.perf_counter() - a) * 1e3, 1)
for rep in range(2):
    for m in range(3):
        plan, tb = tm(lambda: ops.mttkrp_plan(host["dx"], m, wl.R))
        _, te = tm(lambda: ops.mttkrp(plan, host["df"], m, out=host["dout"][m], sync=False))
        _, tc = tm(lambda: plan.close())
        print(f"mode {m}: build {tb} ms exec {te} ms close {tc} ms")
