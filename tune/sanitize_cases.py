"""Small instances of every kernel with a cross-block protocol (decoupled
look-back, tickets, the plan kernel's last-CTA fold, the persistent merge),
for compute-sanitizer (racecheck / synccheck / memcheck):

    compute-sanitizer --tool racecheck python tune/sanitize_cases.py
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1902_03317_b200 import generate, ops  # noqa: E402

torch.cuda.set_device(0)
checks = []


def case(name, fn):
    fn()
    torch.cuda.synchronize()
    checks.append(name)


x = generate.coo([3000, 200, 100], 60_000, 1, [1.2, 0, 0], 0.0, 1.0, [0, 1, 2])
fs = [generate.uniform((d, 32), 1, 10 + k, 0.0, 1.0) for k, d in enumerate(x.dims)]
case("mttkrp segmented CTA tiles (look-back)",
     lambda: ops.mttkrp(x, fs, 0, ops.MTTKRP_SEGMENTED_CTA))
case("mttkrp warp tiles (warp look-back)", lambda: ops.mttkrp(x, fs, 0, ops.MTTKRP_SEGMENTED_WARP))
case("mttkrp atomic", lambda: ops.mttkrp(x, fs, 1, ops.MTTKRP_ATOMIC))
xb = generate.coo([20000, 500, 400], 1_700_000, 2, [1.1, 0, 0], 0.0, 1.0, [0, 1, 2])
fb = [generate.uniform((d, 16), 2, 10 + k, 0.0, 1.0) for k, d in enumerate(xb.dims)]
case("mttkrp persistent async-fold tiles", lambda: ops.mttkrp(xb, fb, 0, ops.MTTKRP_SEGMENTED_CTA))
plan = ops.mttkrp_plan(xb, 1, 16)
case("mttkrp plan (blocked staging, CTA fold, last-CTA grid fold)",
     lambda: ops.mttkrp(plan, fb, 1))
xu = generate.coo([300, 200, 100], 30_000, 3, [0, 0, 0], 0.0, 1.0)  # draw order
fu = [generate.uniform((d, 32), 3, 20 + k, 0.0, 1.0) for k, d in enumerate(xu.dims)]
case("mttkrp AUTO on unsorted input (temporary plan)", lambda: ops.mttkrp(xu, fu, 2))
t = x.clone()
ops.sort_lexicographic(t, ops.mode_last_order(3, 1))
fib = ops.build_fiber_index(t, 1)
v = generate.uniform(t.dims[1], 4, 5, -1.0, 1.0)
u = generate.uniform((t.dims[1], 16), 4, 6, -1.0, 1.0)
case("ttv warp tiles (look-back)", lambda: ops.ttv(t, v, 1, fib))
case("ttm (MTTKRP engine, fiber rows)", lambda: ops.ttm(t, u, 1, fib))
y = generate.coo([3000, 200, 100], 50_000, 7, [0, 0, 0], 0.0, 1.0, [0, 1, 2])
case("tew merge add (persistent, look-back counts)", lambda: ops.tew(x, y, ops.ADD))
case("tew merge mul", lambda: ops.tew(x, y, ops.MUL))
yy = x.clone()
case("tew_eq div (sticky first-failure words)", lambda: ops.tew_eq(x, yy, ops.DIV))
w = generate.coo([3000, 200, 100], 80_000, 8, [0, 0, 0], 0.0, 1.0)
case("sort + coalesce + fiber index", lambda: (ops.sort_lexicographic(w, [2, 0, 1]),
                                               ops.coalesce(w), ops.build_fiber_index(w, 1)))
case("ts", lambda: ops.ts(x, 2.5, ops.SCALAR_MUL))
print("sanitize cases run:", len(checks))
for c in checks:
    print("  ", c)
