"""Run the plan MTTKRP of one config/mode a few times (ncu capture target).

    python tune/run_plan.py c5 [scale] [mode] [reps] [hot:1|0]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1902_03317_b200 import _lib, generate, ops  # noqa: E402

name = sys.argv[1]
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
hot = (sys.argv[5] != "0") if len(sys.argv) > 5 else True
c = generate.CONFIGS[name]
R = c["R"]
x = generate.coo(c["dims"], int(c["nnz"] * scale), 20190210, c["zipf"], 0.0, 1.0, None, 0)
f = [generate.uniform((d, R), 20190210, 100 + k, 0.0, 1.0, 0) for k, d in enumerate(c["dims"])]
plan = ops.mttkrp_plan(x, mode, R, hot=hot)
del x
out = torch.empty((c["dims"][mode], R), device="cuda")
ctx = _lib.Context.get(0)
st = torch.cuda.current_stream().cuda_stream
ts = []
for _ in range(reps):
    _lib.load().spt_l2_flush(ctx.handle, st)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ops.mttkrp(plan, f, mode, out=out, sync=False)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(name, scale, mode, "nhot", plan.nhot, "ms", [round(t, 4) for t in ts])
