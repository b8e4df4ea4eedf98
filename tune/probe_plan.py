"""Plan MTTKRP vs the COO segmented kernel at a BASELINE config: plan build
time, per-mode kernel time (CUDA events, L2 flushed), hot rows, and the max
relative difference between the two outputs.

    python tune/probe_plan.py c5|c4|c1 [scale] [reps]
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1902_03317_b200 import _lib, generate, ops  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
c = generate.CONFIGS[name]
N, R = len(c["dims"]), c["R"]
nnz = int(c["nnz"] * scale)
base = generate.coo(c["dims"], nnz, 20190210, c["zipf"], 0.0, 1.0, None, 0)
f = [generate.uniform((d, R), 20190210, 100 + k, 0.0, 1.0, 0) for k, d in enumerate(c["dims"])]
ctx = _lib.Context.get(0)
lib = _lib.load()
st = torch.cuda.current_stream()


def timeit(fn):
    ts = []
    for i in range(reps + 1):
        lib.spt_l2_flush(ctx.handle, st.cuda_stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if i:
            ts.append(a.elapsed_time(b))
    return sum(ts) / len(ts)


res = {"config": name, "nnz": nnz}
modes = range(N) if len(sys.argv) <= 4 else [int(m) for m in sys.argv[4].split(",")]
for m in modes:
    out_p = torch.empty((c["dims"][m], R), device="cuda")
    t0 = time.time()
    plan = ops.mttkrp_plan(base, m, R)
    torch.cuda.synchronize()
    build = time.time() - t0
    tp = timeit(lambda: ops.mttkrp(plan, f, m, out=out_p, sync=False))
    rec = {"plan_s": round(build, 3), "plan_ms": round(tp, 4), "nhot": plan.nhot,
           "hot_per_level": plan.hot_per_level, "levels": plan.level_modes}
    del plan
    torch.cuda.empty_cache()
    xs = base.clone()
    ops.sort_lexicographic(xs, [m] + [d for d in range(N) if d != m])
    out_s = torch.empty_like(out_p)
    ts = timeit(lambda: ops.mttkrp(xs, f, m, ops.MTTKRP_SEGMENTED, out=out_s, sync=False))
    vplan = ops.mttkrp_plan(xs, m, R, hot=False)
    out_v = torch.empty_like(out_p)
    tv = timeit(lambda: ops.mttkrp(vplan, f, m, out=out_v, sync=False))
    ops.check_deferred(0)
    den = torch.maximum(out_s.abs(), torch.full_like(out_s, 1e-30))
    rec.update({"seg_ms": round(ts, 4), "nohot_ms": round(tv, 4),
                "maxrel_plan_vs_seg": float(((out_p - out_s).abs() / den).max()),
                "maxrel_nohot_vs_seg": float(((out_v - out_s).abs() / den).max())})
    del vplan, xs
    torch.cuda.empty_cache()
    res[f"m{m}"] = rec
    print(json.dumps({f"m{m}": rec}), flush=True)
print(json.dumps(res))
