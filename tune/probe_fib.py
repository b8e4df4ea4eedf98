import torch, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops, _lib
x = generate.coo([10000]*3, 10_000_000, 1, [0,0,0], 0.5, 1.5, None)
ops.sort_lexicographic(x, [0,1,2])
for i in range(5):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record()
    f = ops.build_fiber_index(x, 2)
    b.record(); t1 = time.perf_counter(); torch.cuda.synchronize()
    print(f"event {a.elapsed_time(b)*1e3:.0f} us host {1e6*(t1-t0):.0f} us nfibs {f.nfibs}")
