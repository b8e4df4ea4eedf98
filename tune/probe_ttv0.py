import torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops, _lib
from paper_1902_03317_b200.coo import DeviceCOO
dims, nnz = [50000, 20000, 100000], 20_000_000
mode = int(os.environ.get("MODE", 0))
base = generate.coo(dims, nnz, 1, [1.1, 0, 0], 0, 1, None)
xs = base.clone(); ops.sort_lexicographic(xs, ops.mode_last_order(3, mode))
fib = ops.build_fiber_index(xs, mode)
v = generate.uniform(dims[mode], 1, 6, -1, 1)
zv = DeviceCOO.empty([1, 1], fib.nfibs)
for _ in range(3): ops.ttv(xs, v, mode, fib, out=zv)
torch.cuda.synchronize(); print("ok", fib.nfibs)
