"""Small TEW add/mul runs (debugging aid for the merge kernels)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops
sizes = [int(a) for a in sys.argv[1:]] or [10, 3000, 100000]
for n in sizes:
    x = generate.coo([100, 100, 100], n, 1, [0, 0, 0], 0.5, 1.5, [0, 1, 2])
    y = generate.coo([100, 100, 100], n, 2, [0, 0, 0], 0.5, 1.5, [0, 1, 2])
    for op in (ops.ADD, ops.MUL):
        z = ops.tew(x, y, op)
        torch.cuda.synchronize()
        print(n, op, z.nnz, flush=True)
