import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_1902_03317_b200 import generate, ops
dim = int(sys.argv[1]); n = int(sys.argv[2])
x = generate.coo([dim]*3, n, 1, [0, 0, 0], 0.5, 1.5, [0, 1, 2])
y = generate.coo([dim]*3, n, 2, [0, 0, 0], 0.5, 1.5, [0, 1, 2])
z = ops.tew(x, y, ops.MUL); torch.cuda.synchronize()
print(dim, n, z.nnz, flush=True)
