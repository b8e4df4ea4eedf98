import torch, sys
sys.path.insert(0, '.')
from paper_1902_03317_b200 import generate, ops, _lib
dims, nnz, R = [10000]*3, 10_000_000, 16
x = generate.coo(dims, nnz, 1, [0,0,0], 0, 1, [0,1,2])
f = [generate.uniform((d, R), 1, k, 0, 1) for k, d in enumerate(dims)]
out = torch.empty((dims[0], R), device='cuda')
for i in range(3): ops.mttkrp(x, f, 0, ops.MTTKRP_SEGMENTED, out=out)
torch.cuda.synchronize(); print("ok")
