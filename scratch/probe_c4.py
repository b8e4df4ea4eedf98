import torch, sys
sys.path.insert(0, '.')
from paper_1902_03317_b200 import generate, ops
dims, nnz, R = [2_000_000, 500_000, 100_000, 1000], 20_000_000, 32
x = generate.coo(dims, nnz, 1, [1.2]*4, 0, 1, [0,1,2,3])
f = [generate.uniform((d, R), 1, k, 0, 1) for k, d in enumerate(dims)]
out = torch.empty((dims[0], R), device='cuda')
for i in range(3): ops.mttkrp(x, f, 0, ops.MTTKRP_SEGMENTED, out=out)
torch.cuda.synchronize(); print("ok")
