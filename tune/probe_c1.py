import torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops, _lib
x = generate.coo([1000]*3, 1_000_000, 1, [0,0,0], 0, 1, [0, 1, 2])
f = [generate.uniform((1000, 16), 1, k, 0, 1) for k in range(3)]
out = torch.empty((1000, 16), device='cuda')
for _ in range(4): ops.mttkrp(x, f, 0, ops.MTTKRP_SEGMENTED, out=out, sync=False)
torch.cuda.synchronize(); print("ok")
