import torch, sys
sys.path.insert(0, '.')
from paper_1902_03317_b200 import generate, ops
from paper_1902_03317_b200.coo import DeviceCOO
dims, n = [10000]*3, 10_000_000
x = generate.coo(dims, n, 1, [0,0,0], 0.5, 1.5, [0,1,2])
y = generate.coo(dims, n, 2, [0,0,0], 0.5, 1.5, [0,1,2])
z = DeviceCOO.empty(dims, 2*n)
cnt = torch.zeros(1, dtype=torch.int64, device='cuda')
for i in range(3): ops.tew_device(x, y, ops.ADD, z, cnt)
torch.cuda.synchronize(); print("ok", int(cnt))
