import torch, sys, os, ctypes, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops, _lib
from paper_1902_03317_b200.coo import DeviceCOO
lib = _lib.load()
dims, n = [10000]*3, 10_000_000
x = generate.coo(dims, n, 1, [0,0,0], 0.5, 1.5, [0,1,2])
y = generate.coo(dims, n, 2, [0,0,0], 0.5, 1.5, [0,1,2])
z = DeviceCOO.empty(dims, 2*n)
cnt = torch.zeros(1, dtype=torch.int64, device='cuda')
for op in (ops.ADD, ops.MUL):
    for _ in range(3): ops.tew_device(x, y, op, z, cnt)
    torch.cuda.synchronize()
    nt = (2 * n + 2047) // 2048
    buf = np.zeros(65536 * 8, np.uint64)
    lib.spt_debug_phases(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(65536 * 8))
    ph = buf.reshape(-1, 8)[:nt, :5].astype(np.int64)
    t0 = ph[:, 0].min()
    d = np.diff(ph, axis=1)
    print(f"op {op}: span {(ph[:,4].max()-t0)/1e3:.1f} us  tiles {nt}")
    for k, name in enumerate(["stage", "merge+scan", "lookback", "emit"]):
        print(f"   {name:10s} mean {d[:,k].mean()/1e3:7.2f} us  p50 {np.median(d[:,k])/1e3:7.2f}  p99 {np.percentile(d[:,k],99)/1e3:7.2f}")
    life = (ph[:, 4] - ph[:, 0])
    print(f"   tile lifetime mean {life.mean()/1e3:.2f} us; start spread: first 10 starts (us) {((ph[:10,0]-t0)/1e3).round(2)}")
    conc = []
    for tq in np.linspace(ph[:,0].min(), ph[:,4].max(), 20):
        conc.append(int(((ph[:,0] <= tq) & (ph[:,4] >= tq)).sum()))
    print("   concurrency over time:", conc)
rs = buf.reshape(-1, 8)[:nt, 5].astype(np.int64)
print("lookback rounds mean", (rs & 0xffffffff).mean(), "max", (rs & 0xffffffff).max(), "slides mean", (rs >> 32).mean())
