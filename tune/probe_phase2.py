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
    lib.spt_debug_phases(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(65536 * 8 * 8))
    ph = buf.reshape(-1, 8)[:nt].astype(np.int64)
    t0 = ph[:, 0].min()
    d = np.diff(ph[:, :6], axis=1)
    print(f"op {op}: span {(ph[:,5].max()-t0)/1e3:.1f} us  tiles {nt}  ctas {len(np.unique(ph[:,7]))}")
    for k, name in enumerate(["wait", "pack", "merge+scan", "A->lookback", "emit"]):
        print(f"   {name:10s} mean {d[:,k].mean()/1e3:7.2f} us  p50 {np.median(d[:,k])/1e3:7.2f}  p99 {np.percentile(d[:,k],99)/1e3:7.2f}")
    # first-tile start distribution
    print("   first wait start spread (us):", np.percentile((ph[:,0]-t0)/1e3, [0, 1, 5, 50]).round(2))
    print("   tile end vs tile id monotonic? corr", np.corrcoef(np.arange(nt), ph[:,5])[0,1].round(4))
    st = ph[:, 6]
    polls, dist = st >> 32, st & 0xffffffff
    print("   polls mean", polls[1:].mean().round(2), "p99", np.percentile(polls[1:], 99), " P distance mean", dist[1:].mean().round(1), "p50", np.median(dist[1:]), "p99", np.percentile(dist[1:], 99))
    # when did predecessor publish A vs when this tile's lookback ended
    a_t = ph[:, 3]; lb_start_lower = ph[:, 3]
    lag = (a_t[1:] - a_t[:-1]) / 1e3
    print("   A(t) - A(t-1) us: p1 %.2f p50 %.2f p99 %.2f" % tuple(np.percentile(lag, [1, 50, 99])))
    print("   A(t) - lbdone(t-1): p50 %.2f" % np.median((a_t[1:] - ph[:-1, 4]) / 1e3))
