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
    t0 = ph[:, 1].min()
    print(f"op {op}: span {(ph[:,5].max()-t0)/1e3:.1f} us")
    def st(name, v):
        v = v / 1e3
        print(f"   {name:18s} mean {v.mean():6.2f} p50 {np.median(v):6.2f} p99 {np.percentile(v,99):6.2f}")
    st("pack", ph[:,2]-ph[:,1]); st("merge+scan", ph[:,3]-ph[:,2])
    st("A -> emitter start", ph[:,0]-ph[:,3]); st("lookback", ph[1:,4]-ph[1:,0]); st("emit", ph[:,5]-ph[:,4])
    # consumer gap: from A(t) of previous tile of same CTA to data-ready of this tile
    cta = ph[:,7]; order = np.lexsort((ph[:,1], cta)); o = order
    same = cta[o][1:] == cta[o][:-1]
    gap = (ph[o][1:,1] - ph[o][:-1,3])[same]
    st("A(prev)->ready(next)", gap)
    egap = (ph[o][1:,0] - ph[o][:-1,5])[same]
    st("emit(prev)->estart", egap)
    stt = ph[:, 6]; polls = stt >> 32
    print("   polls mean", polls[1:].mean().round(2))
    lb = (ph[1:,4]-ph[1:,0])/1e3; pl = polls[1:]
    for k in (1,2,3):
        sel = pl == k
        if sel.any(): print(f"   polls=={k}: n={sel.sum()} lookback mean {lb[sel].mean():.2f} p50 {np.median(lb[sel]):.2f}")
    dist = (ph[1:,6] & 0xffffffff)
    print("   dist p50", np.median(dist), "mean", dist.mean().round(1))
    cyc = (ph[1:,6] & 0xffffffff)
    print("   first poll cycles p50", np.median(cyc), "mean", cyc.mean().round(0), "p90", np.percentile(cyc, 90))
