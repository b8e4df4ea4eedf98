import torch, sys, os, ctypes, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_03317_b200 import generate, ops, _lib
from paper_1902_03317_b200.coo import DeviceCOO
lib = _lib.load()
dims, nnz = [50000, 20000, 100000], 20_000_000
base = generate.coo(dims, nnz, 1, [1.1, 0, 0], 0, 1, None)
for mode in (0, 2):
    xs = base.clone(); ops.sort_lexicographic(xs, ops.mode_last_order(3, mode))
    fib = ops.build_fiber_index(xs, mode)
    v = generate.uniform(dims[mode], 1, 5, -1, 1)
    zv = DeviceCOO.empty([1, 1], fib.nfibs)
    for _ in range(3): ops.ttv(xs, v, mode, fib, out=zv)
    torch.cuda.synchronize()
    nt = (nnz + 2047) // 2048
    buf = np.zeros(65536 * 8, np.uint64)
    lib.spt_debug_phases(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(65536 * 8))
    ph = buf.reshape(-1, 8)[:nt, :6].astype(np.int64)
    d = np.diff(ph, axis=1)
    print(f"mode {mode}: span {(ph[:,5].max()-ph[:,0].min())/1e3:.1f} us tiles {nt}")
    for k, name in enumerate(["load+fptr", "search+scan", "meta", "lookback", "emit"]):
        print(f"   {name:12s} mean {d[:,k].mean()/1e3:7.2f} us  p50 {np.median(d[:,k])/1e3:7.2f}  p99 {np.percentile(d[:,k],99)/1e3:7.2f}")
    life = ph[:,5]-ph[:,0]
    conc = [int(((ph[:,0] <= tq) & (ph[:,5] >= tq)).sum()) for tq in np.linspace(ph[:,0].min(), ph[:,5].max(), 12)]
    print("   lifetime", life.mean()/1e3, "concurrency", conc)
