"""Phases of read_tns(path) e2e: file -> pinned -> H2D -> parse."""
import os
import sys
import tempfile
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1902_03317_b200 import generate, tns  # noqa: E402

x = generate.coo([10000] * 3, 10_000_000, 7, [0, 0, 0], 0.5, 1.5, None, 0)
text = generate.tns_text(x)
d = tempfile.mkdtemp(dir="/dev/shm")
path = os.path.join(d, "x.tns")
text.cpu().numpy().tofile(path)
size = os.path.getsize(path)
print("size", size, "cpus", os.cpu_count())
for slice_mb in (4, 8, 32):
    for workers in (4, 8, 16):
        pool = ThreadPoolExecutor(workers)
        host = torch.empty(size, dtype=torch.uint8, pin_memory=True)
        view = memoryview(host.numpy())
        fd = os.open(path, os.O_RDONLY)
        S = slice_mb << 20

        def rd(lo):
            hi = min(size, lo + S)
            got = lo
            while got < hi:
                got += os.preadv(fd, [view[got:hi]], got)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            list(pool.map(rd, range(0, size, S)))
            ts.append(time.perf_counter() - t0)
        os.close(fd)
        print(f"slice {slice_mb} MB workers {workers}: read {1e3 * min(ts):.1f} ms "
              f"({size / min(ts) / 1e9:.1f} GB/s)")
t0 = time.perf_counter()
np_buf = np.empty(size, np.uint8)
t1 = time.perf_counter()
with open(path, "rb") as f:
    f.readinto(memoryview(np_buf))
t2 = time.perf_counter()
print(f"pageable alloc {1e3*(t1-t0):.1f} ms, single readinto {1e3*(t2-t1):.1f} ms")
host = torch.empty(size, dtype=torch.uint8, pin_memory=True)
dev = torch.empty(size, dtype=torch.uint8, device="cuda")
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    print(f"H2D {1e3*(time.perf_counter()-t0):.1f} ms")
for _ in range(2):
    t0 = time.perf_counter()
    h = torch.empty(size, dtype=torch.uint8, pin_memory=True)
    print(f"pinned alloc {1e3*(time.perf_counter()-t0):.1f} ms")
    del h
for _ in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    z = tns.read_tns(path)
    torch.cuda.synchronize()
    print(f"read_tns e2e {1e3*(time.perf_counter()-t0):.1f} ms")
