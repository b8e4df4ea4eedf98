"""Time the device .tns parse on C2's tensor as text (ncu target)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1902_03317_b200 import generate, tns  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
x = generate.coo([10000] * 3, n, 7, [0, 0, 0], 0.5, 1.5, None, 0)
text = generate.tns_text(x)
del x
torch.cuda.synchronize()
for r in range(reps):
    t0 = time.perf_counter()
    z = tns.read_tns_bytes(text, None, 0)
    torch.cuda.synchronize()
    print(f"{text.numel()} bytes {z.nnz} nnz: {1e3 * (time.perf_counter() - t0):.3f} ms")
