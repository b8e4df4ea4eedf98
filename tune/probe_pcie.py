import torch, time
n = 960 * 1024 * 1024 // 4
d = torch.empty(n, dtype=torch.float32, device="cuda")
h = torch.empty(n, dtype=torch.float32).pin_memory()
h2 = torch.empty(n // 2, dtype=torch.float32).pin_memory()
d2 = torch.empty(n // 2, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    torch.cuda.synchronize(); a = time.perf_counter(); fn(); torch.cuda.synchronize(); return time.perf_counter() - a
for _ in range(2):
    td = t(lambda: h.copy_(d, non_blocking=True))
    tu = t(lambda: d2.copy_(h2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
        with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
    tb = t(both)
print(f"D2H {n*4/td/1e9:.1f} GB/s  H2D {n*2/tu/1e9:.1f} GB/s  both (960MB down + 480MB up) {tb*1e3:.1f} ms")
