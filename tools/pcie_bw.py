import torch, time
n = 1 << 30
h1 = torch.empty(n, dtype=torch.int32, pin_memory=True)
h2 = torch.empty(n, dtype=torch.int32, pin_memory=True)
d1 = torch.empty(n, dtype=torch.int32, device="cuda")
d2 = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f):
    torch.cuda.synchronize(); a = time.perf_counter(); f(); torch.cuda.synchronize(); return time.perf_counter() - a
for _ in range(2):
    up = t(lambda: d1.copy_(h1, non_blocking=True))
    dn = t(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    bo = t(both)
    print(f"H2D {4*n/up/1e9:.1f} GB/s  D2H {4*n/dn/1e9:.1f} GB/s  both {2*4*n/bo/1e9:.1f} GB/s total ({bo*1e3:.1f} ms)")
