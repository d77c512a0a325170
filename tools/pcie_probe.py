import torch, time
n = 4_460_000_000
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
a = torch.empty(3_100_000_000, dtype=torch.uint8, pin_memory=True)
da = torch.empty(3_100_000_000, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
print("D2H alone GB/s", n / t(lambda: h.copy_(d, non_blocking=True)) / 1e9)
print("H2D alone GB/s", 3.1e9 / t(lambda: da.copy_(a, non_blocking=True)) / 1e9)
def both():
    with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2): da.copy_(a, non_blocking=True)
print("both, s per pair", t(both))
def chunked():
    c = 1 << 28
    for i in range(0, n, c):
        with torch.cuda.stream(s1 if (i // c) % 2 == 0 else s2):
            h[i:i + c].copy_(d[i:i + c], non_blocking=True)
print("D2H chunked 2 streams GB/s", n / t(chunked) / 1e9)
