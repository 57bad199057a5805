import torch, time
n = 8 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for chunk in (64 << 20, 256 << 20, 768 << 20, 8 << 30):
    torch.cuda.synchronize(); t = time.perf_counter()
    for o in range(0, n, chunk):
        d[o:o+chunk].copy_(h[o:o+chunk], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(chunk >> 20, "MiB chunks:", n / dt / 1e9, "GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t = time.perf_counter()
half = n // 2
with torch.cuda.stream(s1): d[:half].copy_(h[:half], non_blocking=True)
with torch.cuda.stream(s2): d[half:].copy_(h[half:], non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("2 streams:", n / dt / 1e9, "GB/s")
# duplex: H2D of one buffer while D2H of another (the e2e overlap)
h2 = torch.empty(n // 2, dtype=torch.uint8, pin_memory=True)
d2 = torch.empty(n // 2, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("duplex: H2D", n / dt / 1e9, "GB/s with D2H of", (n // 2) / 1e9, "GB")
torch.cuda.synchronize(); t = time.perf_counter()
h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("D2H alone:", (n // 2) / dt / 1e9, "GB/s")
