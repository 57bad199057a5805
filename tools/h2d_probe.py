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
