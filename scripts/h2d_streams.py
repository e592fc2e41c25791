"""Pinned host -> device copy rate with 1, 2, 4 concurrent streams, and H2D with a
concurrent D2H (probe, not product): the link the e2e number is bound by."""
import torch, time
n = 1 << 30  # 4 GiB fp32
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device="cuda")
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        part = n // k
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{k} streams: {4 * n / dt / 1e9:.1f} GB/s")
# D2H while H2D
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1):
    d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d[: n // 4], non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(f"H2D 4 GiB + concurrent D2H 1 GiB: {dt*1e3:.1f} ms (H2D alone at 55.6 GB/s: {4*n/55.6e9*1e3:.1f} ms)")
