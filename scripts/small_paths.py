"""Device time per call (CUDA-graph replay) of each path at small / mid n (not product)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2207_00257_b200 as L

for n in (1024, 16384, 65536, 2**18, 2**20 + 7, 2**22, 2**24):
    x = torch.rand(n, device="cuda")
    y = torch.empty_like(x)
    row = []
    for path in ("small", "two_pass", "fused", "auto"):
        if path == "small" and n > 2**22:
            row.append(f"{path}=   -   ")
            continue
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            L.normalize(y, x, path=path)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for _ in range(50):
                    L.normalize(y, x, path=path)
        torch.cuda.synchronize()
        g.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        row.append(f"{path}={a.elapsed_time(b) * 1e3 / 500:7.2f}us")
    print(f"n={n:>9}: " + "  ".join(row))

# host-side cost per call: eager Python binding vs a replayed NormGraph (n = 2^20 + 7)
import time
n = 2**20 + 7
x = torch.rand(n, device="cuda")
y = torch.empty_like(x)
g = L.NormGraph(y, x)
for f, name in ((lambda: L.normalize(y, x), "eager normalize"), (g.launch, "NormGraph.launch")):
    for _ in range(200):
        f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(2000):
        f()
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t) / 2000 * 1e6:.2f} us/call (host + device, back to back)")
