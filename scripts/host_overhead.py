"""Per-call host overhead of the Python binding + C ABI at small n (not product)."""
import time
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2207_00257_b200 as L

for n in (1024, 2**20 + 7):
    x = torch.rand(n, device="cuda")
    y = torch.empty_like(x)
    for _ in range(100):
        L.normalize(y, x)
    torch.cuda.synchronize()
    t = time.perf_counter()
    K = 2000
    for _ in range(K):
        L.normalize(y, x)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t) / K * 1e6
    # device time of the same call captured in a CUDA graph
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        L.normalize(y, x)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(100):
                L.normalize(y, x)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()
    a.record()
    for _ in range(10):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    dev = a.elapsed_time(b) * 1e3 / 1000
    print(f"n={n}: eager {wall:.2f} us/call (host-bound), graph-replayed {dev:.2f} us/call (device)")
