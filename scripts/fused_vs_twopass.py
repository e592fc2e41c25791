"""Literal normalize, two_pass vs fused, back to back (K calls between events),
over n = 2^27..2^30: the rank-local shape of the sharded step at W = 8 is
n = 2^29 (2 GiB, covered prefix 67 MB)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_2207_00257_b200 as L

sizes = [int(a) * 2**26 for a in os.environ.get("SIZES_X64MI", "2 4 8 9 10 11 12 14 16").split()]
x = torch.empty(max(sizes), device="cuda")
gen.fill_cuda(x, seed=1, dist="unit")
y = torch.empty_like(x)
IDX = os.environ.get("INDEX", "literal")
for n in sizes:
    res = {}
    for path in ("two_pass", "fused"):
        for _ in range(3):
            L.normalize(y[:n], x[:n], index=IDX, path=path)
        K = 50
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(K):
            L.normalize(y[:n], x[:n], index=IDX, path=path)
        b.record()
        torch.cuda.synchronize()
        res[path] = a.elapsed_time(b) / K * 1e3
    cnt, pre = L.coverage(n, IDX)
    print(f"n={n / 2**20:.0f} Mi (prefix {4 * pre / 2**20:.0f} MiB): two_pass {res['two_pass']:8.1f} us  fused {res['fused']:8.1f} us", flush=True)
