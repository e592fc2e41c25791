"""Reduce kernel time vs size (norm_shard_partial = one reduce launch), back to
back (K launches between two events) and isolated (events around each launch):
fits t = t0 + bytes / BW to expose the per-launch fixed cost that bounds the
sharded step at W = 8 (2 GiB per rank)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_2207_00257_b200 as L

nmax = 2**32
x = torch.empty(nmax, device="cuda")
gen.fill_cuda(x, seed=1, dist="unit")
part = torch.empty(1, dtype=torch.float64, device="cuda")
o = L._lib._opts("literal", "auto", None, None, None)
lib = L.lib()
rows = []
for e in range(24, 33):
    n = 2**e
    for _ in range(3):
        lib.norm_shard_partial(part.data_ptr(), x.data_ptr(), n, ctypes.byref(o))
    K = max(5, min(200, 2**32 // n * 2))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(K):
        lib.norm_shard_partial(part.data_ptr(), x.data_ptr(), n, ctypes.byref(o))
    b.record()
    torch.cuda.synchronize()
    bb = a.elapsed_time(b) / K
    iso = []
    for _ in range(10):
        a.record()
        lib.norm_shard_partial(part.data_ptr(), x.data_ptr(), n, ctypes.byref(o))
        b.record()
        torch.cuda.synchronize()
        iso.append(a.elapsed_time(b))
    rows.append((n, bb, float(np.median(iso))))
    print(f"n=2^{e}: back-to-back {bb * 1e3:9.1f} us ({4 * n / bb / 1e6:7.1f} GB/s)  isolated {np.median(iso) * 1e3:9.1f} us", flush=True)
B = np.array([4 * r[0] for r in rows if r[0] >= 2**27], dtype=np.float64)
for col, name in ((1, "back-to-back"), (2, "isolated")):
    T = np.array([r[col] for r in rows if r[0] >= 2**27]) * 1e-3
    A = np.vstack([np.ones_like(B), B]).T
    (t0, inv), *_ = np.linalg.lstsq(A, T, rcond=None)
    print(f"{name}: t = {t0 * 1e6:.1f} us + bytes / {1 / inv / 1e9:.1f} GB/s")
