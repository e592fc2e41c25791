"""Dense two-pass step vs its reduce alone (norm_shard_partial) at several n
(probe, not product): scale time = step - reduce, as GB/s of its 8n bytes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import gen
import paper_2207_00257_b200 as L


def t(fn, k=10):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


for e in [int(a) for a in sys.argv[1:]] or [28, 30, 31, 32]:
    n = 2**e
    x = torch.empty(n, device="cuda")
    gen.fill_cuda(x, seed=1, dist="unit")
    y = torch.empty_like(x)
    part = torch.empty(1, dtype=torch.float64, device="cuda")
    step = t(lambda: L.normalize(y, x, index="dense", path="two_pass"))
    red = t(lambda: L.lib().norm_shard_partial(part.data_ptr(), x.data_ptr(), n, None))
    cp = t(lambda: y.copy_(x))
    sc = step - red
    print(f"2^{e}: step {step:.3f} ms ({12*n/step/1e6:.0f} GB/s)  reduce {red:.3f} ms ({4*n/red/1e6:.0f} GB/s)  "
          f"scale = step - reduce {sc:.3f} ms ({8*n/sc/1e6:.0f} GB/s)  torch copy {cp:.3f} ms ({8*n/cp/1e6:.0f} GB/s)",
          flush=True)
    del x, y
    torch.cuda.empty_cache()
