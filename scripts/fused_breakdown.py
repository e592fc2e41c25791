"""Where the fused path's time goes at n = 2^28 literal (not product): reduce only
(norm_shard_partial), fused, two-pass, each timed per launch after an L2 flush."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_2207_00257_b200 as L
n = 2**28
x = torch.empty(n, device="cuda")
gen.fill_cuda(x, seed=1, dist="unit")
y = torch.empty_like(x)
part = torch.empty(1, dtype=torch.float64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
o = L._lib._opts("literal", "auto", None, None, None)
lib = L.lib()
def t(fn, reps=20):
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return min(ts), sum(ts) / len(ts)
print("reduce only  us (min, mean):", t(lambda: lib.norm_shard_partial(part.data_ptr(), x.data_ptr(), n, ctypes.byref(o))))
print("fused        us (min, mean):", t(lambda: L.normalize(y, x, path="fused")))
print("two_pass     us (min, mean):", t(lambda: L.normalize(y, x, path="two_pass")))
print("empty kernel us (min, mean):", t(lambda: torch.empty(0, device="cuda").zero_()))
