"""Time libnorm's reduce kernel alone (norm_shard_partial = one reduce launch)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_2207_00257_b200 as L
n = 2**32
x = torch.empty(n, device="cuda")
gen.fill_cuda(x, seed=1, dist="unit")
part = torch.empty(1, dtype=torch.float64, device="cuda")
o = L._lib._opts("literal", "auto", None, None, None)
lib = L.lib()
for _ in range(3):
    lib.norm_shard_partial(part.data_ptr(), x.data_ptr(), n, ctypes.byref(o))
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    lib.norm_shard_partial(part.data_ptr(), x.data_ptr(), n, ctypes.byref(o))
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print("reduce only: best %.4f ms (%.1f GB/s), mean %.4f ms" % (min(ts), 4 * n / min(ts) / 1e6, sum(ts) / len(ts)))
