"""Where the dense step's read+write ceiling comes from (probe, not product):
same-box HBM rates of a pure read stream, a pure write stream and read+write
streams over 4 GiB buffers (well beyond the 126 MB L2), each the best of 10
CUDA-event-timed repetitions after 3 warm-ups:
  read   : libnorm reduce (two_pass dense, the reduce share timed alone through
           norm_debug_set_events) and torch.sum
  write  : cudaMemsetAsync (torch zero_) and torch fill_
  r+w    : libnorm scale_bulk_kernel (dense two-pass step minus its reduce),
           cudaMemcpyAsync D2D (torch copy_) and torch's elementwise x * c
Bytes: read-only = 4n, write-only = 4n, read+write = 8n."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2207_00257_b200 as L  # noqa: E402

n = 2**30
x = torch.empty(n, device="cuda")
gen.fill_cuda(x, seed=1, dist="unit")
y = torch.empty_like(x)
st = torch.cuda.current_stream()


def best(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts) / 1e3


def rate(name, nbytes, sec):
    print(f"  {name:44s} {sec * 1e3:8.3f} ms  {nbytes / sec / 1e9:7.0f} GB/s")


print(f"n = 2^30 fp32 (4 GiB per buffer), best of 10")
t_step = best(lambda: L.normalize(y, x, index="dense", path="two_pass"))
ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
reds = []
for _ in range(10):  # the reduce alone: events recorded around it on the launch stream
    L.normalize(y, x, index="dense", path="two_pass", events=ev)
    torch.cuda.synchronize()
    reds.append(ev[0].elapsed_time(ev[1]) / 1e3)
t_red = min(reds)
print("read-only:")
rate("libnorm reduce_dyn_kernel (in the dense step)", 4 * n, t_red)
rate("torch.sum", 4 * n, best(lambda: x.sum()))
print("write-only:")
rate("torch zero_ (cudaMemsetAsync)", 4 * n, best(lambda: y.zero_()))
rate("torch fill_(1.5)", 4 * n, best(lambda: y.fill_(1.5)))
print("read+write:")
rate("libnorm scale (dense step - reduce)", 8 * n, t_step - t_red)
rate("libnorm dense step (reduce + scale, 12n)", 12 * n, t_step)
rate("torch copy_ (cudaMemcpyAsync D2D)", 8 * n, best(lambda: y.copy_(x)))
rate("torch mul(x, c, out=y)", 8 * n, best(lambda: torch.mul(x, 0.5, out=y)))
