"""Device timeline of one two-pass normalize (probe, not product; stands in for
an nsys timeline, which this image lacks): loads the NORM_TIMELINE build of
libnorm (make paper_2207_00257_b200/faults/libnorm_timeline.so), runs the
two-pass path back to back, and prints per-CTA %globaltimer stamps of the last
call relative to the earliest reduce CTA entry:
  reduce_dyn_kernel: entry, streaming done (late PDL trigger), partial published,
                     S written (last CTA)
  scale_bulk_kernel: producer entry, first TMA chunk issued, griddepcontrol.wait
                     returned, first chunk stored, last chunk stored
With PDL (NORM_PDL=late, the default) scale CTAs start on SMs whose reduce CTA has
finished and their producers stream `in` into the ring before the reduce grid
completes; NORM_PDL=off shows the serialised launch for comparison.
  python scripts/pdl_timeline.py [n index] ..."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["LIBNORM_SO"] = os.path.join(ROOT, "paper_2207_00257_b200", "faults", "libnorm_timeline.so")
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2207_00257_b200 as L  # noqa: E402

lib = L.lib()
for f in ("norm_debug_reduce_timeline", "norm_debug_scale_timeline"):
    getattr(lib, f).argtypes = [ctypes.c_void_p, ctypes.c_int]
sms = torch.cuda.get_device_properties(0).multi_processor_count
args = sys.argv[1:] or [str(2**32), "literal", str(2**30), "dense"]
print(f"NORM_PDL={os.environ.get('NORM_PDL', 'late (default)')}")
for n, mode in zip(map(int, args[0::2]), args[1::2]):
    x = torch.empty(n, device="cuda")
    gen.fill_cuda(x, seed=1, dist="unit")
    y = torch.empty_like(x)
    for _ in range(5):
        L.normalize(y, x, index=mode, path="two_pass")
    K = 10
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(K):
        L.normalize(y, x, index=mode, path="two_pass")
    b.record()
    torch.cuda.synchronize()
    per_call = a.elapsed_time(b) / K * 1e3
    rb = np.zeros(sms * 4, dtype=np.uint64)
    sb = np.zeros(sms * 5, dtype=np.uint64)
    assert lib.norm_debug_reduce_timeline(rb.ctypes.data, sms * 4) == 0
    assert lib.norm_debug_scale_timeline(sb.ctypes.data, sms * 5) == 0
    r = rb.reshape(sms, 4).astype(np.int64)
    s = sb.reshape(sms, 5).astype(np.int64)
    t0 = r[:, 0].min()
    last = r[:, 3].max()  # only the last CTA writes stamp 3; others keep older values
    rr, sr = (r - t0) / 1e3, (s - t0) / 1e3
    S_written = (last - t0) / 1e3
    print(f"\n{mode} n={n}: {per_call:.1f} us per call back to back; stamps in us from the first reduce CTA "
          f"entry (min / median / max over {sms} CTAs)")
    for k, nm in enumerate(["reduce entry", "reduce streaming done", "reduce partial published"]):
        print(f"  {nm:30s} {rr[:, k].min():9.2f} {np.median(rr[:, k]):9.2f} {rr[:, k].max():9.2f}")
    print(f"  {'reduce S written (last CTA)':30s} {S_written:9.2f}")
    for k, nm in enumerate(["scale producer entry", "scale first TMA issued", "scale wait returned",
                            "scale first chunk stored", "scale last chunk stored"]):
        print(f"  {nm:30s} {sr[:, k].min():9.2f} {np.median(sr[:, k]):9.2f} {sr[:, k].max():9.2f}")
    early = int((sr[:, 1] < S_written).sum())
    lead = S_written - sr[:, 1]
    print(f"  scale CTAs that issued their first TMA load before the reduce finished: {early} / {sms}; "
          f"lead over S written: median {np.median(lead):.2f} us, max {lead.max():.2f} us")
    print(f"  gap S written -> first scale store: {sr[:, 3].min() - S_written:.2f} us; "
          f"scale span (first wait return -> last store): {sr[:, 4].max() - sr[:, 2].min():.2f} us")
    del x, y
    torch.cuda.empty_cache()
