"""Where the fused kernel's time goes (probe, not product): loads the
NORM_TIMELINE build of libnorm (make paper_2207_00257_b200/faults/libnorm_timeline.so),
runs literal normalize through the fused kernel back to back, and prints per-CTA
%globaltimer phase stamps of the last call relative to the earliest CTA entry:
phase-1 streaming done, grid barrier passed, divisor ready, scale done."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["LIBNORM_SO"] = os.path.join(ROOT, "paper_2207_00257_b200", "faults", "libnorm_timeline.so")
sys.path.insert(0, ROOT)
import numpy as np
import torch

import gen
import paper_2207_00257_b200 as L

lib = L.lib()
lib.norm_debug_fused_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
sms = torch.cuda.get_device_properties(0).multi_processor_count
for n in [int(a) for a in (sys.argv[1:] or [str(2**29), str(2**28)])]:
    x = torch.empty(n, device="cuda")
    gen.fill_cuda(x, seed=1, dist="unit")
    y = torch.empty_like(x)
    for _ in range(5):
        L.normalize(y, x, index="literal", path="fused")
    K = 20
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(K):
        L.normalize(y, x, index="literal", path="fused")
    b.record()
    torch.cuda.synchronize()
    per_call = a.elapsed_time(b) / K * 1e3
    buf = np.zeros(sms * 5, dtype=np.uint64)
    assert lib.norm_debug_fused_timeline(buf.ctypes.data, sms * 5) == 0
    t = buf.reshape(sms, 5).astype(np.int64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    names = ["entry", "phase-1 done", "barrier passed", "divisor ready", "scale done"]
    print(f"n={n}: {per_call:.1f} us per call back to back; per-CTA stamps (us from first entry): min / median / max")
    for k, nm in enumerate(names):
        print(f"  {nm:16s} {rel[:, k].min():8.2f} {np.median(rel[:, k]):8.2f} {rel[:, k].max():8.2f}")

if os.environ.get("DUMP"):
    print("per-CTA (entry, phase-1 done, barrier passed, divisor, scale done) for the 5 earliest and 5 latest phase-1 finishers:")
    order = np.argsort(rel[:, 1])
    for i in list(order[:5]) + list(order[-5:]):
        print("  cta %3d: %s" % (i, " ".join("%8.2f" % v for v in rel[i])))
    print("CTAs whose barrier stamp precedes the last phase-1 stamp:", int((rel[:, 2] < rel[:, 1].max()).sum()))
