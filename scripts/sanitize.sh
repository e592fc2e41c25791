#!/bin/bash
# compute-sanitizer over small launches of every kernel (memcheck, racecheck,
# synccheck, initcheck); summaries into $OUT/sanitize_<tool>.log
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
cat > /tmp/san_driver.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import gen, paper_2207_00257_b200 as L
torch.cuda.set_device(0)
for n, path in [(1000, "small"), (5000, "two_pass"), (2**20 + 7, "two_pass"), (2**20 + 7, "fused"),
                (3 * 2**20 + 5, "two_pass"), (2**22 + 9, "two_pass"), (700, "two_pass"),
                (2**24 + 3, "two_pass"), (2**25, "fused"),  # many chunks per CTA: ring stages reused
                (2**26 + 5, "two_pass"), (2**26 + 5, "fused"),  # dynamic reduce tail: 16 tasks
                (2**20 + 7, "mid"), (3 * 2**20 + 5, "mid"), (5000, "mid"),  # cooperative mid path
                (2**20 + 7, "cluster"), (100000, "cluster"), (1024, "small")]:
    for mode in ("literal", "dense"):
        x = torch.from_numpy(gen.make_host(n, seed=1, dist=0)).cuda()
        y = torch.zeros_like(x)
        s = torch.zeros(1, device="cuda")
        L.normalize(y, x, index=mode, path=path, sum_out=s)
# scale_tile_kernel with a ragged head and tail, out of place and in place
for off in (1, 5):
    for n in (2**21 + 3, 70001):
        base = torch.from_numpy(gen.make_host(n + 8, seed=2, dist=0)).cuda()
        ob = torch.zeros_like(base)
        L.normalize(ob[off:off + n], base[off:off + n], index="dense", path="two_pass")
        L.normalize(base[off:off + n], base[off:off + n], index="literal", path="two_pass")
for form in ("per_thread", "per_block"):
    x = torch.rand(3000, device="cuda"); y = torch.empty_like(x)
    L.normalize_form(y, x, form=form)
for (R, C) in [(300, 4096), (7, 1000), (5, 10000), (9, 512), (3, 4099)]:
    for mode in ("literal", "dense"):
        x = torch.rand(R, C, device="cuda"); y = torch.zeros_like(x)
        L.normalize_rows(y, x, index=mode)
x = torch.randn(64, 2048, device="cuda"); y = torch.empty_like(x)
L.softmax_rows(y, x); L.softmax_rows(y, x, log=True)
t = (torch.rand(64, device="cuda") * 2048).long()
loss, tw = L.nll_forward(y, t)
g = L.nll_backward(torch.ones(1, device="cuda"), (64, 2048), t, tw)
for v in ("printed", "eliminated", "register", "tma"):
    for n_in in (16, 32, 16 * 61, 16 * 4001):
        xi = torch.rand(n_in + 1, device="cuda"); hw = torch.rand(n_in + 1, 17, device="cuda")
        ob = torch.empty(n_in, device="cuda")
        L.bpnn_layerforward(xi, hw, ob, variant=v)
for C in (512, 1024, 8192, 12288):
    x = torch.rand(37, C, device="cuda"); y = torch.zeros_like(x)
    L.normalize_rows(y, x, index="literal")
# gradient kernels (backward.cu): vector (aligned / misaligned, both index modes, in
# place), rows (vector and scalar paths), softmax / log-softmax
for n, off in ((5000, 0), (2**20 + 7, 0), (70001, 1), (100, 0)):
    for mode in ("literal", "dense"):
        xb = torch.rand(n + 8, device="cuda") + 0.1; gb = torch.randn(n + 8, device="cuda")
        yv = xb[off:off + n].clone(); sv = torch.zeros(1, device="cuda")
        L.normalize(yv, yv, index=mode, sum_out=sv)
        gxv = torch.empty(n + 8, device="cuda")[off:off + n]
        L.normalize_backward(gxv, gb[off:off + n], yv, sv, index=mode)
        gi = gb[off:off + n].clone(); L.normalize_backward(gi, gi, yv, sv, index=mode)
for (R, C) in [(300, 4096), (7, 1001), (3, 4099)]:
    xr = torch.rand(R, C, device="cuda") + 0.1; gr = torch.randn(R, C, device="cuda")
    for mode in ("literal", "dense"):
        yr = xr.clone(); sr = torch.zeros(R, device="cuda")
        L.normalize_rows(yr, yr, index=mode, sum_out=sr)
        L.normalize_rows_backward(torch.empty_like(gr), gr, yr, sr, index=mode)
    for lg in (False, True):
        ys = torch.empty_like(xr); L.softmax_rows(ys, xr, log=lg)
        L.softmax_rows_backward(torch.empty_like(gr), gr, ys, log=lg)
h = torch.rand(2**20 + 7).pin_memory(); o = torch.zeros_like(h).pin_memory()
L.normalize_host(o, h)
torch.cuda.synchronize()
print("driver ok")
PY
# --print-limit 0: every report is printed (the default stops at 100).  racecheck
# runs in its default analysis mode (one report per racing pair of source
# locations, with the hazard count) and scripts/racecheck_classify.py assigns
# every report to a documented pattern.  Raw logs go to /tmp (a hazard-level log
# is hundreds of MB); only logs under 8 MB are copied to $OUT.
for tool in memcheck racecheck synccheck initcheck; do
  compute-sanitizer --tool $tool --print-limit 0 --show-backtrace no --error-exitcode 9 \
      python /tmp/san_driver.py > /tmp/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|driver ok' /tmp/sanitize_$tool.log | tr '\n' ' ')"
  if [ $(stat -c %s /tmp/sanitize_$tool.log) -lt 8000000 ]; then cp /tmp/sanitize_$tool.log $OUT/;
  else head -c 2000000 /tmp/sanitize_$tool.log > $OUT/sanitize_$tool.head.log; fi
done
python scripts/racecheck_classify.py /tmp/sanitize_racecheck.log > $OUT/racecheck_classified.txt 2>&1
echo "racecheck classification rc=$? (1 = some report outside the documented patterns)"
