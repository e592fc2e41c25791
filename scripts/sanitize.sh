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
                (2**26 + 5, "two_pass"), (2**26 + 5, "fused")]:  # dynamic reduce tail: 16 tasks
    for mode in ("literal", "dense"):
        x = torch.from_numpy(gen.make_host(n, seed=1, dist=0)).cuda()
        y = torch.zeros_like(x)
        s = torch.zeros(1, device="cuda")
        L.normalize(y, x, index=mode, path=path, sum_out=s)
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
h = torch.rand(2**20 + 7).pin_memory(); o = torch.zeros_like(h).pin_memory()
L.normalize_host(o, h)
torch.cuda.synchronize()
print("driver ok")
PY
for tool in memcheck racecheck synccheck initcheck; do
  compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san_driver.py > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|driver ok' $OUT/sanitize_$tool.log | tr '\n' ' ')"
done
