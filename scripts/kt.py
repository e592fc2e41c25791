"""Kernel timer for same-box A/B probes (with scripts/ab_libs.py or ab_env.sh):
the row and fused workloads, K back-to-back calls between CUDA events, median
of R such groups, one line per workload (µs per call).  Much lighter than
bench.py (no parity, e2e or CPU legs).  KT_WORK selects workloads
(comma-separated: softmax, logsoftmax, nllbwd, fill, dense30, dense30_inplace, rows_dense, rows_literal, fused28, dense28, backprop,
smbwd, lsmbwd, rowsbwd, vecbwd28l, vecbwd28d)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_2207_00257_b200 as L

WORK = os.environ.get("KT_WORK", "softmax,rows_dense,rows_literal,fused28,dense28,backprop").split(",")
K, R = int(os.environ.get("KT_K", "20")), int(os.environ.get("KT_R", "7"))


def timed(fn):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(R):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(K):
            fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / K * 1e3)
    return statistics.median(ts), min(ts)


x = torch.empty(2**28, device="cuda")
y = torch.empty_like(x)
for w in WORK:
    if w in ("softmax", "logsoftmax", "rows_dense", "rows_literal"):
        gen.fill_cuda(x, seed=1, dist="signed" if "softmax" in w else "unit")
        xi, yo = x.view(65536, 4096), y.view(65536, 4096)
        if "softmax" in w:
            lg = w == "logsoftmax"
            fn = lambda: L.softmax_rows(yo, xi, log=lg)  # noqa: E731
        else:
            idx = w.split("_")[1]
            fn = lambda: L.normalize_rows(yo, xi, index=idx)  # noqa: E731
    elif w in ("dense30", "dense30_inplace"):  # in-place vs out-of-place read+write streams
        xs, ys = x[:2**28], y[:2**28]
        gen.fill_cuda(xs, seed=1, dist="unit")
        if w == "dense30":
            fn = lambda: L.normalize(ys, xs, index="dense")  # noqa: E731
        else:
            fn = lambda: L.normalize(xs, xs, index="dense")  # noqa: E731
    elif w in ("fused28", "dense28"):
        gen.fill_cuda(x, seed=1, dist="unit")
        idx = "literal" if w == "fused28" else "dense"
        fn = lambda: L.normalize(y, x, index=idx)  # noqa: E731
    elif w == "nllbwd":  # ClassNLL backward: a 1 GiB write stream (zeros + one value per row)
        nr, nc = 65536, 4096
        tgt = (torch.rand(nr, device="cuda") * nc).long()
        tw = torch.full((1,), float(nr), device="cuda")
        g1 = torch.ones(1, device="cuda")
        grad = y.view(nr, nc)
        fn = lambda: L.nll_backward(g1, (nr, nc), tgt, tw, grad=grad)  # noqa: E731
    elif w == "fill":  # context: torch's own write stream on the same 1 GiB
        fn = lambda: y.fill_(1.5)  # noqa: E731
    elif w == "backprop":
        n_in, hid = 2**22, 16
        inp = torch.rand(n_in + 1, device="cuda")
        hidden = torch.rand((n_in + 1) * (hid + 1), device="cuda")
        outp = torch.empty(n_in, device="cuda")
        fn = lambda: L.bpnn_layerforward(inp, hidden, outp, variant="tma")  # noqa: E731
    elif w in ("smbwd", "lsmbwd", "rowsbwd", "vecbwd28l", "vecbwd28d"):  # gradient kernels
        gen.fill_cuda(x, seed=1, dist="signed")
        gg = torch.empty_like(x)
        gen.fill_cuda(gg, seed=2, dist="signed")
        gxo = torch.empty_like(x)
        if w in ("smbwd", "lsmbwd"):
            lg = w == "lsmbwd"
            L.softmax_rows(y.view(65536, 4096), x.view(65536, 4096), log=lg)
            fn = lambda: L.softmax_rows_backward(gxo.view(65536, 4096), gg.view(65536, 4096),  # noqa: E731
                                                 y.view(65536, 4096), log=lg)
        elif w == "rowsbwd":
            sr = torch.zeros(65536, device="cuda")
            L.normalize_rows(y.view(65536, 4096), x.view(65536, 4096).abs(), index="dense", sum_out=sr)
            fn = lambda: L.normalize_rows_backward(gxo.view(65536, 4096), gg.view(65536, 4096),  # noqa: E731
                                                   y.view(65536, 4096), sr, index="dense")
        else:
            idx = "literal" if w.endswith("l") else "dense"
            sv = torch.zeros(1, device="cuda")
            y.copy_(x.abs())
            L.normalize(y, y, index=idx, sum_out=sv)
            fn = lambda: L.normalize_backward(gxo, gg, y, sv, index=idx)  # noqa: E731
    else:
        continue
    med, mn = timed(fn)
    print(f"{w:14s} median {med:9.2f} us  min {mn:9.2f} us", flush=True)
