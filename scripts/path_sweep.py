"""AUTO-rule evidence (probe, not product): device time per call of every path,
from a CUDA graph of R back-to-back calls (no host in the loop).  hot: the
input stays in L2 between calls when it fits; flushed: each call follows a
256 MiB write + 256 MiB read inside the graph, and the graph of the flushes
alone is subtracted.  Usage: path_sweep.py literal|dense hot|flushed [n ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import gen
import paper_2207_00257_b200 as L

mode = sys.argv[1] if len(sys.argv) > 1 else "literal"
flushed = len(sys.argv) > 2 and sys.argv[2] == "flushed"
sizes = [int(a) for a in sys.argv[3:]] or [2**e + 7 for e in range(12, 26)]
R = 20 if flushed else 50
ws = torch.zeros(L.workspace_bytes(), dtype=torch.uint8, device="cuda")
fw = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
fr = torch.ones(64 << 20, device="cuda")


def flush():
    fw.zero_()
    fr.sum()


def graph_us(body):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        body()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(R):
                body()
    torch.cuda.synchronize()
    g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / (5 * R)


t_flush = graph_us(flush) if flushed else 0.0
for n in sizes:
    x = torch.empty(n, device="cuda")
    gen.fill_cuda(x, seed=1, dist="unit")
    y = torch.empty_like(x)
    row = {"n": n, "mode": mode, "flushed": flushed, "auto": L.choose_path(n, L.coverage(n, mode)[1])}
    for path in ("small", "cluster", "mid", "two_pass", "fused"):
        if path == "small" and n > 2**21:
            continue

        def call():
            L.normalize(y, x, index=mode, path=path, workspace=ws, trusted=True)
        body = (lambda: (flush(), call())) if flushed else call
        row[path + "_us"] = round(graph_us(body) - t_flush, 2)
    print(json.dumps(row), flush=True)
