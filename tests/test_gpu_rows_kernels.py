"""Row kernels at the widths where their launch geometry changes (rows.cu,
rowops.cu: 1024 / 2048 / 2056 / 3000 / 4096 / 8192 / 8200 columns, padded
leading dimensions, in place), against the oracle, with the register row queue
on (default) and off (NORM_ROWS_QUEUE=0, grid-strided rows).  Each
configuration runs in its own process (knobs are read once per process).

norm_rows (reading R10 / P17: row r is Fig. 1's normalize of row r,
PAPER.md:98-119): every row's divisor s_r within 1e-6 of the oracle's exact row
sum (Σ|x| for signed rows, P20), every covered output the bitwise binary32
replay x / s_r, every uncovered and padding element untouched; in-place rows
replayed against the input bits.  Softmax / log-softmax:
within the north_star row tolerance of the oracle's fp64 rows."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import oracle  # noqa: E402

pytestmark = pytest.mark.gpu

SENT = 0x7FC0FFEE
# (rows, cols, ld, index, dist, in place): register kernel with 1, 2 and 4
# vectors per thread (dense), TMA warp-per-row kernel (literal), 8200 columns
CASES = [(4099, 1024, 1024, "dense", 0, False), (1111, 2048, 2048, "literal", 4, False),
         (517, 2056, 2064, "dense", 3, False), (300, 3000, 3000, "literal", 2, True),
         (2000, 4096, 4096, "dense", 1, True), (777, 4096, 4104, "literal", 0, False),
         (129, 8192, 8192, "dense", 4, False), (65, 8192, 8192, "literal", 3, True),
         (9, 8200, 8200, "dense", 0, False)]
SM_CASES = [(3001, 1024, 1024, False, False), (517, 2056, 2064, True, False), (1000, 4096, 4096, False, True),
            (64, 8192, 8192, True, True), (300, 3000, 3000, False, False)]

DRIVER = r"""
import os, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import gen, paper_2207_00257_b200 as L
out_dir = sys.argv[1]
for k, (R, C, ld, index, dist, inplace) in enumerate({cases!r}):
    x = np.zeros((R, ld), np.float32)
    x[:, :C] = gen.make_host(R * C, seed=300 + k, dist=dist).reshape(R, C)
    inp = torch.from_numpy(x).cuda()
    if inplace:
        out = inp
    else:
        out = torch.empty_like(inp)
        out.view(torch.int32).fill_({sent})
    s = torch.zeros(R, device="cuda")
    L.normalize_rows(out[:, :C], inp[:, :C], index=index, sum_out=s)
    torch.cuda.synchronize()
    np.save(os.path.join(out_dir, f"out{{k}}.npy"), out.cpu().numpy())
    np.save(os.path.join(out_dir, f"s{{k}}.npy"), s.cpu().numpy())
for k, (R, C, ld, log, inplace) in enumerate({sm_cases!r}):
    x = np.zeros((R, ld), np.float32)
    x[:, :C] = gen.make_host(R * C, seed=400 + k, dist=3).reshape(R, C) * 8.0
    inp = torch.from_numpy(x).cuda()
    out = inp if inplace else torch.zeros_like(inp)
    L.softmax_rows(out[:, :C], inp[:, :C], log=log)
    torch.cuda.synchronize()
    np.save(os.path.join(out_dir, f"sm{{k}}.npy"), out.cpu().numpy())
print("ok")
"""


@pytest.mark.parametrize("queue", ["1", "0"])
def test_rows_widths(queue, tmp_path):
    code = DRIVER.format(root=ROOT, cases=CASES, sm_cases=SM_CASES, sent=SENT)
    env = dict(os.environ, NORM_ROWS_QUEUE=queue)
    r = subprocess.run([sys.executable, "-c", code, str(tmp_path)], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
    for k, (R, C, ld, index, dist, inplace) in enumerate(CASES):
        x = np.zeros((R, ld), np.float32)
        x[:, :C] = gen.make_host(R * C, seed=300 + k, dist=dist).reshape(R, C)
        o = np.load(tmp_path / f"out{k}.npy")
        sv = np.load(tmp_path / f"s{k}.npy")
        xc = np.ascontiguousarray(x[:, :C])
        S = oracle.rows_sum_exact(xc)
        scale = oracle.rows_sum_exact(np.abs(xc)) if dist == 3 else np.abs(S)
        bad = np.nonzero(np.abs(sv.astype(np.float64) - S) > 1e-6 * scale)[0]
        assert bad.size == 0, (k, bad[:5])
        cov = oracle.covered_mask(C, index)
        q = xc[:, cov] / sv[:, None]
        assert np.array_equal(o[:, :C][:, cov].view(np.uint32), q.view(np.uint32)), k
        prior = x.view(np.uint32) if inplace else np.full(x.shape, SENT, np.uint32)
        assert np.array_equal(o[:, :C][:, ~cov].view(np.uint32), prior[:, :C][:, ~cov]), k
        assert np.array_equal(o[:, C:].view(np.uint32), prior[:, C:]), k
    for k, (R, C, ld, log, inplace) in enumerate(SM_CASES):
        x = gen.make_host(R * C, seed=400 + k, dist=3).reshape(R, C) * np.float32(8.0)
        got = np.load(tmp_path / f"sm{k}.npy")[:, :C].astype(np.float64)
        ref = oracle.softmax_rows(x, log=log)
        ref = ref.astype(np.float64)
        if log:  # the tolerances of test_gpu_rowops.py
            assert np.all(np.abs(got - ref) <= 1e-5 * np.maximum(1.0, np.abs(ref))), k
        else:
            assert np.all(np.abs(got - ref) <= np.maximum(1e-5 * np.abs(ref), 1e-37)), k
            assert np.all(np.abs(got.sum(axis=1) - 1.0) <= 1e-5), k
