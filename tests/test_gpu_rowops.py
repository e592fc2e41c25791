"""GPU parity for the NEXT-2 row ops through the C ABI vs the
fp64 oracle.  Tolerances: softmax per element 1e-5 relative
(absolute 1e-37 below FLT_MIN); log-softmax 1e-5·max(1,|y|); NLL loss and
total weight 1e-6 relative; NLL gradient 1e-6 relative on the target entries
and exact zeros elsewhere; every kernel bitwise repeatable."""
import math
import os

import numpy as np
import pytest
import torch

import gen
import oracle
import paper_2207_00257_b200 as L

pytestmark = pytest.mark.gpu


def logits(R, C, seed, scale):
    return (gen.make_host(R * C, seed=seed, dist="signed").reshape(R, C) * np.float32(scale)).astype(np.float32)


def check_softmax(x, y, log):
    ref = oracle.softmax_rows(x, log=log).astype(np.float64)
    y = y.astype(np.float64)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(y), nan)
    inf = np.isinf(ref)
    assert np.array_equal(y[inf], ref[inf])
    nan = nan | inf
    if log:
        assert np.all(np.abs(y[~nan] - ref[~nan]) <= 1e-5 * np.maximum(1.0, np.abs(ref[~nan])))
    else:
        tol = np.maximum(1e-5 * np.abs(ref[~nan]), 1e-37)
        assert np.all(np.abs(y[~nan] - ref[~nan]) <= tol)


SHAPES = [(65536, 4096, 4096), (5, 1, 1), (7, 33, 33), (3, 4096, 4104), (9, 8192, 8192),
          (4, 10000, 10000), (64, 2048, 2048), (2, 24, 24), (300, 1000, 1000)]


@pytest.mark.parametrize("log", [False, True])
def test_softmax_rows_parity(log):
    for i, (R, C, ld) in enumerate(SHAPES):
        x = np.zeros((R, ld), np.float32)
        x[:, :C] = logits(R, C, seed=i, scale=[1, 4, 20, 60][i % 4])
        inp = torch.from_numpy(x).cuda()
        out = torch.full((R, ld), -7.0, device="cuda")
        L.softmax_rows(out[:, :C], inp[:, :C], log=log)
        out2 = torch.empty_like(out)
        L.softmax_rows(out2[:, :C], inp[:, :C], log=log)
        torch.cuda.synchronize()
        y = out.cpu().numpy()
        assert np.array_equal(y[:, :C], out2[:, :C].cpu().numpy())
        assert np.all(y[:, C:] == -7.0)
        rows = range(R) if R <= 512 else np.random.default_rng(i).integers(0, R, 256)
        rows = np.array(list(rows))
        check_softmax(x[rows, :C], y[rows, :C], log)


def test_softmax_special_and_in_place():
    x = np.array([[0.0, -np.inf, 1.0, 2, 3, 4, 5, 6], [np.nan, 0, 0, 0, 0, 0, 0, 0],
                  [-np.inf] * 8, [88.0, -88.0, 0, 0, 0, 0, 0, 0]], np.float32)
    for log in (False, True):
        t = torch.from_numpy(x).cuda()
        o = torch.empty_like(t)
        L.softmax_rows(o, t, log=log)
        L.softmax_rows(t, t, log=log)  # in place (generic kernel)
        torch.cuda.synchronize()
        check_softmax(x, o.cpu().numpy(), log)
        check_softmax(x, t.cpu().numpy(), log)
    big = logits(1000, 4096, seed=5, scale=10)
    t = torch.from_numpy(big).cuda()
    ref = torch.empty_like(t)
    L.softmax_rows(ref, t)
    L.softmax_rows(t, t)
    torch.cuda.synchronize()
    assert torch.allclose(ref, t, rtol=1e-6, atol=0)


@pytest.mark.parametrize("reduction", ["none", "mean", "sum"])
@pytest.mark.parametrize("weighted", [False, True])
def test_nll_parity(reduction, weighted):
    for N, C in [(1, 1), (300, 37), (65536, 4096), (4099, 1000)]:
        lp = np.log(np.maximum(oracle.softmax_rows(logits(N, C, seed=C, scale=3)), 1e-30)).astype(np.float32)
        t = (gen.make_host(N, seed=N, dist="unit") * C).astype(np.int64)
        t[::13] = -100
        w = (gen.make_host(C, seed=2, dist="unit") + np.float32(0.5)) if weighted else None
        loss_ref, tw_ref = oracle.nll_forward(lp, t, w, reduction)
        lpd, td = torch.from_numpy(lp).cuda(), torch.from_numpy(t).cuda()
        wd = None if w is None else torch.from_numpy(w).cuda()
        loss, tw = L.nll_forward(lpd, td, wd, reduction)
        loss2, _ = L.nll_forward(lpd, td, wd, reduction)
        torch.cuda.synchronize()
        assert torch.equal(loss.view(torch.int32), loss2.view(torch.int32))  # bitwise, NaN too
        lv = loss.cpu().numpy().astype(np.float64)
        np.testing.assert_allclose(lv, loss_ref, rtol=1e-6, atol=0)
        assert abs(tw.item() - tw_ref) <= 1e-6 * tw_ref
        if tw_ref == 0:
            continue
        g = torch.from_numpy(gen.make_host(N, seed=9, dist="unit")).cuda() if reduction == "none" \
            else torch.tensor([0.75], device="cuda")
        grad = L.nll_backward(g, (N, C), td, tw, wd, reduction)
        torch.cuda.synchronize()
        gref = oracle.nll_backward(g.cpu().numpy().astype(np.float64), t, C, w, reduction, -100,
                                   float(np.float32(tw.item())))
        gv = grad.cpu().numpy().astype(np.float64)
        nz = gref != 0
        assert np.all(gv[~nz] == 0)
        assert np.all(np.abs(gv[nz] - gref[nz]) <= 1e-6 * np.abs(gref[nz]))


def test_nll_edges():
    lp = torch.zeros((4, 3), device="cuda")
    t = torch.tensor([-100, -100, -100, -100], device="cuda")
    loss, tw = L.nll_forward(lp, t, None, "mean")
    torch.cuda.synchronize()
    assert math.isnan(loss.item()) and tw.item() == 0
    t = torch.tensor([0, 5, 1, 2], device="cuda")  # 5 out of range, not ignored
    loss, _ = L.nll_forward(lp, t, None, "sum")
    torch.cuda.synchronize()
    assert math.isnan(loss.item())


NLL_DRIVER = r"""
import os, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import gen, paper_2207_00257_b200 as L
out = sys.argv[1]
for k, (N, C, pad, red) in enumerate([(4099, 1000, 16, "none"), (65536, 4096, 0, "mean"), (513, 2056, 8, "sum")]):
    t = (gen.make_host(N, seed=k, dist="unit") * C).astype(np.int64)
    t[::7] = -100
    w = gen.make_host(C, seed=3, dist="unit") + np.float32(0.5)
    buf = torch.full((N, C + pad), 7.0, device="cuda")
    g = torch.from_numpy(gen.make_host(N, seed=11, dist="unit")).cuda() if red == "none" else torch.tensor([0.75], device="cuda")
    tw = torch.tensor([float(N)], device="cuda")
    L.nll_backward(g, (N, C), torch.from_numpy(t).cuda(), tw, torch.from_numpy(w).cuda(), red, grad=buf[:, :C])
    torch.cuda.synchronize()
    np.save(os.path.join(out, f"g{{k}}.npy"), buf.cpu().numpy())
print("ok")
"""


def test_nll_backward_kernels_agree_padded(tmp_path):
    """ClassNLL backward through the zero-fill + scatter pair (default) and the
    persistent row kernel (NORM_NLL_TILE=0): bit-identical gradients, padding
    columns untouched, and equal to the oracle's updateGradInput."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = NLL_DRIVER.format(root=root)
    outs = []
    for v in ("1", "0"):
        d = tmp_path / f"t{v}"
        d.mkdir()
        r = subprocess.run([sys.executable, "-c", code, str(d)], env=dict(os.environ, NORM_NLL_TILE=v),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
        outs.append(d)
    for k, (N, C, pad, red) in enumerate([(4099, 1000, 16, "none"), (65536, 4096, 0, "mean"), (513, 2056, 8, "sum")]):
        a, b = np.load(outs[0] / f"g{k}.npy"), np.load(outs[1] / f"g{k}.npy")
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), k
        assert np.all(a[:, C:] == 7.0), k
        t = (gen.make_host(N, seed=k, dist="unit") * C).astype(np.int64)
        t[::7] = -100
        w = gen.make_host(C, seed=3, dist="unit") + np.float32(0.5)
        g = gen.make_host(N, seed=11, dist="unit").astype(np.float64) if red == "none" else np.array([0.75])
        gref = oracle.nll_backward(g, t, C, w, red, -100, float(N))
        gv = a[:, :C].astype(np.float64)
        nz = gref != 0
        assert np.all(gv[~nz] == 0), k
        assert np.all(np.abs(gv[nz] - gref[nz]) <= 1e-6 * np.abs(gref[nz])), k
