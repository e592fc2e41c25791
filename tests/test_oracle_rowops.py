"""Pins for the NEXT-2 oracle functions (row softmax / log-softmax, ClassNLL),
against independent library implementations (torch fp64 on CPU), closed forms
and invariants — never against the oracle itself."""
import math
from fractions import Fraction

import numpy as np
import pytest
import torch

import gen
import oracle


def logits(R, C, seed, scale=4.0):
    x = gen.make_host(R * C, seed=seed, dist="signed").reshape(R, C) * np.float32(scale)
    return x.astype(np.float32)


@pytest.mark.parametrize("R,C,scale", [(5, 1, 1.0), (7, 33, 4.0), (3, 4096, 8.0), (2, 1000, 80.0)])
def test_softmax_matches_torch_fp64(R, C, scale):
    x = logits(R, C, seed=C, scale=scale)
    ref = torch.softmax(torch.from_numpy(x).double(), dim=1).float().numpy()
    out = oracle.softmax_rows(x)
    np.testing.assert_allclose(out, ref, rtol=2e-7, atol=1e-38)
    lref = torch.log_softmax(torch.from_numpy(x).double(), dim=1).float().numpy()
    np.testing.assert_allclose(oracle.softmax_rows(x, log=True), lref, rtol=2e-7, atol=1e-6)


def test_softmax_closed_forms_and_invariants():
    for C in (1, 2, 3, 64, 1000, 4096):
        u = oracle.softmax_rows(np.full((2, C), 3.25, np.float32))
        assert np.all(u == np.float32(float(Fraction(1, C))))  # uniform row -> 1/C
    x = gen.make_host(4 * 512, seed=1, dist="signed").reshape(4, 512) * 8
    x = (np.round(x * 2.0**12) / 2.0**12).astype(np.float32)  # 2^-12 grid: x + 16 is exact
    sh = (x + np.float32(16.0)).astype(np.float32)
    assert np.array_equal((sh - np.float32(16.0)), x)
    assert np.array_equal(oracle.softmax_rows(sh), oracle.softmax_rows(x))
    y = oracle.softmax_rows(x)
    for r in range(4):
        assert abs(math.fsum(y[r].astype(np.float64)) - 1.0) <= 512 * 2.0**-24
        order = np.argsort(x[r], kind="stable")
        assert np.all(np.diff(y[r][order]) >= 0)  # monotone in the logit
    ly = oracle.softmax_rows(x, log=True)
    np.testing.assert_allclose(np.exp(ly.astype(np.float64)), y, rtol=1e-6)


def test_softmax_nonfinite():
    x = np.array([[0.0, -np.inf, 1.0], [np.nan, 0, 0], [-np.inf] * 3], np.float32)
    y = oracle.softmax_rows(x)
    t = torch.softmax(torch.from_numpy(x).double(), 1).float().numpy()
    assert y[0, 1] == 0 and np.isclose(y[0, 0] + y[0, 2], 1)
    assert np.all(np.isnan(y[1])) and np.all(np.isnan(t[1]))
    assert np.all(np.isnan(y[2])) and np.all(np.isnan(t[2]))


@pytest.mark.parametrize("reduction", ["none", "mean", "sum"])
@pytest.mark.parametrize("weighted", [False, True])
def test_nll_matches_torch_fp64(reduction, weighted):
    N, C = 300, 37
    lp = torch.log_softmax(torch.from_numpy(logits(N, C, seed=3)).double(), 1).float().numpy()
    t = (gen.make_host(N, seed=4, dist="unit") * C).astype(np.int64)
    t[::17] = -100  # ignored
    w = gen.make_host(C, seed=5, dist="unit") + np.float32(0.5) if weighted else None
    loss, tw = oracle.nll_forward(lp, t, w, reduction)
    ref = torch.nn.functional.nll_loss(torch.from_numpy(lp).double(), torch.from_numpy(t),
                                       weight=None if w is None else torch.from_numpy(w).double(),
                                       reduction=reduction, ignore_index=-100)
    np.testing.assert_allclose(loss, ref.numpy(), rtol=1e-12)
    valid = t != -100
    assert tw == pytest.approx(float(w[t[valid]].astype(np.float64).sum()) if weighted else valid.sum(), rel=1e-12)
    # backward: autograd of torch's fp64 nll_loss
    inp = torch.from_numpy(lp).double().requires_grad_()
    out = torch.nn.functional.nll_loss(inp, torch.from_numpy(t),
                                       weight=None if w is None else torch.from_numpy(w).double(),
                                       reduction=reduction, ignore_index=-100)
    g = torch.from_numpy(gen.make_host(N, seed=6, dist="unit").astype(np.float64)) if reduction == "none" \
        else torch.tensor(0.75, dtype=torch.float64)
    out.backward(g)
    grad = oracle.nll_backward(g.numpy(), t, C, w, reduction, -100, tw)
    np.testing.assert_allclose(grad, inp.grad.numpy(), rtol=1e-12, atol=0)


def test_nll_closed_form_and_edges():
    N, C = 64, 10
    lp = np.zeros((N, C), np.float32)
    t = np.arange(N) % C
    k = (np.arange(N) % 7 + 1).astype(np.float32)
    lp[np.arange(N), t] = -k  # loss_i = k_i exactly
    loss, tw = oracle.nll_forward(lp, t, None, "mean")
    assert loss == float(Fraction(int(k.sum()), N)) and tw == N
    assert oracle.nll_forward(lp, t, None, "sum")[0] == float(k.sum())
    all_ign = np.full(N, -100)
    assert math.isnan(oracle.nll_forward(lp, all_ign, None, "mean")[0])
    bad = t.copy()
    bad[3] = C  # out of range, not ignored (reading R17)
    assert math.isnan(oracle.nll_forward(lp, bad, None, "sum")[0])
