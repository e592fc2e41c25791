"""Pins of the oracle's gradients (oracle_normalize_backward,
oracle_softmax_backward_rows) against what the forward definitions fix, not
against their own formulas:
  * central finite differences of the forward maps written out in fp64
    (normalize: covered y_i = x_i / sum x, uncovered y_j = x_j, PAPER.md:108-110;
    softmax / log-softmax: the textbook definitions), for both index modes,
    including the literal residue coverage (n <= 992) and a covered prefix;
  * invariants: y(c x) = y(x) for dense normalize, so sum_j gx_j x_j = 0; the
    softmax rows sum to 1, so sum_j gx_j = 0 (softmax and log-softmax);
  * a constant upstream gradient gives zero for dense normalize and softmax
    (the normalized sum / the softmax row sum is constant)."""
import numpy as np
import pytest

import oracle


def _normalize_f64(x, mode):
    cov = oracle.covered_mask(x.size, mode)
    return np.where(cov, x / x.sum(), x)


def _fd(f, x, g, h):
    gx = np.empty_like(x)
    for j in range(x.size):
        e = np.zeros_like(x)
        e[j] = h * max(1.0, abs(x[j]))
        gx[j] = (g @ f(x + e) - g @ f(x - e)) / (2 * e[j])
    return gx


@pytest.mark.parametrize("mode,n", [("dense", 37), ("dense", 300), ("literal", 100), ("literal", 993),
                                    ("literal", 1500)])
def test_normalize_backward_matches_finite_differences(mode, n):
    rng = np.random.default_rng(n)
    x = rng.random(n) + 0.25
    g = rng.standard_normal(n)
    S = x.sum()
    y = _normalize_f64(x, mode)
    gx = oracle.normalize_backward(g, y, S, mode)
    fd = _fd(lambda v: _normalize_f64(v, mode), x, g, 1e-6)
    assert np.allclose(gx, fd, rtol=1e-6, atol=1e-9 * np.abs(g).max()), np.abs(gx - fd).max()


@pytest.mark.parametrize("log", [False, True])
def test_softmax_backward_matches_finite_differences(log):
    rng = np.random.default_rng(7)
    x = rng.standard_normal((3, 50)) * 3

    def fwd(v):
        m = v.max()
        e = np.exp(v - m)
        return (v - m - np.log(e.sum())) if log else e / e.sum()
    g = rng.standard_normal((3, 50))
    y = np.stack([fwd(r) for r in x])
    gx = oracle.softmax_backward_rows(g, y, log=log)
    for r in range(3):
        fd = _fd(fwd, x[r], g[r], 1e-6)
        assert np.allclose(gx[r], fd, rtol=1e-6, atol=1e-8), np.abs(gx[r] - fd).max()


def test_invariants_and_constant_gradient():
    rng = np.random.default_rng(3)
    x = rng.random(4096) + 0.1
    S = x.sum()
    y = x / S
    g = rng.standard_normal(4096)
    gx = oracle.normalize_backward(g, y, S, "dense")
    assert abs(gx @ x) <= 1e-12 * np.abs(gx).max() * np.abs(x).sum()  # scale invariance
    assert np.abs(oracle.normalize_backward(np.full(4096, 2.5), y, S, "dense")).max() <= 1e-15
    z = rng.standard_normal((4, 256)) * 4
    sm = np.exp(z - z.max(1, keepdims=True))
    sm /= sm.sum(1, keepdims=True)
    lsm = np.log(sm)
    G = rng.standard_normal((4, 256))
    for log, yy in ((False, sm), (True, lsm)):
        gx = oracle.softmax_backward_rows(G, yy, log=log)
        assert np.abs(gx.sum(1)).max() <= 1e-12 * np.abs(G).sum(1).max()
        if not log:  # sum_j softmax_j = 1 is constant (sum_j log-softmax_j is not)
            assert np.abs(oracle.softmax_backward_rows(np.full_like(G, -1.5), yy, log=log)).max() <= 1e-14


def test_literal_uncovered_gradient_is_identity_minus_D():
    """n = 2000: C = [0, 1055); the uncovered outputs are the inputs themselves, so
    their gradient is g_j minus the shared S term (which every element carries)."""
    n = 2000
    rng = np.random.default_rng(11)
    x = rng.random(n) + 0.5
    S = x.sum()
    y = _normalize_f64(x, "literal")
    g = rng.standard_normal(n)
    gx = oracle.normalize_backward(g, y, S, "literal")
    _, L = oracle.coverage_closed(n, "literal")
    D = g[:L] @ (x[:L] / S) / S
    assert L == 1055
    assert np.allclose(gx[L:], g[L:] - D, rtol=0, atol=1e-15)
    assert np.allclose(gx[:L], g[:L] / S - D, rtol=1e-14, atol=1e-16)
