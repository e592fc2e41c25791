"""GPU parity of the gradient kernels (csrc/backward.cu, through the C ABI)
against the oracle's fp64 gradients (oracle_normalize_backward,
oracle_softmax_backward_rows; pinned in tests/test_oracle_backward.py).

Each gradient is a difference of two terms evaluated in fp32 from an fp64 sum
(gx = a - b): the bound per element is 1e-5 (|a| + |b|) with a, b the oracle's
fp64 terms -- a few fp32 roundings of each term, no cancellation credit.  The
reductions run in a fixed order, so results are also checked bitwise run to run
and in place (gx aliasing g) against out of place."""
import numpy as np
import pytest
import torch

import gen
import oracle
import paper_2207_00257_b200 as L

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _forward_normalize(x, mode):
    y = x.clone()
    s = torch.zeros(1, device="cuda")
    L.normalize(y, y, index=mode, sum_out=s)
    return y, s


def _check_normalize(gx, g, y, s, mode):
    g64, y64, S = g.astype(np.float64), y.astype(np.float64), float(s)
    ref = oracle.normalize_backward(g64, y64, S, mode)
    cov = oracle.covered_mask(g.size, mode)
    a = np.where(cov, g64 / S, g64)
    D = float(np.dot(g64[cov], y64[cov]) / S)
    err = np.abs(gx.astype(np.float64) - ref)
    bound = TOL * (np.abs(a) + abs(D)) + 1e-37
    assert np.all(err <= bound), (mode, g.size, float((err / bound).max()))


@pytest.mark.parametrize("mode", ["literal", "dense"])
def test_normalize_backward_parity(mode):
    for i, n in enumerate([1, 5, 33, 100, 993, 1024, 2000, 4099, 2**20 + 7, 2**24 + 3]):
        x = torch.from_numpy(gen.make_host(n, seed=40 + i, dist="unit")).cuda()
        g = torch.from_numpy(gen.make_host(n, seed=80 + i, dist="signed")).cuda()
        y, s = _forward_normalize(x, mode)
        gx = torch.empty_like(g)
        L.normalize_backward(gx, g, y, s, index=mode)
        gx2 = torch.empty_like(g)
        L.normalize_backward(gx2, g, y, s, index=mode)
        gin = g.clone()
        L.normalize_backward(gin, gin, y, s, index=mode)  # in place over g
        torch.cuda.synchronize()
        assert torch.equal(gx, gx2) and torch.equal(gx, gin), (mode, n)
        _check_normalize(gx.cpu().numpy(), g.cpu().numpy(), y.cpu().numpy(), s.item(), mode)


def test_normalize_backward_misaligned_views():
    """Scalar (unaligned) path: views at float offsets 1 and 3."""
    n = 70001
    base = torch.from_numpy(gen.make_host(n + 8, seed=5, dist="unit")).cuda()
    gb = torch.from_numpy(gen.make_host(n + 8, seed=6, dist="signed")).cuda()
    for off, mode in ((1, "dense"), (3, "literal")):
        x, g = base[off:off + n].clone(), gb[off:off + n]
        y, s = _forward_normalize(x, mode)
        gx = torch.empty(n + 8, device="cuda")[off:off + n]
        L.normalize_backward(gx, g, y, s, index=mode)
        torch.cuda.synchronize()
        _check_normalize(gx.cpu().numpy(), g.cpu().numpy(), y.cpu().numpy(), s.item(), mode)


@pytest.mark.parametrize("mode", ["literal", "dense"])
@pytest.mark.parametrize("shape", [(300, 2048), (17, 1000), (5, 4097), (64, 4096)])
def test_rows_normalize_backward_parity(mode, shape):
    R, C = shape
    x = torch.from_numpy(gen.make_host(R * C, seed=R, dist="unit")).cuda().view(R, C)
    g = torch.from_numpy(gen.make_host(R * C, seed=C, dist="signed")).cuda().view(R, C)
    y = x.clone()
    s = torch.zeros(R, device="cuda")
    L.normalize_rows(y, y, index=mode, sum_out=s)
    gx = torch.empty_like(g)
    L.normalize_rows_backward(gx, g, y, s, index=mode)
    torch.cuda.synchronize()
    gh, yh, sh, out = g.cpu().numpy(), y.cpu().numpy(), s.cpu().numpy(), gx.cpu().numpy()
    for r in range(R):
        _check_normalize(out[r], gh[r], yh[r], sh[r], mode)


@pytest.mark.parametrize("log", [False, True])
@pytest.mark.parametrize("shape", [(64, 4096), (300, 1000), (7, 33), (3, 8195)])
def test_softmax_backward_parity(log, shape):
    R, C = shape
    x = torch.from_numpy(gen.make_host(R * C, seed=R + C, dist="signed")).cuda().view(R, C) * 8
    g = torch.from_numpy(gen.make_host(R * C, seed=R * C, dist="signed")).cuda().view(R, C)
    y = torch.empty_like(x)
    L.softmax_rows(y, x, log=log)
    gx = torch.empty_like(g)
    L.softmax_rows_backward(gx, g, y, log=log)
    gin = g.clone()
    L.softmax_rows_backward(gin, gin, y, log=log)
    torch.cuda.synchronize()
    assert torch.equal(gx, gin)
    g64, y64 = g.double().cpu().numpy(), y.double().cpu().numpy()
    ref = oracle.softmax_backward_rows(g64, y64, log=log)
    if log:
        D = g64.sum(1, keepdims=True)
        bound = TOL * (np.abs(g64) + np.exp(y64) * np.abs(D))
    else:
        D = (g64 * y64).sum(1, keepdims=True)
        bound = TOL * np.abs(y64) * (np.abs(g64) + np.abs(D))
    err = np.abs(gx.double().cpu().numpy() - ref)
    assert np.all(err <= bound + 1e-37), float((err / (bound + 1e-37)).max())


def test_softmax_backward_bench_shape_sampled():
    """65536 x 4096 (the bench shape): 128 sampled rows against the oracle, and the
    whole gradient bitwise equal over two runs."""
    R, C = 65536, 4096
    x = torch.empty(R * C, device="cuda")
    gen.fill_cuda(x, seed=2207, dist="signed")
    g = torch.empty_like(x)
    gen.fill_cuda(g, seed=2208, dist="signed")
    x, g = x.view(R, C), g.view(R, C)
    y = torch.empty_like(x)
    L.softmax_rows(y, x)
    gx, gx2 = torch.empty_like(g), torch.empty_like(g)
    L.softmax_rows_backward(gx, g, y)
    L.softmax_rows_backward(gx2, g, y)
    torch.cuda.synchronize()
    assert torch.equal(gx, gx2)
    rows = np.random.default_rng(9).integers(0, R, 128)
    idx = torch.from_numpy(rows).cuda()
    g64, y64 = g[idx].double().cpu().numpy(), y[idx].double().cpu().numpy()
    ref = oracle.softmax_backward_rows(g64, y64)
    D = (g64 * y64).sum(1, keepdims=True)
    bound = TOL * np.abs(y64) * (np.abs(g64) + np.abs(D)) + 1e-37
    assert np.all(np.abs(gx[idx].double().cpu().numpy() - ref) <= bound)


def test_autograd_through_the_torch_ops():
    """torch autograd of the libnorm ops calls the gradient kernels: x.grad equals the
    oracle's gradient at the op's own (y, s)."""
    import paper_2207_00257_b200.torch_ops as T
    for mode in ("dense", "literal"):
        x = torch.from_numpy(gen.make_host(5000, seed=1, dist="unit")).cuda().requires_grad_()
        w = torch.from_numpy(gen.make_host(5000, seed=2, dist="signed")).cuda()
        y, s = torch.ops.libnorm.normalize_fwd(x, mode)
        (y * w).sum().backward()
        _check_normalize(x.grad.cpu().numpy(), w.cpu().numpy(), y.detach().cpu().numpy(), s.item(), mode)
    # rows, through the nn.Module
    xr = torch.from_numpy(gen.make_host(8 * 300, seed=3, dist="unit")).cuda().view(8, 300).requires_grad_()
    wr = torch.from_numpy(gen.make_host(8 * 300, seed=4, dist="signed")).cuda().view(8, 300)
    yr = T.Normalize("dense")(xr)
    (yr * wr).sum().backward()
    sr = xr.detach().double().sum(1).float().cpu().numpy()
    for r in range(8):
        ref = oracle.normalize_backward(wr[r].double().cpu().numpy(), yr[r].detach().double().cpu().numpy(),
                                        float(sr[r]), "dense")
        assert np.allclose(xr.grad[r].double().cpu().numpy(), ref, rtol=1e-4, atol=1e-9)
    # softmax and log-softmax
    for log in (False, True):
        z = (torch.from_numpy(gen.make_host(16 * 512, seed=5, dist="signed")).cuda().view(16, 512) * 4)
        z.requires_grad_()
        v = torch.from_numpy(gen.make_host(16 * 512, seed=6, dist="signed")).cuda().view(16, 512)
        out = torch.ops.libnorm.softmax(z, log)
        (out * v).sum().backward()
        ref = oracle.softmax_backward_rows(v.double().cpu().numpy(), out.detach().double().cpu().numpy(), log=log)
        assert np.allclose(z.grad.double().cpu().numpy(), ref, rtol=1e-4, atol=1e-7), log


def test_backward_argument_errors():
    g = torch.ones(64, device="cuda")
    s = torch.ones(1, device="cuda")
    with pytest.raises(L.NormError):  # partial overlap of gx with g
        big = torch.ones(80, device="cuda")
        L.normalize_backward(big[8:72], big[:64], g, s)
    with pytest.raises(ValueError):
        L.normalize_backward(torch.empty(63, device="cuda"), g, g, s)
    e = torch.empty(0, device="cuda")
    L.normalize_backward(e, e, e, s)  # n == 0: no-op
    torch.cuda.synchronize()


def test_backward_writes_stay_in_bounds():
    """compute-sanitizer is unavailable on this pool: guard regions instead.  gx is a
    view inside a sentinel-filled buffer (64 floats of guard on each side, offsets
    0..3 floats); every gradient entry writes exactly gx and leaves the guards."""
    SENT = 0x7FC0FFEE

    def guarded(n, off):
        buf = torch.empty(n + 128 + 4, dtype=torch.int32, device="cuda").fill_(SENT).view(torch.float32)
        return buf, buf[64 + off:64 + off + n]

    def guards_ok(buf, n, off):
        b = buf.view(torch.int32)
        return bool(torch.all(b[:64 + off] == SENT)) and bool(torch.all(b[64 + off + n:] == SENT))

    for n in (1, 3, 5, 31, 1000, 4099, 70001):
        for off in (0, 1, 3):
            for mode in ("literal", "dense"):
                x = torch.rand(n, device="cuda") + 0.1
                g = torch.randn(n, device="cuda")
                y, s = _forward_normalize(x, mode)
                buf, gx = guarded(n, off)
                L.normalize_backward(gx, g, y, s, index=mode)
                torch.cuda.synchronize()
                assert guards_ok(buf, n, off), (n, off, mode)
                assert not torch.any(gx.view(torch.int32) == SENT)
    for (R, C) in ((7, 1001), (3, 4099), (64, 4096)):
        x = torch.rand(R, C, device="cuda") + 0.1
        g = torch.randn(R, C, device="cuda")
        for kind in ("normalize", "softmax", "log_softmax"):
            buf, gxf = guarded(R * C, 0)
            gx = gxf.view(R, C)
            if kind == "normalize":
                y = x.clone()
                s = torch.zeros(R, device="cuda")
                L.normalize_rows(y, y, index="literal", sum_out=s)
                L.normalize_rows_backward(gx, g, y, s, index="literal")
            else:
                y = torch.empty_like(x)
                L.softmax_rows(y, x, log=kind == "log_softmax")
                L.softmax_rows_backward(gx, g, y, log=kind == "log_softmax")
            torch.cuda.synchronize()
            assert guards_ok(buf, R * C, 0), (R, C, kind)
            assert not torch.any(gx.reshape(-1).view(torch.int32) == SENT)


def test_autograd_under_torch_compile():
    """The differentiable ops trace under torch.compile(fullgraph=True) (fake kernels
    for the forward and the backward ops) and give the eager gradients bit for bit."""
    import paper_2207_00257_b200.torch_ops  # noqa: F401  (registers the ops)

    def f(x, w):
        y, s = torch.ops.libnorm.normalize_fwd(x, "literal")
        return (y * w).sum() + torch.ops.libnorm.softmax(x.view(8, -1), True).sum()

    cf = torch.compile(f, fullgraph=True)
    base = torch.from_numpy(gen.make_host(8 * 512, seed=12, dist="unit")).cuda()
    w = torch.from_numpy(gen.make_host(8 * 512, seed=13, dist="signed")).cuda()
    x1 = base.clone().requires_grad_()
    cf(x1, w).backward()
    x2 = base.clone().requires_grad_()
    f(x2, w).backward()
    torch.cuda.synchronize()
    assert torch.equal(x1.grad, x2.grad)
