"""Randomised parity (fixed seed, 120 cases): random length (incl. ragged tails
around vector/chunk boundaries), index mode, path, distribution, in/out pointer
offsets, in-place, divisor outputs — each checked against the oracle with the
full bitwise replay (covered elements == in ⊘ s, uncovered == sentinel / input
bits) and the 1e-6 bound on s.  Rows get the same treatment with random
shapes, leading dimensions and offsets."""
import random

import numpy as np
import pytest
import torch

import gen
import oracle
import paper_2207_00257_b200 as L

pytestmark = pytest.mark.gpu
SENT = 0x7FC0FFEE


def _len(rng):
    kind = rng.random()
    if kind < 0.25:
        return rng.randrange(0, 2000)
    if kind < 0.5:  # around the 32 KiB / 48 KiB TMA chunks and 8-float vectors
        base = rng.choice([8192, 12288, 2**17, 2**20, 2**22])
        return base * rng.randrange(1, 4) + rng.randrange(-9, 10)
    return rng.randrange(2000, 3 * 2**21)


def test_vector_fuzz():
    rng = random.Random(2207)
    for case in range(120):
        n = max(0, _len(rng))
        mode = rng.choice(["literal", "dense"])
        path = rng.choice(["auto", "auto", "two_pass", "fused", "small", "mid", "cluster"]) if n <= 2**20 else \
            rng.choice(["auto", "two_pass", "fused", "mid", "cluster"])
        dist = rng.randrange(5)
        off_in, off_out = rng.randrange(8), rng.randrange(8)
        in_place = rng.random() < 0.2
        x = gen.make_host(n, seed=case, dist=dist)
        buf_in = torch.zeros(n + 8, device="cuda")
        inp = buf_in[off_in:off_in + n]
        inp.copy_(torch.from_numpy(x))
        if in_place:
            out = inp
            before = x
        else:
            buf_out = torch.empty(n + 8, dtype=torch.int32, device="cuda").fill_(SENT).view(torch.float32)
            out = buf_out[off_out:off_out + n]
            before = np.full(n, SENT, np.uint32).view(np.float32)
        s = torch.zeros(1, device="cuda")
        L.normalize(out, inp, index=mode, path=path, sum_out=s)
        torch.cuda.synchronize()
        if n == 0:
            continue
        o, sv = out.cpu().numpy(), np.float32(s.item())
        S = oracle.sum_exact(x)
        scale = oracle.sum_abs_exact(x) if dist == 3 else abs(S)
        ctx = (case, n, mode, path, dist, off_in, off_out, in_place)
        assert abs(float(sv) - S) <= 1e-6 * scale, ctx
        rep = oracle.replay(x, sv, mode, out=before.copy())
        assert o.view(np.uint32).tobytes() == rep.view(np.uint32).tobytes(), ctx


def test_rows_fuzz():
    rng = random.Random(7)
    for case in range(40):
        R = rng.randrange(1, 300)
        C = rng.choice([rng.randrange(1, 64), rng.randrange(256, 9000), 4096, 1024, 2048])
        ld = C + rng.choice([0, 0, 1, 3, 8, 17])
        mode = rng.choice(["literal", "dense"])
        off = rng.choice([0, 0, 4, 1])
        x = np.zeros((R, ld), np.float32)
        x[:, :C] = gen.make_host(R * C, seed=case, dist=rng.randrange(5)).reshape(R, C)
        flat_in = torch.zeros(R * ld + off, device="cuda")
        flat_in[off:].copy_(torch.from_numpy(x.reshape(-1)))
        inp = flat_in[off:].view(R, ld)[:, :C]
        flat_out = torch.empty(R * ld + off, dtype=torch.int32, device="cuda").fill_(SENT).view(torch.float32)
        out = flat_out[off:].view(R, ld)[:, :C]
        s = torch.zeros(R, device="cuda")
        L.normalize_rows(out, inp, index=mode, sum_out=s)
        torch.cuda.synchronize()
        o = flat_out[off:].view(R, ld).cpu().numpy()
        sv = s.cpu().numpy()
        for r in range(R):
            rep = oracle.replay(x[r, :C], sv[r], mode, out=np.full(C, SENT, np.uint32).view(np.float32))
            assert o[r, :C].view(np.uint32).tobytes() == rep.view(np.uint32).tobytes(), (case, R, C, ld, mode, r)
            S = oracle.sum_exact(x[r, :C])
            assert abs(float(sv[r]) - S) <= 1e-6 * max(abs(S), oracle.sum_abs_exact(x[r, :C])), (case, r)
        assert np.all(o[:, C:].view(np.uint32) == SENT)


def test_rows_fuzz_mixed_strides():
    """Rows whose input and output have different leading dimensions and
    different base offsets (so the two sides are not co-aligned and the kernel
    choice moves between the TMA, register and generic kernels): every row's
    divisor within 1e-6 of its exact sum (P20 for signed rows), every covered
    output the oracle's binary32 replay, everything else untouched."""
    rng = random.Random(11)
    for case in range(30):
        R = rng.randrange(1, 200)
        C = rng.choice([rng.randrange(1, 64), rng.randrange(256, 9000), 4096, 2048])
        ld_in = C + rng.choice([0, 1, 8, 24])
        ld_out = C + rng.choice([0, 3, 8, 40])
        off_in, off_out = rng.choice([0, 8, 1]), rng.choice([0, 8, 5])
        mode = rng.choice(["literal", "dense"])
        dist = rng.randrange(5)
        x = np.zeros((R, ld_in), np.float32)
        x[:, :C] = gen.make_host(R * C, seed=100 + case, dist=dist).reshape(R, C)
        flat_in = torch.zeros(R * ld_in + off_in, device="cuda")
        flat_in[off_in:].copy_(torch.from_numpy(x.reshape(-1)))
        inp = flat_in[off_in:].view(R, ld_in)[:, :C]
        flat_out = torch.empty(R * ld_out + off_out, dtype=torch.int32, device="cuda").fill_(SENT).view(torch.float32)
        out = flat_out[off_out:].view(R, ld_out)[:, :C]
        s = torch.zeros(R, device="cuda")
        L.normalize_rows(out, inp, index=mode, sum_out=s)
        torch.cuda.synchronize()
        o = flat_out.cpu().numpy()
        sv = s.cpu().numpy()
        assert np.all(o[:off_out].view(np.uint32) == SENT), case
        o = o[off_out:].reshape(R, ld_out)
        ctx = (case, R, C, ld_in, ld_out, off_in, off_out, mode)
        for r in range(R):
            rep = oracle.replay(x[r, :C], sv[r], mode, out=np.full(C, SENT, np.uint32).view(np.float32))
            assert o[r, :C].view(np.uint32).tobytes() == rep.view(np.uint32).tobytes(), ctx + (r,)
            S = oracle.sum_exact(x[r, :C])
            assert abs(float(sv[r]) - S) <= 1e-6 * max(abs(S), oracle.sum_abs_exact(x[r, :C])), ctx + (r,)
        assert np.all(o[:, C:].view(np.uint32) == SENT), ctx


def test_softmax_fuzz():
    """Row softmax / log-softmax over random shapes, leading
    dimensions, base offsets and in-place calls (vec, row-queue and generic
    kernels), against the oracle's fp64 rows with DESIGN.md §9's tolerances."""
    rng = random.Random(13)
    for case in range(30):
        R = rng.randrange(1, 300)
        C = rng.choice([rng.randrange(1, 64), rng.randrange(64, 9000), 4096, 1024])
        ld = C + rng.choice([0, 0, 8, 5])
        off = rng.choice([0, 8, 3])
        log = rng.random() < 0.5
        in_place = rng.random() < 0.25
        x = np.zeros((R, ld), np.float32)
        x[:, :C] = gen.make_host(R * C, seed=200 + case, dist="signed").reshape(R, C) * np.float32(rng.choice([1, 8, 30]))
        flat = torch.zeros(R * ld + off, device="cuda")
        flat[off:].copy_(torch.from_numpy(x.reshape(-1)))
        inp = flat[off:].view(R, ld)[:, :C]
        out = inp if in_place else torch.zeros(R, ld, device="cuda")[:, :C]
        L.softmax_rows(out, inp, log=log)
        torch.cuda.synchronize()
        got = out.cpu().numpy().astype(np.float64)
        ref = oracle.softmax_rows(np.ascontiguousarray(x[:, :C]), log=log).astype(np.float64)
        ctx = (case, R, C, ld, off, log, in_place)
        if log:
            assert np.all(np.abs(got - ref) <= 1e-5 * np.maximum(1.0, np.abs(ref))), ctx
        else:
            assert np.all(np.abs(got - ref) <= np.maximum(1e-5 * np.abs(ref), 1e-37)), ctx
