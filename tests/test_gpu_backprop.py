"""GPU parity for NEXT-4 (Rodinia bpnn_layerforward, Fig. backprop): all four
variants bitwise equal to the fp32 step-by-step oracle (same products, same tree
order), in place on `hidden`, bias row/column untouched."""
import numpy as np
import pytest
import torch

import gen
import oracle
import paper_2207_00257_b200 as L

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("variant", ["printed", "eliminated", "register", "tma"])
@pytest.mark.parametrize("n_in", [16, 32, 64, 16 * 31, 16 * 61, 65536, 16 * 70001])
def test_bpnn_parity(variant, n_in):
    x = (gen.make_host(n_in + 1, seed=n_in, dist="signed")).astype(np.float32)
    w = (gen.make_host((n_in + 1) * 17, seed=n_in + 1, dist="wide").reshape(n_in + 1, 17) *
         np.where(gen.make_host((n_in + 1) * 17, seed=3, dist="unit").reshape(n_in + 1, 17) < 0.5, -1, 1)
         ).astype(np.float32)
    hw_ref, out_ref = oracle.bpnn_layerforward(x, w)
    xi = torch.from_numpy(x).cuda()
    hd = torch.from_numpy(w.copy()).cuda()
    od = torch.full((n_in,), -3.0, device="cuda")
    L.bpnn_layerforward(xi, hd, od, variant=variant)
    torch.cuda.synchronize()
    assert od.cpu().numpy().tobytes() == out_ref.tobytes()
    assert hd.cpu().numpy().tobytes() == hw_ref.tobytes()


def test_bpnn_variants_agree_and_reject():
    n_in = 4096
    x = torch.from_numpy(gen.make_host(n_in + 1, seed=1, dist="unit")).cuda()
    w0 = torch.from_numpy(gen.make_host((n_in + 1) * 17, seed=2, dist="unit").reshape(n_in + 1, 17)).cuda()
    res = []
    for v in ("printed", "eliminated", "register", "tma"):
        h = w0.clone()
        o = torch.empty(n_in, device="cuda")
        L.bpnn_layerforward(x, h, o, variant=v)
        res.append((h, o))
    torch.cuda.synchronize()
    for h, o in res[1:]:
        assert torch.equal(h, res[0][0]) and torch.equal(o, res[0][1])
    with pytest.raises(L.NormError):
        L.bpnn_layerforward(x[:18], torch.zeros(18, 17, device="cuda"), torch.zeros(17, device="cuda"))


def test_bpnn_bench_size_tma():
    """The bench's launch configuration (in = 2^22, hid = 16, TMA form, run queue
    over 148 x 2 CTAs): bitwise equal to the fp32 step-by-step oracle, twice in a
    row (the queue counter resets itself between calls)."""
    n_in = 2**22
    x = gen.make_host(n_in + 1, seed=22, dist="signed")
    w = gen.make_host((n_in + 1) * 17, seed=23, dist="unit").reshape(n_in + 1, 17)
    hw_ref, out_ref = oracle.bpnn_layerforward(x, w)
    xi = torch.from_numpy(x).cuda()
    for _ in range(2):
        hd = torch.from_numpy(w.copy()).cuda()
        od = torch.full((n_in,), -3.0, device="cuda")
        L.bpnn_layerforward(xi, hd, od, variant="tma")
        torch.cuda.synchronize()
        assert od.cpu().numpy().tobytes() == out_ref.tobytes()
        assert hd.cpu().numpy().tobytes() == hw_ref.tobytes()
