"""Pins for the NEXT-4 backprop oracle (Fig. backprop)."""
import json
import os

import numpy as np
import pytest

import gen
import oracle
from conftest import GOLDEN


def golden():
    with open(os.path.join(GOLDEN, "backprop_fixture.json")) as f:
        return json.load(f)


def test_all_ones_closed_form():
    g = golden()["all_ones"]
    n_in = 64
    hw0 = np.ones((n_in + 1, 17), np.float32)
    hw, out = oracle.bpnn_layerforward(np.ones(n_in + 1, np.float32), hw0)
    assert np.all(out == g["output"])
    for by in range(n_in // 16):
        rows = hw[16 * by + 1:16 * by + 17, 1:]
        assert np.all(rows == np.array(g["hidden_rows_after_tree"], np.float32)[:, None])
    assert np.all(hw[0] == 1) and np.all(hw[:, 0] == 1)  # bias row / column untouched


def test_integer_inputs_exact():
    # small integers: every product and partial sum is exact in fp32, so the
    # output is the exact column dot product, computed here with Python ints
    rng = np.random.default_rng(3)
    n_in = 160
    x = rng.integers(-7, 8, n_in + 1).astype(np.float32)
    w = rng.integers(-9, 10, (n_in + 1, 17)).astype(np.float32)
    hw, out = oracle.bpnn_layerforward(x, w)
    for by in range(n_in // 16):
        for c in range(16):
            exact = sum(int(x[16 * by + t + 1]) * int(w[16 * by + t + 1, c + 1]) for t in range(16))
            assert out[16 * by + c] == exact
            # row tz-partial sums in the written-back weights
            for t in range(16):
                tz = 4 if t == 0 else min((t & -t).bit_length() - 1, 4)
                part = sum(int(x[16 * by + k + 1]) * int(w[16 * by + k + 1, c + 1]) for k in range(t, t + 2**tz))
                assert hw[16 * by + t + 1, c + 1] == part


def test_tree_order_golden():
    g = golden()["tree_order"]
    w = np.zeros((17, 17), np.float32)
    w[1:, 1] = np.array(g["column"], np.float32)
    hw, out = oracle.bpnn_layerforward(np.full(17, g["node"], np.float32), w)
    assert out[0] == g["output"]


def test_rejects_bad_shapes():
    with pytest.raises(ValueError):
        oracle.bpnn_layerforward(np.ones(18, np.float32), np.ones((18, 17), np.float32))
