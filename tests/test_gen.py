"""Input generator (gen/): determinism, offsets, value sets.  No method arithmetic."""
import numpy as np
import pytest

import gen


@pytest.mark.parametrize("dist", range(5))
def test_deterministic_and_offset(dist):
    a = gen.make_host(5000, seed=7, dist=dist)
    b = gen.make_host(5000, seed=7, dist=dist)
    assert a.tobytes() == b.tobytes()
    c = gen.make_host(1234, seed=7, dist=dist, offset=1000)
    assert c.tobytes() == a[1000:2234].tobytes()
    assert gen.value(7, dist, 4321) == a[4321]


def test_threaded_fill_matches_scalar():
    a = gen.make_host((1 << 20) + 13, seed=2207, dist="unit")  # threaded path
    idx = np.array([0, 1, 12345, (1 << 20) + 12])
    assert all(a[i] == gen.value(2207, "unit", int(i)) for i in idx)


def test_value_sets():
    u = gen.make_host(1 << 16, seed=1, dist="unit").astype(np.float64)
    k = u * 2.0**24
    assert np.all(k == np.floor(k)) and k.min() >= 1 and k.max() < 2**24
    s = gen.make_host(1 << 16, seed=1, dist="signed").astype(np.float64)
    k = s * 2.0**23
    assert np.all(k == np.floor(k)) and s.min() >= -1 and s.max() < 1 and (s < 0).any()
    w = gen.make_host(1 << 16, seed=1, dist="wide").astype(np.float64)
    assert w.min() >= 2.0**-32 and w.max() < 2.0**32
    r = gen.make_host(17, dist="ramp")
    assert list(r) == [1 + (i % 8) for i in range(17)]
    assert np.all(gen.make_host(9, dist="const") == 1.0)


def test_seeds_differ():
    assert gen.make_host(64, seed=0).tobytes() != gen.make_host(64, seed=1).tobytes()
