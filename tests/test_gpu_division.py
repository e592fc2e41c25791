"""libnorm's uniform-divisor division (three FFMAs per element with the refined
reciprocal hoisted) must be bit-identical to __fdiv_rn (IEEE binary32 RN,
reading R13) for ALL 2^32 dividends; checked exhaustively for 28 special and
300 pseudo-random divisors (scripts/verify_division.cu; the full sweep in
profiles/ covers thousands more)."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_division_bit_identical_to_fdiv_rn():
    r = subprocess.run(["make", "-s", "-C", ROOT, "scripts/verify_division"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([os.path.join(ROOT, "scripts", "verify_division"), "300", "7"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches: 0" in r.stdout
