"""The C ABI used from plain C (examples/normalize_c.c): no Python in the loop."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_c_example_runs():
    r = subprocess.run(["make", "-s", "-C", ROOT, "examples"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    for n in ("7", "1048583", "33554437"):
        r = subprocess.run([os.path.join(ROOT, "examples", "normalize_c"), n], capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
