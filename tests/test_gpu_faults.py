"""Fault injection: libnorm rebuilt with one
deliberate mistake at a time (Makefile target `faults`, -DNORM_FAULT=k) must
fail the parity checks, and the product build must pass them:
  1: the sum drops the last element        2: dense index instead of Fig. 1's
  3: approximate (non-IEEE) division       7: covered prefix off by one."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
FAULT_DIR = os.path.join(ROOT, "paper_2207_00257_b200", "faults")


def run_checker(so):
    env = dict(os.environ)
    if so:
        env["LIBNORM_SO"] = so
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "fault_checker.py")],
                       capture_output=True, text=True, env=env, timeout=600)
    return r.returncode, r.stdout + r.stderr


def test_product_build_passes_checker():
    rc, out = run_checker(None)
    assert rc == 0, out


@pytest.mark.parametrize("fault", [1, 2, 3, 7])
def test_fault_is_caught(fault):
    r = subprocess.run(["make", "-s", "-C", ROOT, "-j4", "faults"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rc, out = run_checker(os.path.join(FAULT_DIR, f"libnorm_fault{fault}.so"))
    assert rc == 1, f"fault {fault} was not detected:\n{out}"
