import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")
    # Build (no-op when up to date): the oracle, the generator and libnorm.
    r = subprocess.run(["make", "-s", "-C", ROOT] + os.environ.get("NORM_MAKE_TARGETS", "all").split(), capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("make failed:\n" + r.stdout + r.stderr)


_GPU = None


def _has_gpu():
    """True on a box with a visible NVIDIA GPU.  A fresh box can briefly refuse
    CUDA initialisation right after it is handed over, and the CUDA runtime
    caches that failure for the life of the process, so availability is probed
    in subprocesses (up to ~90 s) before this process touches CUDA; if nvidia-smi
    sees a GPU, the GPU tests run (and fail loudly) rather than being skipped."""
    global _GPU
    if _GPU is not None:
        return _GPU
    try:
        smi = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=60)
        visible = smi.returncode == 0 and "GPU" in smi.stdout
    except Exception:
        visible = False
    if not visible:
        _GPU = False
        return _GPU
    import time
    probe = [sys.executable, "-c", "import torch, sys; sys.exit(0 if torch.cuda.is_available() else 1)"]
    deadline = time.time() + 90
    while time.time() < deadline:
        if subprocess.run(probe, capture_output=True).returncode == 0:
            break
        time.sleep(5)
    _GPU = True
    return _GPU


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
