"""Runs a compact version of the GPU parity checks against whatever libnorm.so
LIBNORM_SO points at; exit 0 = all checks pass, 1 = some check failed.
Used by tests/test_gpu_faults.py (fault-injection sensitivity)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2207_00257_b200 as L  # noqa: E402

SENT = 0x7FC0FFEE


def one(n, mode, path, dist):
    x = gen.make_host(n, seed=n + 3, dist=dist)
    inp = torch.from_numpy(x).cuda()
    out = torch.from_numpy(np.full(n, SENT, np.uint32).view(np.float32)).cuda()
    s = torch.zeros(1, device="cuda")
    L.normalize(out, inp, index=mode, path=path, sum_out=s)
    torch.cuda.synchronize()
    o, sv = out.cpu().numpy(), np.float32(s.item())
    S = oracle.sum_exact(x)
    assert abs(float(sv) - S) <= 1e-6 * abs(S), "sum"
    rep = oracle.replay(x, sv, mode, out=np.full(n, SENT, np.uint32).view(np.float32))
    assert o.view(np.uint32).tobytes() == rep.view(np.uint32).tobytes(), "replay/coverage"
    ref = oracle.normalize(x, mode, out=np.full(n, SENT, np.uint32).view(np.float32))
    cov = oracle.covered_mask(n, mode)
    assert np.all(np.abs(o[cov].astype(np.float64) - ref[cov]) <= 1e-5 * np.abs(ref[cov])), "tolerance"


def main():
    failures = []
    for n in (7, 100, 1025, 2**20 + 7):
        for mode in ("literal", "dense"):
            for path in ("auto", "two_pass"):
                try:
                    one(n, mode, path, 0 if n > 100 else 2)
                except AssertionError as e:
                    failures.append(f"n={n} {mode} {path}: {e}")
    print("\n".join(failures) if failures else "all checks pass")
    sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
