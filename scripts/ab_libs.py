"""Same-box A/B of two libnorm builds (probe): runs scripts/fused_vs_twopass.py
(or bench.py with the given args) under LIBNORM_SO=A and =B, alternating, and
prints both.  Usage: python scripts/ab_libs.py A.so B.so [reps] -- <cmd...>"""
import os
import subprocess
import sys

a, b = sys.argv[1], sys.argv[2]
rest = sys.argv[3:]
reps = 3
if rest and rest[0] != "--":
    reps = int(rest[0])
    rest = rest[1:]
cmd = rest[1:] if rest and rest[0] == "--" else [sys.executable, "scripts/fused_vs_twopass.py"]
for r in range(reps):
    for tag, so in (("A", a), ("B", b)):
        env = dict(os.environ, LIBNORM_SO=os.path.abspath(so))
        out = subprocess.run(cmd, env=env, capture_output=True, text=True).stdout
        for line in out.strip().splitlines():
            print(f"[{tag} rep{r}] {line}", flush=True)
