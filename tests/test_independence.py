"""The oracle and the CUDA path share no code (task rule ③): the product
package never imports `oracle` (or the input generator `gen`), libnorm.so does
not link liboracle / libnormgen, and the oracle's C source includes nothing
from the product tree."""
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2207_00257_b200")


def _sources(top, exts):
    for dp, _, fs in os.walk(top):
        for f in fs:
            if f.endswith(exts):
                yield os.path.join(dp, f)


def test_package_never_imports_oracle_or_gen():
    pat = re.compile(r"^\s*(from|import)\s+(oracle|gen)\b", re.M)
    for p in _sources(PKG, (".py",)):
        assert not pat.search(open(p).read()), p


def test_csrc_includes_nothing_from_oracle_or_gen():
    for p in _sources(os.path.join(PKG, "csrc"), (".cu", ".cuh", ".cpp", ".h")):
        src = open(p).read()
        assert "oracle" not in re.findall(r'#include\s+"([^"]+)"', src).__str__(), p
        assert "norm_gen" not in src, p


def test_oracle_includes_nothing_from_the_product():
    src = open(os.path.join(ROOT, "oracle", "norm_oracle.c")).read()
    for inc in re.findall(r'#include\s+[<"]([^>"]+)[>"]', src):
        assert not inc.startswith(("libnorm", "norm_internal", "device_common", "stream_common")), inc


def test_libnorm_does_not_link_the_oracle():
    so = os.path.join(PKG, "libnorm.so")
    out = subprocess.run(["readelf", "-d", so], capture_output=True, text=True).stdout
    needed = re.findall(r"\(NEEDED\).*\[(.+?)\]", out)
    assert needed, out[:500]
    assert not any("oracle" in n or "normgen" in n for n in needed), needed
    syms = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    assert "oracle_" not in syms


def test_bench_runs_the_oracle_only_in_its_cpu_legs():
    """bench.py may execute oracle/ only in the cpu_baseline leg (which also takes
    the parity record, after every GPU measurement) and the --impl reference arm:
    every function that imports it is one of those, and the GPU arms call the
    parity check only from inside a `not args.no_cpu` block."""
    import ast
    src = open(os.path.join(ROOT, "bench.py")).read()
    tree = ast.parse(src)
    importers = set()
    for fn in ast.walk(tree):
        if isinstance(fn, ast.FunctionDef):
            for node in ast.walk(fn):
                if isinstance(node, ast.Import) and any(a.name == "oracle" for a in node.names):
                    importers.add(fn.name)
    # oracle_bytes / oracle_sample / parity_record: the cpu_baseline leg's helpers;
    # run_reference: the reference arm; run_small / run_licm: their lines' cpu legs
    assert importers <= {"oracle_bytes", "oracle_sample", "parity_record", "run_reference", "run_small",
                         "run_licm"}, importers
    # the module itself never imports it at top level
    assert not any(isinstance(n, ast.Import) and any(a.name == "oracle" for a in n.names) for n in tree.body)
    # parity_record is called only under `if ... not args.no_cpu:`
    calls = [m.start() for m in re.finditer(r"(?<!def )parity_record\(L,", src)]
    assert calls
    for c in calls:
        block = src[:c].rsplit("\n    if ", 1)[-1]
        assert "not args.no_cpu" in block.split("\n")[0], block.split("\n")[0]
