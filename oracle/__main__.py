"""JSON command line for the CPU oracle (TEST INFRASTRUCTURE ONLY).

I/O shape borrowed from SPEC.md:565: {"scalars": {...}, "buffers": {...}}.

  python -m oracle '{"scalars": {}, "buffers": {"in": [1,2,3,4,5,6,7,8]}}' --form hoisted --index dense
  -> {"scalars": {"n": 8, "sum": 36.0, "adds": 8, "covered": 8, "prefix_len": 8},
      "buffers": {"out": [0.0277..., ...]}}

Uncovered outputs are reported as null (untouched by the kernel).  Exit codes:
0 ok, 1 bad input, 2 usage.
"""
import argparse
import json
import sys

import numpy as np

from . import coverage_closed, covered_mask, form_block, form_hoisted, form_thread, sum_exact


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m oracle")
    ap.add_argument("input", help="JSON object {scalars, buffers: {in: [...]}} or @file")
    ap.add_argument("--form", choices=["thread", "block", "hoisted"], default="hoisted")
    ap.add_argument("--index", choices=["literal", "dense"], default="literal")
    args = ap.parse_args(argv)
    try:
        text = open(args.input[1:]).read() if args.input.startswith("@") else args.input
        doc = json.loads(text)
        x = np.asarray(doc["buffers"]["in"], dtype=np.float32)
    except (OSError, ValueError, KeyError, TypeError) as e:
        print(json.dumps({"error": str(e)}))
        return 1
    sentinel = np.full(x.size, np.nan, dtype=np.float32)
    fn = {"thread": form_thread, "block": form_block, "hoisted": form_hoisted}[args.form]
    out, adds = fn(x, args.index, out=sentinel)
    count, prefix = coverage_closed(x.size, args.index)
    res = {"scalars": {"n": int(x.size), "sum": sum_exact(x), "adds": int(adds),
                       "covered": int(count), "prefix_len": int(prefix)},
           "buffers": {"out": [float(v) if c else None
                               for v, c in zip(out, covered_mask(x.size, args.index))]}}
    print(json.dumps(res))
    return 0


if __name__ == "__main__":
    sys.exit(main())
