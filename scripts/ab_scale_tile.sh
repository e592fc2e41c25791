#!/bin/bash
# Same-box A/B of the co-aligned scale kernel (NORM_SCALE_KERNEL=tile | bulk | grid):
# dense two-pass step / reduce / scale split at 2^28, 2^30, 2^32; the literal 2^32
# headline bench line; and the two-pass path at L2-sized n (graph replays).
for r in 1 2; do
  for k in tile bulk; do
    NORM_SCALE_KERNEL=$k python scripts/dense_split.py 28 30 32 | sed "s/^/[$k rep$r] /"
  done
done
for r in 1 2 3; do
  for k in tile bulk; do
    v=$(NORM_SCALE_KERNEL=$k python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --no-parity 2>/dev/null | tail -1 |
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), 'ms', round(d['value'],1), 'GB/s; dense', round(d.get('dense_index',{}).get('ms_per_step',0),4), 'ms', round(d.get('dense_index',{}).get('value',0),1))")
    echo "[$k rep$r] literal 2^32 bench: $v"
  done
done
for k in tile bulk grid; do
  NORM_SCALE_KERNEL=$k python scripts/path_sweep.py literal flushed 1048583 4194311 16777223 | sed "s/^/[$k] /"
  NORM_SCALE_KERNEL=$k python scripts/path_sweep.py dense hot 1048583 4194311 16777223 | sed "s/^/[$k] /"
done
