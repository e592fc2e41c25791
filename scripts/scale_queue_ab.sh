#!/bin/bash
# A/B of the bulk scale's chunk queue (NORM_SCALE_QUEUE=0: grid-strided) on one box.
OUT=${OUT:-gpurun_out}
for rep in 1 2; do
  for q in 0 1; do
    NORM_SCALE_QUEUE=$q python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $OUT/sq_$q.json 2>/dev/null
    python -c "import json; d=json.loads(open('$OUT/sq_$q.json').read().strip().splitlines()[-1]); print('queue=$q literal 2^32: %.1f us  reduce %.1f us  dense %.1f us' % (d['ms_per_step']*1e3, d['roofline']['avg_launch_ms']*1e3, d['dense_index']['ms_per_step']*1e3))"
  done
done
