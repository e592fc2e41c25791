#!/bin/bash
# A/B of the bulk reduce's dynamic tail (NORM_DYN_PCT / NORM_DYN_TC) on one box:
# reduce-only size sweep, the fused kernel's phase timeline at 2^29 and the
# literal 2^32 bench step.
OUT=${OUT:-gpurun_out}
for cfg in ${CFGS:-"0 8" "3 8" "3 16" "5 16" "0 8" "3 8"}; do
  set -- $cfg
  echo "== NORM_DYN_PCT=$1 NORM_DYN_TC=$2"
  NORM_DYN_PCT=$1 NORM_DYN_TC=$2 python scripts/reduce_size_sweep.py 2>&1 | grep -E "2\^29|2\^32|back-to-back:"
  NORM_DYN_PCT=$1 NORM_DYN_TC=$2 python scripts/fused_timeline.py 536870912 2>&1 | grep -E "per call|phase-1|barrier"
  NORM_DYN_PCT=$1 NORM_DYN_TC=$2 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > $OUT/dyn_$1_$2.json 2>/dev/null
  python -c "import json; d=json.loads(open('$OUT/dyn_$1_$2.json').read().strip().splitlines()[-1]); print('bench literal 2^32: %.1f us  reduce %.1f us  dense %.1f us' % (d['ms_per_step']*1e3, d['roofline']['avg_launch_ms']*1e3, d['dense_index']['ms_per_step']*1e3))"
done
