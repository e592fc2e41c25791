#!/bin/bash
# Same-box ablation of the literal / dense n = 2^32 step: each design choice
# switched off in turn through its A/B knob, 2 reps each.
run() {
  local tag="$1"; shift
  env "$@" python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print('%-34s literal %7.1f us  (reduce %7.1f us)   dense %7.1f us' % ('$tag', d['ms_per_step'] * 1e3, d['roofline']['avg_launch_ms'] * 1e3, d['dense_index']['ms_per_step'] * 1e3))"
}
for rep in 1 2; do
  run "all on (default)" X=1
  run "PDL off" NORM_PDL=off
  run "reduce dynamic tail off" NORM_DYN_PCT=0
  run "scale queue off" NORM_SCALE_QUEUE=0
  run "all three off" NORM_PDL=off NORM_DYN_PCT=0 NORM_SCALE_QUEUE=0
done
