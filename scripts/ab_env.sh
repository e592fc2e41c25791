#!/bin/bash
# Same-box A/B of an environment knob: ab_env.sh VAR "valA valB" reps -- cmd...
VAR=$1; VALS=$2; REPS=$3; shift 4
for r in $(seq 1 $REPS); do
  for v in $VALS; do
    echo "[$VAR=$v rep$r] $(env $VAR=$v "$@" 2>/dev/null | tail -1)"
  done
done
