#!/bin/bash
# ncu --set full of ONE workload's dominant kernel and its traffic entry (GPU box, 1 GPU):
#   OUT=... KEY=scale:dense KRE=scale_tile_kernel SKIP=6 bash scripts/ncu_one.sh <bench args>
OUT=${OUT:-gpurun_out/ncu_one}
mkdir -p $OUT
cp profiles/ncu_traffic.json $OUT/ncu_traffic.json
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s ${SKIP:-3} -c 1 -o $OUT/k \
    python bench.py "$@" --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > $OUT/k.bench.log 2>&1
ncu -i $OUT/k.ncu-rep --page raw --csv > $OUT/k_raw.csv 2>/dev/null
ncu -i $OUT/k.ncu-rep --page details --csv > $OUT/k_details.csv 2>/dev/null
rm -f $OUT/k.ncu-rep
python scripts/ncu_traffic_update.py --json $OUT/ncu_traffic.json --capture ${TAG:-round2} $KEY $OUT/k_raw.csv "$KRE"
