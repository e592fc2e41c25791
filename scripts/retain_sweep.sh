#!/bin/bash
# A/B sweep of the two-pass L2 retention window (NORM_RETAIN_BYTES) on one box,
# plus an ncu pass with --cache-control none over consecutive steps to check that
# retained lines do not carry over into the next call (reduce DRAM read = 4n).
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
for rep in 1 2; do
  for R in 0 16777216 33554432 50331648 67108864 100663296; do
    NORM_RETAIN_BYTES=$R timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu \
      > $OUT/retain_${R}_${rep}.json 2> $OUT/retain_${R}_${rep}.err
    python - "$R" "$rep" $OUT/retain_${R}_${rep}.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
print(f"R={int(sys.argv[1])>>20:4d} MiB rep{sys.argv[2]}: literal {d['ms_per_step']*1e3:8.1f} us  {d['value']:7.1f} GB/s  reduce {d['roofline']['avg_launch_ms']*1e3:8.1f} us | dense {d['dense_index']['ms_per_step']*1e3:8.1f} us")
PY
  done
done
ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  -k regex:"reduce_bulk|scale_bulk" -c 16 --csv --log-file $OUT/retain_ncu_steps.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  -k regex:"fused" -c 8 --csv --log-file $OUT/retain_ncu_fused.csv \
  python bench.py --workload paths28 --steps 3 --warmup 3 > /dev/null 2>&1
for R in 0 50331648; do
  for rep in 1 2; do
    NORM_RETAIN_BYTES=$R timeout 300 python bench.py --workload paths28 --steps 50 --warmup 5 > $OUT/retain28_${R}_${rep}.json 2>&1
    python -c "import json,sys; d=json.loads(open('$OUT/retain28_${R}_${rep}.json').read().strip().splitlines()[-1]); print('paths28 R=$R rep$rep', {k:round(v['ms_per_step']*1e3,1) for k,v in d['paths'].items()})"
    NORM_RETAIN_BYTES=$R timeout 300 python bench.py --workload paths28 --index dense --steps 50 --warmup 5 > $OUT/retain28d_${R}_${rep}.json 2>&1
    python -c "import json,sys; d=json.loads(open('$OUT/retain28d_${R}_${rep}.json').read().strip().splitlines()[-1]); print('paths28 dense R=$R rep$rep', {k:round(v['ms_per_step']*1e3,1) for k,v in d['paths'].items()})"
  done
done
