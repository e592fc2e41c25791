#!/bin/bash
# Round-end evidence on one box: the GPU suite + smoke and every bench workload
# (scripts/bench_all.sh) into $D (default gpurun_out/final); NCU_KERNEL=<regex>
# NCU_WORKLOAD=<bench args> additionally re-captures one kernel with ncu --set full
# and records its per-launch traffic (scripts/ncu_traffic_update.py NCU_KEY).
set -x
D=${D:-gpurun_out/final}
mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -q > $D/gpu_tests.log 2>&1; tail -3 $D/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; tail -2 $D/smoke.log
if [ -n "$NCU_KERNEL" ]; then
  OUT=$D/ncu; mkdir -p $OUT; cp profiles/ncu_traffic.json $OUT/ncu_traffic.json
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$NCU_KERNEL -s 3 -c 1 -o $OUT/k \
      python bench.py $NCU_WORKLOAD --steps 3 --warmup 3 > $OUT/k.bench.log 2>&1
  ncu -i $OUT/k.ncu-rep --page raw --csv > $OUT/k_raw.csv 2>/dev/null
  ncu -i $OUT/k.ncu-rep --page details --csv > $OUT/k_details.csv 2>/dev/null
  ncu -i $OUT/k.ncu-rep --page source --csv > $OUT/k_source.csv 2>/dev/null
  rm -f $OUT/k.ncu-rep
  python scripts/ncu_traffic_update.py --json $OUT/ncu_traffic.json --capture ${TAG:-final} $NCU_KEY \
      $OUT/k_raw.csv $NCU_KERNEL
fi
OUT=$D TAG=${TAG:-final} timeout 1500 bash scripts/bench_all.sh > $D/bench_all.log 2>&1
tail -12 $D/bench_all.log | cut -c1-250
