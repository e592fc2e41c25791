#!/bin/bash
# Round-end evidence on one box: the GPU suite + smoke, ncu of kernels changed since the last
# capture (softmax), and every bench workload (scripts/bench_all.sh).
set -x
mkdir -p gpurun_out/final
# 1. full GPU suite + smoke
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final/gpu_tests.log 2>&1; tail -3 gpurun_out/final/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; tail -2 gpurun_out/final/smoke.log
# 2. ncu of the changed softmax kernel -> traffic entry
OUT=gpurun_out/final/ncu; mkdir -p $OUT; cp profiles/ncu_traffic.json $OUT/ncu_traffic.json
timeout 300 ncu --set full --clock-control none --import-source on -k regex:softmax_vec_kernel -s 3 -c 1 -o $OUT/softmax python bench.py --workload softmax --steps 3 --warmup 3 > $OUT/softmax.bench.log 2>&1
ncu -i $OUT/softmax.ncu-rep --page raw --csv > $OUT/softmax_raw.csv 2>/dev/null
ncu -i $OUT/softmax.ncu-rep --page details --csv > $OUT/softmax_details.csv 2>/dev/null
rm -f $OUT/softmax.ncu-rep
python scripts/ncu_traffic_update.py --json $OUT/ncu_traffic.json --capture round2-final softmax:dense $OUT/softmax_raw.csv softmax_vec_kernel
# 3. every bench workload on this box
OUT=gpurun_out/final TAG=final timeout 1500 bash scripts/bench_all.sh > gpurun_out/final/bench_all.log 2>&1
tail -12 gpurun_out/final/bench_all.log | cut -c1-250
