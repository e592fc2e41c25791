#!/bin/bash
# ncu evidence for the bench kernels (run on the GPU box under gpurun; 1 GPU).
# 1) launch list of the bench command (cold-cache, serialised: compare shares)
# 2) one `--set full` capture per hot kernel (reduce, scale, fused, rows)
set -x
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r01}
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/${TAG}_launches_vector.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > $OUT/${TAG}_launches_vector.bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"reduce_dyn_kernel|reduce_bulk_kernel" -s 3 -c 1 \
    -o $OUT/${TAG}_reduce python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:scale_bulk_kernel -s 3 -c 1 \
    -o $OUT/${TAG}_scale python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 3 -c 1 \
    -o $OUT/${TAG}_fused python bench.py --workload paths28 --steps 3 --warmup 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:rows_vec_kernel -s 3 -c 1 \
    -o $OUT/${TAG}_rows_dense python bench.py --workload rows --index dense --steps 3 --warmup 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:rows_vec_kernel -s 3 -c 1 \
    -o $OUT/${TAG}_rows_literal python bench.py --workload rows --index literal --steps 3 --warmup 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:rows_bulk_kernel -s 3 -c 1 \
    -o $OUT/${TAG}_rows_bulk python bench.py --workload rows --index literal --steps 3 --warmup 3 > /dev/null 2>&1
ls -la $OUT
ncu --set full --clock-control none --import-source on -k regex:softmax_vec -s 3 -c 1 \
    -o $OUT/${TAG}_softmax python bench.py --workload softmax --steps 3 --warmup 3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file $OUT/${TAG}_launches_dense.csv \
    python bench.py --index dense --steps 5 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ls -la $OUT
