#!/bin/bash
# Round-2 ncu evidence (run on the GPU box under gpurun; 1 GPU):
# 1) the launch list of the default bench command (cold-cache, serialised)
# 2) --set full captures: the headline reduce (literal 2^32), the dense scale
#    stream (n = 2^30 dense: same kernel and geometry as 2^32, 4 GiB so the
#    replay can save / restore its output) next to torch's copy kernel on the
#    same buffers, and the mid kernel at n = 2^20 + 7.
OUT=${OUT:-gpurun_out/ncu2}
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_vector.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-parity > $OUT/launches_vector.bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"reduce_dyn_kernel" -s 3 -c 1 \
    -o $OUT/reduce python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"scale_bulk_kernel|elementwise" -s 6 -c 3 \
    -o $OUT/scale_dense python bench.py --index dense --numel 1073741824 --steps 3 --warmup 3 --no-e2e \
    --no-cpu --no-parity > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"mid_kernel" -s 20 -c 1 \
    -o $OUT/mid python bench.py --workload small --steps 3 --warmup 3 > /dev/null 2>&1
for f in $OUT/*.ncu-rep; do
  ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null
  ncu -i $f --page details --csv > ${f%.ncu-rep}_details.csv 2>/dev/null
done
ls -la $OUT
