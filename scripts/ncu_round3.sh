#!/bin/bash
# ncu --set full of every bench workload's dominant kernel (run on the GPU box
# under gpurun; 1 GPU), exported to raw/details CSV, and the per-launch DRAM
# traffic recorded into $OUT/ncu_traffic.json bound to the kernels' source hashes
# (scripts/ncu_traffic_update.py; copy the file to profiles/ afterwards).
OUT=${OUT:-gpurun_out/ncu3}
mkdir -p $OUT
cp profiles/ncu_traffic.json $OUT/ncu_traffic.json 2>/dev/null
B="--steps 3 --warmup 3 --no-e2e --no-cpu --no-parity"
cap() {  # name kernel_regex skip bench-args...
  local name=$1 kre=$2 skip=$3; shift 3
  ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c 1 \
      -o $OUT/$name python bench.py "$@" > $OUT/$name.bench.log 2>&1
  ncu -i $OUT/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
  ncu -i $OUT/$name.ncu-rep --page details --csv > $OUT/${name}_details.csv 2>/dev/null
}
cap reduce "reduce_dyn_kernel" 3 $B
cap scale_dense "scale_tile_kernel" 6 --index dense $B
cap fused28 "fused_kernel" 3 --workload paths28 --steps 3 --warmup 3
cap rows_dense "rows_vec_kernel" 3 --workload rows --index dense --steps 3 --warmup 3
cap rows_literal "rows_bulk_kernel" 3 --workload rows --index literal --steps 3 --warmup 3
cap softmax "softmax_vec_kernel" 3 --workload softmax --steps 3 --warmup 3
cap bpnn_tma "bpnn_tma_kernel" 3 --workload backprop --steps 3 --warmup 3
cap mid "mid_kernel" 20 --workload small --steps 3 --warmup 3
U="python scripts/ncu_traffic_update.py --json $OUT/ncu_traffic.json --capture ${TAG:-round2}"
$U vector:literal $OUT/reduce_raw.csv reduce_dyn_kernel
$U vector:dense $OUT/reduce_raw.csv reduce_dyn_kernel
$U scale:dense $OUT/scale_dense_raw.csv scale_tile_kernel
$U paths28:literal $OUT/fused28_raw.csv fused_kernel
$U rows:dense $OUT/rows_dense_raw.csv rows_vec_kernel
$U rows:literal $OUT/rows_literal_raw.csv rows_bulk_kernel
$U softmax:dense $OUT/softmax_raw.csv softmax_vec_kernel
$U backprop:tma $OUT/bpnn_tma_raw.csv bpnn_tma_kernel
$U small:literal $OUT/mid_raw.csv mid_kernel
# keep the two headline reports (source page readable here); the rest live on as CSV
for f in $OUT/*.ncu-rep; do case $f in *reduce*|*scale_dense*) ;; *) rm -f $f ;; esac; done
ls -la $OUT
