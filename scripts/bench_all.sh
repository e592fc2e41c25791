#!/bin/bash
# Every bench workload once (1 GPU), JSON lines into $OUT/bench_<TAG>_*.json
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r04}
mkdir -p $OUT
python bench.py > $OUT/bench_${TAG}_vector_literal.json 2> $OUT/bench_${TAG}_vector_literal.err
python bench.py --index dense --no-e2e --no-cpu > $OUT/bench_${TAG}_vector_dense.json 2>/dev/null
for i in dense literal; do
  python bench.py --workload rows --index $i > $OUT/bench_${TAG}_rows_$i.json 2>/dev/null
  python bench.py --workload paths28 --index $i > $OUT/bench_${TAG}_paths28_$i.json 2>/dev/null
done
python bench.py --workload softmax > $OUT/bench_${TAG}_softmax.json 2>/dev/null
python bench.py --workload licm > $OUT/bench_${TAG}_licm.json 2>/dev/null
python bench.py --workload backprop > $OUT/bench_${TAG}_backprop.json 2>/dev/null
python bench.py --workload small > $OUT/bench_${TAG}_small.json 2>/dev/null
python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_${TAG}_reference.json 2>/dev/null
for f in $OUT/bench_${TAG}_*.json; do echo "$f: $(head -c 300 $f)"; done
