#!/bin/bash
# Probe: build libnorm with each NORM_ST_VARIANT (the scale's 256-bit store
# flavour, device_common.cuh) into paper_2207_00257_b200/faults/, then time the
# dense two-pass step / reduce / scale split (scripts/dense_split.py) under each,
# alternating, same box.  Build here (CPU), run on the GPU box.
#   bash scripts/ab_store.sh build     |     bash scripts/ab_store.sh run [reps]
set -e
PKG=paper_2207_00257_b200
V="0 1 2 3 4 5"
if [ "$1" = build ]; then
  for v in $V; do
    make -s $PKG/libnorm.so > /dev/null
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude \
      -I$(python -c "import sysconfig;print(sysconfig.get_paths()['purelib'])")/nvidia/nccl/include \
      -DNORM_ST_VARIANT=$v -shared -o $PKG/faults/libnorm_st$v.so $PKG/csrc/*.cu $PKG/csrc/*.cpp \
      -L$(python -c "import sysconfig;print(sysconfig.get_paths()['purelib'])")/nvidia/nccl/lib -l:libnccl.so.2 \
      -Xlinker -rpath,$(python -c "import sysconfig;print(sysconfig.get_paths()['purelib'])")/nvidia/nccl/lib &
  done
  wait
  ls -la $PKG/faults/
  exit 0
fi
for r in $(seq ${2:-2}); do
  for v in $V; do
    LIBNORM_SO=$PWD/$PKG/faults/libnorm_st$v.so python scripts/dense_split.py 30 32 | sed "s/^/[st$v rep$r] /"
  done
done
