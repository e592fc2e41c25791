#!/bin/bash
# Keep gpurun_out/ under the 64 MiB copy-back cap: drop the largest .ncu-rep
# files first, then any file over 8 MB, until the tree is below 56 MB.
OUT=${1:-gpurun_out}
size() { du -sm $OUT | cut -f1; }
for f in $(ls -S $(find $OUT -name '*.ncu-rep') 2>/dev/null); do
  [ $(size) -lt 56 ] && break
  echo "trim: $f"; rm -f $f
done
for f in $(find $OUT -type f -size +8M); do
  [ $(size) -lt 56 ] && break
  echo "trim: $f"; rm -f $f
done
du -sm $OUT
