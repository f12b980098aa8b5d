#!/bin/bash
# build A/B variants of libcsaw.so into exp/ (gitignored): name:"-DFLAG=.. -DFLAG=.." pairs
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 $flags -Xcompiler -fPIC,-fvisibility=hidden -shared \
       -o exp/libcsaw_$name.so paper_2009_09103_b200/csrc/*.cu &
done
wait
ls -la exp/
