#!/bin/bash
# cfg3 strong-scaling shares: balanced rounds (every warp the same number of groups) vs resident grid
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in default r4; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  echo "== $v"; timeout 900 python scripts/strong_shares.py cfg3 2>/dev/null | grep "^| cfg3"
done
