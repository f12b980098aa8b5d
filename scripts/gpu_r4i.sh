#!/bin/bash
# k_walk_gb block size A/B (2 warps default vs 1 / 4)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
for v in default g1 g4; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 > /tmp/b_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('/tmp/b_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'])"
done
done
