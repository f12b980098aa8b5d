#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in default ch4 ch64 hub512; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['detail']['cache']['build_ms'])"
done
