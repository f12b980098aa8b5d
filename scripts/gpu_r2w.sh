#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1; do
for v in m4 w4m8 k2m3 k2m4; do
  export CSAW_LIB=$PWD/exp/libcsaw_$v.so
  timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 > gpurun_out/r2w_$v.json 2>&1
  python -c "
import json
for l in open('gpurun_out/r2w_$v.json'):
    if l.startswith('{'): d=json.loads(l); r=d['roofline']; print('$rep $v ms', round(d['ms_per_step'],3), [round(x,2) for x in d['detail']['step_ms']], d['clocks']['sm_mhz'])
"
done
done
