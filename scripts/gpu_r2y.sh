#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_n2v_index.py -x -q 2>&1 | tail -1
for v in default static default static; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 > gpurun_out/r2y_$v.json 2>&1
  python -c "
import json
for l in open('gpurun_out/r2y_$v.json'):
    if l.startswith('{'): d=json.loads(l); r=d['roofline']; print('$v ms', round(d['ms_per_step'],3), 'frac', round(r['frac'],4), r['alg_bytes_per_launch'])
" || tail -3 gpurun_out/r2y_$v.json
done
