#!/bin/bash
# node2vec index: sector-granular member probes A/B (cfg3 default line)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_n2v_index.py -x -q 2>&1 | tail -1
for v in default sec; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 > gpurun_out/r2o_$v.json 2>&1
  python -c "
import json
for l in open('gpurun_out/r2o_$v.json'):
    if l.startswith('{'): d=json.loads(l); r=d['roofline']; print('$v ms', round(d['ms_per_step'],3), 'frac', round(r['frac'],4), 'B/launch', r['alg_bytes_per_launch'])
"
done
