#!/bin/bash
# node2vec index build with hub rank bitmaps: parity + build time
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_n2v_index.py tests/test_gpu_n2v_tri.py -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -k cfg3 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 > gpurun_out/r2q.json 2>&1
python -c "
import json
for l in open('gpurun_out/r2q.json'):
    if l.startswith('{'): d=json.loads(l); c=d['detail']['cache']; print('ms', d['ms_per_step'], 'build_ms', c['build_ms'], 'one_call', c['one_call_seps'], 'bytes', c['graph_device_bytes'])
"
