#!/bin/bash
# MDRW: speculative next block + packed records in memory -- parity, cfg5 in-memory bench, DRAM per launch
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2j_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_oom.py -x -q -k "mdrw or oom" > gpurun_out/r2j_pytest.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2j_pytest.log
timeout 900 python bench.py --config cfg5 --in-memory --no-cpu-baseline --scan-path-steps 0 > gpurun_out/r2j_cfg5.json 2> gpurun_out/r2j_cfg5.err; echo "cfg5 rc=$?"
python -c "
import json
for l in open('gpurun_out/r2j_cfg5.json'):
    if l.startswith('{'): d=json.loads(l); r=d['roofline']; print('cfg5 inmem ms', d['ms_per_step'], 'SEPS', d['value'], 'e2e', d['e2e']['value'], r['kernel'], r['frac'])
"
mkdir -p gpurun_out/prof_r02
timeout 900 ncu --clock-control none --nvtx --nvtx-include csaw_step/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --csv --log-file gpurun_out/prof_r02/cfg5_inmem_launches.csv python bench.py --config cfg5 --in-memory --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --scan-path-steps 0 > /dev/null 2>&1; echo "ncu rc=$?"
grep k_mdrw gpurun_out/prof_r02/cfg5_inmem_launches.csv | awk -F'","' '{print $(NF-2), $NF}'
