#!/bin/bash
# MDRW A/B: speculation, stream hints, record layout (cfg5 in memory)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "mdrw" 2>&1 | tail -1
for v in default ef efkeep; do
  if [ $v = default ]; then unset CSAW_LIB; else export CSAW_LIB=$PWD/exp/libcsaw_$v.so; fi
  timeout 600 python bench.py --config cfg5 --in-memory --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --scan-path-steps 0 > gpurun_out/r2k_$v.json 2>&1
  python -c "
import json
for l in open('gpurun_out/r2k_$v.json'):
    if l.startswith('{'): d=json.loads(l); print('$v ms', round(d['ms_per_step'],3))
"
  timeout 600 ncu --clock-control none --nvtx --nvtx-include csaw_step/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --csv --log-file gpurun_out/r2k_${v}_ll.csv python bench.py --config cfg5 --in-memory --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --scan-path-steps 0 > /dev/null 2>&1
  grep k_mdrw gpurun_out/r2k_${v}_ll.csv | awk -F'","' '{print "   ", $(NF-2), $NF}'
done
unset CSAW_LIB
python - <<'PY'
import torch, sys, time
sys.path.insert(0, '.')
import paper_2009_09103_b200 as cs
from synth import CONFIGS, rmat_csr, mdrw_seeds
cfg = CONFIGS["cfg5"]
PY
