#!/bin/bash
# NEXT-4(i) peer partition store: parity (same-device stand-in), cfg5 OOM partition mode with the store in HBM
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2m_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_oom_peer.py tests/test_gpu_oom.py tests/test_gpu_oom_sample.py -x -q > gpurun_out/r2m_pytest.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2m_pytest.log
timeout 1500 python bench.py --config cfg5 --oom-store peer --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-zerocopy > gpurun_out/r2m_cfg5_peer.json 2> gpurun_out/r2m_cfg5_peer.err; echo "cfg5 peer rc=$?"
python -c "
import json
for l in open('gpurun_out/r2m_cfg5_peer.json'):
    if l.startswith('{'): d=json.loads(l); r=d['roofline']; print('cfg5 OOM peer-store ms', d['ms_per_step'], 'SEPS', d['value'], r)
"
tail -3 gpurun_out/r2m_cfg5_peer.err
