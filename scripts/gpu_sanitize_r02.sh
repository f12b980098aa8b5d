#!/bin/bash
# compute-sanitizer over small cases of the round-2 kernels
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/san
CS="compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20"
timeout 1500 $CS python -m pytest tests/test_gpu_weight.py -k "cfg1 or zero or errors or hub or batched" -x -q > gpurun_out/san/weight.log 2>&1; echo "weight rc=$?"; tail -3 gpurun_out/san/weight.log
timeout 1500 $CS python -m pytest tests/test_gpu_n2v_index.py -x -q > gpurun_out/san/n2x.log 2>&1; echo "n2x rc=$?"; tail -3 gpurun_out/san/n2x.log
timeout 1500 $CS python -m pytest tests/test_gpu_parity.py -k "mdrw" -x -q > gpurun_out/san/mdrw.log 2>&1; echo "mdrw rc=$?"; tail -3 gpurun_out/san/mdrw.log
timeout 1500 $CS python -m pytest tests/test_gpu_oom_peer.py -x -q > gpurun_out/san/peer.log 2>&1; echo "peer rc=$?"; tail -3 gpurun_out/san/peer.log
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_weight.py -k "hub or batched" -x -q > gpurun_out/san/race.log 2>&1; echo "race rc=$?"; tail -3 gpurun_out/san/race.log
