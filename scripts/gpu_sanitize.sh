# compute-sanitizer memcheck / racecheck over small parity cases of the hot kernels
set -x
mkdir -p gpurun_out/san
CS="compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20"
timeout 900 $CS python -m pytest tests/test_gpu_wix.py -k "gtoy or boundaries or isolated" -x -q > gpurun_out/san/wix.log 2>&1; echo "wix rc=$?"; tail -3 gpurun_out/san/wix.log
timeout 900 $CS python -m pytest tests/test_gpu_n2v_tri.py -k "gtoy or asymmetric or medium" -x -q > gpurun_out/san/n2v.log 2>&1; echo "n2v rc=$?"; tail -3 gpurun_out/san/n2v.log
timeout 900 $CS python -m pytest tests/test_gpu_parity.py -k "mdrw or gtoy or forest or layer or pinned" -x -q > gpurun_out/san/parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/san/parity.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -k "gtoy or forest" -x -q > gpurun_out/san/race.log 2>&1; echo "race rc=$?"; tail -3 gpurun_out/san/race.log
