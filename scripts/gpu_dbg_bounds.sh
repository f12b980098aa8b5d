#!/bin/bash
# the GPU suites of the re-entry session's kernels against the bounds-checked debug build
# (CSAW_DEBUG_BOUNDS: device asserts on bucket indices, link searches, MDRW entries, index probes)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export CSAW_LIB=$PWD/exp/libcsaw_dbg.so
mkdir -p gpurun_out/dbg
timeout 1500 python -m pytest tests/test_gpu_buckets.py tests/test_gpu_n2v_index.py tests/test_gpu_batched.py -x -q > gpurun_out/dbg/small.log 2>&1; echo "small rc=$?"; tail -2 gpurun_out/dbg/small.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -k "mdrw" -x -q > gpurun_out/dbg/mdrw.log 2>&1; echo "mdrw rc=$?"; tail -2 gpurun_out/dbg/mdrw.log
timeout 2400 python -m pytest tests/test_gpu_configs.py -x -q -k "cfg2 or cfg3 or cfg5_mdrw" > gpurun_out/dbg/full.log 2>&1; echo "full rc=$?"; tail -2 gpurun_out/dbg/full.log
grep -h "CSAW_DASSERT" gpurun_out/dbg/*.log | head -5
