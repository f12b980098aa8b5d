#!/bin/bash
# round 2: GPU suite with the full-size parity coverage (durations recorded)
set -x
nproc; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests/ -x -q -m gpu -s --durations=25 > gpurun_out/r2a_gputests.log 2>&1
echo "pytest rc=$?"
tail -60 gpurun_out/r2a_gputests.log
