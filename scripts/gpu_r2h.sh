#!/bin/bash
# ncu --set full of the per-step scan kernel on cfg2 (materialised degree-bias stream)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/prof_r02
B="python bench.py --config cfg2 --no-cache --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --scan-path-steps 0"
timeout 900 ncu --clock-control none --nvtx --nvtx-include csaw_step/ --set full --import-source on -k regex:k_walk_vscan -c 1 -o gpurun_out/prof_r02/cfg2_stream $B > gpurun_out/prof_r02/cfg2_stream_full.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_r02/cfg2_stream.ncu-rep --page raw --csv > gpurun_out/prof_r02/cfg2_stream_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_r02/cfg2_stream.ncu-rep --page details --csv > gpurun_out/prof_r02/cfg2_stream_details.csv 2>/dev/null
ncu -i gpurun_out/prof_r02/cfg2_stream.ncu-rep --page source --csv > gpurun_out/prof_r02/cfg2_stream_source.csv 2>/dev/null
ls -la gpurun_out/prof_r02 | grep cfg2
