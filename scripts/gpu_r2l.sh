#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/prof_r02
timeout 900 ncu --clock-control none --nvtx --nvtx-include csaw_step/ --set full --import-source on -k regex:k_mdrw_fast -c 1 -o gpurun_out/prof_r02/cfg5_inmem python bench.py --config cfg5 --in-memory --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --scan-path-steps 0 > gpurun_out/prof_r02/cfg5_full.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/prof_r02/cfg5_inmem.ncu-rep --page raw --csv > gpurun_out/prof_r02/cfg5_inmem_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_r02/cfg5_inmem.ncu-rep --page details --csv > gpurun_out/prof_r02/cfg5_inmem_details.csv 2>/dev/null
ncu -i gpurun_out/prof_r02/cfg5_inmem.ncu-rep --page source --csv > gpurun_out/prof_r02/cfg5_inmem_source.csv 2>/dev/null
ls -la gpurun_out/prof_r02 | grep cfg5
