#!/bin/bash
# default bench (cfg3) + cfg2 with scan-path details; 500-walker cfg2 scan (walker groups)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2i_build.log 2>&1; echo "build rc=$?"
timeout 900 python bench.py > gpurun_out/r2i_bench_cfg3.json 2> gpurun_out/r2i_bench_cfg3.err; echo "cfg3 rc=$?"; tail -c 400 gpurun_out/r2i_bench_cfg3.err
timeout 900 python bench.py --config cfg2 --no-cpu-baseline --scan-path-steps 3 > gpurun_out/r2i_bench_cfg2.json 2> gpurun_out/r2i_bench_cfg2.err; echo "cfg2 rc=$?"
timeout 600 python scripts/walker_groups.py > gpurun_out/r2i_groups.txt 2>&1; echo "groups rc=$?"; cat gpurun_out/r2i_groups.txt
