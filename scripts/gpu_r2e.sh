#!/bin/bash
# round 2 (re-entry): GPU suite, default bench (cfg3, node2vec intersection index), cfg2,
# launch list + one --set full capture of the cfg3 hot kernel
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2e_build.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/ -m gpu -x -q > gpurun_out/r2e_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2e_pytest.log
timeout 900 python bench.py > gpurun_out/r2e_bench_cfg3.json 2> gpurun_out/r2e_bench_cfg3.err; echo "bench rc=$?"
tail -c 600 gpurun_out/r2e_bench_cfg3.err
timeout 600 python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/r2e_bench_cfg2.json 2> gpurun_out/r2e_bench_cfg2.err; echo "cfg2 rc=$?"
mkdir -p gpurun_out/prof_r02
NCU="ncu --clock-control none --nvtx --nvtx-include csaw_step/"
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/prof_r02/cfg3_launches.csv $B > gpurun_out/prof_r02/cfg3_ll.log 2>&1; echo "ll rc=$?"
timeout 900 $NCU --set full --import-source on -k regex:k_node2vec_idx -c 1 -o gpurun_out/prof_r02/cfg3 $B > gpurun_out/prof_r02/cfg3_full.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/prof_r02/cfg3.ncu-rep --page raw --csv > gpurun_out/prof_r02/cfg3_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_r02/cfg3.ncu-rep --page details --csv > gpurun_out/prof_r02/cfg3_details.csv 2>/dev/null
ncu -i gpurun_out/prof_r02/cfg3.ncu-rep --page source --csv > gpurun_out/prof_r02/cfg3_source.csv 2>/dev/null
ls -la gpurun_out/prof_r02
