#!/bin/bash
# node2vec TMA kernel: parity (small + full-size cfg3), smoke, default bench, ncu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_n2v_index.py tests/test_gpu_n2v_tri.py tests/test_gpu_streams.py -x -q 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_gpu_configs.py -x -q -k cfg3 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2x_bench.json 2> gpurun_out/r2x_bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/r2x_dummy > /dev/null 2>&1
mkdir -p gpurun_out/prof3
NCU="ncu --clock-control none --nvtx --nvtx-include csaw_step/"
Q="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --scan-path-steps 0"
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/prof3/cfg3_launches.csv $Q > /dev/null 2>&1
timeout 1200 $NCU --set full --import-source on -k regex:k_node2vec_tma -c 1 -o gpurun_out/prof3/cfg3 $Q > /dev/null 2>&1
ncu -i gpurun_out/prof3/cfg3.ncu-rep --page raw --csv > gpurun_out/prof3/cfg3_raw.csv 2>/dev/null
ncu -i gpurun_out/prof3/cfg3.ncu-rep --page details --csv > gpurun_out/prof3/cfg3_details.csv 2>/dev/null
find gpurun_out/prof3 -name '*.ncu-rep' -size +20M -delete
echo done
