set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "node2vec or hub" > gpurun_out/gpu_n2v.log 2>&1; tail -3 gpurun_out/gpu_n2v.log
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q --timeout 600 -k cfg3 >> gpurun_out/gpu_n2v.log 2>&1; tail -3 gpurun_out/gpu_n2v.log
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; tail -c 1500 gpurun_out/bench_cfg3.json; tail -3 gpurun_out/bench_cfg3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_node2vec -s 0 -c 1 -o gpurun_out/prof_cfg3 python bench.py --config cfg3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cfg3.log 2>&1; tail -2 gpurun_out/ncu_cfg3.log
