set -x
timeout 900 python -m pytest tests/test_gpu_oom.py tests/test_gpu_cache.py tests/test_gpu_parity.py -x -q --timeout 600 > gpurun_out/gpu_c.log 2>&1; tail -5 gpurun_out/gpu_c.log
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_cache.json 2> gpurun_out/bench_cfg2_cache.err; tail -c 2500 gpurun_out/bench_cfg2_cache.json; tail -3 gpurun_out/bench_cfg2_cache.err
for c in cfg1 cfg4_layer; do
timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_${c}_cache.json 2> gpurun_out/bench_${c}_cache.err; tail -c 1200 gpurun_out/bench_${c}_cache.json; tail -3 gpurun_out/bench_${c}_cache.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_walk_cached -s 1 -c 1 -o gpurun_out/prof_cfg2_cache python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cache.log 2>&1; tail -2 gpurun_out/ncu_cache.log
timeout 1500 python bench.py --config cfg5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5_oom.json 2> gpurun_out/bench_cfg5_oom.err; tail -c 2500 gpurun_out/bench_cfg5_oom.json; tail -3 gpurun_out/bench_cfg5_oom.err
