set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cache.py tests/test_gpu_configs.py -x -q --timeout 600 -k "node2vec or cfg3 or hub or cfg2 or cached" > gpurun_out/gpu_i.log 2>&1; tail -3 gpurun_out/gpu_i.log
timeout 300 python scripts/prof_n2v.py 40 > gpurun_out/n2v_mb3.log 2>&1; tail -2 gpurun_out/n2v_mb3.log
CSAW_LIB=exp/libcsaw_mb2.so timeout 300 python scripts/prof_n2v.py 40 > gpurun_out/n2v_mb2.log 2>&1; tail -2 gpurun_out/n2v_mb2.log
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; tail -c 300 gpurun_out/bench_cfg2.json
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --in-memory --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5_inmem.json 2> gpurun_out/bench_cfg5_inmem.err; tail -c 300 gpurun_out/bench_cfg5_inmem.json
timeout 900 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; tail -c 300 gpurun_out/bench_cfg1.json
