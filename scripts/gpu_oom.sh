set -x
timeout 900 python -m pytest tests/test_gpu_oom.py -x -q --timeout 600 > gpurun_out/gpu_oom.log 2>&1; tail -15 gpurun_out/gpu_oom.log
timeout 1500 python bench.py --config cfg5 --steps 1 --warmup 1 --cpu-seconds 10 --no-e2e > gpurun_out/bench_cfg5_oom.json 2> gpurun_out/bench_cfg5_oom.err; tail -c 1500 gpurun_out/bench_cfg5_oom.json; tail -5 gpurun_out/bench_cfg5_oom.err
