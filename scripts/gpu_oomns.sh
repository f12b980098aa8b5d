set -x
timeout 900 python -m pytest tests/test_gpu_oom_sample.py -x -q --timeout 600 > gpurun_out/gpu_oomns.log 2>&1; tail -25 gpurun_out/gpu_oomns.log
timeout 1500 python bench.py --config cfg5_ns --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_cfg5ns.json 2> gpurun_out/bench_cfg5ns.err; tail -c 2500 gpurun_out/bench_cfg5ns.json; tail -5 gpurun_out/bench_cfg5ns.err
