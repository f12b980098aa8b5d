set -x
timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q --timeout 1200 -s > gpurun_out/gpu_configs.log 2>&1; tail -15 gpurun_out/gpu_configs.log
for c in cfg1 cfg3 cfg4_layer cfg4_ff cfg5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 2 --cpu-seconds 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 600 gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err
done
