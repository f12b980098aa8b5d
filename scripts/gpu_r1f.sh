set -x
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/gpu_all.log 2>&1; tail -5 gpurun_out/gpu_all.log
for c in cfg3 cfg1 cfg4_layer cfg4_ff; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 300 gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:node2vec -s 0 -c 1 -o gpurun_out/prof_cfg3 python bench.py --config cfg3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cfg3.log 2>&1; tail -2 gpurun_out/ncu_cfg3.log
