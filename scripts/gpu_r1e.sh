set -x
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/gpu_all.log 2>&1; tail -5 gpurun_out/gpu_all.log
for c in cfg2 cfg1 cfg4_layer cfg4_ff; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 300 gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_walk_cached -s 1 -c 1 -o gpurun_out/prof_cfg2_bt2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bt2.log 2>&1; tail -2 gpurun_out/ncu_bt2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sample_fused -s 2 -c 1 -o gpurun_out/prof_cfg4_layer python bench.py --config cfg4_layer --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_l.log 2>&1; tail -2 gpurun_out/ncu_l.log
