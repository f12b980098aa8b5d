set -x
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/gpu_all.log 2>&1; tail -5 gpurun_out/gpu_all.log
for c in cfg2 cfg1 cfg3 cfg4_layer cfg4_ff; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 400 gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err
done
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 --in-memory --no-cpu-baseline > gpurun_out/bench_cfg5_inmem.json 2> gpurun_out/bench_cfg5_inmem.err; tail -c 400 gpurun_out/bench_cfg5_inmem.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_walk_cached -s 1 -c 1 -o gpurun_out/prof_cfg2_bt python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bt.log 2>&1; tail -2 gpurun_out/ncu_bt.log
timeout 2400 python bench.py --config cfg5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5_oom.json 2> gpurun_out/bench_cfg5_oom.err; tail -c 600 gpurun_out/bench_cfg5_oom.json; tail -3 gpurun_out/bench_cfg5_oom.err
