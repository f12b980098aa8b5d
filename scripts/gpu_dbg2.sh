set -x
timeout 900 python scripts/dbg_n2v.py > gpurun_out/dbg_n2v.log 2>&1; tail -5 gpurun_out/dbg_n2v.log
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/gpu_all.log 2>&1; tail -5 gpurun_out/gpu_all.log
for c in cfg2 cfg3 cfg1 cfg4_layer cfg4_ff; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 300 gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err
done
