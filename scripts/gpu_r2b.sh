#!/bin/bash
# round 2: the new bench (cfg3 default, strong scaling, §8(d) bytes) + stream-ordering tests
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_streams.py -x -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/r2b_bench_cfg3.json 2> gpurun_out/r2b_bench_cfg3.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2b_bench_cfg3.json; tail -5 gpurun_out/r2b_bench_cfg3.err
timeout 600 python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/r2b_bench_cfg2.json 2> gpurun_out/r2b_bench_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --config cfg2 --no-cache --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2b_bench_cfg2_scan.json 2>&1; echo "cfg2 scan rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2b_ref_cfg3.json 2>&1; echo "ref rc=$?"
tail -c 1500 gpurun_out/r2b_ref_cfg3.json
