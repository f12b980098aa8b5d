#!/bin/bash
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_n2v_index.py tests/test_gpu_n2v_tri.py -x -q 2>&1 | tail -15
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_bench_cfg3.json 2> gpurun_out/r2c_bench_cfg3.err; echo "bench rc=$?"
tail -c 2500 gpurun_out/r2c_bench_cfg3.json; tail -5 gpurun_out/r2c_bench_cfg3.err
