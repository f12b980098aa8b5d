#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; mkdir -p gpurun_out/final
true
timeout 900 python bench.py --config cfg4_layer > gpurun_out/final/bench_cfg4_layer.json 2> gpurun_out/final/bench_cfg4_layer.err; echo "cfg4_layer rc=$?"; tail -2 gpurun_out/final/bench_cfg4_layer.err
timeout 900 python bench.py --config cfg2_weight > gpurun_out/final/bench_cfg2_weight.json 2> gpurun_out/final/bench_cfg2_weight.err; echo "cfg2_weight rc=$?"; tail -2 gpurun_out/final/bench_cfg2_weight.err
true
