set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q --timeout 600 -k "node2vec or cfg3 or hub" > gpurun_out/gpu_h.log 2>&1; tail -3 gpurun_out/gpu_h.log
timeout 600 python scripts/prof_n2v.py 40 > gpurun_out/n2v_small.log 2>&1; cat gpurun_out/n2v_small.log | tail -3
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; tail -c 300 gpurun_out/bench_cfg3.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:node2vec -s 1 -c 1 -o gpurun_out/prof_n2v python scripts/prof_n2v.py 40 > gpurun_out/ncu_n2v.log 2>&1; tail -2 gpurun_out/ncu_n2v.log
set -x
timeout 900 python -m pytest tests/test_gpu_walk_variants.py tests/test_gpu_batched.py -x -q --timeout 600 > gpurun_out/gpu_g.log 2>&1; tail -3 gpurun_out/gpu_g.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --gather > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err; tail -c 400 gpurun_out/bench_torchrun1.json; tail -3 gpurun_out/bench_torchrun1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; tail -c 800 gpurun_out/bench_reference.json; tail -3 gpurun_out/bench_reference.err
timeout 900 python scripts/ablation_migration.py --config cfg2 --instances 2000 --fanout 2 2 > gpurun_out/ablation_f2.json 2> gpurun_out/ablation.err; tail -c 1500 gpurun_out/ablation_f2.json; tail -3 gpurun_out/ablation.err
timeout 900 python scripts/ablation_migration.py --config cfg2 --instances 2000 --fanout 8 8 > gpurun_out/ablation_f8.json 2>> gpurun_out/ablation.err; tail -c 600 gpurun_out/ablation_f8.json
