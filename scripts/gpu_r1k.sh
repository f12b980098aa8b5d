set -x
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/gpu_all.log 2>&1; tail -25 gpurun_out/gpu_all.log
timeout 900 python scripts/ablation_oom.py --config cfg2 > gpurun_out/ablation_oom.json 2> gpurun_out/ablation_oom.err; tail -c 3000 gpurun_out/ablation_oom.json; tail -5 gpurun_out/ablation_oom.err
