set -x
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python scripts/dbg_n2v.py > gpurun_out/dbg_n2v.log 2>&1; tail -40 gpurun_out/dbg_n2v.log
