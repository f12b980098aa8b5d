# ncu evidence for every config's hot kernel.  Launch lists are the timed bench steps only
# (NVTX range "csaw_step"); full captures: 1 launch each.  cfg3's full capture is a 1/40
# walker subset (replaying the 1.6 s launch ~40x is too long); its DRAM traffic is taken
# from a metrics-only pass over the full bench launch instead.
set -x
mkdir -p gpurun_out/prof
NCU="ncu --clock-control none --nvtx --nvtx-include csaw_step/"
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-zerocopy"
run() {  # cfg kernel-regex extra-bench-args
  cfg=$1; kre=$2; shift 2
  timeout 900 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/prof/${cfg}_launches.csv $B --config ${cfg%%@*} "$@" > gpurun_out/prof/${cfg}_ll.log 2>&1
  timeout 1200 $NCU --set full --import-source on -k regex:$kre -c 1 -o gpurun_out/prof/${cfg} $B --config ${cfg%%@*} "$@" > gpurun_out/prof/${cfg}_full.log 2>&1
  ncu -i gpurun_out/prof/${cfg}.ncu-rep --page raw --csv > gpurun_out/prof/${cfg}_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof/${cfg}.ncu-rep --page details --csv > gpurun_out/prof/${cfg}_details.csv 2>/dev/null
  ls -la gpurun_out/prof/${cfg}*
}
run cfg2 k_walk_head
run cfg2@scan "^k_walk$" --no-cache
run cfg1 k_sample_fused
run cfg4_layer k_sample_fused
run cfg4_ff k_sample_fused
run cfg5@inmem k_mdrw_fast --in-memory
# cfg3: launch list + DRAM traffic of the full bench launch (metrics-only), full capture of a subset
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/prof/cfg3_launches.csv $B --config cfg3 > gpurun_out/prof/cfg3_ll.log 2>&1
timeout 900 ncu --clock-control none --set full --import-source on -k regex:k_node2vec_tri -c 1 -o gpurun_out/prof/cfg3_subset40 python scripts/prof_n2v.py 40 cache > gpurun_out/prof/cfg3_full.log 2>&1
ncu -i gpurun_out/prof/cfg3_subset40.ncu-rep --page raw --csv > gpurun_out/prof/cfg3_subset40_raw.csv 2>/dev/null
ncu -i gpurun_out/prof/cfg3_subset40.ncu-rep --page details --csv > gpurun_out/prof/cfg3_subset40_details.csv 2>/dev/null
# keep the transfer small: drop reps over 20 MB
find gpurun_out/prof -name '*.ncu-rep' -size +20M -delete
du -sh gpurun_out/prof
