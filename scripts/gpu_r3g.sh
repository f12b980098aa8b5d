#!/bin/bash
# DRAM cost of one random access by size and cache operator (scripts/random_granule.cu)
mkdir -p gpurun_out/r3g
O=gpurun_out/r3g
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rg scripts/random_granule.cu && /tmp/rg > $O/granule.txt
timeout 900 ncu --clock-control none --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum,gpu__time_duration.sum --csv --log-file $O/granule_ncu.csv /tmp/rg > /dev/null 2>&1
cat $O/granule.txt; grep -E "dram__bytes_read|srcunit_tex|time_dur" $O/granule_ncu.csv | awk -F'","' '{print $1, $5, $(NF-2), $NF}'
